#!/usr/bin/env python
"""Benchmark: TokenSelect decode step (Selection Cache -> paged Q.K scoring ->
soft vote -> top-k -> sparse paged attention -> KV append) on B200.

Default workload at N = 1 (BASELINE.json configs[1]):
- one Llama-3-8B attention layer (32 query / 8 KV heads, d = 128);
- a 128K-token paged bf16 KV cache;
- k = 2048 selected tokens, n_init = 128, n_local = 512;
- Selection Cache on at theta = 0.9; batch 1.

The decode query stream is the reference's `rotating` stream
(workload.cpp:261-274) at consecutive similarity 0.95, rescaled to unit
per-element variance. The cache therefore alternates miss / hit, like the
reference's cache-stats experiment. A step is one decode step; the metric is
the mean device microseconds per step over the stream. Like a model's decode
loop, consecutive steps run different layers: 4 layer caches (2.1 GB of K/V,
far larger than the 126 MB L2) are stepped round-robin, so each step's K/V is
cold. The other workloads flush L2 (a 512 MB write) before every step.

With N > 1 (torchrun, one rank per GPU), the workload is configs[3]: the
KV-sequence-sharded decode, with weak scaling of 128K tokens per GPU, so the
context is N x 128K (1M at N = 8). Every rank holds its slice. A step is the
sharded protocol: three NCCL all-gathers over NVLink between four native
launches (paper_2411_02886_b200/sharded.py). The step time is the max over
ranks.

Extra workloads, recorded as evidence but not the driver's line:
- `--workload batched`: configs[2], Qwen2-7B shapes, 16 x 64K, per-request
  page tables, one launch per step;
- `--workload prefill`: configs[4], one 512-row chunk at 128K context.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload ...]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_CTX = 131072
H, H_KV, D = 32, 8, 128
K_SEL, N_INIT, N_LOCAL, THETA = 2048, 128, 512, 0.9
SIMILARITY = 0.95
METRIC = "decode select+sparse-attn µs/step at 128K–1M ctx; HBM GB/s vs peak"
UNIT = "us/step"


# --------------------------------------------------------------- workload
def rotating_stream(steps: int, seed: int, dim: int = H * D, sim: float = SIMILARITY) -> np.ndarray:
    """generate_query_stream kRotating (workload.cpp:261-274), x sqrt(dim)."""
    g = np.random.default_rng(seed)
    e1 = g.standard_normal(dim)
    e1 /= np.linalg.norm(e1)
    e2 = g.standard_normal(dim)
    e2 -= (e2 @ e1) * e1
    e2 /= np.linalg.norm(e2)
    phi = math.acos(sim)
    qs = [(math.cos(phi * t) * e1 + math.sin(phi * t) * e2) * math.sqrt(dim) for t in range(steps)]
    return np.asarray(qs, dtype=np.float32).reshape(steps, 1, dim)


def step_kv(steps: int, seed: int, kv_dim: int = H_KV * D):
    g = np.random.default_rng(seed ^ 0x9E3779B97F4A7C15)
    k = (g.standard_normal((steps, 1, kv_dim)) * 3.0).astype(np.float32)
    v = g.standard_normal((steps, 1, kv_dim)).astype(np.float32)
    return k, v


def cache_decisions(qs: np.ndarray, theta: float):
    """Replays Algorithm 1 (selection_cache.cpp:29-35, fp64 cosine, strict <)
    on the host to label each step hit or miss, for the per-kind breakdown."""
    kinds, cached = [], None
    for q in qs.reshape(len(qs), -1).astype(np.float64):
        if cached is None:
            hit = False
        else:
            c = float(q @ cached) / math.sqrt(float(q @ q) * float(cached @ cached))
            hit = not (c < theta)
        if not hit:
            cached = q
        kinds.append(hit)
    return kinds


def algorithmic_bytes(n_cached: int, miss: bool, h=H, h_kv=H_KV, d=D, k=K_SEL, n_init=N_INIT, n_local=N_LOCAL) -> int:
    """B_miss = T(R+4) + A(2R+4) + 2R + 2*H*d*4 + 2R;
    B_hit = A(2R+4) + 2R + 2*H*d*4 + k*4 + 2R (R = H_kv*d*2 bytes per row)."""
    R = h_kv * d * 2
    T = max(0, n_cached - n_init - n_local)
    A = n_init + min(k, T) + n_local
    common = A * (2 * R + 4) + 2 * R + 2 * h * d * 4 + 2 * R
    return T * (R + 4) + common if miss else common + k * 4


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + clock-event reasons (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# -------------------------------------------------------------- CPU side
def reference_engine(kind: str):
    from oracle.oracle import Oracle, ref_available  # cpu baseline / reference arm only

    if kind == "reference" and not ref_available():
        kind = "port"
    return Oracle(kind), kind


def host_string() -> str:
    """CPU model and core count of this host (hardware_string,
    selattn_bench.cpp:133-145)."""
    model = "unknown CPU"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model}, nproc {os.cpu_count()}"


def reference_pool(seed: int = 1, steps: int = 0):
    o, kind = reference_engine("reference")
    g = np.random.default_rng(seed)
    eng = o.engine(N_CTX + steps + 64, k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=512,
                   theta=THETA, num_heads=H, num_kv_heads=H_KV, head_dim=D, block_size=64)
    chunk = 16384
    for s0 in range(0, N_CTX, chunk):
        kk = (g.standard_normal((chunk, H_KV * D)) * 3.0).astype(np.float32)
        vv = g.standard_normal((chunk, H_KV * D)).astype(np.float32)
        eng.append(kk, vv)
    return eng, kind


def time_reference_split(n_miss: int = 5, n_hit: int = 5, warmup: int = 2, seed: int = 1):
    """The reference's own decode_step (attention.cpp:172-200) on this host at
    the bench's config, with the reference bench's methodology
    (selattn_bench.cpp:147-159, 243-252): median of >= 5 timed calls after 2
    warm-ups (monotonic clock), misses (forced with first_flag, the
    cmd_cache_stats idiom at :439) and hits (the same query again) timed
    separately. Single-threaded by design (README:192-193)."""
    eng, kind = reference_pool(seed, warmup + n_miss + n_hit + 1)
    qs = rotating_stream(warmup + n_miss + 1, seed)
    ks, vs = step_kv(warmup + n_miss + n_hit + 1, seed)
    miss, hit = [], []
    t = 0
    for i in range(warmup + n_miss):
        eng.force_miss()
        t0 = time.perf_counter()
        _, h, _ = eng.decode(qs[i], ks[t], vs[t])
        dt = time.perf_counter() - t0
        assert not h
        t += 1
        if i >= warmup:
            miss.append(dt)
    q_last = qs[warmup + n_miss - 1]
    for i in range(n_hit):
        t0 = time.perf_counter()
        _, h, _ = eng.decode(q_last, ks[t], vs[t])
        dt = time.perf_counter() - t0
        assert h
        t += 1
        hit.append(dt)
    return 1e6 * statistics.median(miss), 1e6 * statistics.median(hit), kind


def cpu_baseline_line(kinds, n_miss=5, n_hit=5, warmup=2):
    """cpu_baseline object: the reference's median miss / hit step, weighted
    by the hit rate of the GPU arm's own stream."""
    miss_us, hit_us, kind = time_reference_split(n_miss, n_hit, warmup)
    n_h = sum(kinds)
    value = (miss_us * (len(kinds) - n_h) + hit_us * n_h) / len(kinds)
    sample = (f"reference decode_step at {N_CTX // 1024}K context: median of {n_miss} forced misses and of {n_hit} "
              f"hits after {warmup} warm-ups, weighted by this stream's {len(kinds) - n_h} misses / {n_h} hits; "
              f"1 of {os.cpu_count()} host cores ({host_string()})")
    return {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
            "miss_us": round(miss_us, 1), "hit_us": round(hit_us, 1), "host": host_string()}


def time_reference(steps: int, warmup: int, seed: int = 1):
    """--impl reference: the reference's decode_step over the bench's own
    rotating stream (same config, metric and step count as our arm)."""
    eng, kind = reference_pool(seed, warmup + steps)
    qs = rotating_stream(warmup + steps, seed)
    ks, vs = step_kv(warmup + steps, seed)
    times, hits = [], 0
    for t in range(warmup + steps):
        t0 = time.perf_counter()
        _, hit, _ = eng.decode(qs[t], ks[t], vs[t])
        dt = time.perf_counter() - t0
        if t >= warmup:
            times.append(dt)
            hits += int(hit)
    us = 1e6 * sum(times) / len(times)
    sample = (f"{len(times)} reference decode_step calls at {N_CTX // 1024}K context after {warmup} warm-up, "
              f"rotating stream sim {SIMILARITY}, theta {THETA}: {len(times) - hits} misses / {hits} hits; "
              f"1 of {os.cpu_count()} host cores ({host_string()})")
    return us, kind, sample


# ------------------------------------------------------------------ GPU
def fill_bf16(append, n, kv_dim, dev, seed, chunk=16384, seq=None):
    import torch

    gen = torch.Generator(device=dev).manual_seed(seed)
    for s0 in range(0, n, chunk):
        m = min(chunk, n - s0)
        kk = (torch.randn(m, kv_dim, device=dev, generator=gen) * 3.0).to(torch.bfloat16)
        vv = torch.randn(m, kv_dim, device=dev, generator=gen).to(torch.bfloat16)
        if seq is None:
            append(kk, vv)
        else:
            append(kk, vv, seq)


def timed_steps(stream, flush, run_step, steps, warmup, local_rank, world, counter=None):
    """W untimed steps, then K steps each bracketed by CUDA events on `stream`,
    each preceded by an L2 flush (512 MB write) unless `flush` is empty
    (inputs larger than L2); barrier + synchronize on both sides. The timed
    steps are queued ahead of the GPU (behind a device sleep), so a step's
    time is its device time. Returns per-step device us and the clock summary."""
    import torch

    dev = torch.device("cuda", local_rank)
    for i in range(warmup):
        if flush.numel():
            with torch.cuda.stream(stream):
                flush.zero_()
        run_step(i)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    evs = []
    c0 = counter() if counter else 0
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize(dev)
        # the K steps are queued behind a device-side sleep, so they run
        # back to back on the GPU (as in a captured decode loop) and no step's
        # events include the host's launch latency; the sleep itself is
        # outside every step's event pair
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(2e6 + 2e5 * steps * (8 if world > 1 else 1)))  # ~1 ms + 0.1 ms/step (cycles)
        for t in range(steps):
            if flush.numel():
                with torch.cuda.stream(stream):
                    flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step(warmup + t)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
    launches = (counter() - c0) if counter else None  # our kernels launched in the timed region
    if world > 1:
        torch.distributed.barrier()
    return [a.elapsed_time(b) * 1000.0 for a, b in evs], clk.summary(), launches


def split_by_kind(step_us, kinds):
    miss = [u for u, h in zip(step_us, kinds) if not h]
    hit = [u for u, h in zip(step_us, kinds) if h]
    return (statistics.mean(miss) if miss else None), (statistics.mean(hit) if hit else None)


LAYERS = 4  # decode workload: layer caches stepped round-robin (2.1 GB of K/V > 126 MB L2)


def run_decode_single(args, local_rank, n_ctx=N_CTX):
    """configs[1]: the fused single-launch decode step (N = 1).

    Like a model's decode loop, consecutive steps run different layers:
    LAYERS independent layer caches (each 128K tokens, its own Selection
    Cache and query stream) are stepped round-robin, so every step's K/V is
    cold in L2 (the other layers streamed >1.6 GB through it), while the
    kernel's code stays resident as it would across a real model's layers."""
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2411_02886_b200 import selattn as sa

    dev = torch.device("cuda", local_rank)
    total = args.warmup + args.steps
    per_layer = (total + LAYERS - 1) // LAYERS
    engines, streams = [], []
    for L in range(LAYERS):
        eng = sa.Engine(n_ctx + 2 * per_layer + 16, k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=512,
                        theta=THETA, num_heads=H, num_kv_heads=H_KV, head_dim=D, block_size=64)
        fill_bf16(eng.append_bf16, n_ctx, H_KV * D, dev, 1234 + L)
        engines.append(eng)
    qs_h = [rotating_stream(per_layer, 1234 + L) for L in range(LAYERS)]
    kv_h = [step_kv(per_layer, 1234 + L) for L in range(LAYERS)]
    qs = [torch.from_numpy(x).to(dev) for x in qs_h]
    ks = [torch.from_numpy(x[0]).to(dev) for x in kv_h]
    vs = [torch.from_numpy(x[1]).to(dev) for x in kv_h]
    out = torch.empty(1, H * D, device=dev)
    no_flush = torch.empty(0, dtype=torch.uint8, device=dev)  # inputs > L2: no flush needed
    stream = torch.cuda.Stream(dev)
    for eng in engines:
        eng.set_stream(stream.cuda_stream)

    def step(i):
        L, t = i % LAYERS, i // LAYERS
        engines[L].decode_async(qs[L][t], ks[L][t], vs[L][t], out)

    st0 = [eng.stats() for eng in engines]
    step_us, clocks, launches = timed_steps(stream, no_flush, step, args.steps, args.warmup, local_rank, 1,
                                            sa.launch_count)
    st1 = [eng.stats() for eng in engines]
    kinds_l = [cache_decisions(q, THETA) for q in qs_h]
    all_kinds = [kinds_l[i % LAYERS][i // LAYERS] for i in range(total)]
    kinds = all_kinds[args.warmup:]
    # the device's own Selection Cache counters must agree with the host replay
    dev_hits = sum(b["hits"] - a["hits"] for a, b in zip(st0, st1))
    assert dev_hits == sum(all_kinds), (dev_hits, sum(all_kinds))
    hits, lookups = sum(kinds), len(kinds)
    miss_us, hit_us = split_by_kind(step_us, kinds)
    n_mean = n_ctx + per_layer
    alg = sum(algorithmic_bytes(n_mean, not h) for h in kinds) / len(kinds)

    # end-to-end: host buffers through the public C ABI (H2D + D2H inside the call)
    for eng in engines:
        eng.set_stream(None)
    e_steps = (args.steps + LAYERS - 1) // LAYERS
    qs_e = [rotating_stream(e_steps, 77 + L) for L in range(LAYERS)]
    kv_e = [step_kv(e_steps, 77 + L) for L in range(LAYERS)]
    out_h = np.zeros((1, H * D), np.float32)
    hit_h = np.zeros(1, np.int32)
    e2e = []
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        L, t = i % LAYERS, i // LAYERS
        t0 = time.perf_counter()
        engines[L].decode_into(qs_e[L][t], kv_e[L][0][t], kv_e[L][1][t], out_h, hit_h)
        e2e.append(time.perf_counter() - t0)
    return {"step_us": statistics.mean(step_us), "miss_us": miss_us, "hit_us": hit_us, "hits": hits,
            "lookups": lookups, "kinds": kinds, "alg_bytes": alg, "launches": launches, "clocks": clocks,
            "e2e_us": 1e6 * statistics.mean(e2e), "h2d": (H * D + 2 * H_KV * D) * 4, "d2h": H * D * 4 + 48,
            "miss_bytes": algorithmic_bytes(n_mean, True), "hit_bytes": algorithmic_bytes(n_mean, False),
            "n_ctx": n_ctx, "per_gpu_bytes_div": 1}


def run_decode_sharded(args, rank, world, local_rank):
    """configs[3]: KV-sequence-sharded decode, 128K tokens per GPU (weak scaling)."""
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2411_02886_b200 import sharded
    from paper_2411_02886_b200 import selattn as sa

    dev = torch.device("cuda", local_rank)
    total = args.warmup + args.steps
    n_global = args.context or N_CTX * world
    ranges = sharded.shard_ranges(n_global, world, N_INIT, N_LOCAL)
    rr = ranges[rank]
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        shard = sharded.NativeShard(rank, world, rr.length + 2 * total + 16, k=K_SEL, n_local=N_LOCAL,
                                    n_init=N_INIT, chunk_size=512, theta=THETA, num_heads=H, num_kv_heads=H_KV,
                                    head_dim=D, block_size=64)
    fill_bf16(shard.append_bf16, rr.length, H_KV * D, dev, 1234 + rank)
    seed = 1234  # q / k_t / v_t replicated on every rank
    qs_h = rotating_stream(total, seed)
    ks_h, vs_h = step_kv(total, seed)
    qs, ks, vs = (torch.from_numpy(x).to(dev) for x in (qs_h, ks_h, vs_h))
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    comm = sharded.LibraryComm(rank, world)  # the library's own NCCL communicator
    out_d = torch.empty(1, H * D, dtype=torch.float32, device=dev)

    def step(i):
        with torch.cuda.stream(stream):
            sharded.decode_step_native(shard, comm, qs[i].view(-1), ks[i].view(-1), vs[i].view(-1), rr.base,
                                       n_global + i, out_d)

    step_us, clocks, launches = timed_steps(stream, flush, step, args.steps, args.warmup, local_rank, world,
                                            sa.launch_count)
    kinds = cache_decisions(qs_h, THETA)[args.warmup:]
    # end-to-end: host q/k/v -> H2D, the sharded step, D2H of the output
    qs_e = rotating_stream(args.steps, seed + 7)
    ks_e, vs_e = step_kv(args.steps, seed + 7)
    e2e = []
    pins = [torch.empty(x[0].size, dtype=torch.float32).pin_memory() for x in (qs_e, ks_e, vs_e)]
    for t in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        torch.distributed.barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for pin, x in zip(pins, (qs_e[t], ks_e[t], vs_e[t])):
                pin.copy_(torch.from_numpy(x).view(-1))  # host buffer -> pinned staging
            q, k, v = (pin.to(dev, non_blocking=True) for pin in pins)
            sharded.decode_step_native(shard, comm, q, k, v, rr.base, n_global + total + t, out_d).cpu()
        e2e.append(time.perf_counter() - t0)
    mt = torch.tensor(step_us + [1e6 * statistics.mean(e2e)], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(mt, op=torch.distributed.ReduceOp.MAX)  # max over ranks, per step
    vals = mt.tolist()
    step_us, e2e_us = vals[:-1], vals[-1]
    miss_us, hit_us = split_by_kind(step_us, kinds)
    n_mean = n_global + args.warmup + args.steps // 2
    alg = sum(algorithmic_bytes(n_mean, not h) for h in kinds) / len(kinds)
    return {"step_us": statistics.mean(step_us), "miss_us": miss_us, "hit_us": hit_us, "hits": sum(kinds),
            "lookups": len(kinds), "alg_bytes": alg, "launches": launches, "clocks": clocks, "e2e_us": e2e_us,
            "h2d": (H * D + 2 * H_KV * D) * 4, "d2h": H * D * 4, "miss_bytes": algorithmic_bytes(n_mean, True),
            "hit_bytes": algorithmic_bytes(n_mean, False), "n_ctx": n_global, "per_gpu_bytes_div": world}


def run_batched(args, local_rank):
    """configs[2]: Qwen2-7B shapes, 16 requests x 64K context, one launch per step."""
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2411_02886_b200 import selattn as sa

    dev = torch.device("cuda", local_rank)
    B, n, h, hkv, d = 16, 65536, 28, 4, 128
    total = args.warmup + args.steps
    eng = sa.Engine(n + total + 16, k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=512, theta=THETA,
                    num_heads=h, num_kv_heads=hkv, head_dim=d, block_size=64, n_seqs=B)
    for b in range(B):
        fill_bf16(eng.append_bf16, n, hkv * d, dev, 99 + b, seq=b)
    qs_h = np.concatenate([rotating_stream(total, 500 + b, h * d) for b in range(B)], axis=1)  # [steps, B, h*d]
    kv = [step_kv(total, 500 + b, hkv * d) for b in range(B)]
    ks_h = np.concatenate([x[0] for x in kv], axis=1)
    vs_h = np.concatenate([x[1] for x in kv], axis=1)
    qs, ks, vs = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (qs_h, ks_h, vs_h))
    out = torch.empty(B, h * d, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    eng.set_stream(stream.cuda_stream)
    step_us, clocks, launches = timed_steps(stream, flush, lambda i: eng.decode_async(qs[i], ks[i], vs[i], out),
                                            args.steps, args.warmup, local_rank, 1, sa.launch_count)
    kinds_b = [cache_decisions(qs_h[:, b], THETA)[args.warmup:] for b in range(B)]
    n_mean = n + args.warmup + args.steps // 2
    alg = sum(sum(algorithmic_bytes(n_mean, not kb[t], h, hkv, d) for kb in kinds_b)
              for t in range(args.steps)) / args.steps
    return {"step_us": statistics.mean(step_us), "miss_us": None, "hit_us": None,
            "hits": sum(sum(k) for k in kinds_b), "lookups": B * args.steps, "alg_bytes": alg, "launches": launches,
            "clocks": clocks, "e2e_us": None, "h2d": 0, "d2h": 0,
            "miss_bytes": B * algorithmic_bytes(n_mean, True, h, hkv, d),
            "hit_bytes": B * algorithmic_bytes(n_mean, False, h, hkv, d), "n_ctx": n, "per_gpu_bytes_div": 1}


def run_prefill(args, local_rank):
    """configs[4]: one 512-row prefill chunk at 128K context (select_for_chunk
    with the chunk-mean query, sparse causal attention, append)."""
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2411_02886_b200 import selattn as sa

    dev = torch.device("cuda", local_rank)
    C = 512
    total = args.warmup + args.steps
    eng = sa.Engine(N_CTX + C * total + 16, k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=C, theta=THETA,
                    num_heads=H, num_kv_heads=H_KV, head_dim=D, block_size=64)
    fill_bf16(eng.append_bf16, N_CTX, H_KV * D, dev, 1234)
    g = torch.Generator(device=dev).manual_seed(7)
    q = torch.randn(total, C, H * D, device=dev, generator=g)
    k = (torch.randn(total, C, H_KV * D, device=dev, generator=g) * 3.0).to(torch.bfloat16).float()
    v = torch.randn(total, C, H_KV * D, device=dev, generator=g).to(torch.bfloat16).float()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    eng.set_stream(stream.cuda_stream)
    out = torch.empty(C, H * D, device=dev)
    # device time: the stream-ordered entry (the synchronous one would put the
    # host's launch and sync latency between the steps' events)
    step_us, clocks, launches = timed_steps(stream, flush, lambda i: eng.prefill_async(q[i], k[i], v[i], out),
                                            args.steps, args.warmup, local_rank, 1, sa.launch_count)
    eng.sync()
    # end to end: the synchronous prefill with host buffers (H2D of the chunk's
    # q/k/v and D2H of its output inside the call)
    n_e = max(3, min(args.steps, 10))
    e_eng = sa.Engine(N_CTX + C * (n_e + 1) + 16, k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=C, theta=THETA,
                      num_heads=H, num_kv_heads=H_KV, head_dim=D, block_size=64)
    del eng
    fill_bf16(e_eng.append_bf16, N_CTX, H_KV * D, dev, 1234)
    # host buffers in pinned memory (what a serving host stages activations
    # in), so the copies run at DMA speed
    def pinned(x):
        return x.cpu().pin_memory().numpy()

    qh = [pinned(q[i % total]) for i in range(n_e + 1)]
    kh = [pinned(k[i % total]) for i in range(n_e + 1)]
    vh = [pinned(v[i % total]) for i in range(n_e + 1)]
    oh = torch.empty(C, H * D).pin_memory().numpy()
    e_eng.prefill(qh[0], kh[0], vh[0], out=oh)  # warm-up
    e2e = []
    for i in range(1, n_e + 1):
        t0 = time.perf_counter()
        e_eng.prefill(qh[i], kh[i], vh[i], out=oh)
        e2e.append(time.perf_counter() - t0)
    R = H_KV * D * 2
    T = N_CTX - N_INIT - N_LOCAL
    alg = T * (R + 4) + C * H * D * 4 + (N_INIT + K_SEL + N_LOCAL) * 2 * R + 2 * C * R + C * H * D * 4
    return {"step_us": statistics.mean(step_us), "miss_us": None, "hit_us": None, "hits": 0, "lookups": 0,
            "alg_bytes": alg, "launches": launches, "clocks": clocks, "e2e_us": 1e6 * statistics.median(e2e),
            "h2d": C * (H * D + 2 * H_KV * D) * 4, "d2h": C * H * D * 4,
            "miss_bytes": alg, "hit_bytes": alg, "n_ctx": N_CTX, "per_gpu_bytes_div": 1,
            "flops": 2 * H * sum(N_INIT + K_SEL + N_LOCAL + i + 1 for i in range(C)) * D * 2}


def run_full(args, local_rank):
    """The full-attention baseline (reference bench-attn's full path,
    selattn_bench.cpp:214-226: sdpa_full over the whole cache + the current
    token) on the same kernels: an engine with k = 0 and a local window
    covering the whole context attends all N + 1 rows every step. Same
    4-layer rotation as the decode workload; the ratio of the two is the
    B200 speed-up of selective over full attention."""
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2411_02886_b200 import selattn as sa

    dev = torch.device("cuda", local_rank)
    total = args.warmup + args.steps
    per_layer = (total + LAYERS - 1) // LAYERS
    engines = []
    for L in range(LAYERS):
        eng = sa.Engine(N_CTX + 2 * per_layer + 16, k=0, n_local=N_CTX + 2 * per_layer + 16, n_init=0,
                        chunk_size=512, theta=THETA, num_heads=H, num_kv_heads=H_KV, head_dim=D, block_size=64)
        fill_bf16(eng.append_bf16, N_CTX, H_KV * D, dev, 1234 + L)
        engines.append(eng)
    qs = [torch.from_numpy(rotating_stream(per_layer, 1234 + L)).to(dev) for L in range(LAYERS)]
    kv = [step_kv(per_layer, 1234 + L) for L in range(LAYERS)]
    ks = [torch.from_numpy(x[0]).to(dev) for x in kv]
    vs = [torch.from_numpy(x[1]).to(dev) for x in kv]
    out = torch.empty(1, H * D, device=dev)
    no_flush = torch.empty(0, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    for eng in engines:
        eng.set_stream(stream.cuda_stream)

    def step(i):
        L, t = i % LAYERS, i // LAYERS
        engines[L].decode_async(qs[L][t], ks[L][t], vs[L][t], out)

    step_us, clocks, launches = timed_steps(stream, no_flush, step, args.steps, args.warmup, local_rank, 1,
                                            sa.launch_count)
    n_mean = N_CTX + per_layer
    R = H_KV * D * 2
    alg = n_mean * (2 * R + 4) + 2 * R + H * D * 4 * 2 + 2 * R  # all rows' K + V + page table, current, q, out, append
    return {"step_us": statistics.mean(step_us), "miss_us": None, "hit_us": None, "hits": 0, "lookups": 0,
            "kinds": [], "alg_bytes": alg, "launches": launches, "clocks": clocks, "e2e_us": None, "h2d": 0,
            "d2h": 0, "miss_bytes": alg, "hit_bytes": alg, "n_ctx": N_CTX, "per_gpu_bytes_div": 1}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1632.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def traffic_per_launch():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


WORKLOADS = {
    "decode": "Llama-3-8B layer decode, 128K paged bf16 KV, k=2048, Selection Cache theta=0.9 (configs[1])",
    "sharded": "Llama-3-8B layer decode, KV-sequence-sharded over N GPUs (N x 128K tokens, weak scaling, 1M at "
               "N=8; --context 1048576: 1M at every N), one library call per step: 4 shard launches + 3 "
               "ncclAllGather of stats / top-k / LSE partials on the engine stream (configs[3])",
    "batched": "Qwen2-7B layer decode, 16 requests x 64K, per-request page tables, one launch (configs[2])",
    "prefill": "Llama-3-8B chunked-prefill step: one 512-query chunk over a 128K context (configs[4])",
    "full": "Llama-3-8B layer decode with FULL attention over the 128K paged bf16 KV (the reference bench-attn "
            "full baseline, selattn_bench.cpp:214-226), same kernels, no selection",
}


_OUT = None  # the process's real stdout: only the one JSON line goes there


def emit(line: dict):
    os.write(_OUT if _OUT is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _OUT
    # everything else the process prints (NCCL's INFO lines and version banner,
    # library diagnostics) goes to stderr: fd 1 is pointed at fd 2, the JSON
    # line is written to a private duplicate of the original stdout
    sys.stdout.flush()
    _OUT = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--context", type=int, default=0,
                    help="sharded workload: total context tokens (strong scaling, e.g. 1048576 for configs[3] "
                         "at every N); default N x 128K (weak scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-execute under
        # torch.distributed.run, one rank per GPU (rank 0 prints the line)
        import socket

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.dup2(_OUT, 1)  # the launcher's ranks write the line to the real stdout
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    workload = args.workload or ("sharded" if world > 1 else "decode")
    shapes = (28, 4, 128) if workload == "batched" else (H, H_KV, D)  # configs[2] is Qwen2-7B
    config = {"workload": WORKLOADS[workload], "num_heads": shapes[0], "num_kv_heads": shapes[1], "head_dim": shapes[2],
              "k": K_SEL,
              "n_init": N_INIT, "n_local": N_LOCAL, "theta": THETA,
              "stream": f"rotating, consecutive cos {SIMILARITY}",
              "parallelism": f"KV-sequence shards x{world}" if workload == "sharded" else "single GPU",
              "l2": (f"no flush: {LAYERS} layer caches stepped round-robin, {LAYERS * 2 * N_CTX * H_KV * D * 2 >> 20} MB "
                     f"of K/V > 126 MB L2" if workload in ("decode", "full")
                     else "flushed (512 MB write) before every timed step")}

    if args.impl == "reference":
        if rank != 0:
            return
        steps = min(args.steps, 100)  # our arm's step count (bounded: ~1.8 s per reference miss)
        us, kind, sample = time_reference(steps, 2)
        config["context_tokens"] = N_CTX
        line = {"impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": UNIT, "n_gpus": args.gpus,
                "steps": steps, "warmup": 2, "ms_per_step": round(us / 1000, 3), "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": 1, "kind": kind, "sample": sample},
                "e2e": {"value": round(us, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        emit(line)
        return

    if world > 1 or workload == "sharded":
        import torch

        torch.cuda.set_device(local_rank)
        # NCCL's communicator lines (transport, NVLS, ranks) go to stderr; stdout
        # stays the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        torch.distributed.init_process_group("nccl", rank=rank, world_size=world,
                                             device_id=torch.device("cuda", local_rank))
    if workload == "sharded" and world == 1 and args.context:
        # strong scaling's N = 1 point: the whole context on one GPU, fused kernel
        r = run_decode_single(args, local_rank, args.context)
    elif workload == "sharded":
        r = run_decode_sharded(args, rank, world, local_rank)
    elif workload == "batched":
        r = run_batched(args, local_rank)
    elif workload == "prefill":
        r = run_prefill(args, local_rank)
    elif workload == "full":
        r = run_full(args, local_rank)
    else:
        r = run_decode_single(args, local_rank)
    config["context_tokens"] = r["n_ctx"]
    hbm, tflops, peak_kind = peaks()
    div = r["per_gpu_bytes_div"]
    achieved = r["alg_bytes"] / div / (r["step_us"] * 1e-6) / 1e9  # per GPU
    miss_ach = r["miss_bytes"] / div / (r["miss_us"] * 1e-6) / 1e9 if r["miss_us"] else None
    traffic = traffic_per_launch() if workload == "decode" else None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "peak_kind": peak_kind, "per": "GPU",
            "traffic": (int((r["lookups"] - r["hits"]) / max(r["lookups"], 1) * traffic["miss_bytes_per_launch"]
                            + r["hits"] / max(r["lookups"], 1) * traffic["hit_bytes_per_launch"])
                        if traffic else None),
            "traffic_source": traffic.get("source") if traffic else None,
            "algorithmic_bytes_per_step": int(r["alg_bytes"])}
    if miss_ach:
        roof["miss_step"] = {"achieved": round(miss_ach, 1), "frac": round(miss_ach / hbm, 4),
                             "algorithmic_bytes": r["miss_bytes"]}
    if "flops" in r:
        tf = r["flops"] / (r["step_us"] * 1e-6) / 1e12
        roof["tensor"] = {"achieved": round(tf, 2), "peak": tflops, "unit": "TFLOP/s", "frac": round(tf / tflops, 4),
                          "flops_per_step": r["flops"]}
    line = {
        "metric": METRIC, "value": round(r["step_us"], 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["step_us"] / 1000, 5), "higher_is_better": False,
        "scaling": "strong" if (workload == "sharded" and args.context) else "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random bf16 KV, rotating query stream)", "config": config,
        "cache": {"lookups": r["lookups"], "hits": r["hits"]},
        "miss_step_us": round(r["miss_us"], 2) if r["miss_us"] else None,
        "hit_step_us": round(r["hit_us"], 2) if r["hit_us"] else None,
        "roofline": roof,
        "e2e": ({"value": round(r["e2e_us"], 2), "unit": UNIT, "h2d_bytes_per_step": r["h2d"],
                 "d2h_bytes_per_step": r["d2h"]} if r["e2e_us"] else None),
        "clocks": r["clocks"], "gpu_launches": r["launches"], "gpus_active": world,
    }
    if rank == 0 and world == 1 and workload == "decode" and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_line(r["kinds"])
        except Exception as e:  # the oracle build is test infrastructure; report, do not fail the bench
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        emit(line)
    if world > 1 or workload == "sharded":
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

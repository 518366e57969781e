"""Where the end-to-end decode call spends its time (dev tool).

Times, at N tokens (default 131072), always-miss and always-hit streams:
  e2e    Engine.decode_into with host numpy buffers (the bench's e2e leg)
  sync   decode_async on device tensors + torch.cuda.synchronize
  b2b    decode_async back to back (device step time, no host waits)
and prints the library's host-side split (TS_HOST_PROF) at engine teardown.
"""
import os
import statistics
import sys
import time

os.environ.setdefault("TS_HOST_PROF", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
REPS = 200
H, Hkv, d = 32, 8, 128
rng = np.random.default_rng(0)


def run(theta, label):
    eng = sa.Engine(N + 4 * REPS + 64, k=2048, n_local=512, n_init=128, num_heads=H, num_kv_heads=Hkv, head_dim=d)
    K = torch.randn(N, Hkv * d, device="cuda").to(torch.bfloat16)
    eng.append_bf16(K, K)
    del K
    eng.set_theta(theta)
    q = rng.standard_normal((1, H * d), dtype=np.float32)
    k = rng.standard_normal((1, Hkv * d), dtype=np.float32)
    out = np.zeros((1, H * d), np.float32)
    hit = np.zeros(1, np.int32)
    for _ in range(5):
        eng.decode_into(q, k, k, out, hit)
    e2e = []
    for _ in range(REPS):
        t0 = time.perf_counter()
        eng.decode_into(q, k, k, out, hit)
        e2e.append(time.perf_counter() - t0)
    qd = torch.from_numpy(q).cuda()
    kd = torch.from_numpy(k).cuda()
    od = torch.empty_like(qd)
    eng.set_stream(torch.cuda.current_stream().cuda_stream or 1)
    sync = []
    for _ in range(REPS):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.decode_async(qd, kd, kd, od)
        torch.cuda.synchronize()
        sync.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(REPS):
        eng.decode_async(qd, kd, kd, od)
    torch.cuda.synchronize()
    b2b = (time.perf_counter() - t0) / REPS
    med = lambda xs: 1e6 * statistics.median(xs)
    print(f"{label}: e2e median {med(e2e):.1f} us (mean {1e6 * statistics.mean(e2e):.1f}); "
          f"async+sync {med(sync):.1f} us; back-to-back {1e6 * b2b:.1f} us/step; hit={int(hit[0])}", flush=True)
    del eng


run(2.0, "miss")
run(-2.0, "hit")
import ctypes as C  # noqa: E402
from paper_2411_02886_b200._native import lib  # noqa: E402

t0 = time.perf_counter()
for _ in range(10000):
    lib.ts_launch_count()
print(f"ctypes no-arg call: {1e6 * (time.perf_counter() - t0) / 10000:.2f} us")
a = np.zeros(4096, np.float32)
t0 = time.perf_counter()
for _ in range(10000):
    a.ctypes.data_as(C.c_void_p)
print(f"numpy ctypes.data_as: {1e6 * (time.perf_counter() - t0) / 10000:.2f} us")
# torch's own small pinned H2D in this process, for scale
hp = torch.empty(6144, dtype=torch.float32).pin_memory()
dd = torch.empty(6144, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for _ in range(20):
    with torch.cuda.stream(s):
        dd.copy_(hp, non_blocking=True)
s.synchronize()
api, tot = [], []
for _ in range(300):
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        dd.copy_(hp, non_blocking=True)
    t1 = time.perf_counter()
    s.synchronize()
    api.append(t1 - t0)
    tot.append(time.perf_counter() - t0)
print(f"torch pinned H2D 24KB: call {1e6 * statistics.median(api):.2f} us, +sync {1e6 * statistics.median(tot):.2f} us")
if os.path.exists(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ubench", "libcopyapi.so")):
    print("--- tools/ubench/copyapi in this process", flush=True)
    C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ubench", "libcopyapi.so")).bench_main()

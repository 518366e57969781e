"""Generates tests/golden/*.npz from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Runs only in the build container, where /root/reference exists: `make -C oracle`
compiles the reference sources (/root/reference/proj/src) behind
oracle/ref_shim.cpp into oracle/_ref/libselattn_ref.so, and every array below is
the reference's own output on seeded, bf16-representable inputs. The fixtures
are small (< 1 MB in total) and pin the C restatement (oracle/tsoracle.c) in
tests/test_oracle_golden.py wherever the reference cannot be built (the GPU box).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, build  # noqa: E402
from tests.helpers import bf16_round, rng_normal  # noqa: E402


def score_cases(ref):
    out = {}
    # (H, H_kv, d, n, page_size, shuffle, block)
    cases = [(4, 2, 16, 50, 1, 0, 64), (4, 2, 16, 50, 4, 9, 7), (6, 3, 8, 77, 1, 5, 1),
             (8, 2, 32, 120, 2, 3, 64), (32, 8, 128, 40, 1, 0, 64), (28, 4, 128, 33, 1, 2, 16)]
    for i, (H, H_kv, d, n, ps, sh, blk) in enumerate(cases):
        k = bf16_round(rng_normal(1000 + i, (n, H_kv * d), 3.0))
        q = rng_normal(2000 + i, (H, d))
        g = np.random.default_rng(3000 + i)
        cand = np.sort(g.choice(n, size=max(1, n // 2), replace=False)).astype(np.uint32)
        s = ref.score_paged(q, k, H_kv, cand, block_size=blk, page_size=ps, shuffle_seed=sh)
        out.update({f"c{i}_q": q, f"c{i}_k": k, f"c{i}_cand": cand, f"c{i}_S": s,
                    f"c{i}_meta": np.array([H, H_kv, d, n, ps, sh, blk], np.int64)})
    out["n"] = np.array(len(cases))
    return out


def select_cases(ref):
    out = {}
    cases = []
    # the reference's known answer (test_selector.cpp:128-141, acceptance.cpp:155-169)
    cases.append((np.array([[5, 4.5, 0, 0], [0, 0, 500, 480]], np.float32), 2))
    cases.append((np.full((3, 5), 1.25, np.float32), 2))          # uniform ties (test_selector.cpp:215-221)
    cases.append((rng_normal(11, (4, 200), 20.0), 17))
    cases.append((rng_normal(12, (8, 1000), 5.0), 100))
    cases.append((rng_normal(13, (2, 30), 50.0), 40))              # k > T
    S = rng_normal(14, (5, 300), 3.0)
    S[:, 100:110] = S[:, 100:101]                                   # planted exact ties
    cases.append((S, 50))
    i = 0
    for S, k in cases:
        H, T = S.shape
        cand = (np.arange(T, dtype=np.uint32) * 3 + 7).astype(np.uint32)
        out[f"c{i}_S"] = S
        out[f"c{i}_cand"] = cand
        out[f"c{i}_k"] = np.array(k)
        for m in ("topk", "head_vote", "head_soft_vote"):
            sel, crit = ref.select(S, cand, k, m)
            out[f"c{i}_{m}_sel"] = sel
            out[f"c{i}_{m}_crit"] = crit
        i += 1
    out["n"] = np.array(i)
    return out


def primitive_cases(ref):
    out = {}
    tk = [np.array([5, 1, 9], np.float64), np.array([7, 7, 7], np.float64),
          np.random.default_rng(5).integers(0, 20, 1000).astype(np.float64)]
    for i, (s, k) in enumerate(zip(tk, (2, 2, 100))):
        out[f"topk{i}_s"] = s
        out[f"topk{i}_k"] = np.array(k)
        out[f"topk{i}_out"] = ref.topk_indices(s, k)
    pairs = [(rng_normal(20, 4096), rng_normal(21, 4096))]
    a = rng_normal(22, 3584)
    pairs += [(a, a), (a, -a), (a, a * 0.5 + rng_normal(23, 3584) * 0.1)]
    for i, (u, v) in enumerate(pairs):
        out[f"cos{i}_u"], out[f"cos{i}_v"] = u, v
        out[f"cos{i}_out"] = np.array(ref.cosine(u, v))
    m = rng_normal(30, (6, 50), 10.0)
    out["softmax_in"], out["softmax_out"] = m, ref.softmax_rows(m)
    qc = rng_normal(31, (37, 96))
    out["cmean_in"], out["cmean_out"] = qc, ref.chunk_mean(qc)
    wins = [(100, 4, 8, [2, 5, 6, 90]), (6, 4, 4, []), (2000, 128, 512, list(range(100, 2000, 7))),
            (10, 4, 4, [4, 5]), (640, 128, 512, [0, 1])]
    for i, (cached, ni, nl, sel) in enumerate(wins):
        out[f"win{i}_args"] = np.array([cached, ni, nl], np.int64)
        out[f"win{i}_sel"] = np.array(sel, np.uint32)
        out[f"win{i}_merged"] = ref.make_windows(cached, ni, nl, sel)
    return out


def attention_cases(ref):
    out = {}
    cases = [(1, 4, 2, 8, 20), (3, 4, 2, 8, 20), (7, 2, 1, 16, 0), (1, 32, 8, 128, 50), (16, 6, 3, 32, 64)]
    for i, (C, H, H_kv, d, n) in enumerate(cases):
        q = rng_normal(40 + i, (C, H * d))
        k = bf16_round(rng_normal(50 + i, (n + C, H_kv * d), 2.0))
        v = bf16_round(rng_normal(60 + i, (n + C, H_kv * d)))
        out.update({f"c{i}_q": q, f"c{i}_k": k, f"c{i}_v": v, f"c{i}_H": np.array(H),
                    f"c{i}_out": ref.sdpa_full(q, k, v, H)})
    out["n"] = np.array(len(cases))
    return out


def engine_kv(i, n, H_kv, d):
    return (bf16_round(rng_normal(70 + i, (n, H_kv * d), 3.0)), bf16_round(rng_normal(80 + i, (n, H_kv * d))))


def kv_sha(K, V):
    import hashlib

    return hashlib.sha256(K.tobytes() + V.tobytes()).hexdigest()


def engine_cases(ref):
    """decode streams (Selection Cache hits and misses) + chunked prefill."""
    out = {}
    cfgs = [dict(n=200, H=4, H_kv=2, d=16, k=16, n_init=4, n_local=8, theta=0.9, method="head_soft_vote"),
            dict(n=300, H=8, H_kv=2, d=32, k=40, n_init=8, n_local=16, theta=0.5, method="topk"),
            dict(n=2100, H=32, H_kv=8, d=128, k=256, n_init=16, n_local=64, theta=0.9,
                 method="head_soft_vote")]
    for i, c in enumerate(cfgs):
        H, H_kv, d, n = c["H"], c["H_kv"], c["d"], c["n"]
        K, V = engine_kv(i, n, H_kv, d)
        eng = ref.engine(n + 64, k=c["k"], n_local=c["n_local"], n_init=c["n_init"], chunk_size=64,
                         theta=c["theta"], num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64,
                         selection_method=c["method"])
        eng.append(K, V)
        g = np.random.default_rng(90 + i)
        base = g.standard_normal(H * d).astype(np.float32)
        qs, ks, vs, outs, hits, sels = [], [], [], [], [], []
        for step in range(8):
            q = (base + (0.02 if step % 2 else 2.0) * g.standard_normal(H * d)).astype(np.float32)
            if step % 2 == 0:
                base = q
            kt = bf16_round(rng_normal(100 * i + step, (1, H_kv * d), 3.0))
            vt = bf16_round(rng_normal(100 * i + 50 + step, (1, H_kv * d)))
            o, hit, sel = eng.decode(q.reshape(1, -1), kt, vt)
            qs.append(q)
            ks.append(kt[0])
            vs.append(vt[0])
            outs.append(o[0])
            hits.append(hit)
            sel_p = np.full(c["k"], 0xFFFFFFFF, np.uint32)
            sel_p[: len(sel)] = sel
            sels.append(sel_p)
        # K/V are regenerated from their seeds by the test (numpy PCG64 is
        # stream-stable); the sha256 of their bytes pins that they match.
        out.update({f"d{i}_kv_sha": np.array(kv_sha(K, V)), f"d{i}_q": np.array(qs), f"d{i}_kt": np.array(ks),
                    f"d{i}_vt": np.array(vs), f"d{i}_out": np.array(outs), f"d{i}_hit": np.array(hits),
                    f"d{i}_sel": np.array(sels),
                    f"d{i}_cfg": np.array([n, H, H_kv, d, c["k"], c["n_init"], c["n_local"],
                                           {"topk": 0, "head_vote": 1, "head_soft_vote": 2}[c["method"]]],
                                          np.int64),
                    f"d{i}_theta": np.array(c["theta"])})
    out["nd"] = np.array(len(cfgs))
    # chunked prefill (attention.cpp:135-170)
    pcs = [dict(n=30, H=2, H_kv=2, d=4, chunk=8, k=4, n_init=2, n_local=4),
           dict(n=400, H=4, H_kv=2, d=32, chunk=64, k=32, n_init=8, n_local=16)]
    for i, c in enumerate(pcs):
        H, H_kv, d, n = c["H"], c["H_kv"], c["d"], c["n"]
        q = rng_normal(120 + i, (n, H * d))
        K = bf16_round(rng_normal(130 + i, (n, H_kv * d)))
        V = bf16_round(rng_normal(140 + i, (n, H_kv * d)))
        eng = ref.engine(n + 4, k=c["k"], n_local=c["n_local"], n_init=c["n_init"], chunk_size=c["chunk"],
                         theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=8)
        o, trace = eng.prefill(q, K, V, trace=True)
        out.update({f"p{i}_q": q, f"p{i}_K": K, f"p{i}_V": V, f"p{i}_out": o,
                    f"p{i}_trace": np.concatenate(trace) if trace else np.zeros(0, np.uint32),
                    f"p{i}_counts": np.array([len(t) for t in trace], np.int64),
                    f"p{i}_cfg": np.array([n, H, H_kv, d, c["chunk"], c["k"], c["n_init"], c["n_local"]],
                                          np.int64)})
    out["np"] = np.array(len(pcs))
    return out


def main():
    build()
    ref = Oracle("reference")
    for name, fn in (("score", score_cases), ("select", select_cases), ("primitives", primitive_cases),
                     ("attention", attention_cases), ("engine", engine_cases)):
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **fn(ref))
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()

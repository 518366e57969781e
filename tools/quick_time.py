"""Quick decode-step timing (dev tool): Llama-3-8B layer, N tokens, miss-only and hit-only streams,
R steps back to back between CUDA events (host launch overlapped)."""
import sys
import time

import numpy as np
import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H, Hkv, d = 32, 8, 128
R = 20
eng = sa.Engine(N + 512, k=2048, n_local=512, n_init=128, num_heads=H, num_kv_heads=Hkv, head_dim=d)
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn(N, Hkv * d, device="cuda", generator=g) * 3).to(torch.bfloat16)
V = torch.randn(N, Hkv * d, device="cuda", generator=g).to(torch.bfloat16)
eng.append_bf16(K, V)
del K, V
q = torch.randn(1, H * d, device="cuda", generator=g)
kt = torch.randn(1, Hkv * d, device="cuda", generator=g)
vt = torch.randn(1, Hkv * d, device="cuda", generator=g)
out = torch.empty(1, H * d, device="cuda")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")
for mode, theta in (("miss", 2.0), ("hit", -2.0)):
    eng.set_theta(theta)
    eng.decode_async(q, kt, vt, out)
    torch.cuda.synchronize()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        for it in range(R):
            eng.decode_async(q, kt, vt, out)
        e1.record(st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{mode}: {e0.elapsed_time(e1) * 1000 / R:.1f} us/step (gpu, back-to-back, L2 warm); host {1e6 * (t1 - t0) / R:.1f} us/launch")
    print(eng.stats())
if os.environ.get("QT_NOTRACE"):
    sys.exit(0)
eng.set_trace(True)
for mode, theta in (("miss", 2.0), ("hit", -2.0)):
    eng.set_theta(theta)
    for _ in range(3):
        eng.decode_async(q, kt, vt, out)
    torch.cuda.synchronize()
    print(mode, "phase trace (us):", {k: round(v, 2) for k, v in eng.read_trace().items()},
          f"SM clock {eng._trace_rate:.3f} GHz")
# all-CTA phase statistics of one miss and one hit step (start-relative us)
for mode, theta in (("miss", 2.0), ("hit", -2.0)):
    eng.set_theta(theta)
    for _ in range(3):
        eng.decode_async(q, kt, vt, out)
    torch.cuda.synchronize()
    a = eng.read_trace(all_ctas=True)
    names = eng.trace_names()
    print(f"{mode}: all-CTA stamps (us from earliest start): phase: min / median / max")
    for i, nm in sorted(names.items(), key=lambda kv: np.nanmedian(a[:, kv[0]]) if np.any(~np.isnan(a[:, kv[0]])) else 1e9):
        col = a[:, i]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"  {i:2d} {nm:18s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}  (n={col.size})")
    # QT_DIFF="a,b,c": per-CTA differences of consecutive listed slots (median / max over CTAs, us)
    if os.environ.get("QT_DIFF"):
        sl = [int(x) for x in os.environ["QT_DIFF"].split(",")]
        for x, y in zip(sl, sl[1:]):
            dd = a[:, y] - a[:, x]
            dd = dd[~np.isnan(dd)]
            if dd.size:
                print(f"  {mode} {names.get(x, x)} -> {names.get(y, y)}: median {np.median(dd):.2f} max {dd.max():.2f} us")

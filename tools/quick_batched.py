"""Phase trace of the batched decode (configs[2]: Qwen2-7B, 16 x 64K) (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402

B, n, h, hkv, d = 16, 65536, 28, 4, 128
eng = sa.Engine(n + 64, k=2048, n_local=512, n_init=128, num_heads=h, num_kv_heads=hkv, head_dim=d, n_seqs=B)
for b in range(B):
    g = torch.Generator(device="cuda").manual_seed(b)
    K = (torch.randn(n, hkv * d, device="cuda", generator=g) * 3).to(torch.bfloat16)
    eng.append_bf16(K, K, b)
del K
q = torch.randn(B, h * d, device="cuda")
kt = torch.randn(B, hkv * d, device="cuda")
out = torch.empty(B, h * d, device="cuda")
for theta in (2.0, -2.0):
    for s in range(B):
        eng.set_theta(theta, s)
    eng.decode_async(q, kt, kt, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        eng.decode_async(q, kt, kt, out)
    e1.record()
    torch.cuda.synchronize()
    print("theta", theta, "us/step", e0.elapsed_time(e1) * 1000 / 5)
    eng.set_trace(True)
    eng.decode_async(q, kt, kt, out)
    torch.cuda.synchronize()
    a = eng.read_trace(all_ctas=True)
    names = dict(enumerate(sa.Engine.TRACE_POINTS))
    names.update(sa.Engine.SUB_POINTS)
    for i, nm in sorted(names.items(), key=lambda kv: np.nanmedian(a[:, kv[0]]) if np.any(~np.isnan(a[:, kv[0]])) else 1e9):
        col = a[:, i]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"  {i:2d} {nm:18s} {col.min():9.2f} {np.median(col):9.2f} {col.max():9.2f}  (n={col.size})")
    eng.set_trace(False)

"""Dev: one batched (Qwen2-7B, 16 x 64K) miss launch for ncu (run with TS_DEBUG_FLAGS=512 to stop after the scan)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402

B, n, h, hkv, d = 16, 65536, 28, 4, 128
eng = sa.Engine(n + 64, k=2048, n_local=512, n_init=128, num_heads=h, num_kv_heads=hkv, head_dim=d, n_seqs=B)
for b in range(B):
    g = torch.Generator(device="cuda").manual_seed(b)
    K = (torch.randn(n, hkv * d, device="cuda", generator=g) * 3).to(torch.bfloat16)
    eng.append_bf16(K, K, b)
q = torch.randn(B, h * d, device="cuda")
kt = torch.randn(B, hkv * d, device="cuda")
out = torch.empty(B, h * d, device="cuda")
for s in range(B):
    eng.set_theta(2.0, s)
for _ in range(3):
    eng.decode_async(q, kt, kt, out)
eng.sync()

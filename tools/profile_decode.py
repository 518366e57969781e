"""Profiling driver (dev tool): 2 warm-up misses, then 1 miss step and 1 hit step
of the fused decode kernel at N tokens (Llama-3-8B layer). Run under ncu with
-k regex:decode_kernel -s 2 -c 2."""
import sys

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H, Hkv, d = 32, 8, 128
eng = sa.Engine(N + 64, k=2048, n_local=512, n_init=128, num_heads=H, num_kv_heads=Hkv, head_dim=d)
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn(N, Hkv * d, device="cuda", generator=g) * 3).to(torch.bfloat16)
V = torch.randn(N, Hkv * d, device="cuda", generator=g).to(torch.bfloat16)
eng.append_bf16(K, V)
del K, V
q = torch.randn(1, H * d, device="cuda", generator=g)
kt = torch.randn(1, Hkv * d, device="cuda", generator=g)
vt = torch.randn(1, Hkv * d, device="cuda", generator=g)
out = torch.empty(1, H * d, device="cuda")
eng.set_theta(2.0)  # theta > 1: every lookup misses
for _ in range(3):  # 2 warm-up misses + the profiled miss
    eng.decode_async(q, kt, vt, out)
eng.set_theta(-2.0)  # theta < -1: every lookup hits
eng.decode_async(q, kt, vt, out)  # the profiled hit
eng.sync()
print(eng.stats())

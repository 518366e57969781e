"""Host-side cost of one decode_async call (dev tool): Python ctypes vs the C-ABI."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402
from paper_2411_02886_b200._native import lib  # noqa: E402
import ctypes as C  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H, Hkv, d = 32, 8, 128
eng = sa.Engine(N + 4096, k=2048, n_local=512, n_init=128, num_heads=H, num_kv_heads=Hkv, head_dim=d)
K = torch.randn(N, Hkv * d, device="cuda").to(torch.bfloat16)
eng.append_bf16(K, K)
q = torch.randn(1, H * d, device="cuda")
kt = torch.randn(1, Hkv * d, device="cuda")
out = torch.empty(1, H * d, device="cuda")
eng.set_theta(-2.0)
args = [eng._h] + [C.c_void_p(t.data_ptr()) for t in (q, kt, kt, out)]
for _ in range(10):
    lib.ts_engine_decode_async(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000):
    lib.ts_engine_decode_async(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per call: {1e6 * (t1 - t0) / 1000:.2f} us; gpu drain {1e3 * (t2 - t1):.1f} ms")

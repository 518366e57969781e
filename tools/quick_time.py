"""Quick decode-step timing (dev tool): Llama-3-8B layer, N tokens, miss and hit steps."""
import sys
import time

import numpy as np
import torch

from paper_2411_02886_b200 import selattn as sa

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H, Hkv, d = 32, 8, 128
eng = sa.Engine(N + 256, k=2048, n_local=512, n_init=128, num_heads=H, num_kv_heads=Hkv, head_dim=d)
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn(N, Hkv * d, device="cuda", generator=g) * 3).to(torch.bfloat16)
V = torch.randn(N, Hkv * d, device="cuda", generator=g).to(torch.bfloat16)
eng.append_bf16(K, V)
q = torch.randn(1, H * d, device="cuda", generator=g)
kt = torch.randn(1, Hkv * d, device="cuda", generator=g)
vt = torch.randn(1, Hkv * d, device="cuda", generator=g)
out = torch.empty(1, H * d, device="cuda")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
for mode in ("miss", "hit"):
    ts = []
    for it in range(12):
        if mode == "miss":
            eng.force_miss()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        eng.decode_async(q, kt, vt, out)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    print(mode, "us/step median", np.median(ts[2:]), "min", min(ts[2:]), eng.stats())

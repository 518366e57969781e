"""Phase trace of the sharded decode's stats launch at world 1, 128K (dev tool):
why it is slower than the one-GPU step's scan."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_02886_b200 import selattn as sa  # noqa: E402
from paper_2411_02886_b200 import sharded  # noqa: E402
from paper_2411_02886_b200._native import lib, check  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H, Hkv, d = 32, 8, 128
os.environ.setdefault("TS_DEBUG_TMA", "1")
shard = sharded.NativeShard(0, 1, N + 64, k=2048, n_local=512, n_init=128, chunk_size=512, theta=2.0, num_heads=H,
                            num_kv_heads=Hkv, head_dim=d, block_size=64)
K = torch.randn(N, Hkv * d, device="cuda").to(torch.bfloat16).view(torch.uint16)
shard.append_bf16(K, K)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(H * d, device="cuda", generator=g)
kt = torch.randn(Hkv * d, device="cuda", generator=g)
check(lib.ts_engine_set_trace(shard._h, 1))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(4):
    torch.cuda.synchronize()
    ev[0].record()
    st = shard.stats(q, kt, kt, 0, N + i)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"stats launch {i}: {ev[0].elapsed_time(ev[1]) * 1000:.1f} us")
    cands = shard.select(st)
    part, ml = shard.attend(cands)
    torch.cuda.synchronize()
shard.TRACE_POINTS = sa.Engine.TRACE_POINTS
st = shard.stats(q, kt, kt, 0, N + 4)
torch.cuda.synchronize()
print("stats phase trace (us):", sa.Engine.read_trace(shard))
cands = shard.select(st)
torch.cuda.synchronize()
print("select phase trace (us):", sa.Engine.read_trace(shard))
part, ml = shard.attend(cands)
torch.cuda.synchronize()
print("attend phase trace (us):", sa.Engine.read_trace(shard))
for name, fn in (("select", lambda: shard.select(st)), ("attend", lambda: shard.attend(cands))):
    torch.cuda.synchronize()
    ev[0].record()
    fn()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{name} launch: {ev[0].elapsed_time(ev[1]) * 1000:.1f} us")

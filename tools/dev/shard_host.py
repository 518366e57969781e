"""Host time of one sharded decode step's calls at world 1 over NCCL (dev tool)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_02886_b200 import sharded  # noqa: E402

N = 131072
H, Hkv, d = 32, 8, 128
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29571", rank=0, world_size=1)
torch.cuda.set_device(0)
shard = sharded.NativeShard(0, 1, N + 4096, k=2048, n_local=512, n_init=128, chunk_size=512, theta=-2.0, num_heads=H,
                            num_kv_heads=Hkv, head_dim=d, block_size=64)
K = torch.randn(N, Hkv * d, device="cuda").to(torch.bfloat16).view(torch.uint16)
shard.append_bf16(K, K)
ex = sharded.TorchDistExchange()
if os.environ.get("FORCE_NCCL_GATHER"):  # time the NCCL all-gather even at world 1
    class _Ex(sharded.TorchDistExchange):
        def all_gather(self, t):
            w, self.world = self.world, 2
            try:
                out = torch.empty(t.numel(), dtype=t.dtype, device=t.device)
                self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
                return out
            finally:
                self.world = w
    ex = _Ex()
q = torch.randn(H * d, device="cuda")
kt = torch.randn(Hkv * d, device="cuda")
names = ["stats", "gather stats", "select", "gather cands", "attend", "gather partials", "combine"]
acc = [0.0] * len(names)
n = 0
for i in range(300):
    t = [time.perf_counter()]
    st = shard.stats(q, kt, kt, 0, N + i)
    t.append(time.perf_counter())
    a = ex.all_gather(st)
    t.append(time.perf_counter())
    c = shard.select(a)
    t.append(time.perf_counter())
    ac = ex.all_gather(c)
    t.append(time.perf_counter())
    pm = shard.attend_packed(ac)
    t.append(time.perf_counter())
    ap = ex.all_gather(pm)
    t.append(time.perf_counter())
    shard.combine_packed(ap)
    t.append(time.perf_counter())
    if i >= 50:
        n += 1
        for j in range(len(names)):
            acc[j] += t[j + 1] - t[j]
    if i % 10 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("host us per call (hit stream):", {k: round(1e6 * v / n, 1) for k, v in zip(names, acc)},
      "total", round(1e6 * sum(acc) / n, 1))
dist.destroy_process_group()

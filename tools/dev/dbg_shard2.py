import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from tests.helpers import bf16_round, rng_normal
from oracle.oracle import Oracle
from paper_2411_02886_b200 import sharded
from tests.test_gpu_sharded import global_selection
orc = Oracle("port")
world = 2
n, H, H_kv, d, k, n_init, n_local = 6000, 32, 8, 128, 256, 16, 64
K = bf16_round(rng_normal(11, (n, H_kv * d), 3.0)); V = bf16_round(rng_normal(12, (n, H_kv * d)))
kw = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
ranges = sharded.shard_ranges(n, world, n_init, n_local)
shards = []
for r in ranges:
    s = sharded.NativeShard(r.rank, world, r.length + 64, **kw)
    s.append(torch.from_numpy(K[r.base:r.base + r.length]).cuda(), torch.from_numpy(V[r.base:r.base + r.length]).cuda())
    shards.append(s)
g = np.random.default_rng(5)
base_q = g.standard_normal(H * d).astype(np.float32)
q = (base_q + 3.0 * g.standard_normal(H * d)).astype(np.float32).reshape(1, -1)
kt = bf16_round(rng_normal(700, (1, H_kv * d), 3.0)); vt = bf16_round(rng_normal(800, (1, H_kv * d)))
qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, kt, vt))
outs, all_cands = sharded.simulate_step(shards, [(qd, kd, vd)] * world, [r.base for r in ranges], n)
torch.cuda.synchronize()
a = all_cands.cpu().numpy().view(np.uint32).reshape(world, 2 * k + 1)
def key_float(kk):
    kk = np.asarray(kk, np.uint32)
    b = np.where(kk & 0x80000000, kk & 0x7fffffff, ~kk)
    return b.astype(np.uint32).view(np.float32)
cand = np.arange(n_init, n - n_local, dtype=np.uint32)
S = orc.score_paged(q.reshape(H, d), K, H_kv, cand)
crit = orc.criticality(S, k)
posmap = {int(t): i for i, t in enumerate(cand)}
for r in range(world):
    nn = a[r, 2*k]
    idx = a[r, :nn]; cr = key_float(a[r, k:k+nn])
    print("rank", r, "n", nn, "4119 in", 4119 in idx, "max ours", cr.max(), "n ours >0.5:", (cr > 0.5).sum())
    ref_hi = [t for t in range(ranges[r].base, ranges[r].base + ranges[r].length) if t in posmap and crit[posmap[t]] > 0.5]
    print("  oracle tokens with crit>0.5 in this range:", len(ref_hi), ref_hi[:10])
    print("  ours crit of those:", [float(cr[list(idx).index(t)]) if t in idx else None for t in ref_hi[:10]])
print("4119 oracle crit", crit[posmap[4119]], "S max head", S[:, posmap[4119]].max(), "per-head M", S.max(axis=1)[:4])

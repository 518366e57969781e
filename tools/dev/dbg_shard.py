import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from tests.helpers import bf16_round, rng_normal
from oracle.oracle import Oracle
from paper_2411_02886_b200 import sharded
from tests.test_gpu_sharded import global_selection
orc = Oracle("port")
n, H, H_kv, d, k, n_init, n_local = 6000, 32, 8, 128, 256, 16, 64
K = bf16_round(rng_normal(11, (n, H_kv * d), 3.0)); V = bf16_round(rng_normal(12, (n, H_kv * d)))
kw = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
for world in (1, 2):
    ranges = sharded.shard_ranges(n, world, n_init, n_local)
    shards = []
    for r in ranges:
        s = sharded.NativeShard(r.rank, world, r.length + 64, **kw)
        s.append(torch.from_numpy(K[r.base:r.base + r.length]).cuda(), torch.from_numpy(V[r.base:r.base + r.length]).cuda())
        shards.append(s)
    g = np.random.default_rng(5)
    q = (g.standard_normal(H * d) * 1.0).astype(np.float32).reshape(1, -1)
    kt = bf16_round(rng_normal(700, (1, H_kv * d), 3.0)); vt = bf16_round(rng_normal(800, (1, H_kv * d)))
    qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, kt, vt))
    stats = [s.stats(qd, kd, vd, r.base, n) for s, r in zip(shards, ranges)]
    all_stats = torch.cat(stats); torch.cuda.synchronize()
    print("world", world, "stats rank0 h0..2", all_stats[:6].cpu().numpy(), "last", all_stats[-6:].cpu().numpy())
    cands = [s.select(all_stats) for s in shards]
    all_cands = torch.cat(cands); torch.cuda.synchronize()
    a = all_cands.cpu().numpy().view(np.uint32).reshape(world, 2 * k + 1)
    for r in range(world):
        nn = a[r, 2*k]; print(" rank", r, "count", nn, "first idx", a[r, :5], "keys", [hex(x) for x in a[r, k:k+3]], "has4119", 4119 in a[r, :nn])
    cand = np.arange(n_init, n - n_local, dtype=np.uint32)
    S = orc.score_paged(q.reshape(H, d), K, H_kv, cand)
    crit = orc.criticality(S, k)
    top = np.argsort(-crit)[:5]
    print(" oracle top crit", cand[top], crit[top])
    # oracle per-head stats
    m = S.max(axis=1); z = np.exp(S - m[:, None]).sum(axis=1)
    print(" oracle M,Z h0..2", m[:3], z[:3])
    def key_float(kk):
        kk = np.asarray(kk, np.uint32)
        b = np.where(kk & 0x80000000, kk & 0x7fffffff, ~kk)
        return b.astype(np.uint32).view(np.float32)
    ours = []
    for r in range(world):
        nn = a[r, 2*k]; ours += list(zip(a[r, :nn], key_float(a[r, k:k+nn])))
    od = dict((int(i), float(c)) for i, c in ours)
    posmap = {int(t): i for i, t in enumerate(cand)}
    topk = set(int(cand[i]) for i in np.argsort(-crit, kind='stable')[:k])
    miss = [t for t in topk if t not in od]
    print(" missing from ours:", len(miss), [(t, crit[posmap[t]]) for t in sorted(miss, key=lambda t: -crit[posmap[t]])[:8]])
    print(" ours crit for oracle top:", [(int(t), od.get(int(t))) for t in cand[top]])

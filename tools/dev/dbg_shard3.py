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
ref = orc.engine(n + 64, **kw); ref.append(K, V)
ranges = sharded.shard_ranges(n, world, n_init, n_local)
shards = []
for r in ranges:
    s = sharded.NativeShard(r.rank, world, r.length + 64, **kw)
    s.append(torch.from_numpy(K[r.base:r.base + r.length]).cuda(), torch.from_numpy(V[r.base:r.base + r.length]).cuda())
    shards.append(s)
g = np.random.default_rng(5)
base_q = g.standard_normal(H * d).astype(np.float32)
for step in range(6):
    q = (base_q + (0.01 if step % 2 else 3.0) * g.standard_normal(H * d)).astype(np.float32).reshape(1, -1)
    if step % 2 == 0: base_q = q.ravel()
    kt = bf16_round(rng_normal(700 + step, (1, H_kv * d), 3.0)); vt = bf16_round(rng_normal(800 + step, (1, H_kv * d)))
    N = n + step
    o_ref, hit_ref, sel_ref = ref.decode(q, kt, vt)
    qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, kt, vt))
    stats = [s.stats(qd, kd, vd, r.base, N) for s, r in zip(shards, ranges)]
    torch.cuda.synchronize()
    import ctypes as C
    from paper_2411_02886_b200._native import lib
    for s in shards:
        a_, b_, c_, h_, cs_ = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_int(), C.c_double()
        rc = lib.ts_engine_stats(s._h, 0, C.byref(a_), C.byref(b_), C.byref(c_), C.byref(h_), C.byref(cs_))
        print(f"   rank {s.rank}: rc {rc} lookups {a_.value} hits {b_.value} len {c_.value} last_hit {h_.value} cos {cs_.value:.4f}")
    print("   stats nan:", [bool(torch.isnan(x).any()) for x in stats])
    all_stats = torch.cat(stats)
    cands = [s.select(all_stats) for s in shards]
    all_cands = torch.cat(cands)
    torch.cuda.synchronize()
    for s in shards:
        kk = 256
        sel_ = np.zeros(kk, np.uint32); cr_ = np.zeros(kk, np.float64); n_ = C.c_size_t()
        lib.ts_engine_cached_selection(s._h, 0, sel_.ctypes.data_as(C.c_void_p), cr_.ctypes.data_as(C.c_void_p), C.byref(n_))
        print(f"   cands count slot rank {s.rank}:", int(cands[s.rank][512].item()), "first", cands[s.rank][:3].tolist(), "keys", [hex(x & 0xffffffff) for x in cands[s.rank][256:259].tolist()])
        print(f"   after select rank {s.rank}: n_sel {n_.value} sel {sel_[:4]} crit {cr_[:4]} max crit {cr_[:n_.value].max() if n_.value else None}")
    parts = [s.attend(all_cands) for s in shards]
    torch.cuda.synchronize()
    sel = global_selection(all_cands, world, k, N, n_init, n_local)
    a = all_cands.cpu().numpy().view(np.uint32).reshape(world, 2 * k + 1)
    st = [sh.torch for sh in shards]
    d1 = set(sel.tolist()) - set(int(x) for x in sel_ref); d2 = set(int(x) for x in sel_ref) - set(sel.tolist())
    print(f"step {step} N {N} hit_ref {hit_ref} counts {[int(a[r, 2*k]) for r in range(world)]} ours-ref {sorted(d1)[:6]} ref-ours {sorted(d2)[:6]} 4119 in ref {4119 in set(int(x) for x in sel_ref)}")

"""Sharded decode (config 4) on one GPU: `world` shard engines of one sequence
in one process, exchanges by concatenation in rank order (the bytes NCCL
would deliver). Checked against the CPU oracle's unsharded decode_step:

* every rank's output is bit-identical (deterministic rank-order combines);
* Selection Cache decisions identical to the oracle;
* the global selection (recovered from the exchanged candidates exactly as
  the merge kernel ranks them) equals the oracle's except at criticality ties
  within 1e-4 relative + 1e-30 absolute;
* the output equals the oracle's sparse attention over that selection within
  rel. Frobenius 1e-5, max-abs 1e-4.
"""
import numpy as np
import pytest

from tests.helpers import bf16_round, check_selection, rng_normal

pytestmark = pytest.mark.gpu


def global_selection(all_cands, world, k, N, n_init, n_local):
    """The merge kernel's ranking (aux.cu shard_merge_kernel) on the host."""
    a = all_cands.cpu().numpy().view(np.uint32).reshape(world, 2 * k + 1)
    idx, key = [], []
    for r in range(world):
        n = int(a[r, 2 * k])
        idx.append(a[r, :n])
        key.append(a[r, k:k + n] >> 8)
    idx = np.concatenate(idx).astype(np.int64)
    key = np.concatenate(key).astype(np.int64)
    order = np.lexsort((idx, -key))[:k]
    sel = np.sort(idx[order])
    return sel


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decode_matches_oracle(world):
    import torch

    from oracle.oracle import Oracle
    from paper_2411_02886_b200 import sharded

    orc = Oracle("port")
    n, H, H_kv, d, k, n_init, n_local = 6000, 32, 8, 128, 256, 16, 64
    K = bf16_round(rng_normal(11, (n, H_kv * d), 3.0))
    V = bf16_round(rng_normal(12, (n, H_kv * d)))
    kw = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv,
              head_dim=d, block_size=64)
    ref = orc.engine(n + 64, **kw)
    ref.append(K, V)
    ranges = sharded.shard_ranges(n, world, n_init, n_local)
    shards = []
    for r in ranges:
        s = sharded.NativeShard(r.rank, world, r.length + 64, **kw)
        s.append(torch.from_numpy(K[r.base:r.base + r.length]).cuda(), torch.from_numpy(V[r.base:r.base + r.length]).cuda())
        shards.append(s)
    bases = [r.base for r in ranges]
    g = np.random.default_rng(5)
    base_q = g.standard_normal(H * d).astype(np.float32)
    hits = []
    q_sel = None  # the query the current selection was made with (the last miss)
    for step in range(6):
        q = (base_q + (0.01 if step % 2 else 3.0) * g.standard_normal(H * d)).astype(np.float32).reshape(1, -1)
        if step % 2 == 0:
            base_q = q.ravel()
        kt = bf16_round(rng_normal(700 + step, (1, H_kv * d), 3.0))
        vt = bf16_round(rng_normal(800 + step, (1, H_kv * d)))
        N = n + step
        o_ref, hit_ref, sel_ref = ref.decode(q, kt, vt)
        qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, kt, vt))
        outs, all_cands, all_packed = sharded.simulate_step(shards, [(qd, kd, vd)] * world, bases, N,
                                                            return_packed=True)
        torch.cuda.synchronize()
        # the two-array combine over the same blocks is the same merge
        blocks = all_packed.view(world, -1)
        two = shards[0].combine(blocks[:, : H * d].reshape(-1), blocks[:, H * d:].reshape(-1))
        assert torch.equal(two, outs[0]), "packed and two-array combines disagree"
        outs = [o.cpu().numpy() for o in outs]
        for o in outs[1:]:
            assert np.array_equal(o, outs[0]), "ranks disagree"
        sel = global_selection(all_cands, world, k, N, n_init, n_local)
        cand = np.arange(n_init, N - n_local, dtype=np.uint32)
        K_all = np.vstack([K] + [bf16_round(rng_normal(700 + s, (1, H_kv * d), 3.0)) for s in range(step)])
        V_all = np.vstack([V] + [bf16_round(rng_normal(800 + s, (1, H_kv * d))) for s in range(step)])
        if not hit_ref:
            q_sel, N_sel = q, N
        if not np.array_equal(sel, np.asarray(sel_ref, np.int64)):
            # ties are judged on the criticality the selection was made with
            cand_sel = np.arange(n_init, N_sel - n_local, dtype=np.uint32)
            S = orc.score_paged(q_sel.reshape(H, d), K_all[:N_sel], H_kv, cand_sel)
            check_selection(sel, sel_ref, orc.criticality(S, k), cand_sel)
        att = orc.make_windows(N, n_init, n_local, sel.astype(np.uint32))
        want = orc.sparse_attend(q, kt, vt, K_all[:N], V_all[:N], H, H_kv, att)
        err = np.linalg.norm(outs[0] - want) / np.linalg.norm(want)
        assert err <= 1e-5 and np.abs(outs[0] - want).max() <= 1e-4, (step, err)
        hits.append(hit_ref)
    assert any(hits) and not all(hits)


def test_shard_decode_step_native_world1_matches_oracle():
    """ts_shard_decode_step (the one-call in-library path the bench runs) at
    world 1: the four shard launches with their exchanges on the engine's
    stream, against the oracle's decode_step over a miss / hit stream."""
    import torch

    from oracle.oracle import Oracle
    from paper_2411_02886_b200 import sharded

    orc = Oracle("port")
    n, H, H_kv, d, k, n_init, n_local = 9000, 32, 8, 128, 512, 64, 128
    K = bf16_round(rng_normal(21, (n + 8, H_kv * d), 3.0))
    V = bf16_round(rng_normal(22, (n + 8, H_kv * d)))
    kw = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv,
              head_dim=d, block_size=64)
    ref = orc.engine(n + 64, **kw)
    ref.append(K[:n], V[:n])
    shard = sharded.NativeShard(0, 1, n + 64, **kw)
    shard.append(torch.from_numpy(K[:n]).cuda(), torch.from_numpy(V[:n]).cuda())
    comm = sharded.LibraryComm(0, 1)
    g = np.random.default_rng(23)
    base_q = g.standard_normal(H * d).astype(np.float32)
    hits = []
    for step in range(5):
        q = (base_q + (0.01 if step % 2 else 3.0) * g.standard_normal(H * d)).astype(np.float32).reshape(1, -1)
        if step % 2 == 0:
            base_q = q.ravel()
        kt, vt = K[n + step:n + step + 1], V[n + step:n + step + 1]
        o2, h2, s2 = ref.decode(q, kt, vt)
        qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).cuda().view(-1) for x in (q, kt, vt))
        o1 = sharded.decode_step_native(shard, comm, qd, kd, vd, 0, n + step).cpu().numpy()
        hits.append(h2)
        if step == 0 or not h2:
            q_sel, N_sel = q, n + step
        st = shard_stats(shard)
        assert st["last_hit"] == int(h2), (step, st, h2)
        cand = np.arange(n_init, N_sel - n_local, dtype=np.uint32)
        sel = np.asarray(shard_selection(shard), np.int64)
        want = o2
        if not np.array_equal(sel, np.asarray(s2, np.int64)):
            S = orc.score_paged(q_sel.reshape(H, d), K[:N_sel], H_kv, cand)
            check_selection(sel, s2, orc.criticality(S, k), cand)
            att = orc.make_windows(n + step, n_init, n_local, sel.astype(np.uint32))
            want = orc.sparse_attend(q, kt, vt, K[:n + step], V[:n + step], H, H_kv, att)
        err = np.linalg.norm(o1 - want) / np.linalg.norm(want)
        assert err <= 1e-5 and np.abs(o1 - want).max() <= 1e-4, (step, err)
    assert any(hits) and not all(hits)


def shard_stats(shard):
    import ctypes as C

    from paper_2411_02886_b200._native import check, lib

    a, b, c, h, cs = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_int(), C.c_double()
    check(lib.ts_engine_stats(shard._h, 0, C.byref(a), C.byref(b), C.byref(c), C.byref(h), C.byref(cs)))
    return {"lookups": a.value, "hits": b.value, "len": c.value, "last_hit": h.value}


def shard_selection(shard):
    import ctypes as C

    from paper_2411_02886_b200._native import check, lib

    sel = np.zeros(max(shard.k, 1), np.uint32)
    crit = np.zeros(max(shard.k, 1), np.float64)
    n = C.c_size_t()
    check(lib.ts_engine_cached_selection(shard._h, 0, sel.ctypes.data_as(C.c_void_p), crit.ctypes.data_as(C.c_void_p),
                                         C.byref(n)))
    return [int(x) for x in sel[: n.value]]

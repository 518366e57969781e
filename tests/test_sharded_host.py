"""Host-side logic of the sharded decode (config 4) on CPU, world_size 2 over
gloo: sharded.decode_step's call sequence and rank-order all-gathers, and
shard_ranges' layout rules.

The per-shard compute is a float64 numpy stand-in for the four native calls
(`NumpyShard`, test infrastructure only). It implements the same exchange
contract: (m, z) stats, local top-k (index, key, count), (o, M, L) partials.
The output of the two gloo processes must equal the CPU oracle's unsharded
decode_step. The native kernels behind the same protocol are checked on the
GPU in tests/test_gpu_sharded.py.
"""
import socket

import numpy as np
import pytest

from tests.helpers import bf16_round, rng_normal

N, H, H_KV, D, K, N_INIT, N_LOCAL = 700, 4, 2, 16, 24, 8, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpyShard:
    """float64 stand-in for one rank's ts_shard_* calls (same buffers)."""

    def __init__(self, rank, world, K_rows, V_rows, base):
        import torch

        self.torch = torch
        self.rank, self.world = rank, world
        self.K, self.V, self.base = K_rows.astype(np.float64), V_rows.astype(np.float64), base

    def stats(self, q, k, v, base, n_global):
        t = self.torch
        self.q = q.numpy().reshape(H, D).astype(np.float64)
        self.kt, self.vt = k.numpy().astype(np.float64), v.numpy().astype(np.float64)
        self.n_global = n_global
        n_r = self.K.shape[0]
        lo = N_INIT if self.rank == 0 else 0
        hi = n_r - N_LOCAL if self.rank == self.world - 1 else n_r
        self.cand = np.arange(lo, max(lo, hi))
        kh = self.K[self.cand].reshape(len(self.cand), H_KV, D)
        # h mod H_kv (selector.cpp:51), no 1/sqrt(d) (selector.cpp:59-63)
        self.S = np.stack([kh[:, h % H_KV, :] @ self.q[h] for h in range(H)]) if len(self.cand) else np.zeros((H, 0))
        m = self.S.max(axis=1) if len(self.cand) else np.full(H, -np.inf)
        z = np.exp(self.S - m[:, None]).sum(axis=1) if len(self.cand) else np.zeros(H)
        return t.tensor(np.stack([m, z], 1).ravel(), dtype=t.float64)

    def select(self, all_stats):
        t = self.torch
        st = all_stats.numpy().reshape(self.world, H, 2)
        M = st[:, :, 0].max(axis=0)
        Z = (st[:, :, 1] * np.exp(st[:, :, 0] - M)).sum(axis=0)
        crit = (np.exp(self.S - M[:, None]) / Z[:, None]).sum(axis=0)
        order = np.lexsort((self.cand, -crit))[:K]
        pick = np.sort(order)
        out = np.zeros(2 * K + 1)
        out[: len(pick)] = self.cand[pick] + self.base
        out[K:K + len(pick)] = crit[pick]
        out[2 * K] = len(pick)
        return t.tensor(out, dtype=t.float64)

    def attend(self, all_cands):
        t = self.torch
        a = all_cands.numpy().reshape(self.world, 2 * K + 1)
        idx = np.concatenate([a[r, : int(a[r, 2 * K])] for r in range(self.world)]).astype(np.int64)
        crit = np.concatenate([a[r, K:K + int(a[r, 2 * K])] for r in range(self.world)])
        sel = np.sort(idx[np.lexsort((idx, -crit))[:K]])
        Ng = self.n_global
        ie, lbs = min(N_INIT, Ng), max(Ng - min(N_LOCAL, Ng), min(N_INIT, Ng))
        rows = [i for i in range(ie)] + [int(s) for s in sel if ie <= s < lbs] + list(range(lbs, Ng))
        own = [r - self.base for r in rows if self.base <= r < self.base + self.K.shape[0]]
        keys = self.K[own].reshape(len(own), H_KV, D)
        vals = self.V[own].reshape(len(own), H_KV, D)
        last = self.rank == self.world - 1
        o = np.zeros((H, D))
        ml = np.zeros((H, 2))
        for h in range(H):
            s = keys[:, h % H_KV, :] @ self.q[h] / np.sqrt(D)
            vv = vals[:, h % H_KV, :]
            if last:
                s = np.append(s, self.kt.reshape(H_KV, D)[h % H_KV] @ self.q[h] / np.sqrt(D))
                vv = np.vstack([vv, self.vt.reshape(H_KV, D)[h % H_KV]])
            if len(s) == 0:
                ml[h] = (-np.inf, 0.0)
                continue
            m = s.max()
            w = np.exp(s - m)
            o[h] = w @ vv / w.sum()
            ml[h] = (m, w.sum())
        if last:
            self.K = np.vstack([self.K, self.kt])
            self.V = np.vstack([self.V, self.vt])
        return t.tensor(o.ravel(), dtype=t.float64), t.tensor(ml.ravel(), dtype=t.float64)

    def attend_packed(self, all_cands):
        o, ml = self.attend(all_cands)
        return self.torch.cat([o, ml])

    def combine_packed(self, all_packed):
        a = all_packed.reshape(self.world, H * D + 2 * H)
        return self.combine(a[:, : H * D].reshape(-1), a[:, H * D:].reshape(-1))

    def combine(self, all_part, all_ml):
        t = self.torch
        o = all_part.numpy().reshape(self.world, H, D)
        ml = all_ml.numpy().reshape(self.world, H, 2)
        M = ml[:, :, 0].max(axis=0)
        w = np.where(ml[:, :, 1] > 0, np.exp(ml[:, :, 0] - M) * ml[:, :, 1], 0.0)
        out = (w[:, :, None] * o).sum(axis=0) / w.sum(axis=0)[:, None]
        return t.tensor(out.reshape(1, -1))


def _data():
    K_all = bf16_round(rng_normal(3, (N + 8, H_KV * D), 2.0))
    V_all = bf16_round(rng_normal(4, (N + 8, H_KV * D)))
    q = rng_normal(5, (3, 1, H * D))
    return K_all, V_all, q


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    from paper_2411_02886_b200 import sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    K_all, V_all, qs = _data()
    r = sharded.shard_ranges(N, world, N_INIT, N_LOCAL)[rank]
    shard = NumpyShard(rank, world, K_all[r.base:r.base + r.length], V_all[r.base:r.base + r.length], r.base)
    ex = sharded.TorchDistExchange()
    outs = []
    for step in range(3):
        kt = torch.from_numpy(K_all[N + step:N + step + 1])
        vt = torch.from_numpy(V_all[N + step:N + step + 1])
        outs.append(sharded.decode_step(shard, ex, torch.from_numpy(qs[step]), kt, vt, r.base, N + step).numpy())
    np.save(out_path, np.array(outs))
    dist.destroy_process_group()


def test_shard_ranges_layout():
    from paper_2411_02886_b200 import sharded

    rs = sharded.shard_ranges(1000, 3, 128, 300)
    assert [(r.base, r.length) for r in rs] == [(0, 333), (333, 333), (666, 334)]
    assert sum(r.length for r in rs) == 1000
    with pytest.raises(ValueError):
        sharded.shard_ranges(1000, 4, 128, 512)  # last shard (250) cannot hold the local window
    with pytest.raises(ValueError):
        sharded.shard_ranges(200, 2, 128, 16)  # shard 0 (100) cannot hold the init window
    assert [(r.base, r.length) for r in sharded.shard_ranges(50, 1, 128, 512)] == [(0, 50)]


def test_sharded_decode_gloo_world2_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    from oracle.oracle import Oracle

    world, port = 2, _free_port()
    paths = [str(tmp_path / f"out{r}.npy") for r in range(world)]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, paths[r])) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    outs = [np.load(p) for p in paths]
    assert np.array_equal(outs[0], outs[1]), "ranks disagree"
    K_all, V_all, qs = _data()
    ref = Oracle("port").engine(N + 16, k=K, n_local=N_LOCAL, n_init=N_INIT, chunk_size=64, theta=2.0, num_heads=H,
                                num_kv_heads=H_KV, head_dim=D, block_size=8)  # theta > 1: every step selects
    ref.append(K_all[:N], V_all[:N])
    for step in range(3):
        want, hit, _ = ref.decode(qs[step], K_all[N + step:N + step + 1], V_all[N + step:N + step + 1])
        assert not hit
        err = np.linalg.norm(outs[0][step] - want) / np.linalg.norm(want)
        assert err <= 1e-5, (step, err)

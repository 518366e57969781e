"""Dev: chunk_size = 1 prefill row-1 mismatch -- variations."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.helpers import rng_normal, bf16_round
from oracle.oracle import Oracle
from paper_2411_02886_b200 import selattn as sa
import torch
orc = Oracle("port")
def run(H, H_kv, n, chunk, n_init, n_local, k, dev=False):
    d = 128
    kw = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=chunk, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
    q = rng_normal(71, (n, H * d)); kk = bf16_round(rng_normal(72, (n, H_kv * d))); vv = bf16_round(rng_normal(73, (n, H_kv * d)))
    e = sa.Engine(n + 4, **kw)
    if dev:
        got = e.prefill(torch.from_numpy(q).cuda(), torch.from_numpy(kk).cuda(), torch.from_numpy(vv).cuda())
        got = got.cpu().numpy() if hasattr(got, "cpu") else got
    else:
        got = e.prefill(q, kk, vv)
    want = orc.engine(n + 4, **kw).prefill(q, kk, vv)
    err = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-30)
    print(f"H{H}/{H_kv} n{n} chunk{chunk} init{n_init} local{n_local} k{k} dev{dev}: bad rows {np.nonzero(err > 1e-4)[0][:10]}")
run(8, 1, 4, 1, 16, 64, 256)
run(8, 1, 4, 1, 16, 64, 256, dev=True)
run(8, 1, 4, 1, 0, 64, 256)
run(8, 1, 4, 1, 16, 0, 256)
run(8, 2, 4, 1, 16, 64, 256)
run(32, 8, 4, 1, 16, 64, 256)
run(8, 1, 6, 2, 16, 64, 256)
run(8, 1, 6, 3, 16, 64, 256)

"""Dev: prefill over a pre-filled cache of n0 rows, chunk of C rows -- which (n0, C) mismatch the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.helpers import rng_normal, bf16_round
from oracle.oracle import Oracle
from paper_2411_02886_b200 import selattn as sa
orc = Oracle("port")
H, H_kv, d = 8, 1, 128
for n0, C in [(1, 1), (1, 4), (2, 1), (3, 1), (1, 2), (65, 1), (63, 1), (64, 1)]:
    kw = dict(k=256, n_local=64, n_init=16, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
    k0 = bf16_round(rng_normal(1, (n0, H_kv * d))); v0 = bf16_round(rng_normal(2, (n0, H_kv * d)))
    q = rng_normal(3, (C, H * d)); kk = bf16_round(rng_normal(4, (C, H_kv * d))); vv = bf16_round(rng_normal(5, (C, H_kv * d)))
    e = sa.Engine(n0 + C + 4, **kw); e.append(k0, v0)
    r = orc.engine(n0 + C + 4, **kw); r.append(k0, v0)
    got = e.prefill(q, kk, vv); want = r.prefill(q, kk, vv)
    err = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-30)
    print(f"n0 {n0} C {C}: max row err {err.max():.2e}, bad rows {np.nonzero(err > 1e-4)[0][:8]}")

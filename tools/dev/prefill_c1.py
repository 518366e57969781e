"""Dev: chunk_size = 1 prefill vs the oracle -- which rows differ, and their selections."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.helpers import rng_normal, bf16_round
from oracle.oracle import Oracle
from paper_2411_02886_b200 import selattn as sa
H, H_kv, d, n, chunk = 8, 1, 128, 700, int(sys.argv[1]) if len(sys.argv) > 1 else 1
kw = dict(k=256, n_local=64, n_init=16, chunk_size=chunk, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
q = rng_normal(71, (n, H * d))
kk = bf16_round(rng_normal(72, (n, H_kv * d)))
vv = bf16_round(rng_normal(73, (n, H_kv * d)))
got, tr1 = sa.Engine(n + 4, **kw).prefill(q, kk, vv, trace=True)
orc = Oracle("port")
want, tr2 = orc.engine(n + 4, **kw).prefill(q, kk, vv, trace=True)
err = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-30)
bad = np.nonzero(err > 1e-4)[0]
print("chunk", chunk, "bad rows", len(bad), bad[:20])
for r in bad[:3]:
    c = r // chunk
    a, b = list(tr1[c]), [int(x) for x in tr2[c]]
    print("row", r, "chunk", c, "err", err[r], "sel len", len(a), len(b), "sel equal", a == b,
          "diff", sorted(set(a) ^ set(b))[:10])
if chunk == 1:
    G = H // H_kv
    g1 = got[1].reshape(H, d); w1 = want[1].reshape(H, d)
    v0 = vv[0].reshape(H_kv, d); v1 = vv[1].reshape(H_kv, d)
    print("got[1] head0 ~ v1?", np.abs(g1[0] - v1[0]).max(), " ~ v0?", np.abs(g1[0] - v0[0]).max(), " want-v1", np.abs(w1[0] - v1[0]).max())
    # the oracle's own attention over {0, 1}
    import math
    qh = q[1].reshape(H, d)[0]; k0 = kk[0].reshape(H_kv, d)[0]; k1 = kk[1].reshape(H_kv, d)[0]
    s0, s1 = qh @ k0 / math.sqrt(d), qh @ k1 / math.sqrt(d)
    m = max(s0, s1); e0, e1 = math.exp(s0 - m), math.exp(s1 - m)
    manual = (e0 * v0[0] + e1 * v1[0]) / (e0 + e1)
    print("manual vs want", np.abs(manual - w1[0]).max(), "manual vs got", np.abs(manual - g1[0]).max())
    for r in range(0, 6):
        print("row", r, "err", err[r])

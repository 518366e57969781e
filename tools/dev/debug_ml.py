"""Dev: isolate the multi-layer selection mismatch (general kernel, H_kv=2 rows)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.helpers import bf16_round, rng_normal
from oracle.oracle import Oracle
from paper_2411_02886_b200 import selattn as sa

orc = Oracle("port")
H, H_kv, d, n, k = 8, 2, 128, 3000, 128
kw = dict(k=k, n_local=64, n_init=16, chunk_size=512, theta=0.9, num_heads=H, num_kv_heads=H_kv, head_dim=d,
          block_size=64)
cand = np.arange(16, n - 64, dtype=np.uint32)


def run(L, B, tag):
    eng = sa.Engine(n + 16, n_seqs=B, n_layers=L, **kw)
    data = {}
    g = np.random.default_rng(5)
    for l in range(L):
        eng.set_layer(l)
        for b in range(B):
            K = bf16_round(rng_normal(1000 + 10 * l + b, (n, H_kv * d), 3.0))
            V = bf16_round(rng_normal(2000 + 10 * l + b, (n, H_kv * d)))
            eng.append(K, V, b)
            data[l, b] = K
    qs = {key: g.standard_normal(H * d).astype(np.float32) for key in data}
    bad = 0
    for l in range(L):
        eng.set_layer(l)
        q = np.stack([qs[l, b] for b in range(B)])
        kt = bf16_round(rng_normal(300 + l, (B, H_kv * d), 3.0))
        vt = bf16_round(rng_normal(400 + l, (B, H_kv * d)))
        o, h, s = eng.decode(q, kt, vt)
        if B == 1:
            s = [s]
        for b in range(B):
            S = orc.score_paged(qs[l, b].reshape(H, d), data[l, b], H_kv, cand)
            want, _ = orc.select(S, cand, k)
            diff = set(s[b]) ^ set(int(x) for x in want)
            if diff:
                bad += 1
            print(tag, "layer", l, "seq", b, "diff", len(diff))
    return bad


print("TS_NO_TMA", os.environ.get("TS_NO_TMA"))
run(1, 2, "single-layer B=2")
run(3, 1, "3 layers B=1")
run(3, 2, "3 layers B=2")

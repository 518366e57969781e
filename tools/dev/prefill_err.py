"""Dev: output error of the 128K prefill chunk (configs[4]) vs the oracle, for
the current prefill kernel (run twice: default, TS_PREFILL_MMA_SYNC=1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.test_gpu_configs import kv_rows, append_chunked, rel_fro, L_H, L_HKV, D, K_SEL, N_INIT, N_LOCAL
from tests.helpers import rng_normal
from oracle.oracle import Oracle
from paper_2411_02886_b200 import selattn as sa

n, C = int(sys.argv[1]) if len(sys.argv) > 1 else 131072, 512
orc = Oracle("port")
K, V = kv_rows(5050, n + C, L_HKV * D)
kw = dict(k=K_SEL, n_local=N_LOCAL, n_init=N_INIT, chunk_size=C, theta=0.9, num_heads=L_H, num_kv_heads=L_HKV,
          head_dim=D, block_size=64)
eng = sa.Engine(n + C + 16, **kw)
ref = orc.engine(n + C + 16, **kw)
append_chunked(eng.append, K[:n], V[:n])
append_chunked(ref.append, K[:n], V[:n])
q = rng_normal(5051, (C, L_H * D))
got, tr1 = eng.prefill(q, K[n:], V[n:], trace=True)
want, tr2 = ref.prefill(q, K[n:], V[n:], trace=True)
print(os.environ.get("TS_PREFILL_MMA_SYNC") and "mma.sync" or "tcgen05", "sel equal", list(tr1[0]) == [int(x) for x in tr2[0]],
      "rel_fro %.3e" % rel_fro(got, want), "max abs %.3e" % np.abs(got - want).max())

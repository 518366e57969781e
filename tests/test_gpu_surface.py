"""The reference Python module's surface (proj/python/bindings.cpp:60-116) on
the device: softmax_rows, topk_indices, cosine, chunk_mean, sdpa_full -- the
checks of the reference's own smoke test (proj/tests/python/smoke_test.py:8-101)
plus oracle parity on random inputs.

Deviation: the pool stores bf16, so the smoke test's pool /
scoring / engine checks are run here on bf16-representable K/V (the
reference's fp32 pool round-trips any fp32 value).

Tolerances: softmax_rows and sdpa_full are fp64 on both sides -> rel 1e-6;
topk_indices exact; cosine within 1e-12 (fp64 summation order); chunk_mean
bit-exact (fp64 column sums in row order, like the reference).
"""
import numpy as np
import pytest

from tests.helpers import bf16_round

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sa():
    from paper_2411_02886_b200 import selattn

    return selattn


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle

    return Oracle("port")


# --- smoke_test.py:8-23, 25-28
def test_softmax_rows_smoke(sa):
    m = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 3.0]], dtype=np.float32)
    p = sa.softmax_rows(m)
    assert p.shape == (2, 3)
    assert np.allclose(p.sum(axis=1), 1.0, atol=1e-6)
    assert np.allclose(p[0], 1.0 / 3.0, atol=1e-6)


def test_topk_ties_and_order_smoke(sa):
    assert sa.topk_indices(np.array([5.0, 1.0, 9.0]), 2) == [0, 2]
    assert sa.topk_indices(np.array([7.0, 7.0, 7.0]), 2) == [0, 1]


def test_cosine_smoke(sa):
    v = np.array([1.0, 2.0, -3.0])
    assert sa.cosine(v, v) == 1.0
    assert abs(sa.cosine(np.array([1.0, 0.0]), np.array([0.0, 1.0]))) < 1e-12
    with pytest.raises(ValueError, match="zero-norm"):
        sa.cosine(np.zeros(3), v)


def test_topk_errors(sa):
    with pytest.raises(ValueError, match="empty"):
        sa.topk_indices(np.zeros(0), 2)
    with pytest.raises(ValueError, match="k must be"):
        sa.topk_indices(np.ones(3), 0)


# --- oracle parity on random inputs
@pytest.mark.parametrize("rows,cols,scale", [(1, 1, 1.0), (3, 1000, 5.0), (32, 20000, 30.0)])
def test_softmax_rows_vs_oracle(sa, orc, rows, cols, scale):
    m = (np.random.default_rng(cols).standard_normal((rows, cols)) * scale).astype(np.float32)
    got = sa.softmax_rows(m)
    want = orc.softmax_rows(m)
    assert np.all(np.abs(got - want) <= 1e-6 * np.abs(want) + 1e-37)


@pytest.mark.parametrize("n,k", [(1, 1), (10, 3), (1000, 100), (130000, 2048), (500, 600)])
def test_topk_vs_oracle(sa, orc, n, k):
    g = np.random.default_rng(n + k)
    s = g.standard_normal(n)
    s[::7] = s[0]  # exact ties
    assert sa.topk_indices(s, k) == [int(x) for x in orc.topk_indices(s, k)]


def test_cosine_vs_oracle(sa, orc):
    g = np.random.default_rng(5)
    for n in (1, 7, 4096, 100000):
        # fp32 inputs: the oracle restates the fp32 instantiation (the Selection
        # Cache's, tensor.cpp:92-113); ours reads them as exact doubles
        u, v = g.standard_normal(n).astype(np.float32), g.standard_normal(n).astype(np.float32)
        assert abs(sa.cosine(u, v) - orc.cosine(u, v)) <= 1e-12
        w = (-2.5 * u).astype(np.float32)
        assert abs(sa.cosine(u, w) - orc.cosine(u, w)) <= 1e-12


@pytest.mark.parametrize("c,w", [(1, 64), (7, 4096), (512, 4096), (700, 4096), (300, 37), (257, 100)])
def test_chunk_mean_vs_oracle(sa, orc, c, w):
    q = np.random.default_rng(c).standard_normal((c, w)).astype(np.float32)
    assert np.array_equal(sa.chunk_mean(q), orc.chunk_mean(q))


@pytest.mark.parametrize("C,N,H,H_kv,d", [(1, 1, 1, 1, 4), (3, 50, 4, 2, 8), (16, 300, 8, 2, 32), (1, 2000, 32, 8, 128)])
def test_sdpa_full_vs_oracle(sa, orc, C, N, H, H_kv, d):
    g = np.random.default_rng(N)
    q = g.standard_normal((C, H * d)).astype(np.float32)
    k = g.standard_normal((N, H_kv * d)).astype(np.float32)
    v = g.standard_normal((N, H_kv * d)).astype(np.float32)
    got = sa.sdpa_full(q, k, v, H)
    want = orc.sdpa_full(q, k, v, H)
    assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)


# --- smoke_test.py:43-101 on bf16-representable K/V (the pool stores bf16)
def test_score_and_select_smoke(sa):
    rng = np.random.default_rng(1)
    pool = sa.PagedKvPool(32, 1, 1, 8)
    seq = pool.create_sequence()
    k = bf16_round(rng.standard_normal((16, 8), dtype=np.float32))
    v = bf16_round(rng.standard_normal((16, 8), dtype=np.float32))
    pool.append_kv(seq, k, v)
    q = rng.standard_normal((2, 8), dtype=np.float32)
    scores, candidates = sa.score_paged(q, pool, seq, list(range(16)), block_size=4)
    assert scores.shape == (2, 16)
    assert np.allclose(scores, q.astype(np.float64) @ k.astype(np.float64).T, atol=1e-4)
    selected, criticality = sa.select(scores, candidates, 4, "head_soft_vote")
    assert len(selected) == 4 and sorted(selected) == list(selected) and len(criticality) == 4


def test_engine_select_all_matches_full_attention_smoke(sa):
    rng = np.random.default_rng(2)
    n = 48
    q = rng.standard_normal((n, 16), dtype=np.float32)
    k = bf16_round(rng.standard_normal((n, 16), dtype=np.float32))
    v = bf16_round(rng.standard_normal((n, 16), dtype=np.float32))
    engine = sa.Engine(n + 8, k=n, n_local=4, n_init=4, chunk_size=16, num_heads=2, num_kv_heads=2, head_dim=8,
                       block_size=8)
    sparse = engine.prefill(q, k, v)
    full = sa.sdpa_full(q, k, v, 2)
    assert np.linalg.norm(full - sparse) / np.linalg.norm(full) <= 1e-5
    assert len(engine) == n


def test_engine_decode_cache_smoke(sa):
    rng = np.random.default_rng(3)
    n = 64
    engine = sa.Engine(n + 16, k=8, n_local=8, n_init=4, chunk_size=32, num_heads=1, num_kv_heads=1, head_dim=8,
                       block_size=8, theta=0.9)
    engine.prefill(rng.standard_normal((n, 8), dtype=np.float32),
                   bf16_round(rng.standard_normal((n, 8), dtype=np.float32)),
                   bf16_round(rng.standard_normal((n, 8), dtype=np.float32)))
    q = rng.standard_normal((1, 8), dtype=np.float32)
    kt = rng.standard_normal((1, 8), dtype=np.float32)
    vt = rng.standard_normal((1, 8), dtype=np.float32)
    out1, hit1, sel1 = engine.decode(q, kt, vt)
    out2, hit2, sel2 = engine.decode(q, kt, vt)
    assert not hit1 and hit2 and sel1 == sel2 and out1.shape == (1, 8) and engine.cache_hits == 1


def test_prefill_async_matches_prefill(sa):
    """ts_engine_prefill_async (stream-ordered, device buffers) computes what
    the synchronous ts_engine_prefill does: same outputs, same pool state."""
    import torch

    rng = np.random.default_rng(11)
    H, H_kv, d, n0, n = 8, 2, 128, 3000, 700
    kw = dict(k=256, n_local=64, n_init=16, chunk_size=256, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
    k0 = bf16_round(rng.standard_normal((n0, H_kv * d), dtype=np.float32))
    v0 = bf16_round(rng.standard_normal((n0, H_kv * d), dtype=np.float32))
    q = rng.standard_normal((n, H * d), dtype=np.float32)
    k = rng.standard_normal((n, H_kv * d), dtype=np.float32)
    v = rng.standard_normal((n, H_kv * d), dtype=np.float32)
    a = sa.Engine(n0 + n + 8, **kw)
    b = sa.Engine(n0 + n + 8, **kw)
    for e in (a, b):
        e.append(k0, v0)
    want = a.prefill(q, k, v)
    out = torch.empty(n, H * d, device="cuda")
    b.prefill_async(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), out)
    b.sync()
    assert np.array_equal(out.cpu().numpy(), want)
    assert len(a) == len(b) == n0 + n
    with pytest.raises(ValueError):
        b.prefill_async(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v), out)


def test_prefill_pinned_host_buffers(sa):
    """Host-buffer prefill over several chunks (the chunk K/V copies run on
    the engine's copy stream, overlapping the selection): pinned and pageable
    inputs, a caller-provided pinned output, all equal to the device-buffer
    path; a wrongly shaped `out` is rejected."""
    import torch

    rng = np.random.default_rng(12)
    H, H_kv, d, n0, n = 8, 2, 128, 3000, 700
    kw = dict(k=256, n_local=64, n_init=16, chunk_size=256, num_heads=H, num_kv_heads=H_kv, head_dim=d, block_size=64)
    k0 = bf16_round(rng.standard_normal((n0, H_kv * d), dtype=np.float32))
    v0 = bf16_round(rng.standard_normal((n0, H_kv * d), dtype=np.float32))
    q = rng.standard_normal((n, H * d), dtype=np.float32)
    k = rng.standard_normal((n, H_kv * d), dtype=np.float32)
    v = rng.standard_normal((n, H_kv * d), dtype=np.float32)
    engines = [sa.Engine(n0 + n + 8, **kw) for _ in range(3)]
    for e in engines:
        e.append(k0, v0)
    dev_out = torch.empty(n, H * d, device="cuda")
    engines[0].prefill_async(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), dev_out)
    engines[0].sync()
    want = dev_out.cpu().numpy()
    pin = lambda x: torch.from_numpy(x).pin_memory().numpy()  # noqa: E731
    out = torch.empty(n, H * d).pin_memory().numpy()
    got = engines[1].prefill(pin(q), pin(k), pin(v), out=out)
    assert got is out and np.array_equal(out, want)
    assert np.array_equal(engines[2].prefill(q, k, v), want)
    with pytest.raises(ValueError):
        engines[2].prefill(q, k, v, out=np.empty((n, H * d + 1), np.float32))

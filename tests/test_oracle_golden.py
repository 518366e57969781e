"""Pins the CPU oracle (oracle/tsoracle.c, "port") to the reference.

1. against the golden fixtures in tests/golden/*.npz — outputs of the UNMODIFIED
   reference sources (tests/golden/make_golden.py), committed so this runs
   anywhere: bit-identical for every array (the port uses the reference's loop
   order and fp64 accumulation, compiled without FMA contraction);
2. against oracle/_ref (the reference library compiled from /root/reference)
   on fresh random inputs, when that library is present.

CPU only: no GPU, no product code.
"""
import hashlib
import os

import numpy as np
import pytest

from tests.helpers import bf16_round, rng_normal

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
METHODS = ("topk", "head_vote", "head_soft_vote")


@pytest.fixture(scope="module")
def port():
    from oracle.oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref (reference built from /root/reference) not present")
    return Oracle("reference")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


# ------------------------------------------------------------ golden vectors
def test_golden_score_bit_exact(port):
    g = load("score")
    for i in range(int(g["n"])):
        H, H_kv, d, n, ps, sh, blk = (int(x) for x in g[f"c{i}_meta"])
        got = port.score_paged(g[f"c{i}_q"], g[f"c{i}_k"], H_kv, g[f"c{i}_cand"])
        # page_size / shuffle / block_size of the reference run do not change S
        assert np.array_equal(got, g[f"c{i}_S"]), f"case {i}"


@pytest.mark.parametrize("method", METHODS)
def test_golden_select_bit_exact(port, method):
    g = load("select")
    for i in range(int(g["n"])):
        sel, crit = port.select(g[f"c{i}_S"], g[f"c{i}_cand"], int(g[f"c{i}_k"]), method)
        assert np.array_equal(sel, g[f"c{i}_{method}_sel"]), f"case {i}"
        assert np.array_equal(crit, g[f"c{i}_{method}_crit"]), f"case {i}"


def test_golden_known_answers_in_fixtures():
    # test_selector.cpp:128-141 / acceptance.cpp:155-169: raw sum -> {2,3}, soft vote -> {0,2}
    g = load("select")
    cand = g["c0_cand"]
    assert [int(cand.tolist().index(x)) for x in g["c0_topk_sel"]] == [2, 3]
    assert [int(cand.tolist().index(x)) for x in g["c0_head_soft_vote_sel"]] == [0, 2]
    # uniform -> {0,1}, crit = H/T (test_selector.cpp:215-221)
    assert [int(cand.tolist().index(x)) for x in g["c1_head_soft_vote_sel"]] == [0, 1]
    assert np.allclose(g["c1_head_soft_vote_crit"], 3 / 5, rtol=1e-6)


def test_golden_primitives(port):
    g = load("primitives")
    for i in range(3):
        assert np.array_equal(port.topk_indices(g[f"topk{i}_s"], int(g[f"topk{i}_k"])), g[f"topk{i}_out"])
    assert g["topk0_out"].tolist() == [0, 2] and g["topk1_out"].tolist() == [0, 1]  # test_tensor.cpp:102-112
    for i in range(4):
        assert port.cosine(g[f"cos{i}_u"], g[f"cos{i}_v"]) == float(g[f"cos{i}_out"])
    assert float(g["cos1_out"]) == 1.0 and float(g["cos2_out"]) == -1.0  # exact +-1 clamp (tensor.cpp:108)
    assert np.array_equal(port.softmax_rows(g["softmax_in"]), g["softmax_out"])
    assert np.array_equal(port.chunk_mean(g["cmean_in"]), g["cmean_out"])
    for i in range(5):
        cached, ni, nl = (int(x) for x in g[f"win{i}_args"])
        assert np.array_equal(port.make_windows(cached, ni, nl, g[f"win{i}_sel"]), g[f"win{i}_merged"]), i
    # test_attention.cpp:238-252
    assert g["win1_merged"].tolist() == list(range(6))


def test_golden_sdpa(port):
    g = load("attention")
    for i in range(int(g["n"])):
        got = port.sdpa_full(g[f"c{i}_q"], g[f"c{i}_k"], g[f"c{i}_v"], int(g[f"c{i}_H"]))
        assert np.array_equal(got, g[f"c{i}_out"]), f"case {i}"


def engine_kv(i, n, H_kv, d):
    # tests/golden/make_golden.py:engine_kv
    return (bf16_round(rng_normal(70 + i, (n, H_kv * d), 3.0)), bf16_round(rng_normal(80 + i, (n, H_kv * d))))


def golden_decode_case(g, i):
    n, H, H_kv, d, k, n_init, n_local, method = (int(x) for x in g[f"d{i}_cfg"])
    K, V = engine_kv(i, n, H_kv, d)
    assert hashlib.sha256(K.tobytes() + V.tobytes()).hexdigest() == str(g[f"d{i}_kv_sha"]), \
        "regenerated K/V differ from the fixture's inputs"
    cfg = dict(k=k, n_local=n_local, n_init=n_init, chunk_size=64, theta=float(g[f"d{i}_theta"]), num_heads=H,
               num_kv_heads=H_kv, head_dim=d, block_size=64, selection_method=METHODS[method])
    return n, K, V, cfg


def test_golden_decode_stream(port):
    g = load("engine")
    for i in range(int(g["nd"])):
        n, K, V, cfg = golden_decode_case(g, i)
        eng = port.engine(n + 64, **cfg)
        eng.append(K, V)
        for s in range(len(g[f"d{i}_q"])):
            o, hit, sel = eng.decode(g[f"d{i}_q"][s].reshape(1, -1), g[f"d{i}_kt"][s:s + 1], g[f"d{i}_vt"][s:s + 1])
            assert hit == bool(g[f"d{i}_hit"][s]), (i, s)
            want = g[f"d{i}_sel"][s]
            assert np.array_equal(sel, want[want != 0xFFFFFFFF]), (i, s)
            assert np.array_equal(o[0], g[f"d{i}_out"][s]), (i, s)
        assert any(g[f"d{i}_hit"]) and not all(g[f"d{i}_hit"])


def test_golden_prefill(port):
    g = load("engine")
    for i in range(int(g["np"])):
        n, H, H_kv, d, chunk, k, n_init, n_local = (int(x) for x in g[f"p{i}_cfg"])
        eng = port.engine(n + 4, k=k, n_local=n_local, n_init=n_init, chunk_size=chunk, theta=0.9, num_heads=H,
                          num_kv_heads=H_kv, head_dim=d, block_size=8)
        o, trace = eng.prefill(g[f"p{i}_q"], g[f"p{i}_K"], g[f"p{i}_V"], trace=True)
        assert np.array_equal(o, g[f"p{i}_out"])
        assert [len(t) for t in trace] == g[f"p{i}_counts"].tolist()
        assert np.array_equal(np.concatenate(trace) if trace else np.zeros(0, np.uint32), g[f"p{i}_trace"])


# ------------------------------------------------- port vs live reference
@pytest.mark.parametrize("seed", range(6))
def test_port_vs_reference_random(port, ref, seed):
    rng = np.random.default_rng(seed)
    H_kv = int(rng.integers(1, 5))
    H = H_kv * int(rng.integers(1, 5))
    d = int(rng.choice([4, 8, 16, 64, 128]))
    n = int(rng.integers(5, 400))
    k = bf16_round(rng_normal(seed, (n, H_kv * d), 3.0))
    q = rng_normal(seed + 100, (H, d))
    cand = np.sort(rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False)).astype(np.uint32)
    S = port.score_paged(q, k, H_kv, cand)
    for ps, sh, blk in ((1, 0, 64), (3, seed + 1, 1), (2, 7, int(cand.size))):
        assert np.array_equal(S, ref.score_paged(q, k, H_kv, cand, block_size=blk, page_size=ps, shuffle_seed=sh))
    kk = int(rng.integers(1, cand.size + 3))
    for m in METHODS:
        a = port.select(S, cand, kk, m)
        b = ref.select(S, cand, kk, m)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), m


def test_port_vs_reference_decode_and_prefill(port, ref):
    H, H_kv, d, n = 8, 4, 32, 700
    K = bf16_round(rng_normal(1, (n, H_kv * d), 3.0))
    V = bf16_round(rng_normal(2, (n, H_kv * d)))
    cfg = dict(k=64, n_local=32, n_init=16, chunk_size=128, theta=0.8, num_heads=H, num_kv_heads=H_kv,
               head_dim=d, block_size=16)
    a, b = port.engine(n + 16, **cfg), ref.engine(n + 16, **cfg)
    oa = a.prefill(rng_normal(3, (n, H * d)), K, V)
    ob = b.prefill(rng_normal(3, (n, H * d)), K, V)
    assert np.array_equal(oa, ob)
    g = np.random.default_rng(4)
    base = g.standard_normal(H * d).astype(np.float32)
    for s in range(6):
        q = (base + (0.05 if s % 2 else 1.5) * g.standard_normal(H * d)).astype(np.float32).reshape(1, -1)
        kt, vt = rng_normal(10 + s, (1, H_kv * d)), rng_normal(20 + s, (1, H_kv * d))
        x, y = a.decode(q, kt, vt), b.decode(q, kt, vt)
        assert np.array_equal(x[0], y[0]) and x[1] == y[1] and np.array_equal(x[2], y[2]), s
    assert a.stats() == b.stats()


def test_error_contract_matches_reference(port, ref):
    # score_paged: H not a multiple of H_kv -> invalid_argument; bad index -> out_of_range
    from oracle.oracle import OracleError

    k = rng_normal(1, (8, 8))
    for o in (port, ref):
        with pytest.raises(OracleError) as e:
            o.score_paged(rng_normal(2, (3, 4)), k, 2, np.array([0], np.uint32))
        assert e.value.code == 1
        with pytest.raises(OracleError) as e:
            o.score_paged(rng_normal(2, (2, 4)), k, 2, np.array([1, 9], np.uint32))
        assert e.value.code == 2

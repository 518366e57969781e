"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end to the CPU oracle.

Two interchangeable back ends with one API:

* ``Oracle("port")``      -> oracle/_build/libtsoracle.so, the plain-C restatement
  (oracle/tsoracle.c) of the reference's decode selection + sparse attention.
* ``Oracle("reference")`` -> oracle/_ref/libselattn_ref.so, the UNMODIFIED
  reference sources (/root/reference/proj/src) behind oracle/ref_shim.cpp.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libtsoracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libselattn_ref.so")

METHODS = {"topk": 0, "head_vote": 1, "head_soft_vote": 2}

_sz = C.c_size_t
_p = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def build():
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a):
    return a.ctypes.data_as(_p)


class Oracle:
    """Same calls on either back end; arrays are numpy, results numpy."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.pre = "oc_" if kind == "port" else "ref_"
        err = getattr(self.lib, self.pre + "last_error")
        err.restype = C.c_char_p
        self._err = err
        if kind == "port":
            self.lib.oc_make_windows.restype = _sz
            self.lib.oc_selection_candidates.restype = _sz

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # ------------------------------------------------------------- scoring
    def score_paged(self, q, k_rows, H_kv, cand, block_size=64, page_size=1, shuffle_seed=0):
        q = _f32(q)
        H, d = q.shape
        k_rows = _f32(k_rows)
        cand = _u32(cand)
        T = cand.size
        out = np.zeros((H, T), np.float32)
        if self.kind == "port":
            self._check(self._fn("score")(_ptr(q), _sz(H), _sz(d), _ptr(k_rows), _sz(k_rows.shape[0]),
                                          _sz(H_kv), _ptr(cand), _sz(T), _ptr(out)))
        else:
            self._check(self._fn("score_paged")(_ptr(q), _sz(H), _sz(d), _ptr(k_rows),
                                                _sz(k_rows.shape[0]), _sz(H_kv), _sz(page_size),
                                                C.c_uint64(shuffle_seed), _ptr(cand), _sz(T),
                                                _sz(block_size), _ptr(out)))
        return out

    def select(self, per_head, cand, k, method="head_soft_vote"):
        per_head = _f32(per_head)
        H, T = per_head.shape
        cand = _u32(cand)
        sel = np.zeros(max(T, 1), np.uint32)
        crit = np.zeros(max(T, 1), np.float64)
        n = _sz(0)
        self._check(self._fn("select")(_ptr(per_head), _sz(H), _sz(T), _ptr(cand), _sz(k),
                                       C.c_int(METHODS[method]), _ptr(sel), _ptr(crit), C.byref(n)))
        return sel[: n.value].copy(), crit[: n.value].copy()

    def criticality(self, per_head, k, method="head_soft_vote"):
        assert self.kind == "port"
        per_head = _f32(per_head)
        H, T = per_head.shape
        crit = np.zeros(max(T, 1), np.float64)
        self._check(self._fn("criticality")(_ptr(per_head), _sz(H), _sz(T), _sz(k),
                                            C.c_int(METHODS[method]), _ptr(crit)))
        return crit[:T]

    def topk_indices(self, scores, k):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        out = np.zeros(max(s.size, 1), np.uint32)
        n = _sz(0)
        name = "topk_indices_f64" if self.kind == "port" else "topk_indices"
        self._check(self._fn(name)(_ptr(s), _sz(s.size), _sz(k), _ptr(out), C.byref(n)))
        return out[: n.value].copy()

    def cosine(self, u, v):
        u, v = _f32(u).ravel(), _f32(v).ravel()
        out = C.c_double(0)
        self._check(self._fn("cosine_f32")(_ptr(u), _ptr(v), _sz(u.size), C.byref(out)))
        return out.value

    def softmax_rows(self, m):
        m = _f32(m)
        out = np.zeros_like(m)
        fn = self._fn("softmax_rows")
        r = fn(_ptr(m), _sz(m.shape[0]), _sz(m.shape[1]), _ptr(out))
        if self.kind == "reference":
            self._check(r)
        return out

    def chunk_mean(self, q):
        q = _f32(q)
        out = np.zeros(q.shape[1], np.float32)
        self._check(self._fn("chunk_mean")(_ptr(q), _sz(q.shape[0]), _sz(q.shape[1]), _ptr(out)))
        return out

    def make_windows(self, cached, n_init, n_local, selected):
        sel = _u32(selected)
        merged = np.zeros(cached + sel.size + 1, np.uint32)
        if self.kind == "port":
            kept = _sz(0)
            n = self._fn("make_windows")(_sz(cached), _sz(n_init), _sz(n_local), _ptr(sel),
                                         _sz(sel.size), _ptr(merged), C.byref(kept))
            return merged[:n].copy()
        n, a, b, c = _sz(0), _sz(0), _sz(0), _sz(0)
        self._check(self._fn("make_windows")(_sz(cached), _sz(n_init), _sz(n_local), _ptr(sel),
                                             _sz(sel.size), _ptr(merged), C.byref(n), C.byref(a),
                                             C.byref(b), C.byref(c)))
        return merged[: n.value].copy()

    def sdpa_full(self, q, k_all, v_all, num_heads):
        q, k_all, v_all = _f32(q), _f32(k_all), _f32(v_all)
        out = np.zeros_like(q)
        Cq, qw = q.shape
        rows, kw = k_all.shape
        if self.kind == "port":
            d = qw // num_heads
            self._check(self._fn("sdpa")(_ptr(q), _sz(Cq), _sz(num_heads), _sz(d), _ptr(k_all),
                                         _ptr(v_all), _sz(rows), _sz(kw // d), _ptr(out)))
        else:
            self._check(self._fn("sdpa_full")(_ptr(q), _sz(Cq), _sz(qw), _ptr(k_all), _ptr(v_all),
                                              _sz(rows), _sz(kw), _sz(num_heads), _ptr(out)))
        return out

    def sparse_attend(self, q, k_cur, v_cur, k_rows, v_rows, H, H_kv, attended):
        q, k_cur, v_cur = _f32(q), _f32(k_cur), _f32(v_cur)
        k_rows, v_rows = _f32(k_rows), _f32(v_rows)
        att = _u32(attended)
        Cq = q.shape[0]
        d = q.shape[1] // H
        out = np.zeros_like(q)
        if self.kind == "port":
            self._check(self._fn("sparse_attend")(_ptr(q), _ptr(k_cur), _ptr(v_cur), _sz(Cq),
                                                  _ptr(k_rows), _ptr(v_rows), _sz(k_rows.shape[0]),
                                                  _sz(H), _sz(H_kv), _sz(d), _ptr(att), _sz(att.size),
                                                  _ptr(out)))
        else:
            empty = np.zeros(1, np.uint32)
            self._check(self._fn("sparse_attend")(_ptr(q), _ptr(k_cur), _ptr(v_cur), _sz(Cq),
                                                  _ptr(k_rows), _ptr(v_rows), _sz(k_rows.shape[0]),
                                                  _sz(H), _sz(H_kv), _sz(d), _ptr(empty), _sz(0),
                                                  _ptr(att), _sz(att.size), _ptr(empty), _sz(0),
                                                  _ptr(out)))
        return out

    def engine(self, capacity_tokens, k=2048, n_local=512, n_init=128, chunk_size=512, theta=0.9,
               num_heads=8, num_kv_heads=8, head_dim=64, block_size=64,
               selection_method="head_soft_vote"):
        return OracleEngine(self, capacity_tokens, k, n_local, n_init, chunk_size, theta, num_heads,
                            num_kv_heads, head_dim, block_size, selection_method)


class OracleEngine:
    """AttentionEngine restated (attention.cpp:218-232) on either back end."""

    def __init__(self, o: Oracle, capacity, k, n_local, n_init, chunk_size, theta, H, H_kv, d,
                 block, method):
        self.o = o
        self.H, self.H_kv, self.d, self.k, self.chunk_size = H, H_kv, d, k, chunk_size
        create = o._fn("engine_create")
        create.restype = _p
        create.argtypes = [_sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz, C.c_int, _sz]
        self.h = create(k, n_local, n_init, chunk_size, theta, H, H_kv, d, block,
                        METHODS[method], capacity)
        if not self.h:
            raise OracleError(1, o._err().decode())
        self.h = _p(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._fn("engine_destroy")(self.h)
            self.h = None

    def append(self, k, v):
        k, v = _f32(k), _f32(v)
        self.o._check(self.o._fn("engine_append")(self.h, _ptr(k), _ptr(v), _sz(k.shape[0])))

    def decode(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        out = np.zeros((1, self.H * self.d), np.float32)
        hit = C.c_int(0)
        sel = np.zeros(max(self.k, 1), np.uint32)
        n = _sz(0)
        if self.o.kind == "port":
            cosv = C.c_double(0)
            self.o._check(self.o._fn("engine_decode")(self.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                                      C.byref(hit), _ptr(sel), C.byref(n),
                                                      C.byref(cosv)))
        else:
            self.o._check(self.o._fn("engine_decode")(self.h, _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                                      C.byref(hit), _ptr(sel), C.byref(n)))
        return out, bool(hit.value), sel[: n.value].copy()

    def force_miss(self):
        self.o._fn("engine_force_miss")(self.h)

    def prefill(self, q, k, v, trace=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n = q.shape[0]
        out = np.zeros_like(q)
        if not trace:
            if self.o.kind == "port":
                self.o._check(self.o._fn("engine_prefill")(self.h, _ptr(q), _ptr(k), _ptr(v), _sz(n),
                                                           _ptr(out), None, None, _sz(0)))
            else:
                self.o._check(self.o._fn("engine_prefill")(self.h, _ptr(q), _ptr(k), _ptr(v), _sz(n),
                                                           _ptr(out)))
            return out
        chunks = (n + self.chunk_size - 1) // self.chunk_size
        counts = np.zeros(chunks, np.uint64)
        flat = np.zeros(chunks * max(self.k, 1), np.uint32)
        fn = "engine_prefill" if self.o.kind == "port" else "engine_prefill_trace"
        self.o._check(self.o._fn(fn)(self.h, _ptr(q), _ptr(k), _ptr(v), _sz(n), _ptr(out),
                                     _ptr(flat), _ptr(counts), _sz(chunks)))
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return out, [flat[offs[i]:offs[i + 1]].copy() for i in range(chunks)]

    def stats(self):
        a, b, c = _sz(0), _sz(0), _sz(0)
        self.o._fn("engine_stats")(self.h, C.byref(a), C.byref(b), C.byref(c))
        return {"lookups": a.value, "hits": b.value, "len": c.value}

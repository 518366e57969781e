"""Python mirror of the reference's ``selattn`` module (proj/python/bindings.cpp:57-228)
over the native B200 library — same names, argument meaning and error types:

    std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
    selattn::capacity_error -> CapacityError (a RuntimeError).

Arrays may be numpy arrays (host) or torch CUDA tensors (device); results come
back in the same kind. All compute runs in sm_100a kernels (include/tokenselect.h).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import CapacityError, EngineConfig, check, lib

_sz = C.c_size_t
METHODS = {"topk": 0, "head_vote": 1, "head_soft_vote": 2}

__all__ = ["PagedKvPool", "Engine", "score_paged", "select", "select_for_chunk", "sparse_attend",
           "CapacityError", "METHODS", "version", "softmax_rows", "topk_indices", "cosine", "chunk_mean",
           "sdpa_full"]


def version() -> str:
    return lib.ts_version().decode()


def _is_torch_cuda(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


class _Arg:
    """A contiguous array argument: pointer + keep-alive + where it lives."""

    def __init__(self, x, dtype, ndim=None, name="array"):
        if x is None:
            self.ptr, self.obj, self.cuda, self.shape = None, None, False, (0,)
            return
        if _is_torch_cuda(x):
            import torch

            want = {np.float32: torch.float32, np.uint32: torch.int32, np.uint16: torch.int16}[dtype]
            if dtype is np.uint32 and x.dtype in (torch.int64, torch.int32, torch.uint32):
                x = x.to(torch.int32)
            elif dtype is np.uint16 and x.dtype == torch.bfloat16:
                x = x.view(torch.int16)
            elif x.dtype != want:
                x = x.to(want)
            x = x.contiguous()
            torch.cuda.current_stream().synchronize()
            self.obj, self.cuda, self.ptr, self.shape = x, True, C.c_void_p(x.data_ptr()), tuple(x.shape)
        else:
            a = np.ascontiguousarray(x, dtype=dtype)
            self.obj, self.cuda, self.shape = a, False, a.shape
            self.ptr = a.ctypes.data_as(C.c_void_p)
        if ndim is not None and len(self.shape) != ndim:
            raise ValueError(f"expected a {ndim}-D {name}")


def _out(shape, like_cuda, dtype=np.float32):
    if like_cuda:
        import torch

        t = torch.empty(shape, dtype={np.float32: torch.float32}[dtype], device="cuda")
        return t, C.c_void_p(t.data_ptr())
    a = np.zeros(shape, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)


def _idx_list(idx) -> _Arg:
    if _is_torch_cuda(idx):
        return _Arg(idx, np.uint32)
    return _Arg(np.asarray(list(idx) if not isinstance(idx, np.ndarray) else idx, dtype=np.int64).astype(np.uint32),
                np.uint32)


# ------------------------------------------------------------------- pool
class PagedKvPool:
    """PagedKvPool (kv_pool.hpp:33-95): bf16 K/V pages in HBM."""

    def __init__(self, capacity_tokens, page_size, num_kv_heads, head_dim, _handle=None):
        if _handle is not None:
            self._h, self._owned = _handle, False
        else:
            h = C.c_void_p()
            check(lib.ts_pool_create(capacity_tokens, page_size, num_kv_heads, head_dim, C.byref(h)))
            self._h, self._owned = h, True
        self.num_kv_heads = lib.ts_pool_num_kv_heads(self._h)
        self.head_dim = lib.ts_pool_head_dim(self._h)
        self.row_width = self.num_kv_heads * self.head_dim

    def __del__(self):
        if getattr(self, "_owned", False) and self._h and lib is not None:
            lib.ts_pool_destroy(self._h)
            self._h = None

    def create_sequence(self) -> int:
        s = C.c_uint32()
        check(lib.ts_pool_create_sequence(self._h, C.byref(s)))
        return s.value

    def append_kv(self, seq, k_new, v_new):
        k = _Arg(k_new, np.float32, 2, "float32 array")
        v = _Arg(v_new, np.float32, 2, "float32 array")
        if k.shape[1] != self.row_width or v.shape[1] != self.row_width or k.shape[0] != v.shape[0]:
            raise ValueError("append_kv: rows must be [t x (H_kv * d_h)]")
        first, last = _sz(), _sz()
        check(lib.ts_pool_append_kv(self._h, seq, k.ptr, v.ptr, k.shape[0], C.byref(first), C.byref(last)))
        return first.value, last.value

    def append_kv_bf16(self, seq, k_bits, v_bits):
        k = _Arg(k_bits, np.uint16, 2)
        v = _Arg(v_bits, np.uint16, 2)
        first, last = _sz(), _sz()
        check(lib.ts_pool_append_kv_bf16(self._h, seq, k.ptr, v.ptr, k.shape[0], C.byref(first), C.byref(last)))
        return first.value, last.value

    def gather(self, seq, idx):
        ia = _idx_list(idx)
        n = ia.shape[0] if ia.shape else 0
        k, kp = _out((n, self.row_width), ia.cuda)
        v, vp = _out((n, self.row_width), ia.cuda)
        check(lib.ts_pool_gather(self._h, seq, ia.ptr, n, kp, vp))
        return k, v

    def release(self, seq):
        check(lib.ts_pool_release(self._h, seq))

    def logical_len(self, seq) -> int:
        n = _sz()
        check(lib.ts_pool_logical_len(self._h, seq, C.byref(n)))
        return n.value

    def shuffle_free_frames(self, seed):
        check(lib.ts_pool_shuffle_free_frames(self._h, seed))

    def page_table_json(self, seq) -> str:
        need = _sz()
        check(lib.ts_pool_page_table_json(self._h, seq, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib.ts_pool_page_table_json(self._h, seq, buf, need.value, C.byref(need)))
        return buf.value.decode()

    @property
    def total_frames(self) -> int:
        return lib.ts_pool_total_frames(self._h)

    @property
    def free_frames(self) -> int:
        return lib.ts_pool_free_frames(self._h)

    @property
    def page_size(self) -> int:
        return lib.ts_pool_page_size(self._h)


# -------------------------------------------------------------- selection
def score_paged(q, pool: PagedKvPool, seq, candidates, block_size=64):
    """score_paged (selector.cpp:26-68) -> (scores [H x T], candidates)."""
    qa = _Arg(q, np.float32, 2, "float32 array")
    ca = _idx_list(candidates)
    H, d = qa.shape
    T = ca.shape[0]
    s, sp = _out((H, T), qa.cuda)
    check(lib.ts_score_paged(pool._h, seq, qa.ptr, H, d, ca.ptr, T, block_size, sp))
    return s, (candidates if _is_torch_cuda(candidates) else [int(x) for x in np.asarray(ca.obj)])


def select(per_head, candidate_idx, k, method="head_soft_vote"):
    """select_with (selector.cpp:128-135) -> (selected, criticality)."""
    if method not in METHODS:
        raise ValueError("unknown selection method: " + str(method))
    sa = _Arg(per_head, np.float32, 2, "float32 array")
    ca = _idx_list(candidate_idx)
    H, T = sa.shape
    if ca.shape[0] != T:
        raise ValueError("candidate_idx length must match score columns")
    n_max = max(min(k, T), 1)
    sel = np.zeros(n_max, np.uint32)
    crit = np.zeros(n_max, np.float64)
    n = _sz()
    check(lib.ts_select(sa.ptr, H, T, ca.ptr, k, METHODS[method], sel.ctypes.data_as(C.c_void_p),
                        crit.ctypes.data_as(C.c_void_p), C.byref(n)))
    return [int(x) for x in sel[: n.value]], [float(x) for x in crit[: n.value]]


def select_for_chunk(q_chunk, pool: PagedKvPool, seq, candidates, k, method="head_soft_vote", block_size=64):
    """select_for_chunk (selector.cpp:137-150) -> (selected, criticality)."""
    if method not in METHODS:
        raise ValueError("unknown selection method: " + str(method))
    qa = _Arg(q_chunk, np.float32, 2, "float32 array")
    ca = _idx_list(candidates)
    c, width = qa.shape
    T = ca.shape[0]
    n_max = max(min(k, T), 1)
    sel = np.zeros(n_max, np.uint32)
    crit = np.zeros(n_max, np.float64)
    n = _sz()
    check(lib.ts_select_for_chunk(pool._h, seq, qa.ptr, c, width, ca.ptr, T, k, METHODS[method], block_size,
                                  sel.ctypes.data_as(C.c_void_p), crit.ctypes.data_as(C.c_void_p), C.byref(n)))
    return [int(x) for x in sel[: n.value]], [float(x) for x in crit[: n.value]]


def sparse_attend(q, k_cur, v_cur, pool: PagedKvPool, seq, forced_init=(), selected=(), forced_local=(),
                  num_heads=None):
    """sparse_attend (attention.cpp:114-123) with AttentionWindows given as three lists."""
    qa = _Arg(q, np.float32, 2, "float32 array")
    ka = _Arg(k_cur, np.float32, 2, "float32 array")
    va = _Arg(v_cur, np.float32, 2, "float32 array")
    if ka.shape[0] != qa.shape[0] or va.shape[0] != qa.shape[0]:
        raise ValueError("sparse_attend: current KV rows must match query rows")
    H = num_heads if num_heads is not None else qa.shape[1] // pool.head_dim
    if H == 0 or qa.shape[1] % H != 0:
        raise ValueError("sdpa_full: q must be [C x (H * d_h)]")
    if qa.shape[1] // H != pool.head_dim:
        raise ValueError("sdpa_full: K/V must be [(N + C) x (H_kv * d_h)]")
    lists = [_idx_list(x) for x in (forced_init, selected, forced_local)]
    o, op = _out(qa.shape, qa.cuda)
    check(lib.ts_sparse_attend(pool._h, seq, qa.ptr, ka.ptr, va.ptr, qa.shape[0], H,
                               lists[0].ptr, lists[0].shape[0], lists[1].ptr, lists[1].shape[0],
                               lists[2].ptr, lists[2].shape[0], op))
    return o


# ----------------------------------------------------------------- engine
# ---------------------------------------------------- tensor utilities
# (the free functions of the reference's module, bindings.cpp:60-116; on the device)
def softmax_rows(m):
    """softmax_rows (tensor.cpp:31-52) -> [rows x cols] fp32."""
    a = _Arg(m, np.float32, 2)
    o, op = _out(a.shape, a.cuda)
    check(lib.ts_softmax_rows(a.ptr, a.shape[0], a.shape[1], op))
    return o


def topk_indices(scores, k):
    """topk_indices (tensor.cpp:68-90): the min(k, n) largest, ties to the
    smaller index, ascending."""
    a = _Arg(np.ravel(np.asarray(scores, np.float64)), np.float64, 1)
    n = a.shape[0]
    out = np.zeros(max(1, min(int(k), n)), np.uint32)
    m = _sz()
    check(lib.ts_topk_indices(a.ptr, n, int(k), out.ctypes.data_as(C.c_void_p), C.byref(m)))
    return [int(x) for x in out[: m.value]]


def cosine(u, v):
    """cosine (tensor.cpp:92-113), fp64."""
    a = _Arg(np.ravel(np.asarray(u, np.float64)), np.float64, 1)
    b = _Arg(np.ravel(np.asarray(v, np.float64)), np.float64, 1)
    if a.shape[0] != b.shape[0]:
        raise ValueError("cosine: length mismatch")
    r = C.c_double()
    check(lib.ts_cosine(a.ptr, b.ptr, a.shape[0], C.byref(r)))
    return r.value


def chunk_mean(q_chunk):
    """chunk_mean (tensor.cpp:133-150) -> [H*d] fp32."""
    a = _Arg(q_chunk, np.float32, 2)
    o, op = _out((a.shape[1],), a.cuda)
    check(lib.ts_chunk_mean(a.ptr, a.shape[0], a.shape[1], op))
    return o


def sdpa_full(q, k_all, v_all, num_heads):
    """sdpa_full (attention.cpp:54-112): q [C x H*d] over k_all / v_all
    [(N + C) x H_kv*d], causal within the last C rows."""
    qa = _Arg(q, np.float32, 2)
    ka = _Arg(k_all, np.float32, 2)
    va = _Arg(v_all, np.float32, 2)
    if ka.shape != va.shape:
        raise ValueError("sdpa_full: K/V must be [(N + C) x (H_kv * d_h)]")
    o, op = _out(qa.shape, qa.cuda)
    check(lib.ts_sdpa_full(qa.ptr, qa.shape[0], qa.shape[1], ka.ptr, va.ptr, ka.shape[0], ka.shape[1],
                           int(num_heads), op))
    return o


class Engine:
    """AttentionEngine (attention.hpp:94-115) on the device, optionally over
    ``n_seqs`` sequences decoded together (per-request page tables)."""

    def __init__(self, capacity_tokens, k=2048, n_local=512, n_init=128, chunk_size=512, theta=0.9,
                 num_heads=8, num_kv_heads=8, head_dim=64, block_size=64, selection_method="head_soft_vote",
                 n_seqs=1, n_layers=1):
        if selection_method not in METHODS:
            raise ValueError("unknown selection method: " + str(selection_method))
        cfg = EngineConfig(k, n_local, n_init, chunk_size, theta, num_heads, num_kv_heads, head_dim, block_size,
                           METHODS[selection_method])
        self.cfg = cfg
        self.n_seqs = n_seqs
        self.model_dim = num_heads * head_dim
        self.kv_dim = num_kv_heads * head_dim
        h = C.c_void_p()
        check(lib.ts_engine_create_layers(C.byref(cfg), capacity_tokens, n_seqs, n_layers, C.byref(h)))
        self._h = h
        self.n_layers = n_layers
        self.pool = PagedKvPool(0, 1, 1, 1, _handle=C.c_void_p(lib.ts_engine_pool(h)))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ts_engine_destroy(self._h)
            self._h = None

    def sequence(self, i=0) -> int:
        return lib.ts_engine_sequence(self._h, i)

    def set_layer(self, layer):
        """Multi-layer engine: the layer the following calls act on (each
        (layer, sequence) has its own KV cache and Selection Cache entry)."""
        check(lib.ts_engine_set_layer(self._h, layer))

    def set_stream(self, stream_ptr):
        check(lib.ts_engine_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def append(self, k, v, seq=0):
        """Raw KV fill (PagedKvPool::append_kv on the engine's sequence)."""
        ka = _Arg(k, np.float32, 2)
        va = _Arg(v, np.float32, 2)
        check(lib.ts_engine_append(self._h, seq, ka.ptr, va.ptr, ka.shape[0]))

    def append_bf16(self, k_bits, v_bits, seq=0):
        ka = _Arg(k_bits, np.uint16, 2)
        va = _Arg(v_bits, np.uint16, 2)
        check(lib.ts_engine_append_bf16(self._h, seq, ka.ptr, va.ptr, ka.shape[0]))

    def prefill(self, q, k, v, seq=0, trace=False, out=None):
        """prefill (attention.cpp:135-170) -> output [n x H*d] (and the chunk
        traces with trace=True). `out`: an optional preallocated float32
        [n x H*d] array (host, e.g. a view of pinned memory, or a CUDA tensor)
        the output is written into and returned."""
        qa = _Arg(q, np.float32, 2)
        ka = _Arg(k, np.float32, 2)
        va = _Arg(v, np.float32, 2)
        n = qa.shape[0]
        if n == 0:
            raise ValueError("prefill: empty input")
        if qa.shape[1] != self.model_dim or ka.shape[1] != self.kv_dim or ka.shape != va.shape or ka.shape[0] != n:
            raise ValueError("prefill: inconsistent input shapes")
        if out is None:
            o, op = _out(qa.shape, qa.cuda)
        else:
            oa = _Arg(out, np.float32, 2)
            if oa.shape != qa.shape or (isinstance(out, np.ndarray) and oa.obj is not out):
                raise ValueError("prefill: out must be a contiguous float32 array shaped like q")
            o, op = out, oa.ptr
        if not trace:
            check(lib.ts_engine_prefill(self._h, seq, qa.ptr, ka.ptr, va.ptr, n, op, None, None, 0))
            return o
        chunks = (n + self.cfg.chunk_size - 1) // self.cfg.chunk_size
        counts = np.zeros(chunks, np.uint64)
        flat = np.zeros(max(chunks * max(self.cfg.k, 1), 1), np.uint32)
        check(lib.ts_engine_prefill(self._h, seq, qa.ptr, ka.ptr, va.ptr, n, op, flat.ctypes.data_as(C.c_void_p),
                                    counts.ctypes.data_as(C.c_void_p), chunks))
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return o, [[int(x) for x in flat[offs[i]:offs[i + 1]]] for i in range(chunks)]

    def prefill_async(self, q, k, v, out, seq=0):
        """Stream-ordered prefill on device tensors (no host sync): q [n x H*d],
        k/v [n x H_kv*d], out [n x H*d], all float32 CUDA tensors."""
        n = q.shape[0]
        check(lib.ts_engine_prefill_async(self._h, seq, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                          C.c_void_p(v.data_ptr()), n, C.c_void_p(out.data_ptr())))

    def decode(self, q, k, v):
        """decode_step (attention.cpp:172-200) -> (output, cache_hit, selected).

        With n_seqs > 1, q is [B x H*d] and the result holds per-sequence lists."""
        qa = _Arg(q, np.float32, 2)
        ka = _Arg(k, np.float32, 2)
        va = _Arg(v, np.float32, 2)
        B = self.n_seqs
        if qa.shape != (B, self.model_dim):
            raise ValueError("decode_step: q must be [1 x (H * d_h)]")
        if ka.shape != (B, self.kv_dim) or va.shape != ka.shape:
            raise ValueError("decode_step: KV must be [1 x (H_kv * d_h)]")
        o, op = _out(qa.shape, qa.cuda)
        hits = np.zeros(B, np.int32)
        kk = max(self.cfg.k, 1)
        sel = np.zeros(B * kk, np.uint32)
        nsel = np.zeros(B, np.uint64)
        check(lib.ts_engine_decode(self._h, qa.ptr, ka.ptr, va.ptr, op, hits.ctypes.data_as(C.c_void_p),
                                   sel.ctypes.data_as(C.c_void_p), nsel.ctypes.data_as(C.c_void_p)))
        sels = [[int(x) for x in sel[b * kk: b * kk + int(nsel[b])]] for b in range(B)]
        if B == 1:
            return o, bool(hits[0]), sels[0]
        return o, [bool(h) for h in hits], sels

    def decode_into(self, q, k, v, out, hits=None, sel=None, n_sel=None):
        """decode_step through the C ABI with caller-owned host buffers (no
        Python-side conversion): q/k/v/out are C-contiguous float32 numpy
        arrays; optional hits (int32[B]), sel (uint32[B*k]), n_sel (uint64[B])."""
        # plain addresses: c_void_p argtypes take ints (ndarray.ctypes.data_as
        # costs about twice as much per array)
        ptr = lambda a: None if a is None else a.ctypes.data
        check(lib.ts_engine_decode(self._h, ptr(q), ptr(k), ptr(v), ptr(out), ptr(hits), ptr(sel), ptr(n_sel)))

    def decode_async(self, q, k, v, out):
        """Stream-ordered decode on device tensors (no host sync)."""
        check(lib.ts_engine_decode_async(self._h, C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                         C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr())))

    def force_miss(self, seq=0):
        check(lib.ts_engine_force_miss(self._h, seq))

    # the single-sequence step kernel (csrc/step.cu; slot 63 = 2)
    STEP_TRACE_POINTS = ["start", "decision", "scan", "stats", "sync1", "crit", "radix1", "radix2", "select",
                         "att_rows", "attend", "sync4", "merge"]
    STEP_SUB_POINTS = {13: "crit:stats", 14: "crit:tmem_done", 16: "radix:find1", 17: "radix:hist2", 18: "radix:B3",
                       19: "att:scores", 20: "att:softmax", 21: "att:pv", 22: "merge:loaded", 23: "merge:weights",
                       24: "p0:loads_issued", 25: "p0:decided"}

    def trace_names(self):
        """Slot -> name for read_trace(all_ctas=True) of the last step read."""
        if getattr(self, "_trace_kid", 0) == 2:
            names = dict(enumerate(self.STEP_TRACE_POINTS))
            names.update(self.STEP_SUB_POINTS)
        else:
            names = dict(enumerate(self.TRACE_POINTS))
            names.update(self.SUB_POINTS)
        return names

    TRACE_POINTS = ["start", "decision", "scan", "softmax_partials", "sync1", "crit", "radix1", "radix2",
                    "compact", "sync4", "sel_out", "attend", "merge"]
    # sub-phase stamps (slots 13..63, 29 / 30 reserved) of read_trace(all_ctas=True)
    SUB_POINTS = {13: "crit:stats_staged", 14: "crit:f_done", 15: "radix:hist1", 16: "radix:find1",
                  17: "radix:hist2", 18: "radix:find2", 19: "radix:ties", 20: "att:ridx", 21: "att:data",
                  22: "att:scores", 23: "att:softmax", 24: "att:pv", 25: "att:end", 27: "dec:done", 28: "merge:all_in", 31: "merge:end", 32: "crit:hist_zeroed",
                  33: "find1:loaded", 36: "find2:loaded", 38: "hist2:zeroed", 39: "hist2:counted",
                  40: "compact:iter", 41: "sel_out:prefix", 42: "merge:loaded", 43: "merge:weights",
                  26: "dec:issued", 44: "dev:att_rep",
                  45: "p0:dec_loads", 46: "p0:frames", 47: "p0:hit_prep", 48: "crit:tmem_done", 49: "crit:keys"}

    def set_trace(self, enable=True):
        check(lib.ts_engine_set_trace(self._h, 1 if enable else 0))

    def read_trace(self, all_ctas=False):
        """Per-phase device time (us) of the last decode step from CTA 0's
        stamps (or, with all_ctas, a [ctas x 32] array of stamps in us
        relative to the earliest CTA start; NaN where a CTA did not pass).

        Stamps are SM clock64 values; slot 0 / 30 hold %globaltimer (ns) at the
        start / end (slot 12) and slot 29 the start clock, which align the CTAs
        and give each CTA's clock rate."""
        st = np.zeros(64 * 1024, np.uint64)
        check(lib.ts_engine_read_trace(self._h, st.ctypes.data_as(C.c_void_p), st.size))
        raw = st.reshape(1024, 64).astype(np.int64)
        raw = raw[: int(np.count_nonzero(raw[:, 0]))]
        self._trace_kid = int(raw[0, 63])  # 2: the step kernel (csrc/step.cu)
        # rebase before going to float64 (ns since the epoch exceed its 2^53 mantissa)
        gmin, cmin = raw[:, 0].min(), raw[:, 29].min()
        a = np.where(raw == 0, 0.0, (raw - cmin).astype(np.float64))
        a[:, 0] = (raw[:, 0] - gmin).astype(np.float64)
        a[:, 30] = np.where(raw[:, 30] == 0, 0.0, (raw[:, 30] - gmin).astype(np.float64))
        g0, c0, c_end, g_end = a[:, 0], a[:, 29], a[:, 12], a[:, 30]
        ok = (g_end > g0) & (c_end > c0)
        rate = np.where(ok, (c_end - c0) / np.where(ok, g_end - g0, 1.0), np.nan)  # cycles per ns
        r = np.nanmedian(rate) if np.any(ok) else 1.9
        self._trace_rate = float(r)  # SM cycles per ns over the launch
        ns = g0[:, None] + (a - c0[:, None]) / r
        ns[:, 0] = g0
        ns[raw == 0] = np.nan
        ns[:, 29] = np.nan
        ns[:, 30] = np.nan
        ns[:, 63] = np.nan  # kernel id
        us = ns / 1000.0
        if all_ctas:
            return us
        t = us[0]
        names = self.STEP_TRACE_POINTS if raw[0, 63] == 2 else self.TRACE_POINTS  # slot 63: kernel id
        out, prev = {}, 0.0
        for i, name in enumerate(names[1:], start=1):
            if not np.isnan(t[i]):
                out[name] = round(t[i] - prev, 3)
                prev = t[i]
        out["total"] = prev
        for i in range(len(self.TRACE_POINTS), 63):  # optional sub-phase stamps, relative to start
            if i not in (29, 30) and not np.isnan(t[i]):
                out[f"t{i}@"] = round(t[i], 3)
        return out

    def set_theta(self, theta, seq=0):
        check(lib.ts_engine_set_theta(self._h, seq, theta))

    def sync(self):
        check(lib.ts_engine_sync(self._h))

    def stats(self, seq=0):
        a, b, c, h, cs = _sz(), _sz(), _sz(), C.c_int(), C.c_double()
        check(lib.ts_engine_stats(self._h, seq, C.byref(a), C.byref(b), C.byref(c), C.byref(h), C.byref(cs)))
        return {"lookups": a.value, "hits": b.value, "len": c.value, "last_hit": h.value, "last_cos": cs.value}

    def cached_selection(self, seq=0):
        kk = max(self.cfg.k, 1)
        sel = np.zeros(kk, np.uint32)
        crit = np.zeros(kk, np.float64)
        n = _sz()
        check(lib.ts_engine_cached_selection(self._h, seq, sel.ctypes.data_as(C.c_void_p),
                                             crit.ctypes.data_as(C.c_void_p), C.byref(n)))
        return sel[: n.value].copy(), crit[: n.value].copy()

    def __len__(self):
        return self.stats(0)["len"]

    @property
    def cache_lookups(self):
        return self.stats(0)["lookups"]

    @property
    def cache_hits(self):
        return self.stats(0)["hits"]


def launch_count() -> int:
    return int(lib.ts_launch_count())

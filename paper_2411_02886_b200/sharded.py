"""KV-sequence-sharded TokenSelect decode (BASELINE config 4: 1M-token context
over 2/4/8 B200s).

One sequence is split into contiguous shards, one per rank. Every rank holds
its range [base, base + len) in its own engine (bf16 pages in its HBM):
- rank 0 holds the init window;
- the last rank holds the local window and the current token, and receives
  every append.

A decode step is four native calls per rank (include/tokenselect.h,
ts_shard_*) with three all-gathers in between:

    stats   [H][2]       per-head (m, z) of the rank's scores -> global softmax stats
    cands   [2k + 1]     the rank's local top-k (global index, key, count) -> exact global top-k
    partial [H*d | H*2]  the rank's attention (o, then M, L), one packed block -> log-sum-exp combine

The Selection Cache decision needs no exchange: q and the cached query are
replicated, so every rank decides identically.

Transport:
- ``LibraryComm`` + ``decode_step_native``: the library's own NCCL
  communicator; the whole step (launches + all-gathers) is one C call,
  ts_shard_decode_step, on the engine's stream (the bench's path);
- ``TorchDistExchange`` + ``decode_step``: the same protocol phase by phase
  over torch.distributed (gloo on CPU for the host-logic tests);
- ``simulate_step`` runs all shards of one sequence inside one process.

All device work is the library's sm_100a kernels. This module only sequences
the calls and moves three small buffers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence

from ._native import EngineConfig, check, lib
from .selattn import METHODS


@dataclass(frozen=True)
class ShardRange:
    rank: int
    base: int
    length: int


def shard_ranges(n_tokens: int, world: int, n_init: int, n_local: int) -> List[ShardRange]:
    """Contiguous near-equal split of the cached prefix. Rank 0 must hold the
    init window and the last rank the local window (validated); appends go to
    the last rank, so its range grows by one token per step."""
    if world < 1:
        raise ValueError("world must be >= 1")
    per = n_tokens // world
    out, base = [], 0
    for r in range(world):
        length = per if r < world - 1 else n_tokens - base
        out.append(ShardRange(r, base, length))
        base += length
    if world > 1:
        if out[0].length < min(n_init, n_tokens):
            raise ValueError("shard 0 must hold the whole init window")
        if out[-1].length < min(n_local, n_tokens):
            raise ValueError("the last shard must hold the whole local window")
    return out


class NativeShard:
    """One rank's shard engine (ts_shard_*), on the current torch CUDA stream."""

    def __init__(self, rank: int, world: int, capacity_tokens: int, k=2048, n_local=512, n_init=128, chunk_size=512,
                 theta=0.9, num_heads=32, num_kv_heads=8, head_dim=128, block_size=64,
                 selection_method="head_soft_vote"):
        import torch

        self.torch = torch
        self.rank, self.world = rank, world
        self.cfg = EngineConfig(k, n_local, n_init, chunk_size, theta, num_heads, num_kv_heads, head_dim, block_size,
                                METHODS[selection_method])
        h = C.c_void_p()
        check(lib.ts_shard_engine_create(C.byref(self.cfg), capacity_tokens, rank, world, C.byref(h)))
        self._h = h
        self.H, self.H_kv, self.d, self.k = num_heads, num_kv_heads, head_dim, k
        dev = torch.device("cuda", torch.cuda.current_device())
        self._stats = torch.empty(num_heads * 2, dtype=torch.float32, device=dev)
        self._cands = torch.empty(2 * k + 1, dtype=torch.int32, device=dev)
        # partial output and (M, L) pairs are one block, so a step needs one
        # all-gather for both (ts_shard_combine_packed)
        self._pm = torch.empty(num_heads * head_dim + num_heads * 2, dtype=torch.float32, device=dev)
        self._part = self._pm[: num_heads * head_dim]
        self._ml = self._pm[num_heads * head_dim:]
        # torch's default stream has handle 0, which the C ABI reads as "the
        # engine's own stream": pass cudaStreamLegacy (0x1) instead so both
        # sides order on the same stream
        st = torch.cuda.current_stream().cuda_stream or 1
        self._stream = C.c_void_p(st)
        check(lib.ts_engine_set_stream(self._h, self._stream))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ts_engine_destroy(self._h)
            self._h = None

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def append_bf16(self, k_bits, v_bits):
        check(lib.ts_engine_append_bf16(self._h, 0, self._p(k_bits), self._p(v_bits), k_bits.shape[0]))

    def append(self, k, v):
        check(lib.ts_engine_append(self._h, 0, self._p(k), self._p(v), k.shape[0]))

    def set_theta(self, theta):
        check(lib.ts_engine_set_theta(self._h, 0, theta))

    # -- the four phases ----------------------------------------------------
    def _follow_stream(self):
        """Every phase runs on the caller's current stream, the one the
        all-gathers between the phases are ordered on."""
        st = self.torch.cuda.current_stream().cuda_stream or 1
        if st != self._stream.value:
            self._stream = C.c_void_p(st)
            check(lib.ts_engine_set_stream(self._h, self._stream))

    def stats(self, q, k, v, base: int, n_global: int):
        self._follow_stream()
        out = self._stats
        check(lib.ts_shard_stats(self._h, self._p(q), self._p(k), self._p(v), base, n_global, self._p(out)))
        self._qkv = (q, k, v)  # keep alive until attend
        return out

    def select(self, all_stats):
        self._follow_stream()
        out = self._cands
        check(lib.ts_shard_select(self._h, self._p(all_stats), self._p(out)))
        return out

    def attend(self, all_cands):
        self._follow_stream()
        part, ml = self._part, self._ml
        check(lib.ts_shard_attend(self._h, self._p(all_cands), self._p(part), self._p(ml)))
        return part, ml

    def attend_packed(self, all_cands):
        """attend, returning the [H*d | H*2] block (a view reused next step)."""
        self.attend(all_cands)
        return self._pm

    def combine_packed(self, all_packed):
        """The step's [1 x H*d] output, a fresh tensor (callers may keep
        per-step outputs), on the stream of the other phases."""
        self._follow_stream()
        out = self.torch.empty(1, self.H * self.d, dtype=self.torch.float32, device=all_packed.device)
        check(lib.ts_shard_combine_packed(self._p(all_packed), self.world, self.H, self.d, self._p(out),
                                          self._stream))
        return out

    def combine(self, all_part, all_ml):
        out = self.torch.empty(1, self.H * self.d, dtype=self.torch.float32, device=all_part.device)
        check(lib.ts_shard_combine(self._p(all_part), self._p(all_ml), self.world, self.H, self.d, self._p(out),
                                   C.c_void_p(self.torch.cuda.current_stream().cuda_stream)))
        return out


class LibraryComm:
    """The library's own NCCL communicator (ts_comm_*): rank 0 makes the
    unique id, torch.distributed broadcasts it (bootstrap only), and the
    library then calls ncclAllGather itself on the engine's stream inside
    ts_shard_decode_step. world == 1 needs no NCCL at all."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world = rank, world
        idb = (C.c_uint8 * 128)()
        if world > 1:
            import torch.distributed as dist

            if rank == 0:
                check(lib.ts_comm_unique_id(C.cast(idb, C.c_void_p)))
            obj = [bytes(idb)]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(idb, obj[0], 128)
        h = C.c_void_p()
        check(lib.ts_comm_create(C.cast(idb, C.c_void_p), world, rank, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ts_comm_destroy(self._h)
            self._h = None


def decode_step_native(shard, comm: LibraryComm, q, k, v, base: int, n_global: int, out=None):
    """One sharded decode step in ONE library call (ts_shard_decode_step):
    the four shard launches and the three ncclAllGather exchanges are issued
    by the library on the shard's stream. Returns the [1 x H*d] output."""
    torch = shard.torch
    shard._follow_stream()
    if out is None:
        out = torch.empty(1, shard.H * shard.d, dtype=torch.float32, device=q.device)
    check(lib.ts_shard_decode_step(shard._h, comm._h, shard._p(q), shard._p(k), shard._p(v), base, n_global,
                                   shard._p(out)))
    shard._qkv = (q, k, v)
    return out


class TorchDistExchange:
    """all-gather of one flat tensor per rank via torch.distributed (rank
    order): all_gather_into_tensor on NCCL (one collective, into a reused
    output buffer per shape), the list form elsewhere (gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.nccl = dist.get_backend(group) == "nccl"
        self.world = dist.get_world_size(group)
        self._out = {}

    def all_gather(self, t):
        import torch

        t = t.contiguous()
        if self.world == 1:
            return t  # a one-rank all-gather is the identity
        if self.nccl:
            key = (t.numel(), t.dtype, t.device)
            out = self._out.get(key)
            if out is None:
                out = self._out[key] = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.cat(parts)


def decode_step(shard, exchange, q, k, v, base: int, n_global: int):
    """One sharded decode step on this rank (every rank calls it in lockstep);
    returns the [1 x H*d] output, identical on every rank."""
    stats = shard.stats(q, k, v, base, n_global)
    cands = shard.select(exchange.all_gather(stats))
    packed = shard.attend_packed(exchange.all_gather(cands))
    return shard.combine_packed(exchange.all_gather(packed))


def simulate_step(shards: Sequence, qkv_per_shard, bases: Sequence[int], n_global: int, return_packed=False):
    """All shards of one sequence in one process (single GPU): the exchanges
    are concatenations in rank order -- the same bytes NCCL would deliver
    (each shard's phase outputs are copied before the next shard reuses its
    buffers)."""
    import torch

    stats = [s.stats(*qkv_per_shard[i], bases[i], n_global).clone() for i, s in enumerate(shards)]
    all_stats = torch.cat(stats)
    cands = [s.select(all_stats).clone() for s in shards]
    all_cands = torch.cat(cands)
    all_packed = torch.cat([s.attend_packed(all_cands).clone() for s in shards])
    outs = [s.combine_packed(all_packed) for s in shards]
    # return_packed: also the gathered [world][H*d | H*2] partial blocks
    return (outs, all_cands, all_packed) if return_packed else (outs, all_cands)

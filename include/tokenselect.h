/* tokenselect.h — C ABI of the B200-native TokenSelect decode path.
 *
 * Drop-in boundary for the reference's hot path (decode-time Selection Cache
 * -> paged Q.K scoring -> per-head soft vote -> top-k -> sparse attention ->
 * KV append). Every entry point replaces one reference interface, cited as
 * /root/reference/proj/<file>:<line>. Plain pointers and sizes only; array
 * arguments may be HOST or DEVICE (CUDA) pointers — the library detects the
 * kind per pointer. Shapes are implied by the sizes passed (row-major).
 *
 * Errors: every call returns a ts_status mirroring the reference's exception
 * types; ts_last_error() holds the reference's message text (thread-local).
 * A failed call leaves pool/engine state exactly as the reference would.
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns TS_CUDA_ERROR.
 */
#ifndef TOKENSELECT_H
#define TOKENSELECT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum ts_status {
  TS_OK = 0,
  TS_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  TS_OUT_OF_RANGE = 2,     /* std::out_of_range */
  TS_CAPACITY = 3,         /* selattn::capacity_error (kv_pool.hpp:15-17) */
  TS_CUDA_ERROR = 4        /* no device / CUDA failure */
} ts_status;

/* SelectionMethod, selector.hpp:12 */
typedef enum ts_method { TS_TOPK = 0, TS_HEAD_VOTE = 1, TS_HEAD_SOFT_VOTE = 2 } ts_method;

typedef struct ts_pool ts_pool;
typedef struct ts_engine ts_engine;

/* EngineConfig, attention.hpp:12-27 (same fields, same defaults). */
typedef struct ts_engine_config {
  size_t k;            /* 2048 */
  size_t n_local;      /* 512 */
  size_t n_init;       /* 128 */
  size_t chunk_size;   /* 512 */
  double theta;        /* 0.9 */
  size_t num_heads;    /* 8 */
  size_t num_kv_heads; /* 8 */
  size_t head_dim;     /* 64 */
  size_t block_size;   /* 64 */
  int selection_method; /* TS_HEAD_SOFT_VOTE */
} ts_engine_config;

const char* ts_last_error(void);
const char* ts_version(void);
/* Fills cfg with EngineConfig's defaults (attention.hpp:13-22). */
void ts_engine_config_default(ts_engine_config* cfg);
/* EngineConfig::validate, attention.cpp:10-19. */
ts_status ts_engine_config_validate(const ts_engine_config* cfg);

/* ------------------------------------------------------------------------
 * PagedKvPool — kv_pool.hpp:33-95. bf16 K/V slabs in HBM, device page table
 * per sequence, host LIFO frame allocator (kv_pool.cpp:12-28, :73-76).
 * ---------------------------------------------------------------------- */
/* PagedKvPool::PagedKvPool, kv_pool.cpp:12-28 */
ts_status ts_pool_create(size_t capacity_tokens, size_t page_size, size_t num_kv_heads,
                         size_t head_dim, ts_pool** out);
void ts_pool_destroy(ts_pool* pool);
/* PagedKvPool::create_sequence, kv_pool.cpp:30-34 */
ts_status ts_pool_create_sequence(ts_pool* pool, uint32_t* seq_id);
/* PagedKvPool::append_kv, kv_pool.cpp:55-85: k, v are [t x (H_kv*d)] fp32
 * (stored as bf16); all-or-nothing; returns the range [first, last). */
ts_status ts_pool_append_kv(ts_pool* pool, uint32_t seq, const float* k, const float* v,
                            size_t t, size_t* first, size_t* last);
/* Same, from bf16 rows (bit patterns) — no rounding step. */
ts_status ts_pool_append_kv_bf16(ts_pool* pool, uint32_t seq, const uint16_t* k,
                                 const uint16_t* v, size_t t, size_t* first, size_t* last);
/* PagedKvPool::gather, kv_pool.cpp:87-101: rows idx[j] -> k_out/v_out [n x row] fp32 */
ts_status ts_pool_gather(const ts_pool* pool, uint32_t seq, const uint32_t* idx, size_t n,
                         float* k_out, float* v_out);
/* PagedKvPool::release, kv_pool.cpp:103-111 */
ts_status ts_pool_release(ts_pool* pool, uint32_t seq);
/* PagedKvPool::logical_len, kv_pool.cpp:113 */
ts_status ts_pool_logical_len(const ts_pool* pool, uint32_t seq, size_t* len);
/* PagedKvPool::shuffle_free_frames, kv_pool.cpp:133-138 (same permutation) */
ts_status ts_pool_shuffle_free_frames(ts_pool* pool, uint64_t seed);
/* PagedKvPool::page_table_json, kv_pool.cpp:140-147. *needed = strlen+1. */
ts_status ts_pool_page_table_json(const ts_pool* pool, uint32_t seq, char* buf, size_t cap,
                                  size_t* needed);
/* kv_pool.hpp:60-65 accessors */
size_t ts_pool_total_frames(const ts_pool* pool);
size_t ts_pool_free_frames(const ts_pool* pool);
size_t ts_pool_page_size(const ts_pool* pool);
size_t ts_pool_num_kv_heads(const ts_pool* pool);
size_t ts_pool_head_dim(const ts_pool* pool);
/* Device address of the bf16 K / V slabs and of a sequence's int32 page
 * table (replaces key_row/value_row raw pointers, kv_pool.hpp:57-58). */
ts_status ts_pool_device_views(const ts_pool* pool, uint32_t seq, const void** k_slab,
                               const void** v_slab, const int32_t** page_table);

/* ------------------------------------------------------------------------
 * Selection — selector.hpp:32-54
 * ---------------------------------------------------------------------- */
/* score_paged, selector.cpp:26-68: s_out [H x T] fp32, q [H x d]. */
ts_status ts_score_paged(const ts_pool* pool, uint32_t seq, const float* q, size_t num_heads,
                         size_t head_dim, const uint32_t* candidates, size_t T,
                         size_t block_size, float* s_out);
/* select_with, selector.cpp:128-135 (+ select_topk / select_head_vote /
 * select_head_soft_vote :89-126, pick :72-85). sel_out/crit_out need
 * min(k, T) slots; *n_out receives the count. */
ts_status ts_select(const float* per_head, size_t num_heads, size_t T,
                    const uint32_t* candidate_idx, size_t k, int method, uint32_t* sel_out,
                    double* crit_out, size_t* n_out);
/* select_for_chunk, selector.cpp:137-150: q_chunk [c x width]. */
ts_status ts_select_for_chunk(const ts_pool* pool, uint32_t seq, const float* q_chunk, size_t c,
                              size_t width, const uint32_t* candidates, size_t T, size_t k,
                              int method, size_t block_size, uint32_t* sel_out, double* crit_out,
                              size_t* n_out);

/* ------------------------------------------------------------------------
 * Attention — attention.hpp:35-59
 * ---------------------------------------------------------------------- */
/* sparse_attend, attention.cpp:114-123: windows given as the three lists of
 * AttentionWindows (merged = sorted dedup union, attention.cpp:21-23).
 * q [C x H*d], k_cur/v_cur [C x H_kv*d], out [C x H*d]. */
ts_status ts_sparse_attend(const ts_pool* pool, uint32_t seq, const float* q,
                           const float* k_cur, const float* v_cur, size_t C, size_t num_heads,
                           const uint32_t* forced_init, size_t n_init, const uint32_t* selected,
                           size_t n_sel, const uint32_t* forced_local, size_t n_local,
                           float* out);

/* ------------------------------------------------------------------------
 * AttentionEngine — attention.hpp:94-115, attention.cpp:218-232, generalised
 * to n_seqs independent sequences (per-request page tables, one Selection
 * Cache entry each) that decode together in one launch.
 * ---------------------------------------------------------------------- */
ts_status ts_engine_create(const ts_engine_config* cfg, size_t capacity_tokens, size_t n_seqs,
                           ts_engine** out);
void ts_engine_destroy(ts_engine* eng);
/* Runs subsequent work on a caller-owned cudaStream_t (NULL: engine stream). */
ts_status ts_engine_set_stream(ts_engine* eng, void* stream);
/* Raw KV fill without attention (PagedKvPool::append_kv on the engine's
 * sequence) — fp32 or bf16 rows, host or device. */
ts_status ts_engine_append(ts_engine* eng, size_t seq, const float* k, const float* v, size_t t);
ts_status ts_engine_append_bf16(ts_engine* eng, size_t seq, const uint16_t* k,
                                const uint16_t* v, size_t t);
/* AttentionEngine::prefill / prefill(), attention.cpp:135-170 for sequence
 * `seq`: q [n x H*d], k/v [n x H_kv*d], out [n x H*d]. Optional trace: the
 * selection of every chunk concatenated in trace_sel (k per chunk max) with
 * per-chunk counts in trace_counts (max_chunks entries). */
ts_status ts_engine_prefill(ts_engine* eng, size_t seq, const float* q, const float* k,
                            const float* v, size_t n, float* out, uint32_t* trace_sel,
                            size_t* trace_counts, size_t max_chunks);
/* Stream-ordered prefill (no host sync, no trace): q/k/v/out must be device
 * buffers; errors of the queued work surface at the next ts_engine_sync.
 * Same computation as ts_engine_prefill (attention.cpp:135-170). */
ts_status ts_engine_prefill_async(ts_engine* eng, size_t seq, const float* q, const float* k,
                                  const float* v, size_t n, float* out);
/* AttentionEngine::decode / decode_step, attention.cpp:172-200, for all
 * n_seqs sequences at once: q [B x H*d], k/v [B x H_kv*d], out [B x H*d].
 * cache_hit [B] (optional), selected: if sel_out != NULL, B x k slots and
 * n_sel [B] — the raw (unfiltered) selection, attention.cpp:195. Blocks until
 * the step finished. */
ts_status ts_engine_decode(ts_engine* eng, const float* q, const float* k, const float* v,
                           float* out, int* cache_hit, uint32_t* sel_out, size_t* n_sel);
/* Stream-ordered variant for device-resident inputs/outputs: no host sync,
 * no D2H. Query validity (non-zero) is checked on the device: a zero query
 * makes the step append nothing and leave the Selection Cache untouched
 * (the reference throws before any mutation, selection_cache.cpp:18-27).
 * The next ts_engine_sync / ts_engine_stats call (before another step) rolls
 * the host's length back and returns TS_INVALID_ARGUMENT. ts_engine_decode
 * (blocking) reports it from the same call. */
ts_status ts_engine_decode_async(ts_engine* eng, const float* q, const float* k, const float* v,
                                 float* out);
/* Forces the next lookup of sequence `seq` to miss (first_flag = true,
 * selattn_bench.cpp:439 idiom). */
ts_status ts_engine_force_miss(ts_engine* eng, size_t seq);
/* Device phase trace of the fused decode kernel (tracing subsystem): when
 * enabled, thread 0 of every CTA stamps its SM clock64 at the phase
 * boundaries of the decode step into stamps[cta * 64 + phase]; slots 0 and 30
 * hold %globaltimer (ns) at the start and at the end (slot 12), slot 29 the
 * start clock. ts_engine_read_trace copies the first n stamps of the last
 * step (n <= 65536). */
ts_status ts_engine_set_trace(ts_engine* eng, int enable);
ts_status ts_engine_read_trace(ts_engine* eng, uint64_t* stamps, size_t n);
/* SelectionCacheEntry::theta of sequence `seq` (the reference reads theta
 * from the entry, selection_cache.cpp:34; the bench sets it by hand,
 * selattn_bench.cpp:239). */
ts_status ts_engine_set_theta(ts_engine* eng, size_t seq, double theta);
/* CacheStats + logical length (attention.hpp:102-103); blocks on the stream.
 * last_hit: -1 when the last step ran no lookup. */
ts_status ts_engine_stats(const ts_engine* eng, size_t seq, size_t* lookups, size_t* hits,
                          size_t* len, int* last_hit, double* last_cos);
/* The current cached selection (SelectionCacheEntry::cached_result) of `seq`. */
ts_status ts_engine_cached_selection(const ts_engine* eng, size_t seq, uint32_t* sel_out,
                                     double* crit_out, size_t* n_out);
/* SelectionCacheEntry of `seq` (selection_cache.hpp:23-29) beyond the cached
 * selection: the cached query [H*d] (nullable), first_flag and theta. */
ts_status ts_engine_cache_entry(const ts_engine* eng, size_t seq, float* cached_q, int* first_flag, double* theta);
ts_status ts_engine_sync(ts_engine* eng);
ts_pool* ts_engine_pool(ts_engine* eng);
uint32_t ts_engine_sequence(const ts_engine* eng, size_t seq);
/* Multi-layer engine (AttentionEngine generalised to a model's layers,
 * attention.cpp:218-232): n_layers x n_seqs sequences in one
 * pool, each (layer, sequence) with its own KV cache and Selection Cache
 * entry. Every engine call acts on the current layer (initially 0);
 * ts_engine_create is ts_engine_create_layers with n_layers = 1. */
ts_status ts_engine_create_layers(const ts_engine_config* cfg, size_t capacity_tokens, size_t n_seqs,
                                  size_t n_layers, ts_engine** out);
ts_status ts_engine_set_layer(ts_engine* eng, size_t layer);
size_t ts_engine_num_layers(const ts_engine* eng);
/* ------------------------------------------------------------------------
 * Tensor utilities (the free functions of the reference's Python module,
 * proj/python/bindings.cpp:60-116), computed on the device in fp64 like the
 * reference. Arrays may be host or device pointers; every call blocks.
 * ---------------------------------------------------------------------- */
/* softmax_rows, tensor.cpp:31-52: m and out are [rows x cols] fp32. */
ts_status ts_softmax_rows(const float* m, size_t rows, size_t cols, float* out);
/* topk_indices, tensor.cpp:68-90: the min(k, n) largest scores (the smaller
 * index wins a tie), indices ascending. n == 0 or k == 0: TS_INVALID_ARGUMENT. */
ts_status ts_topk_indices(const double* scores, size_t n, size_t k, uint32_t* out, size_t* n_out);
/* cosine, tensor.cpp:92-113 (fp64; +-1 exactly when dot^2 >= |u|^2 |v|^2;
 * a zero-norm input is TS_INVALID_ARGUMENT). */
ts_status ts_cosine(const double* u, const double* v, size_t n, double* out);
/* chunk_mean, tensor.cpp:133-150: column mean of q_chunk [c x width] in fp64,
 * rounded to fp32 (c == 1: identity). */
ts_status ts_chunk_mean(const float* q_chunk, size_t c, size_t width, float* out);
/* sdpa_full, attention.cpp:54-112: q [C x width] (width = H * d) over
 * k_all / v_all [N x kv_width] (N >= C, the last C rows are the current
 * tokens, causal among them), out [C x width]. */
ts_status ts_sdpa_full(const float* q, size_t C, size_t width, const float* k_all, const float* v_all, size_t N,
                       size_t kv_width, size_t num_heads, float* out);
/* ------------------------------------------------------------------------
 * KV-sequence-sharded decode (BASELINE config 4). Each
 * shard (rank) owns a contiguous range [base, base + len) of one sequence in
 * its own engine: rank 0 holds the init window, the last rank the local
 * window, the current token and every append. A decode step is four calls
 * on every rank with three all-gathers in between (NCCL over NVLink, or any
 * transport), all on device buffers and the engine's stream:
 *   ts_shard_stats      -> stats  [H][2]        all-gather -> [world][H][2]
 *   ts_shard_select     -> cands  [2k + 1] u32  all-gather -> [world][2k + 1]
 *   ts_shard_attend     -> out    [H*d], ml [H][2]  all-gather both (or, packed
 *                          into one [H*d + 2H] block, one all-gather)
 *   ts_shard_combine[_packed] -> the step's output [H*d] (identical on every rank)
 * The Selection Cache decision needs no exchange (q is replicated). Global
 * softmax statistics are combined in rank order, the global top-k is exact
 * (it is a subset of the union of the shards' local top-k), and outputs
 * merge by log-sum-exp: the result equals the unsharded decode_step
 * (attention.cpp:172-200) up to fp32 summation order.
 * ---------------------------------------------------------------------- */
ts_status ts_shard_engine_create(const ts_engine_config* cfg, size_t capacity_tokens, int rank, int world,
                                 ts_engine** out);
/* q, k, v: device [H*d], [H_kv*d]; n_global: the sequence length before the step. */
ts_status ts_shard_stats(ts_engine* eng, const float* q, const float* k, const float* v, size_t base,
                         size_t n_global, float* stats_out);
ts_status ts_shard_select(ts_engine* eng, const float* all_stats, uint32_t* cands_out);
ts_status ts_shard_attend(ts_engine* eng, const uint32_t* all_cands, float* out_partial, float* ml_out);
ts_status ts_shard_combine(const float* o_all, const float* ml_all, int world, size_t num_heads,
                           size_t head_dim, float* out, void* stream);
/* ts_shard_combine over one all-gather instead of two: every rank's block is
 * [H*d partial output | H x (M, L)], i.e. ts_shard_attend called with
 * ml_out = out_partial + H*d; packed_all is [world][H*d + 2H]. */
ts_status ts_shard_combine_packed(const float* packed_all, int world, size_t num_heads, size_t head_dim,
                                  float* out, void* stream);

/* Kernel launches issued by this library since process start (evidence
 * counter for the benchmark's gpu_launches field). */
/* In-library data plane of the sharded decode: an NCCL communicator the
 * library drives itself (libnccl resolved at run time: the copy already in
 * the process, else libnccl.so.2). Rank 0 makes the 128-byte unique id, the
 * host broadcasts it (any bootstrap), every rank creates its communicator.
 * world == 1 needs no id (id128 may be NULL). */
typedef struct ts_comm ts_comm;
ts_status ts_comm_unique_id(uint8_t* id128);
ts_status ts_comm_create(const uint8_t* id128, int world, int rank, ts_comm** out);
void ts_comm_destroy(ts_comm* comm);
/* One whole sharded decode step on this rank: ts_shard_stats -> all-gather ->
 * ts_shard_select -> all-gather -> ts_shard_attend -> all-gather ->
 * ts_shard_combine_packed, launches and ncclAllGather calls all on the
 * engine's stream, no host synchronisation (unless out is a host pointer).
 * out [H*d] is identical on every rank. comm may be NULL at world 1. */
ts_status ts_shard_decode_step(ts_engine* eng, ts_comm* comm, const float* q, const float* k, const float* v,
                               size_t base, size_t n_global, float* out);
uint64_t ts_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* TOKENSELECT_H */

// Launch descriptors shared by the host C-ABI layer (abi.cpp) and the
// kernels. Plain structs only: they are copied to the device per launch.
#pragma once

#include <cstdint>

namespace tsb {

// Selection Cache entry state (selection_cache.hpp:11-29), device resident.
struct CacheState {
  double theta;                  // selection_cache.cpp:34 reads theta from the entry
  double last_cos;               // cosine of the last lookup (NaN on first/forced miss)
  unsigned long long lookups;    // CacheStats::lookups
  unsigned long long hits;       // CacheStats::hits
  int first_flag;                // SelectionCacheEntry::first_flag
  int n_sel;                     // size of the cached SelectionResult
  int last_hit;                  // output of the last lookup (-1: no lookup this step)
  int error;                     // nonzero: zero query (lookup_or_select :18-27)
};

enum Mode : int {
  kModeCache = 1,    // run the Selection Cache test (Alg. 1) before selecting
  kModeScore = 2,    // compute S = q.K over the candidates (Alg. 2)
  kModeSelect = 4,   // per-head soft vote / raw sum + top-k
  kModeAttend = 8,   // sparse flash-decoding over the windows (+ current token)
  kModeAppend = 16,  // write the current token's K/V row into the pool
  kModeSOut = 32,    // also write S [H x T] to SeqDesc::s_out (score_paged API)
  kModeSIn = 64,     // S is given in SeqDesc::s_in (select API), skip the scan
  // KV-sequence-sharded decode (config 4), one launch per exchange phase:
  kModeShardStats = 128,   // stop after the scan: this shard's per-head (m, z) -> shard_stats
  kModeShardSelect = 256,  // resume from the spilled e^(S-m): global stats in, local top-k out
  kModeUseCached = 512,    // attend over the cache entry's selection (decided by an earlier launch)
};

// One sequence (request) of a launch. Everything is a device pointer.
struct SeqDesc {
  int32_t* page_table;         // frame per logical page
  int32_t n_cached;            // N: cached tokens at step start
  int32_t cand_begin;          // implicit candidate range [cand_begin, cand_begin + n_cand)
  int32_t n_cand;              // T
  const uint32_t* cand;        // explicit candidate list (nullptr: implicit range)
  int32_t select;              // 1: selection runs this step for this sequence
  const float* q;              // [H * d] query (decode row or chunk mean)
  const float* k_new;          // [H_kv * d] current token K (fp32)
  const float* v_new;          // [H_kv * d] current token V (fp32)
  float* out;                  // [H * d] attention output
  int32_t append_frame;        // frame that receives logical position n_cached (-1: none)
  int32_t append_slot;         // slot inside that frame
  int32_t append_page;         // page-table index of position n_cached
  int32_t init_end;            // implicit windows: [0, init_end) ...
  int32_t local_begin;         // ... and [max(local_begin, init_end), n_cached)
  const uint32_t* att_list;    // explicit attended (merged) list; nullptr: implicit windows
  int32_t n_att;
  // Selection Cache entry / selection result
  CacheState* cache;
  float* cached_q;             // [H * d]
  uint32_t* sel;               // [k] selected logical indices (the cached SelectionResult)
  float* sel_crit;             // [k] their criticality
  int32_t* sel_rows;           // [k] their slab rows (nullptr: resolve through the page table)
  // optional I/O for the standalone APIs
  float* s_out;                // [H x n_cand] scores out (kModeSOut)
  const float* s_in;           // [H x n_cand] scores in (kModeSIn)
  // sharded decode (kModeShard*, explicit-list attention)
  int32_t shard_base;          // global position of local position 0
  int32_t shard_world;         // number of shards
  float* shard_stats;          // out [H][2]: this shard's (m, z) per head
  const float* shard_all;      // in [world][H][2]: every shard's (m, z)
  uint32_t* shard_cands;       // out [2k + 1]: global indices, keys, count
  const int32_t* n_att_dev;    // device count of att_list (overrides n_att)
  float* ml_out;               // out [H][2]: (M, L) of the normalised output
  int32_t no_cur;              // 1: the current token belongs to another shard
  // synchronous host-buffer API: host-visible (mapped pinned) copy of the
  // cache entry, written by the sequence's CTA 0 at the end of the launch
  // (nullptr: none); `out` may then point into mapped pinned memory too
  CacheState* cache_mirror;
};

constexpr int kMaxSeqPerLaunch = 16;

struct DecodeParams {
  const uint16_t* k_slab;      // bf16 bits [frames][page_size][H_kv][d]
  const uint16_t* v_slab;
  uint16_t* k_slab_w;
  uint16_t* v_slab_w;
  int page_size;
  int H, H_kv, d;
  int k;                       // selection budget
  int method;                  // 0 topk (raw sum), 2 head_soft_vote
  int mode;
  float attn_scale;            // 1/sqrt(d) (attention.cpp:72)
  int n_seq;
  int ctas_per_seq;            // CTAs working on each sequence
  int tpc;                     // candidate tokens per CTA (max over sequences)
  int s_in_smem;               // S lives in shared memory (else ws_s)
  float* ws_s;                 // [n_ctas][H][tpc] S / exp(S - m) spill
  uint32_t* ws_keys;           // [n_ctas][tpc] selection keys spill
  float* ws_m;                 // [n_seq][H][stats_stride] per-CTA head max
  float* ws_z;                 // [n_seq][H][stats_stride] per-CTA head sum exp(S - m)
  uint32_t* ws_hist;           // [n_seq][2][kRadixBins] radix histograms (pass 1, pass 2)
  uint32_t* ws_cnt;            // [n_ctas] per-CTA count of keys tied at the threshold
  uint32_t* ws_nsel;           // [n_ctas] per-CTA count of selected candidates
  uint32_t* ws_sel_tok;        // [n_ctas][tpc] per-CTA selected token indices (ascending)
  float* ws_sel_crit;          // [n_ctas][tpc] their criticality
  int32_t* ws_sel_row;         // [n_ctas][tpc] their slab rows
  float* ws_att;               // [n_seq][H_kv][chunks][G][att_stride(d)] attention partials (o, m, l)
  unsigned int* ws_acnt;       // [n_seq][H_kv] arrival counters of the attention merge (self-resetting)
  unsigned int* bar;           // grid barrier counters: bar[0] / bar[32] alternate per launch
  int bar_slot;                // 0 or 32: this launch's counter (the other one is reset)
  int ring_bytes;              // shared-memory K ring (>= kRingBudget)
  int att_bytes;               // attention staging: the ring + the (then dead) S/keys region
  int debug_flags;             // dev timing: n << 8 ends the launch at stop point n (decode.cu)
  unsigned long long* trace;   // optional phase trace, [CTA][kTraceStride] clock64 stamps
  SeqDesc seqs[kMaxSeqPerLaunch];  // passed by value in the kernel parameter space
  // (kept last: the fields above keep their constant-bank offsets)
  // TMA tensor map (device memory) viewing the K slab as [128-B chunk][slab
  // row][64 bf16] with the 128B swizzle: one op brings a whole 16-row stage
  // (abi.cpp, encode_k_tmap); used by the general kernel when every stage is
  // 16 consecutive slab rows. nullptr: row-by-row copies.
  const void* k_tmap;
  int scan_tma;
  int any_select;  // some sequence of the launch selects (seqs[b].select)
  int any_radix;   // some selecting sequence has more candidates than k
};

}  // namespace tsb

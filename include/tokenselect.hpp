// tokenselect.hpp — header-only C++ drop-in for the reference's hot-path API
// (/root/reference/proj/include/selattn/{kv_pool,selector,attention}.hpp) over
// the C ABI in tokenselect.h.
//
// Same class / function names and argument meaning as namespace selattn, in
// namespace tokenselect; errors re-thrown with the reference's exception
// types and message text: std::invalid_argument, std::out_of_range and
// tokenselect::capacity_error (a std::runtime_error, like
// selattn::capacity_error, kv_pool.hpp:15-17). Matrices are row-major fp32
// host buffers as in selattn::Matrix (tensor.hpp:19-37); everything runs in
// the sm_100a kernels of libtokenselect.so (no CPU path).
//
// Source-compatible, not ABI-compatible: the reference's PagedKvPool keeps
// std::vector slabs in its private members (kv_pool.hpp:90-93); ours are bf16
// slabs in HBM behind an opaque handle.
#ifndef TOKENSELECT_HPP
#define TOKENSELECT_HPP

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tokenselect.h"

namespace tokenselect {

struct capacity_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(ts_status rc) {
  switch (rc) {
    case TS_OK: return;
    case TS_INVALID_ARGUMENT: throw std::invalid_argument(ts_last_error());
    case TS_OUT_OF_RANGE: throw std::out_of_range(ts_last_error());
    case TS_CAPACITY: throw capacity_error(ts_last_error());
    default: throw std::runtime_error(ts_last_error());
  }
}

using TokenIndex = std::uint32_t;
using IndexList = std::vector<TokenIndex>;

// selattn::Matrix (tensor.hpp:19-37): row-major fp32.
struct Matrix {
  std::size_t rows = 0, cols = 0;
  std::vector<float> data;
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.f) {}
  float* row(std::size_t i) { return data.data() + i * cols; }
  const float* row(std::size_t i) const { return data.data() + i * cols; }
};

enum class SelectionMethod { kTopK = TS_TOPK, kHeadVote = TS_HEAD_VOTE, kHeadSoftVote = TS_HEAD_SOFT_VOTE };

struct SequenceHandle {
  std::uint32_t seq_id = 0;
};

// PagedKvPool (kv_pool.hpp:33-95)
class PagedKvPool {
 public:
  PagedKvPool(std::size_t capacity_tokens, std::size_t page_size, std::size_t num_kv_heads,
              std::size_t head_dim) {
    check(ts_pool_create(capacity_tokens, page_size, num_kv_heads, head_dim, &h_));
  }
  explicit PagedKvPool(ts_pool* borrowed) : h_(borrowed), owned_(false) {}
  ~PagedKvPool() {
    if (owned_ && h_) ts_pool_destroy(h_);
  }
  PagedKvPool(const PagedKvPool&) = delete;
  PagedKvPool& operator=(const PagedKvPool&) = delete;

  SequenceHandle create_sequence() {
    SequenceHandle s;
    check(ts_pool_create_sequence(h_, &s.seq_id));
    return s;
  }
  std::pair<std::size_t, std::size_t> append_kv(SequenceHandle seq, const Matrix& k_new, const Matrix& v_new) {
    if (k_new.cols != row_width() || v_new.cols != row_width() || k_new.rows != v_new.rows)
      throw std::invalid_argument("append_kv: rows must be [t x (H_kv * d_h)]");
    std::size_t first = 0, last = 0;
    check(ts_pool_append_kv(h_, seq.seq_id, k_new.data.data(), v_new.data.data(), k_new.rows, &first, &last));
    return {first, last};
  }
  std::pair<Matrix, Matrix> gather(SequenceHandle seq, const IndexList& idx) const {
    Matrix k(idx.size(), row_width()), v(idx.size(), row_width());
    check(ts_pool_gather(h_, seq.seq_id, idx.data(), idx.size(), k.data.data(), v.data.data()));
    return {std::move(k), std::move(v)};
  }
  void release(SequenceHandle seq) { check(ts_pool_release(h_, seq.seq_id)); }
  std::size_t logical_len(SequenceHandle seq) const {
    std::size_t n = 0;
    check(ts_pool_logical_len(h_, seq.seq_id, &n));
    return n;
  }
  void shuffle_free_frames(std::uint64_t seed) { check(ts_pool_shuffle_free_frames(h_, seed)); }
  std::size_t page_size() const { return ts_pool_page_size(h_); }
  std::size_t num_kv_heads() const { return ts_pool_num_kv_heads(h_); }
  std::size_t head_dim() const { return ts_pool_head_dim(h_); }
  std::size_t row_width() const { return num_kv_heads() * head_dim(); }
  std::size_t total_frames() const { return ts_pool_total_frames(h_); }
  std::size_t free_frames() const { return ts_pool_free_frames(h_); }
  ts_pool* handle() const { return h_; }

 private:
  ts_pool* h_ = nullptr;
  bool owned_ = true;
};

// CriticalityScores / SelectionResult (selector.hpp:16-30)
struct CriticalityScores {
  Matrix per_head;  // [H x T]
  IndexList candidate_idx;
};
struct SelectionResult {
  IndexList selected;              // ascending
  std::vector<double> criticality;  // same order
};

// score_paged (selector.cpp:26-68)
inline CriticalityScores score_paged(const Matrix& q, const PagedKvPool& pool, SequenceHandle seq,
                                     const IndexList& candidates, std::size_t block_size) {
  CriticalityScores s;
  s.per_head = Matrix(q.rows, candidates.size());
  s.candidate_idx = candidates;
  check(ts_score_paged(pool.handle(), seq.seq_id, q.data.data(), q.rows, q.cols, candidates.data(),
                       candidates.size(), block_size, s.per_head.data.data()));
  return s;
}

// select_with (selector.cpp:128-135)
inline SelectionResult select_with(const CriticalityScores& s, std::size_t k, SelectionMethod method) {
  SelectionResult r;
  const std::size_t T = s.candidate_idx.size();
  r.selected.resize(std::max<std::size_t>(std::min(k, T), 1));
  r.criticality.resize(r.selected.size());
  std::size_t n = 0;
  check(ts_select(s.per_head.data.data(), s.per_head.rows, T, s.candidate_idx.data(), k, static_cast<int>(method),
                  r.selected.data(), r.criticality.data(), &n));
  r.selected.resize(n);
  r.criticality.resize(n);
  return r;
}

// select_for_chunk (selector.cpp:137-150)
inline SelectionResult select_for_chunk(const Matrix& q_chunk, const PagedKvPool& pool, SequenceHandle seq,
                                        const IndexList& candidates, std::size_t k, SelectionMethod method,
                                        std::size_t block_size) {
  SelectionResult r;
  r.selected.resize(std::max<std::size_t>(std::min(k, candidates.size()), 1));
  r.criticality.resize(r.selected.size());
  std::size_t n = 0;
  check(ts_select_for_chunk(pool.handle(), seq.seq_id, q_chunk.data.data(), q_chunk.rows, q_chunk.cols,
                            candidates.data(), candidates.size(), k, static_cast<int>(method), block_size,
                            r.selected.data(), r.criticality.data(), &n));
  r.selected.resize(n);
  r.criticality.resize(n);
  return r;
}

// ---------------------------------------------------------------- tensor utilities
// (tensor.hpp; computed on the device, fp64 like the reference)
inline Matrix softmax_rows(const Matrix& m) {
  Matrix out(m.rows, m.cols);
  check(ts_softmax_rows(m.data.data(), m.rows, m.cols, out.data.data()));
  return out;
}
inline IndexList topk_indices(const std::vector<double>& scores, std::size_t k) {
  IndexList out(std::max<std::size_t>(std::min(k, scores.size()), 1));
  std::size_t n = 0;
  check(ts_topk_indices(scores.data(), scores.size(), k, out.data(), &n));
  out.resize(n);
  return out;
}
template <typename T>
inline double cosine(const std::vector<T>& u, const std::vector<T>& v) {
  if (u.size() != v.size()) throw std::invalid_argument("cosine: length mismatch");
  std::vector<double> a(u.begin(), u.end()), b(v.begin(), v.end());
  double r = 0.0;
  check(ts_cosine(a.data(), b.data(), a.size(), &r));
  return r;
}
inline std::vector<float> chunk_mean(const Matrix& q_chunk) {
  std::vector<float> out(q_chunk.cols);
  check(ts_chunk_mean(q_chunk.data.data(), q_chunk.rows, q_chunk.cols, out.data()));
  return out;
}
// sdpa_full (attention.cpp:54-112)
inline Matrix sdpa_full(const Matrix& q, const Matrix& k_all, const Matrix& v_all, std::size_t num_heads) {
  if (k_all.rows != v_all.rows || k_all.cols != v_all.cols)
    throw std::invalid_argument("sdpa_full: K/V must be [(N + C) x (H_kv * d_h)]");
  Matrix out(q.rows, q.cols);
  check(ts_sdpa_full(q.data.data(), q.rows, q.cols, k_all.data.data(), v_all.data.data(), k_all.rows, k_all.cols,
                     num_heads, out.data.data()));
  return out;
}

// AttentionWindows (attention.hpp:32-39)
struct AttentionWindows {
  IndexList forced_init, selected, forced_local;
  // deduped ascending union (attention.cpp:21-33, tensor.cpp:159-168)
  IndexList merged() const {
    IndexList m;
    m.reserve(forced_init.size() + selected.size() + forced_local.size());
    m.insert(m.end(), forced_init.begin(), forced_init.end());
    m.insert(m.end(), selected.begin(), selected.end());
    m.insert(m.end(), forced_local.begin(), forced_local.end());
    std::sort(m.begin(), m.end());
    m.erase(std::unique(m.begin(), m.end()), m.end());
    return m;
  }
};

// selection_candidates / make_windows (attention.cpp:35-52): index-list
// plumbing on the host, as in the reference (the fused device decode keeps
// these ranges implicit)
inline IndexList selection_candidates(std::size_t cached_len, std::size_t n_init, std::size_t n_local) {
  IndexList c;
  if (cached_len <= n_init + n_local) return c;
  for (std::size_t i = n_init; i < cached_len - n_local; ++i) c.push_back(static_cast<TokenIndex>(i));
  return c;
}
inline AttentionWindows make_windows(std::size_t cached_len, std::size_t n_init, std::size_t n_local, IndexList selected) {
  AttentionWindows w;
  const std::size_t init_end = std::min(n_init, cached_len);
  const std::size_t local_begin = std::max(cached_len - std::min(n_local, cached_len), init_end);
  for (std::size_t i = 0; i < init_end; ++i) w.forced_init.push_back(static_cast<TokenIndex>(i));
  for (std::size_t i = local_begin; i < cached_len; ++i) w.forced_local.push_back(static_cast<TokenIndex>(i));
  for (TokenIndex t : selected)
    if (t >= init_end && t < local_begin) w.selected.push_back(t);
  return w;
}

// sparse_attend (attention.cpp:114-123)
inline Matrix sparse_attend(const Matrix& q, const Matrix& k_cur, const Matrix& v_cur, const PagedKvPool& pool,
                            SequenceHandle seq, const AttentionWindows& w, std::size_t num_heads) {
  Matrix out(q.rows, q.cols);
  check(ts_sparse_attend(pool.handle(), seq.seq_id, q.data.data(), k_cur.data.data(), v_cur.data.data(), q.rows,
                         num_heads, w.forced_init.data(), w.forced_init.size(), w.selected.data(), w.selected.size(),
                         w.forced_local.data(), w.forced_local.size(), out.data.data()));
  return out;
}

// EngineConfig (attention.hpp:12-27)
struct EngineConfig {
  std::size_t k = 2048, n_local = 512, n_init = 128, chunk_size = 512;
  double theta = 0.9;
  std::size_t num_heads = 8, num_kv_heads = 8, head_dim = 64, block_size = 64;
  SelectionMethod selection_method = SelectionMethod::kHeadSoftVote;
  std::size_t model_dim() const { return num_heads * head_dim; }
  std::size_t kv_dim() const { return num_kv_heads * head_dim; }
  ts_engine_config c() const {
    return ts_engine_config{k, n_local, n_init, chunk_size, theta, num_heads, num_kv_heads, head_dim, block_size,
                            static_cast<int>(selection_method)};
  }
  void validate() const {
    const ts_engine_config cc = c();
    check(ts_engine_config_validate(&cc));
  }
};

struct CacheStats {
  std::size_t lookups = 0, hits = 0;
};
// hit_rate (selection_cache.cpp:9-14)
inline double hit_rate(const CacheStats& s) {
  if (s.lookups == 0) throw std::invalid_argument("hit_rate: no lookups recorded");
  return static_cast<double>(s.hits) / static_cast<double>(s.lookups);
}

// SelectionCacheEntry / lookup_or_select (selection_cache.hpp:23-36,
// selection_cache.cpp:16-44): the generic host-callback form; the cosine
// runs on the device. (The engine's own entry lives on the device and is
// decided inside the fused decode kernel.)
struct SelectionCacheEntry {
  std::vector<float> cached_query;
  SelectionResult cached_result;
  bool first_flag = true;
  double theta = 0.9;
  CacheStats stats;
};
using SelectorFn = std::function<SelectionResult(const Matrix& q, std::size_t k)>;

inline std::pair<SelectionResult, bool> lookup_or_select(const Matrix& q, SelectionCacheEntry& entry, std::size_t k,
                                                         const SelectorFn& selector_fn) {
  bool all_zero = true;
  for (float x : q.data)
    if (x != 0.0f) {
      all_zero = false;
      break;
    }
  if (q.data.empty() || all_zero) throw std::invalid_argument("lookup_or_select: zero query vector");
  entry.stats.lookups += 1;
  bool miss = entry.first_flag;
  if (!miss) miss = cosine(q.data, entry.cached_query) < entry.theta;  // strict <
  if (miss) {
    entry.cached_result = selector_fn(q, k);
    entry.cached_query = q.data;
    entry.first_flag = false;
    return {entry.cached_result, false};
  }
  entry.stats.hits += 1;
  return {entry.cached_result, true};
}

// DecodeStep (attention.hpp:74-78)
struct DecodeStep {
  Matrix output;
  bool cache_hit = false;
  IndexList selected;
};

// ChunkTrace (attention.hpp:61-65)
struct ChunkTrace {
  std::size_t chunk_begin = 0, chunk_len = 0;
  IndexList selected;
};

namespace detail {
inline Matrix slice_rows(const Matrix& m, std::size_t begin, std::size_t count) {
  Matrix out(count, m.cols);
  std::copy(m.row(begin), m.row(begin) + count * m.cols, out.data.begin());
  return out;
}
}  // namespace detail

// prefill over a caller's pool (attention.cpp:135-170): per chunk,
// select_for_chunk -> make_windows -> sparse_attend -> append_kv, each step on
// the device
inline Matrix prefill(const Matrix& q_full, const Matrix& k_full, const Matrix& v_full, const EngineConfig& cfg,
                      PagedKvPool& pool, SequenceHandle seq, std::vector<ChunkTrace>* trace = nullptr) {
  cfg.validate();
  if (q_full.rows == 0) throw std::invalid_argument("prefill: empty input");
  if (q_full.cols != cfg.model_dim() || k_full.cols != cfg.kv_dim() || k_full.rows != v_full.rows ||
      k_full.cols != v_full.cols || k_full.rows != q_full.rows)
    throw std::invalid_argument("prefill: inconsistent input shapes");
  Matrix out(q_full.rows, q_full.cols);
  for (std::size_t begin = 0; begin < q_full.rows; begin += cfg.chunk_size) {
    const std::size_t len = std::min(cfg.chunk_size, q_full.rows - begin);
    Matrix qc = detail::slice_rows(q_full, begin, len), kc = detail::slice_rows(k_full, begin, len),
           vc = detail::slice_rows(v_full, begin, len);
    const std::size_t cached = pool.logical_len(seq);
    SelectionResult sel;
    if (cfg.k > 0) {
      IndexList cand = selection_candidates(cached, cfg.n_init, cfg.n_local);
      if (!cand.empty()) sel = select_for_chunk(qc, pool, seq, cand, cfg.k, cfg.selection_method, cfg.block_size);
    }
    if (trace) trace->push_back(ChunkTrace{begin, len, sel.selected});
    Matrix oc = sparse_attend(qc, kc, vc, pool, seq, make_windows(cached, cfg.n_init, cfg.n_local, sel.selected),
                              cfg.num_heads);
    std::copy(oc.data.begin(), oc.data.end(), out.row(begin));
    pool.append_kv(seq, kc, vc);
  }
  return out;
}

// decode_step over a caller's pool and cache entry (attention.cpp:172-200),
// each step on the device
inline DecodeStep decode_step(const Matrix& q_t, const Matrix& k_t, const Matrix& v_t, const EngineConfig& cfg,
                              PagedKvPool& pool, SequenceHandle seq, SelectionCacheEntry& cache) {
  cfg.validate();
  if (q_t.rows != 1 || q_t.cols != cfg.model_dim()) throw std::invalid_argument("decode_step: q must be [1 x (H * d_h)]");
  if (k_t.rows != 1 || k_t.cols != cfg.kv_dim() || v_t.rows != 1 || v_t.cols != cfg.kv_dim())
    throw std::invalid_argument("decode_step: KV must be [1 x (H_kv * d_h)]");
  const std::size_t cached = pool.logical_len(seq);
  DecodeStep step;
  SelectionResult sel;
  if (cfg.k > 0 && cached > cfg.n_init + cfg.n_local) {
    auto fn = [&](const Matrix& q, std::size_t k) {
      return select_for_chunk(q, pool, seq, selection_candidates(cached, cfg.n_init, cfg.n_local), k,
                              cfg.selection_method, cfg.block_size);
    };
    auto r = lookup_or_select(q_t, cache, cfg.k, fn);
    sel = std::move(r.first);
    step.cache_hit = r.second;
  }
  step.selected = sel.selected;
  step.output = sparse_attend(q_t, k_t, v_t, pool, seq, make_windows(cached, cfg.n_init, cfg.n_local, sel.selected),
                              cfg.num_heads);
  pool.append_kv(seq, k_t, v_t);
  return step;
}

// AttentionEngine (attention.hpp:94-115, attention.cpp:218-232)
class AttentionEngine {
 public:
  AttentionEngine(EngineConfig cfg, std::size_t capacity_tokens) : cfg_(cfg) {
    const ts_engine_config c = cfg_.c();
    check(ts_engine_create(&c, capacity_tokens, 1, &h_));
    pool_ = std::make_unique<PagedKvPool>(ts_engine_pool(h_));
  }
  ~AttentionEngine() {
    if (h_) ts_engine_destroy(h_);
  }
  AttentionEngine(const AttentionEngine&) = delete;
  AttentionEngine& operator=(const AttentionEngine&) = delete;

  Matrix prefill(const Matrix& q, const Matrix& k, const Matrix& v, std::vector<ChunkTrace>* trace = nullptr) {
    Matrix out(q.rows, q.cols);
    if (!trace) {
      check(ts_engine_prefill(h_, 0, q.data.data(), k.data.data(), v.data.data(), q.rows, out.data.data(), nullptr,
                              nullptr, 0));
      return out;
    }
    const std::size_t chunks = (q.rows + cfg_.chunk_size - 1) / std::max<std::size_t>(cfg_.chunk_size, 1);
    std::vector<std::size_t> counts(chunks);
    IndexList flat(std::max<std::size_t>(chunks * std::max<std::size_t>(cfg_.k, 1), 1));
    check(ts_engine_prefill(h_, 0, q.data.data(), k.data.data(), v.data.data(), q.rows, out.data.data(), flat.data(),
                            counts.data(), chunks));
    std::size_t off = 0;
    for (std::size_t c = 0; c < chunks; ++c) {
      const std::size_t b = c * cfg_.chunk_size;
      trace->push_back(ChunkTrace{b, std::min(cfg_.chunk_size, q.rows - b),
                                  IndexList(flat.begin() + off, flat.begin() + off + counts[c])});
      off += counts[c];
    }
    return out;
  }
  DecodeStep decode(const Matrix& q, const Matrix& k, const Matrix& v) {
    if (q.rows != 1 || q.cols != cfg_.model_dim()) throw std::invalid_argument("decode_step: q must be [1 x (H * d_h)]");
    if (k.rows != 1 || v.rows != 1 || k.cols != cfg_.kv_dim() || v.cols != cfg_.kv_dim())
      throw std::invalid_argument("decode_step: KV must be [1 x (H_kv * d_h)]");
    DecodeStep s;
    s.output = Matrix(1, cfg_.model_dim());
    s.selected.resize(std::max<std::size_t>(cfg_.k, 1));
    int hit = 0;
    std::size_t n = 0;
    check(ts_engine_decode(h_, q.data.data(), k.data.data(), v.data.data(), s.output.data.data(), &hit,
                           s.selected.data(), &n));
    s.selected.resize(n);
    s.cache_hit = hit != 0;
    return s;
  }
  std::size_t len() const { return stats().second; }
  CacheStats cache_stats() const {
    CacheStats c;
    std::size_t len = 0;
    int last = 0;
    double cs = 0;
    check(ts_engine_stats(h_, 0, &c.lookups, &c.hits, &len, &last, &cs));
    return c;
  }
  const EngineConfig& config() const { return cfg_; }
  ts_engine* handle() const { return h_; }
  // the device-resident SelectionCacheEntry, read back (attention.hpp:104)
  SelectionCacheEntry cache_entry() const {
    SelectionCacheEntry c;
    c.cached_query.resize(cfg_.model_dim());
    int ff = 1;
    check(ts_engine_cache_entry(h_, 0, c.cached_query.data(), &ff, &c.theta));
    c.first_flag = ff != 0;
    c.stats = cache_stats();
    IndexList sel(std::max<std::size_t>(cfg_.k, 1));
    std::vector<double> crit(sel.size());
    std::size_t n = 0;
    check(ts_engine_cached_selection(h_, 0, sel.data(), crit.data(), &n));
    sel.resize(n);
    crit.resize(n);
    c.cached_result = SelectionResult{sel, crit};
    return c;
  }
  // the engine's pool (borrowed) and sequence (attention.hpp:105-107)
  PagedKvPool& pool() { return *pool_; }
  SequenceHandle sequence() const { return SequenceHandle{ts_engine_sequence(h_, 0)}; }

 private:
  std::pair<std::size_t, std::size_t> stats() const {
    std::size_t lk = 0, hits = 0, len = 0;
    int last = 0;
    double cs = 0;
    check(ts_engine_stats(h_, 0, &lk, &hits, &len, &last, &cs));
    return {lk, len};
  }
  EngineConfig cfg_;
  ts_engine* h_ = nullptr;
  std::unique_ptr<PagedKvPool> pool_;  // borrowed view, made once the engine exists
};

}  // namespace tokenselect

#endif  // TOKENSELECT_HPP

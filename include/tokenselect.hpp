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

#include <cstddef>
#include <cstdint>
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

// AttentionWindows (attention.hpp:32-39)
struct AttentionWindows {
  IndexList forced_init, selected, forced_local;
};

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

// DecodeStep (attention.hpp:74-78)
struct DecodeStep {
  Matrix output;
  bool cache_hit = false;
  IndexList selected;
};

// AttentionEngine (attention.hpp:94-115, attention.cpp:218-232)
class AttentionEngine {
 public:
  AttentionEngine(EngineConfig cfg, std::size_t capacity_tokens) : cfg_(cfg) {
    const ts_engine_config c = cfg_.c();
    check(ts_engine_create(&c, capacity_tokens, 1, &h_));
  }
  ~AttentionEngine() {
    if (h_) ts_engine_destroy(h_);
  }
  AttentionEngine(const AttentionEngine&) = delete;
  AttentionEngine& operator=(const AttentionEngine&) = delete;

  Matrix prefill(const Matrix& q, const Matrix& k, const Matrix& v) {
    Matrix out(q.rows, q.cols);
    check(ts_engine_prefill(h_, 0, q.data.data(), k.data.data(), v.data.data(), q.rows, out.data.data(), nullptr,
                            nullptr, 0));
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
};

}  // namespace tokenselect

#endif  // TOKENSELECT_HPP

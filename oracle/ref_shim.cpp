// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/src/{tensor,kv_pool,selector,selection_cache,attention}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libselattn_ref.so. It lets the
// Python tests, the golden-vector generator and bench.py's cpu_baseline /
// --impl reference leg call the reference's own code path:
//   decode_step            attention.cpp:172-200
//   prefill                attention.cpp:135-170
//   score_paged            selector.cpp:26-68
//   select_with            selector.cpp:128-135
//   select_for_chunk       selector.cpp:137-150
//   lookup_or_select       selection_cache.cpp:16-44
//   sdpa_full              attention.cpp:54-112
//   sparse_attend          attention.cpp:114-123
//   topk_indices / cosine / softmax_rows / chunk_mean   tensor.cpp
// Every entry point returns 0 on success or a nonzero code and leaves the
// exception text in ref_last_error():
//   1 invalid_argument, 2 out_of_range, 3 capacity_error, 9 other.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "selattn/attention.hpp"
#include "selattn/kv_pool.hpp"
#include "selattn/selection_cache.hpp"
#include "selattn/selector.hpp"
#include "selattn/tensor.hpp"

using namespace selattn;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const capacity_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Matrix mat(const float* p, std::size_t r, std::size_t c) {
  Matrix m(r, c);
  if (r * c) std::memcpy(m.data.data(), p, r * c * sizeof(float));
  return m;
}

IndexList idx(const std::uint32_t* p, std::size_t n) { return IndexList(p, p + n); }

struct RefEngine {
  EngineConfig cfg;
  std::unique_ptr<AttentionEngine> eng;
};

SelectionMethod method_of(int m) {
  switch (m) {
    case 0: return SelectionMethod::kTopK;
    case 1: return SelectionMethod::kHeadVote;
    case 2: return SelectionMethod::kHeadSoftVote;
  }
  throw std::invalid_argument("ref_shim: bad method id");
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- pool-level helpers: the pool is rebuilt from logical rows per call so
// the physical layout is the reference allocator's (optionally shuffled).
int ref_score_paged(const float* q, std::size_t H, std::size_t d, const float* k_rows,
                    std::size_t n_tokens, std::size_t H_kv, std::size_t page_size,
                    std::uint64_t shuffle_seed, const std::uint32_t* cand, std::size_t T,
                    std::size_t block, float* s_out) {
  return guarded([&] {
    PagedKvPool pool(n_tokens + 1, page_size, H_kv, d);
    if (shuffle_seed) pool.shuffle_free_frames(shuffle_seed);
    SequenceHandle seq = pool.create_sequence();
    Matrix k = mat(k_rows, n_tokens, H_kv * d);
    pool.append_kv(seq, k, k);
    CriticalityScores s = score_paged(mat(q, H, d), pool, seq, idx(cand, T), block);
    if (!s.per_head.data.empty())
      std::memcpy(s_out, s.per_head.data.data(), s.per_head.data.size() * sizeof(float));
  });
}

int ref_select(const float* per_head, std::size_t H, std::size_t T, const std::uint32_t* cand,
               std::size_t k, int method, std::uint32_t* sel_out, double* crit_out,
               std::size_t* n_out) {
  return guarded([&] {
    CriticalityScores s;
    s.per_head = mat(per_head, H, T);
    s.candidate_idx = idx(cand, T);
    SelectionResult r = select_with(s, k, method_of(method));
    *n_out = r.selected.size();
    for (std::size_t i = 0; i < r.selected.size(); ++i) {
      sel_out[i] = r.selected[i];
      crit_out[i] = r.criticality[i];
    }
  });
}

int ref_select_for_chunk(const float* q_chunk, std::size_t c, std::size_t width,
                         const float* k_rows, std::size_t n_tokens, std::size_t H_kv,
                         std::size_t d, const std::uint32_t* cand, std::size_t T, std::size_t k,
                         int method, std::size_t block, std::uint32_t* sel_out, double* crit_out,
                         std::size_t* n_out) {
  return guarded([&] {
    PagedKvPool pool(n_tokens + 1, 1, H_kv, d);
    SequenceHandle seq = pool.create_sequence();
    Matrix kk = mat(k_rows, n_tokens, H_kv * d);
    pool.append_kv(seq, kk, kk);
    SelectionResult r = select_for_chunk(mat(q_chunk, c, width), pool, seq, idx(cand, T), k,
                                         method_of(method), block);
    *n_out = r.selected.size();
    for (std::size_t i = 0; i < r.selected.size(); ++i) {
      sel_out[i] = r.selected[i];
      crit_out[i] = r.criticality[i];
    }
  });
}

int ref_topk_indices(const double* scores, std::size_t n, std::size_t k, std::uint32_t* out,
                     std::size_t* n_out) {
  return guarded([&] {
    IndexList r = topk_indices(std::span<const double>(scores, n), k);
    *n_out = r.size();
    std::memcpy(out, r.data(), r.size() * sizeof(std::uint32_t));
  });
}

int ref_cosine_f32(const float* u, const float* v, std::size_t n, double* out) {
  return guarded([&] { *out = cosine(std::span<const float>(u, n), std::span<const float>(v, n)); });
}

int ref_softmax_rows(const float* m, std::size_t r, std::size_t c, float* out) {
  return guarded([&] {
    Matrix p = softmax_rows(mat(m, r, c));
    if (r * c) std::memcpy(out, p.data.data(), r * c * sizeof(float));
  });
}

int ref_chunk_mean(const float* q, std::size_t c, std::size_t width, float* out) {
  return guarded([&] {
    std::vector<float> m = chunk_mean(mat(q, c, width));
    std::memcpy(out, m.data(), m.size() * sizeof(float));
  });
}

int ref_sdpa_full(const float* q, std::size_t C, std::size_t q_width, const float* k_all,
                  const float* v_all, std::size_t rows, std::size_t kv_width, std::size_t H,
                  float* out) {
  return guarded([&] {
    Matrix o = sdpa_full(mat(q, C, q_width), mat(k_all, rows, kv_width), mat(v_all, rows, kv_width), H);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// Windows: writes the merged (deduped ascending) list; returns sizes of the
// three disjoint parts too.
int ref_make_windows(std::size_t cached, std::size_t n_init, std::size_t n_local,
                     const std::uint32_t* sel, std::size_t n_sel, std::uint32_t* merged_out,
                     std::size_t* n_merged, std::size_t* n_init_out, std::size_t* n_sel_out,
                     std::size_t* n_local_out) {
  return guarded([&] {
    AttentionWindows w = make_windows(cached, n_init, n_local, idx(sel, n_sel));
    IndexList m = w.merged();
    *n_merged = m.size();
    std::memcpy(merged_out, m.data(), m.size() * sizeof(std::uint32_t));
    *n_init_out = w.forced_init.size();
    *n_sel_out = w.selected.size();
    *n_local_out = w.forced_local.size();
  });
}

int ref_selection_candidates(std::size_t cached, std::size_t n_init, std::size_t n_local,
                             std::size_t* begin, std::size_t* count) {
  return guarded([&] {
    IndexList c = selection_candidates(cached, n_init, n_local);
    *count = c.size();
    *begin = c.empty() ? 0 : c.front();
  });
}

// sparse_attend over a freshly built pool holding n_tokens logical rows.
int ref_sparse_attend(const float* q, const float* k_cur, const float* v_cur, std::size_t C,
                      const float* k_rows, const float* v_rows, std::size_t n_tokens,
                      std::size_t H, std::size_t H_kv, std::size_t d, const std::uint32_t* init,
                      std::size_t n_init, const std::uint32_t* sel, std::size_t n_sel,
                      const std::uint32_t* local, std::size_t n_local, float* out) {
  return guarded([&] {
    PagedKvPool pool(n_tokens + 1, 1, H_kv, d);
    SequenceHandle seq = pool.create_sequence();
    pool.append_kv(seq, mat(k_rows, n_tokens, H_kv * d), mat(v_rows, n_tokens, H_kv * d));
    AttentionWindows w;
    w.forced_init = idx(init, n_init);
    w.selected = idx(sel, n_sel);
    w.forced_local = idx(local, n_local);
    Matrix o = sparse_attend(mat(q, C, H * d), mat(k_cur, C, H_kv * d), mat(v_cur, C, H_kv * d),
                             pool, seq, w, H);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// ---- engine: AttentionEngine (attention.cpp:218-232), page_size 1.
void* ref_engine_create(std::size_t k, std::size_t n_local, std::size_t n_init,
                        std::size_t chunk_size, double theta, std::size_t H, std::size_t H_kv,
                        std::size_t d, std::size_t block, int method, std::size_t capacity) {
  void* out = nullptr;
  int rc = guarded([&] {
    auto* e = new RefEngine;
    e->cfg.k = k;
    e->cfg.n_local = n_local;
    e->cfg.n_init = n_init;
    e->cfg.chunk_size = chunk_size;
    e->cfg.theta = theta;
    e->cfg.num_heads = H;
    e->cfg.num_kv_heads = H_kv;
    e->cfg.head_dim = d;
    e->cfg.block_size = block;
    e->cfg.selection_method = method_of(method);
    e->eng = std::make_unique<AttentionEngine>(e->cfg, capacity);
    out = e;
  });
  return rc == 0 ? out : nullptr;
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

// Raw KV fill (no attention): PagedKvPool::append_kv on the engine's sequence.
int ref_engine_append(void* h, const float* k, const float* v, std::size_t t) {
  return guarded([&] {
    auto* e = static_cast<RefEngine*>(h);
    e->eng->pool().append_kv(e->eng->sequence(), mat(k, t, e->cfg.kv_dim()), mat(v, t, e->cfg.kv_dim()));
  });
}

int ref_engine_decode(void* h, const float* q, const float* k, const float* v, float* out,
                      int* hit, std::uint32_t* sel_out, std::size_t* n_sel) {
  return guarded([&] {
    auto* e = static_cast<RefEngine*>(h);
    DecodeStep s = e->eng->decode(mat(q, 1, e->cfg.model_dim()), mat(k, 1, e->cfg.kv_dim()),
                                  mat(v, 1, e->cfg.kv_dim()));
    std::memcpy(out, s.output.data.data(), s.output.data.size() * sizeof(float));
    *hit = s.cache_hit ? 1 : 0;
    if (n_sel) *n_sel = s.selected.size();
    if (sel_out) std::memcpy(sel_out, s.selected.data(), s.selected.size() * sizeof(std::uint32_t));
  });
}

// decode_step against the engine's pool with an externally held cache entry
// flag: force_miss sets first_flag (selattn_bench.cpp:439 idiom).
int ref_engine_force_miss(void* h) {
  return guarded([&] {
    auto* e = static_cast<RefEngine*>(h);
    const_cast<SelectionCacheEntry&>(e->eng->cache_entry()).first_flag = true;
  });
}

int ref_engine_prefill(void* h, const float* q, const float* k, const float* v, std::size_t n,
                       float* out) {
  return guarded([&] {
    auto* e = static_cast<RefEngine*>(h);
    Matrix o = e->eng->prefill(mat(q, n, e->cfg.model_dim()), mat(k, n, e->cfg.kv_dim()),
                               mat(v, n, e->cfg.kv_dim()));
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

int ref_engine_prefill_trace(void* h, const float* q, const float* k, const float* v,
                             std::size_t n, float* out, std::uint32_t* sel_flat,
                             std::size_t* sel_counts, std::size_t max_chunks) {
  return guarded([&] {
    auto* e = static_cast<RefEngine*>(h);
    std::vector<ChunkTrace> trace;
    Matrix o = e->eng->prefill(mat(q, n, e->cfg.model_dim()), mat(k, n, e->cfg.kv_dim()),
                               mat(v, n, e->cfg.kv_dim()), &trace);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    std::size_t off = 0;
    for (std::size_t c = 0; c < trace.size() && c < max_chunks; ++c) {
      sel_counts[c] = trace[c].selected.size();
      std::memcpy(sel_flat + off, trace[c].selected.data(),
                  trace[c].selected.size() * sizeof(std::uint32_t));
      off += trace[c].selected.size();
    }
  });
}

void ref_engine_stats(void* h, std::size_t* lookups, std::size_t* hits, std::size_t* len) {
  auto* e = static_cast<RefEngine*>(h);
  *lookups = e->eng->cache_stats().lookups;
  *hits = e->eng->cache_stats().hits;
  *len = e->eng->len();
}

// lookup_or_select with a stub selector returning a distinct set per call
// (test_selection_cache.cpp CountingSelector pattern) — pins Alg. 1 alone.
void* ref_cache_create(double theta) {
  auto* c = new SelectionCacheEntry;
  c->theta = theta;
  return c;
}
void ref_cache_destroy(void* c) { delete static_cast<SelectionCacheEntry*>(c); }
int ref_cache_lookup(void* c, const float* q, std::size_t n, int* hit, std::uint64_t* selector_calls) {
  return guarded([&] {
    auto* e = static_cast<SelectionCacheEntry*>(c);
    SelectorFn fn = [&](const Matrix&, std::size_t kk) {
      ++*selector_calls;
      SelectionResult r;
      for (std::size_t i = 0; i < kk; ++i) r.selected.push_back(static_cast<TokenIndex>(100 * *selector_calls + i));
      r.criticality.assign(kk, static_cast<double>(*selector_calls));
      return r;
    };
    auto res = lookup_or_select(mat(q, 1, n), *e, 2, fn);
    *hit = res.second ? 1 : 0;
  });
}
void ref_cache_stats(void* c, std::size_t* lookups, std::size_t* hits) {
  auto* e = static_cast<SelectionCacheEntry*>(c);
  *lookups = e->stats.lookups;
  *hits = e->stats.hits;
}

}  // extern "C"

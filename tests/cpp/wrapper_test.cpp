// Drives the header-only C++ drop-in (include/tokenselect.hpp) the way the
// reference's own tests drive selattn (test_selector.cpp:47-55,
// test_kv_pool.cpp:82-111, test_attention.cpp:341-372): prints one line per
// check and exits non-zero on the first failure. Built and run by
// tests/test_cpp_wrapper.py (GPU).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "tokenselect.hpp"

using namespace tokenselect;

#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                               \
    }                                                         \
  } while (0)

int main() {
  // score_paged known answer: q = k = (1,2,3,4) -> 30
  {
    PagedKvPool pool(4, 1, 1, 4);
    SequenceHandle s = pool.create_sequence();
    Matrix q(1, 4);
    for (int i = 0; i < 4; ++i) q.data[i] = float(i + 1);
    pool.append_kv(s, q, q);
    CriticalityScores c = score_paged(q, pool, s, IndexList{0}, 8);
    CHECK(c.per_head.data[0] == 30.f);
    std::printf("ok score_paged known answer\n");
  }
  // out_of_range with the reference's message, capacity_error with no partial append
  {
    PagedKvPool pool(8, 1, 1, 4);
    SequenceHandle s = pool.create_sequence();
    Matrix k(6, 4);
    pool.append_kv(s, k, k);
    bool thrown = false;
    try {
      pool.gather(s, IndexList{2, 7});
    } catch (const std::out_of_range& e) {
      thrown = std::strstr(e.what(), "index 7") != nullptr;
    }
    CHECK(thrown);
    thrown = false;
    try {
      Matrix k3(3, 4);
      pool.append_kv(s, k3, k3);
    } catch (const capacity_error&) {
      thrown = true;
    }
    CHECK(thrown && pool.logical_len(s) == 6 && pool.free_frames() == 2);
    std::printf("ok error contract\n");
  }
  // select_with known answers (test_selector.cpp:128-141)
  {
    CriticalityScores c;
    c.per_head = Matrix(2, 4);
    const float v[8] = {5, 4.5f, 0, 0, 0, 0, 500, 480};
    std::memcpy(c.per_head.data.data(), v, sizeof v);
    c.candidate_idx = {0, 1, 2, 3};
    CHECK((select_with(c, 2, SelectionMethod::kTopK).selected == IndexList{2, 3}));
    CHECK((select_with(c, 2, SelectionMethod::kHeadSoftVote).selected == IndexList{0, 2}));
    std::printf("ok select_with known answers\n");
  }
  // engine: identical queries hit and return identical output
  {
    EngineConfig cfg;
    cfg.k = 8; cfg.n_init = 4; cfg.n_local = 0; cfg.chunk_size = 16; cfg.num_heads = 2; cfg.num_kv_heads = 2;
    cfg.head_dim = 4; cfg.block_size = 8;
    AttentionEngine eng(cfg, 96);
    std::mt19937 g(7);
    std::normal_distribution<float> n01;
    Matrix q(64, 8), k(64, 8), v(64, 8);
    for (auto* m : {&q, &k, &v})
      for (float& x : m->data) x = n01(g);
    eng.prefill(q, k, v);
    Matrix qt(1, 8), kt(1, 8), vt(1, 8);
    for (auto* m : {&qt, &kt, &vt})
      for (float& x : m->data) x = n01(g);
    DecodeStep a = eng.decode(qt, kt, vt);
    DecodeStep b = eng.decode(qt, kt, vt);
    CHECK(!a.cache_hit && b.cache_hit && a.selected == b.selected && a.output.data == b.output.data);
    CHECK(eng.cache_stats().lookups == 2 && eng.cache_stats().hits == 1 && eng.len() == 66);
    std::printf("ok engine decode hit\n");
  }
  // windows known answers (test_attention.cpp:233-252)
  {
    CHECK((selection_candidates(10, 4, 4) == IndexList{4, 5}));
    AttentionWindows w = make_windows(100, 4, 8, IndexList{2, 5, 6, 90});
    CHECK((w.selected == IndexList{5, 6, 90}) && w.forced_local.front() == 92 && w.forced_init.size() == 4);
    AttentionWindows w2 = make_windows(6, 4, 4, IndexList{});
    CHECK((w2.merged() == IndexList{0, 1, 2, 3, 4, 5}));
    std::printf("ok windows\n");
  }
  // tensor utilities on the device (tensor.cpp; smoke_test.py:8-28)
  {
    CHECK((topk_indices(std::vector<double>{5, 1, 9}, 2) == IndexList{0, 2}));
    CHECK((topk_indices(std::vector<double>{7, 7, 7}, 2) == IndexList{0, 1}));
    CHECK(cosine(std::vector<float>{1, 2, -3}, std::vector<float>{1, 2, -3}) == 1.0);
    Matrix m(1, 3);
    m.data = {1, 2, 3};
    Matrix p = softmax_rows(m);
    CHECK(std::fabs(p.data[0] + p.data[1] + p.data[2] - 1.0f) < 1e-6f && p.data[2] > p.data[1]);
    std::printf("ok tensor utilities\n");
  }
  // lookup_or_select semantics with a stub selector (test_selection_cache.cpp:34-82)
  {
    SelectionCacheEntry e;
    e.theta = 0.5;
    int calls = 0;
    SelectorFn stub = [&](const Matrix&, std::size_t k) {
      ++calls;
      SelectionResult r;
      for (std::size_t i = 0; i < k; ++i) r.selected.push_back(static_cast<TokenIndex>(i + calls));
      r.criticality.assign(k, 1.0);
      return r;
    };
    Matrix a(1, 2), b(1, 2), c(1, 2), z(1, 2);
    a.data = {1, 0};
    b.data = {1, 1};   // cos(a, b) = 0.7071 >= 0.5: hit
    c.data = {0, 1};   // cos(a, c) = 0: miss
    auto r1 = lookup_or_select(a, e, 2, stub);
    auto r2 = lookup_or_select(b, e, 2, stub);
    auto r3 = lookup_or_select(c, e, 2, stub);
    CHECK(!r1.second && r2.second && !r3.second && calls == 2 && e.stats.lookups == 3 && e.stats.hits == 1);
    bool thrown = false;
    try {
      lookup_or_select(z, e, 2, stub);
    } catch (const std::invalid_argument& ex) {
      thrown = std::strstr(ex.what(), "zero query") != nullptr;
    }
    CHECK(thrown && e.stats.lookups == 3);
    std::printf("ok lookup_or_select\n");
  }
  // free decode_step / prefill over a caller's pool == the engine (attention.cpp:135-200)
  {
    EngineConfig cfg;
    cfg.k = 16; cfg.n_init = 4; cfg.n_local = 8; cfg.chunk_size = 32; cfg.num_heads = 4; cfg.num_kv_heads = 2;
    cfg.head_dim = 32; cfg.block_size = 8;
    std::mt19937 g(11);
    std::normal_distribution<float> n01;
    auto bf16 = [](float x) {  // bf16-representable inputs: both paths store bf16
      std::uint32_t u;
      std::memcpy(&u, &x, 4);
      u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
      std::memcpy(&x, &u, 4);
      return x;
    };
    const std::size_t n = 200;
    Matrix q(n, 128), k(n, 64), v(n, 64);
    for (float& x : q.data) x = n01(g);
    for (float& x : k.data) x = bf16(n01(g));
    for (float& x : v.data) x = bf16(n01(g));
    AttentionEngine eng(cfg, n + 16);
    std::vector<ChunkTrace> t1, t2;
    Matrix o1 = eng.prefill(q, k, v, &t1);
    PagedKvPool pool(n + 16, 1, 2, 32);
    SequenceHandle s = pool.create_sequence();
    Matrix o2 = prefill(q, k, v, cfg, pool, s, &t2);
    CHECK(t1.size() == t2.size() && t1.size() == 7);
    double err = 0, ref = 0;
    for (std::size_t i = 0; i < o1.data.size(); ++i) {
      err += (o1.data[i] - o2.data[i]) * double(o1.data[i] - o2.data[i]);
      ref += double(o2.data[i]) * o2.data[i];
    }
    CHECK(std::sqrt(err / ref) <= 1e-5);
    SelectionCacheEntry cache;
    cache.theta = cfg.theta;
    Matrix qt(1, 128), kt(1, 64), vt(1, 64);
    for (int step = 0; step < 3; ++step) {
      if (step != 1)
        for (float& x : qt.data) x = n01(g);
      for (float& x : kt.data) x = bf16(n01(g));
      for (float& x : vt.data) x = bf16(n01(g));
      DecodeStep a = eng.decode(qt, kt, vt);
      DecodeStep b = decode_step(qt, kt, vt, cfg, pool, s, cache);
      CHECK(a.cache_hit == b.cache_hit && a.cache_hit == (step == 1));
      double e2 = 0, r2 = 0;
      for (std::size_t i = 0; i < a.output.data.size(); ++i) {
        e2 += (a.output.data[i] - b.output.data[i]) * double(a.output.data[i] - b.output.data[i]);
        r2 += double(b.output.data[i]) * b.output.data[i];
      }
      CHECK(std::sqrt(e2 / r2) <= 1e-5);
    }
    SelectionCacheEntry ce = eng.cache_entry();
    CHECK(ce.stats.lookups == 3 && ce.stats.hits == 1 && !ce.first_flag && ce.cached_query.size() == 128);
    CHECK(ce.cached_result.selected.size() == cfg.k && eng.pool().logical_len(eng.sequence()) == n + 3);
    std::printf("ok free decode_step / prefill\n");
  }
  std::printf("ALL OK\n");
  return 0;
}

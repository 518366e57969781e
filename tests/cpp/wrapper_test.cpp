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
  std::printf("ALL OK\n");
  return 0;
}

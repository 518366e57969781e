/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, loaded by,
 * or called from the product library (paper_2411_02886_b200/).
 *
 * Plain-C restatement of the reference's decode selection + sparse-attention
 * path (/root/reference/proj/src/*.cpp). Storage fp32, every dot product and
 * softmax sum accumulated in fp64, exactly as the reference does, in the same
 * loop order, so the restatement is bit-identical to the reference when both
 * are built with the same flags (pinned by tests/test_oracle_*.py against
 * oracle/_ref and tests/golden/).
 *
 * Status codes mirror the reference's exception types:
 *   0 ok, 1 invalid_argument, 2 out_of_range, 3 capacity_error.
 */
#ifndef TSORACLE_H
#define TSORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oc_last_error(void);

/* selector.cpp:26-68 (score_paged, Alg. 2): S[h][j] = sum_d q[h][d]*K[cand[j]][h mod H_kv][d].
 * k_rows holds the LOGICAL rows [n_tokens x H_kv*d]; physical paging is
 * unobservable by construction (kv_pool.hpp:24-29). */
int oc_score(const float* q, size_t H, size_t d, const float* k_rows, size_t n_tokens,
             size_t H_kv, const uint32_t* cand, size_t T, float* s_out);

/* tensor.cpp:31-52 */
void oc_softmax_rows(const float* m, size_t rows, size_t cols, float* out);

/* tensor.cpp:68-90: k largest, ties to the smaller index, output ascending. */
int oc_topk_indices_f64(const double* s, size_t n, size_t k, uint32_t* out, size_t* n_out);
int oc_topk_indices_f32(const float* s, size_t n, size_t k, uint32_t* out, size_t* n_out);

/* selector.cpp:72-135: method 0 = topk (Eq. 5), 1 = head_vote (Eq. 6),
 * 2 = head_soft_vote (Eq. 7). Writes min(k,T) selected indices (ascending)
 * and their criticality. */
int oc_select(const float* per_head, size_t H, size_t T, const uint32_t* cand, size_t k,
              int method, uint32_t* sel_out, double* crit_out, size_t* n_out);

/* Full criticality vector (length T) for a method, before pick(). */
int oc_criticality(const float* per_head, size_t H, size_t T, size_t k, int method,
                   double* crit_out);

/* tensor.cpp:92-113 */
int oc_cosine_f32(const float* u, const float* v, size_t n, double* out);

/* tensor.cpp:133-150 */
int oc_chunk_mean(const float* q, size_t c, size_t width, float* out);

/* attention.cpp:25-33 — returns count; *begin set when count > 0. */
size_t oc_selection_candidates(size_t cached, size_t n_init, size_t n_local, size_t* begin);

/* attention.cpp:35-52 + merged() :21-23. merged_out needs n_init+n_sel+n_local slots. */
size_t oc_make_windows(size_t cached, size_t n_init, size_t n_local, const uint32_t* sel,
                       size_t n_sel, uint32_t* merged_out, size_t* n_sel_kept);

/* attention.cpp:54-112 over gathered rows: q [C x H*d], k_all/v_all
 * [(N+C) x H_kv*d] (cached rows first, current rows last), causal among the
 * current rows. */
int oc_sdpa(const float* q, size_t C, size_t H, size_t d, const float* k_all,
            const float* v_all, size_t rows, size_t H_kv, float* out);

/* attention.cpp:114-123: gather `attended` from logical rows, append the
 * current C rows, then oc_sdpa. */
int oc_sparse_attend(const float* q, const float* k_cur, const float* v_cur, size_t C,
                     const float* k_rows, const float* v_rows, size_t n_tokens, size_t H,
                     size_t H_kv, size_t d, const uint32_t* attended, size_t n_att, float* out);

/* ---- engine: AttentionEngine + decode_step + prefill (attention.cpp:135-232)
 * with the Selection Cache (selection_cache.cpp:16-44). */
typedef struct oc_engine oc_engine;

oc_engine* oc_engine_create(size_t k, size_t n_local, size_t n_init, size_t chunk_size,
                            double theta, size_t H, size_t H_kv, size_t d, size_t block,
                            int method, size_t capacity);
void oc_engine_destroy(oc_engine* e);
int oc_engine_append(oc_engine* e, const float* k, const float* v, size_t t);
int oc_engine_decode(oc_engine* e, const float* q, const float* k, const float* v, float* out,
                     int* hit, uint32_t* sel_out, size_t* n_sel, double* cos_out);
int oc_engine_prefill(oc_engine* e, const float* q, const float* k, const float* v, size_t n,
                      float* out, uint32_t* sel_flat, size_t* sel_counts, size_t max_chunks);
void oc_engine_force_miss(oc_engine* e);
void oc_engine_stats(const oc_engine* e, size_t* lookups, size_t* hits, size_t* len);
const float* oc_engine_k_rows(const oc_engine* e);
const float* oc_engine_v_rows(const oc_engine* e);

#ifdef __cplusplus
}
#endif
#endif

/* TEST INFRASTRUCTURE ONLY — CPU oracle (see tsoracle.h). Plain C restatement
 * of /root/reference/proj/src/{tensor,selector,selection_cache,attention}.cpp.
 * Each function cites the reference lines it follows. Compiled with the same
 * flags as oracle/_ref (-O2, no FMA contraction) so results are bit-identical.
 */
#include "tsoracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* oc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---------------------------------------------------------------- scoring */
/* selector.cpp:26-68. block_size only tiles the loop (Alg. 2),
 * so it is not a parameter here: the per-(h,j) fp64 sum is order-identical. */
int oc_score(const float* q, size_t H, size_t d, const float* k_rows, size_t n_tokens,
             size_t H_kv, const uint32_t* cand, size_t T, float* s_out) {
  if (H == 0 || H_kv == 0 || H % H_kv != 0)
    return fail(1, "score_paged: H must be a positive multiple of H_kv");
  const size_t row = H_kv * d;
  for (size_t j = 0; j < T; ++j)
    if (cand[j] >= n_tokens) return fail(2, "key_row: index out of range");
  for (size_t h = 0; h < H; ++h) {
    const float* qh = q + h * d;
    const size_t off = (h % H_kv) * d; /* selector.cpp:51 — h mod H_kv */
    for (size_t j = 0; j < T; ++j) {
      const float* key = k_rows + (size_t)cand[j] * row + off;
      double acc = 0.0;
      for (size_t t = 0; t < d; ++t) acc += (double)qh[t] * (double)key[t];
      s_out[h * T + j] = (float)acc;
    }
  }
  return 0;
}

/* tensor.cpp:31-52 */
void oc_softmax_rows(const float* m, size_t rows, size_t cols, float* out) {
  for (size_t i = 0; i < rows; ++i) {
    const float* src = m + i * cols;
    float* dst = out + i * cols;
    double mx = -HUGE_VAL;
    for (size_t j = 0; j < cols; ++j) mx = fmax(mx, (double)src[j]);
    double sum = 0.0;
    for (size_t j = 0; j < cols; ++j) {
      double e = exp((double)src[j] - mx);
      dst[j] = (float)e;
      sum += e;
    }
    double inv = 1.0 / sum;
    for (size_t j = 0; j < cols; ++j) dst[j] = (float)((double)dst[j] * inv);
  }
}

/* ------------------------------------------------------------------ top-k */
/* tensor.cpp:68-90: order (score desc, index asc); take min(k,n); sort
 * ascending. qsort with that total order yields the same set as the
 * reference's partial_sort. */
static const double* g_sd;
static const float* g_sf;
static int cmp_better_d(const void* a, const void* b) {
  uint32_t l = *(const uint32_t*)a, r = *(const uint32_t*)b;
  if (g_sd[l] != g_sd[r]) return g_sd[l] > g_sd[r] ? -1 : 1;
  return l < r ? -1 : (l > r);
}
static int cmp_better_f(const void* a, const void* b) {
  uint32_t l = *(const uint32_t*)a, r = *(const uint32_t*)b;
  if (g_sf[l] != g_sf[r]) return g_sf[l] > g_sf[r] ? -1 : 1;
  return l < r ? -1 : (l > r);
}
static int cmp_u32(const void* a, const void* b) {
  uint32_t l = *(const uint32_t*)a, r = *(const uint32_t*)b;
  return l < r ? -1 : (l > r);
}

static int topk_common(size_t n, size_t k, uint32_t* out, size_t* n_out, int is_double,
                       const void* s) {
  if (n == 0) return fail(1, "topk_indices: empty scores");
  if (k == 0) return fail(1, "topk_indices: k must be >= 1");
  uint32_t* order = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  if (is_double) {
    g_sd = (const double*)s;
    qsort(order, n, sizeof(uint32_t), cmp_better_d);
  } else {
    g_sf = (const float*)s;
    qsort(order, n, sizeof(uint32_t), cmp_better_f);
  }
  const size_t take = k < n ? k : n;
  memcpy(out, order, take * sizeof(uint32_t));
  qsort(out, take, sizeof(uint32_t), cmp_u32);
  *n_out = take;
  free(order);
  return 0;
}

int oc_topk_indices_f64(const double* s, size_t n, size_t k, uint32_t* out, size_t* n_out) {
  return topk_common(n, k, out, n_out, 1, s);
}
int oc_topk_indices_f32(const float* s, size_t n, size_t k, uint32_t* out, size_t* n_out) {
  return topk_common(n, k, out, n_out, 0, s);
}

/* ------------------------------------------------------------- selection */
/* selector.cpp:89-126 — criticality per method. */
int oc_criticality(const float* S, size_t H, size_t T, size_t k, int method, double* crit) {
  for (size_t j = 0; j < T; ++j) crit[j] = 0.0;
  if (T == 0) return 0;
  if (method == 0) { /* select_topk :89-99 raw logit sum */
    for (size_t h = 0; h < H; ++h)
      for (size_t j = 0; j < T; ++j) crit[j] += (double)S[h * T + j];
  } else if (method == 1) { /* select_head_vote :101-111 */
    uint32_t* top = (uint32_t*)malloc(T * sizeof(uint32_t));
    for (size_t h = 0; h < H; ++h) {
      size_t n = 0;
      int rc = oc_topk_indices_f32(S + h * T, T, k, top, &n);
      if (rc) {
        free(top);
        return rc;
      }
      for (size_t i = 0; i < n; ++i) crit[top[i]] += 1.0;
    }
    free(top);
  } else if (method == 2) { /* select_head_soft_vote :113-126 */
    float* p = (float*)malloc(H * T * sizeof(float));
    oc_softmax_rows(S, H, T, p);
    for (size_t h = 0; h < H; ++h)
      for (size_t j = 0; j < T; ++j) crit[j] += (double)p[h * T + j];
    free(p);
  } else {
    return fail(1, "select_with: bad method");
  }
  return 0;
}

/* selector.cpp:72-85 pick() over the criticality vector. */
int oc_select(const float* S, size_t H, size_t T, const uint32_t* cand, size_t k, int method,
              uint32_t* sel_out, double* crit_out, size_t* n_out) {
  *n_out = 0;
  if (T == 0) {
    if (method < 0 || method > 2) return fail(1, "select_with: bad method");
    return 0; /* :75 empty criticality -> empty result */
  }
  double* crit = (double*)malloc(T * sizeof(double));
  int rc = oc_criticality(S, H, T, k, method, crit);
  if (rc == 0) {
    uint32_t* cols = (uint32_t*)malloc(T * sizeof(uint32_t));
    size_t n = 0;
    rc = oc_topk_indices_f64(crit, T, k, cols, &n);
    if (rc == 0) {
      for (size_t i = 0; i < n; ++i) {
        sel_out[i] = cand[cols[i]];
        crit_out[i] = crit[cols[i]];
      }
      *n_out = n;
    }
    free(cols);
  }
  free(crit);
  return rc;
}

/* tensor.cpp:92-113 */
int oc_cosine_f32(const float* u, const float* v, size_t n, double* out) {
  double dot = 0.0, nu = 0.0, nv = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double a = (double)u[i], b = (double)v[i];
    dot += a * b;
    nu += a * a;
    nv += b * b;
  }
  if (nu == 0.0 || nv == 0.0) return fail(1, "cosine: zero-norm input");
  if (dot * dot >= nu * nv) {
    *out = dot >= 0.0 ? 1.0 : -1.0;
    return 0;
  }
  *out = dot / sqrt(nu * nv);
  return 0;
}

/* tensor.cpp:133-150 */
int oc_chunk_mean(const float* q, size_t c, size_t width, float* out) {
  if (c == 0) return fail(1, "chunk_mean: empty chunk");
  double* acc = (double*)calloc(width, sizeof(double));
  for (size_t i = 0; i < c; ++i)
    for (size_t j = 0; j < width; ++j) acc[j] += (double)q[i * width + j];
  const double inv = 1.0 / (double)c;
  for (size_t j = 0; j < width; ++j) out[j] = (float)(acc[j] * inv);
  free(acc);
  return 0;
}

/* ---------------------------------------------------------------- windows */
/* attention.cpp:25-33 */
size_t oc_selection_candidates(size_t cached, size_t n_init, size_t n_local, size_t* begin) {
  if (cached <= n_init + n_local) return 0;
  *begin = n_init;
  return cached - n_local - n_init;
}

/* attention.cpp:35-52 and merged() = merge_dedup (tensor.cpp:159-168). The
 * three lists are disjoint by construction, so the dedup is a merge. */
size_t oc_make_windows(size_t cached, size_t n_init, size_t n_local, const uint32_t* sel,
                       size_t n_sel, uint32_t* merged, size_t* n_sel_kept) {
  const size_t init_end = n_init < cached ? n_init : cached;
  const size_t local_begin = cached - (n_local < cached ? n_local : cached);
  size_t n = 0, kept = 0;
  uint32_t* tmp = (uint32_t*)malloc((init_end + n_sel + cached + 1) * sizeof(uint32_t));
  for (size_t i = 0; i < init_end; ++i) tmp[n++] = (uint32_t)i;
  for (size_t i = 0; i < n_sel; ++i) {
    uint32_t t = sel[i];
    if (t >= init_end && (t < local_begin || t >= cached)) {
      tmp[n++] = t;
      ++kept;
    }
  }
  size_t lb = local_begin > init_end ? local_begin : init_end;
  for (size_t i = lb; i < cached; ++i) tmp[n++] = (uint32_t)i;
  qsort(tmp, n, sizeof(uint32_t), cmp_u32);
  size_t m = 0;
  for (size_t i = 0; i < n; ++i)
    if (m == 0 || tmp[i] != merged[m - 1]) merged[m++] = tmp[i];
  free(tmp);
  if (n_sel_kept) *n_sel_kept = kept;
  return m;
}

/* -------------------------------------------------------------- attention */
/* attention.cpp:54-112 */
int oc_sdpa(const float* q, size_t C, size_t H, size_t d, const float* k_all,
            const float* v_all, size_t rows, size_t H_kv, float* out) {
  if (H == 0 || d == 0) return fail(1, "sdpa_full: q must be [C x (H * d_h)]");
  if (H_kv == 0 || H % H_kv != 0) return fail(1, "sdpa_full: H must be a multiple of H_kv");
  if (rows < C) return fail(1, "sdpa_full: fewer KV rows than query rows");
  const size_t qw = H * d, kw = H_kv * d;
  const size_t n_cached = rows - C;
  const double scale = 1.0 / sqrt((double)d);
  double* logits = (double*)malloc((rows ? rows : 1) * sizeof(double));
  double* acc = (double*)malloc(d * sizeof(double));
  for (size_t h = 0; h < H; ++h) {
    const size_t kv_off = (h % H_kv) * d, q_off = h * d;
    for (size_t i = 0; i < C; ++i) {
      const float* q_row = q + i * qw + q_off;
      const size_t attended = n_cached + i + 1;
      double mx = -HUGE_VAL;
      for (size_t j = 0; j < attended; ++j) {
        const float* k_row = k_all + j * kw + kv_off;
        double dot = 0.0;
        for (size_t t = 0; t < d; ++t) dot += (double)q_row[t] * (double)k_row[t];
        logits[j] = dot * scale;
        mx = fmax(mx, logits[j]);
      }
      double denom = 0.0;
      for (size_t j = 0; j < attended; ++j) {
        logits[j] = exp(logits[j] - mx);
        denom += logits[j];
      }
      for (size_t t = 0; t < d; ++t) acc[t] = 0.0;
      for (size_t j = 0; j < attended; ++j) {
        const double w = logits[j] / denom;
        const float* v_row = v_all + j * kw + kv_off;
        for (size_t t = 0; t < d; ++t) acc[t] += w * (double)v_row[t];
      }
      float* o = out + i * qw + q_off;
      for (size_t t = 0; t < d; ++t) o[t] = (float)acc[t];
    }
  }
  free(logits);
  free(acc);
  return 0;
}

/* attention.cpp:114-123 (gather kv_pool.cpp:87-101 + vstack tensor.cpp:54-64) */
int oc_sparse_attend(const float* q, const float* k_cur, const float* v_cur, size_t C,
                     const float* k_rows, const float* v_rows, size_t n_tokens, size_t H,
                     size_t H_kv, size_t d, const uint32_t* att, size_t n_att, float* out) {
  const size_t kw = H_kv * d;
  for (size_t j = 0; j < n_att; ++j) {
    if (att[j] >= n_tokens) {
      snprintf(g_err, sizeof g_err, "gather: index %u out of range (logical_len %zu)", att[j],
               n_tokens);
      return 2;
    }
  }
  const size_t rows = n_att + C;
  float* ka = (float*)malloc((rows ? rows : 1) * kw * sizeof(float));
  float* va = (float*)malloc((rows ? rows : 1) * kw * sizeof(float));
  for (size_t j = 0; j < n_att; ++j) {
    memcpy(ka + j * kw, k_rows + (size_t)att[j] * kw, kw * sizeof(float));
    memcpy(va + j * kw, v_rows + (size_t)att[j] * kw, kw * sizeof(float));
  }
  memcpy(ka + n_att * kw, k_cur, C * kw * sizeof(float));
  memcpy(va + n_att * kw, v_cur, C * kw * sizeof(float));
  int rc = oc_sdpa(q, C, H, d, ka, va, rows, H_kv, out);
  free(ka);
  free(va);
  return rc;
}

/* ----------------------------------------------------------------- engine */
struct oc_engine {
  size_t k, n_local, n_init, chunk, H, H_kv, d, block, cap, len;
  int method;
  /* SelectionCacheEntry (selection_cache.hpp:23-29) */
  double theta;
  int first_flag;
  float* cached_q;
  uint32_t* cached_sel;
  double* cached_crit;
  size_t cached_n;
  size_t lookups, hits;
  float* K;
  float* V;
};

oc_engine* oc_engine_create(size_t k, size_t n_local, size_t n_init, size_t chunk, double theta,
                            size_t H, size_t H_kv, size_t d, size_t block, int method,
                            size_t capacity) {
  /* EngineConfig::validate attention.cpp:10-19 */
  if (H == 0 || H_kv == 0 || d == 0 || H % H_kv != 0 || chunk == 0 || block == 0 ||
      method < 0 || method > 2) {
    fail(1, "EngineConfig: invalid configuration");
    return NULL;
  }
  oc_engine* e = (oc_engine*)calloc(1, sizeof(oc_engine));
  e->k = k;
  e->n_local = n_local;
  e->n_init = n_init;
  e->chunk = chunk;
  e->theta = theta; /* attention.cpp:222 */
  e->H = H;
  e->H_kv = H_kv;
  e->d = d;
  e->block = block;
  e->method = method;
  e->cap = capacity;
  e->first_flag = 1;
  e->cached_q = (float*)malloc(H * d * sizeof(float));
  e->cached_sel = (uint32_t*)malloc((k ? k : 1) * sizeof(uint32_t));
  e->cached_crit = (double*)malloc((k ? k : 1) * sizeof(double));
  e->K = (float*)malloc((capacity ? capacity : 1) * H_kv * d * sizeof(float));
  e->V = (float*)malloc((capacity ? capacity : 1) * H_kv * d * sizeof(float));
  return e;
}

void oc_engine_destroy(oc_engine* e) {
  if (!e) return;
  free(e->cached_q);
  free(e->cached_sel);
  free(e->cached_crit);
  free(e->K);
  free(e->V);
  free(e);
}

/* kv_pool.cpp:55-85: all-or-nothing capacity check (page_size 1). */
int oc_engine_append(oc_engine* e, const float* k, const float* v, size_t t) {
  if (e->len + t > e->cap) return fail(3, "append_kv: pool exhausted");
  const size_t kw = e->H_kv * e->d;
  memcpy(e->K + e->len * kw, k, t * kw * sizeof(float));
  memcpy(e->V + e->len * kw, v, t * kw * sizeof(float));
  e->len += t;
  return 0;
}

/* select_for_chunk selector.cpp:137-150 over candidates [begin, begin+T). */
static int select_chunk(oc_engine* e, const float* q_chunk, size_t c, size_t begin, size_t T,
                        uint32_t* sel, double* crit, size_t* n) {
  const size_t width = e->H * e->d;
  float* mean = (float*)malloc(width * sizeof(float));
  int rc = oc_chunk_mean(q_chunk, c, width, mean);
  if (rc) {
    free(mean);
    return rc;
  }
  uint32_t* cand = (uint32_t*)malloc((T ? T : 1) * sizeof(uint32_t));
  for (size_t j = 0; j < T; ++j) cand[j] = (uint32_t)(begin + j);
  float* S = (float*)malloc((e->H * T ? e->H * T : 1) * sizeof(float));
  rc = oc_score(mean, e->H, e->d, e->K, e->len, e->H_kv, cand, T, S);
  if (rc == 0) rc = oc_select(S, e->H, T, cand, e->k, e->method, sel, crit, n);
  free(S);
  free(cand);
  free(mean);
  return rc;
}

/* decode_step attention.cpp:172-200 with lookup_or_select selection_cache.cpp:16-44 */
int oc_engine_decode(oc_engine* e, const float* q, const float* k, const float* v, float* out,
                     int* hit, uint32_t* sel_out, size_t* n_sel, double* cos_out) {
  const size_t width = e->H * e->d;
  const size_t cached = e->len;
  *hit = 0;
  if (cos_out) *cos_out = NAN;
  uint32_t* sel = NULL;
  size_t n = 0;
  if (e->k > 0 && cached > e->n_init + e->n_local) {
    int all_zero = 1;
    for (size_t i = 0; i < width; ++i)
      if (q[i] != 0.0f) {
        all_zero = 0;
        break;
      }
    if (all_zero) return fail(1, "lookup_or_select: zero query vector");
    e->lookups += 1;
    int miss = e->first_flag;
    if (!miss) {
      double c = 0.0;
      int rc = oc_cosine_f32(q, e->cached_q, width, &c);
      if (rc) return rc;
      if (cos_out) *cos_out = c;
      miss = c < e->theta;
    }
    if (miss) {
      size_t begin = 0;
      size_t T = oc_selection_candidates(cached, e->n_init, e->n_local, &begin);
      size_t cn = 0;
      int rc = select_chunk(e, q, 1, begin, T, e->cached_sel, e->cached_crit, &cn);
      if (rc) return rc;
      e->cached_n = cn;
      memcpy(e->cached_q, q, width * sizeof(float));
      e->first_flag = 0;
    } else {
      e->hits += 1;
      *hit = 1;
    }
    sel = e->cached_sel;
    n = e->cached_n;
  }
  if (n_sel) *n_sel = n;
  if (sel_out && n) memcpy(sel_out, sel, n * sizeof(uint32_t));
  uint32_t* merged = (uint32_t*)malloc((cached + n + 1) * sizeof(uint32_t));
  size_t m = oc_make_windows(cached, e->n_init, e->n_local, sel, n, merged, NULL);
  int rc = oc_sparse_attend(q, k, v, 1, e->K, e->V, e->len, e->H, e->H_kv, e->d, merged, m, out);
  free(merged);
  if (rc) return rc;
  return oc_engine_append(e, k, v, 1);
}

/* prefill attention.cpp:135-170 */
int oc_engine_prefill(oc_engine* e, const float* q, const float* k, const float* v, size_t n_in,
                      float* out, uint32_t* sel_flat, size_t* sel_counts, size_t max_chunks) {
  if (n_in == 0) return fail(1, "prefill: empty input");
  const size_t qw = e->H * e->d, kw = e->H_kv * e->d;
  size_t chunk_id = 0, flat_off = 0;
  uint32_t* sel = (uint32_t*)malloc((e->k ? e->k : 1) * sizeof(uint32_t));
  double* crit = (double*)malloc((e->k ? e->k : 1) * sizeof(double));
  int rc = 0;
  for (size_t b = 0; b < n_in; b += e->chunk, ++chunk_id) {
    const size_t len = e->chunk < n_in - b ? e->chunk : n_in - b;
    const size_t cached = e->len;
    size_t n = 0;
    if (e->k > 0) {
      size_t begin = 0;
      size_t T = oc_selection_candidates(cached, e->n_init, e->n_local, &begin);
      if (T > 0) {
        rc = select_chunk(e, q + b * qw, len, begin, T, sel, crit, &n);
        if (rc) break;
      }
    }
    if (sel_counts && chunk_id < max_chunks) {
      sel_counts[chunk_id] = n;
      memcpy(sel_flat + flat_off, sel, n * sizeof(uint32_t));
      flat_off += n;
    }
    uint32_t* merged = (uint32_t*)malloc((cached + n + 1) * sizeof(uint32_t));
    size_t m = oc_make_windows(cached, e->n_init, e->n_local, sel, n, merged, NULL);
    rc = oc_sparse_attend(q + b * qw, k + b * kw, v + b * kw, len, e->K, e->V, e->len, e->H,
                          e->H_kv, e->d, merged, m, out + b * qw);
    free(merged);
    if (rc) break;
    rc = oc_engine_append(e, k + b * kw, v + b * kw, len);
    if (rc) break;
  }
  free(sel);
  free(crit);
  return rc;
}

void oc_engine_force_miss(oc_engine* e) { e->first_flag = 1; }

void oc_engine_stats(const oc_engine* e, size_t* lookups, size_t* hits, size_t* len) {
  *lookups = e->lookups;
  *hits = e->hits;
  *len = e->len;
}

const float* oc_engine_k_rows(const oc_engine* e) { return e->K; }
const float* oc_engine_v_rows(const oc_engine* e) { return e->V; }

// Single-sequence decode step (sm_100a): the engine's TokenSelect decode step
// (decode_step, reference attention.cpp:172-200) in ONE cooperative launch of
// one CTA per SM, built so that as little as possible happens after the K
// scan, which is the HBM roofline:
//
//   phase 0  Selection Cache test, fp64 cosine vs the cached query
//            (selection_cache.cpp:16-44, tensor.cpp:92-113), evaluated
//            bit-identically by every CTA; slab rows of the CTA's candidates;
//            append of the current token's K/V row (kv_pool.cpp:55-85).
//   phase 1  miss: K scan S = q.K over the CTA's candidates (selector.cpp:26-68)
//            -- 16-token x 2 KB rows streamed by the TMA engine through an
//            mbarrier ring, mma.sync with q split exactly into three bf16
//            parts. The softmax statistics (tensor.cpp:31-52) are formed ON
//            THE FLY: per consumer warp and head a stage-wise reference max
//            m_ref and z = sum e^(S - m_ref); e = e^(S - m_ref) (not S) goes to
//            tensor memory, m_ref of every stage to shared memory.
//            -> (m, z) per head published, grid barrier B1.
//   phase 2  global (M_h, Z_h); crit[j] = sum_h e_hj e^(m_ref - M_h) / Z_h
//            (select_head_soft_vote, selector.cpp:113-126) -- one FMA per
//            score, the exponentials were paid during the scan; 12-bit radix
//            histogram, B2; second 12-bit pass only when the boundary bin is
//            split (B3); ties at the 24-bit threshold ranked by position
//            (B3b, only when they straddle k): tensor.cpp:68-90.
//   phase 3  attention (sdpa_full over make_windows, attention.cpp:35-123)
//            WITHOUT a compaction barrier: every CTA attends the rows it
//            owns -- its own selected candidates (miss) or its slice of the
//            cached selection (hit), plus its slice of init U local U current
//            -- to an unnormalised partial (o, m, l) per head, fp32 CUDA cores.
//            B4; every CTA merges a slice of the H*d outputs by log-sum-exp
//            over all CTAs' partials; the SelectionResult is written in
//            ascending order from the per-CTA counts.
//
// A hit runs phase 0, phase 3 and B4 only: no scan grid work, no TMEM.
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "step.h"

namespace tsb {

namespace {

constexpr float kL2E = 1.4426950408889634f;
constexpr int kD = 128;
constexpr int kCons = kDecodeConsumers;      // 16
constexpr int kNW = kDecodeWarps;            // 17
constexpr int kRB = kStepRowsPerBatch;
constexpr int kMaxWinSlice = 64;             // window rows per CTA (host-checked)
constexpr int kMaxHitSlice = 64;             // cached-selection entries per CTA (host-checked)

// own: what this step does for the sequence (every CTA decides identically)
constexpr int kOwnNone = 0, kOwnMiss = 1, kOwnHit = 2, kOwnZero = 3;

__device__ __forceinline__ void trace_at(const StepParams& p, int i) {
  if (p.trace && threadIdx.x == 0) {
    unsigned long long* t = p.trace + blockIdx.x * kTraceStride;
    const unsigned long long c = clock64();
    if (i == 0 || i == 12) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      t[i == 0 ? 0 : 30] = g;
      t[i == 0 ? 29 : 12] = c;
      if (i == 0) t[63] = 2;  // kernel id: the step kernel (selattn.read_trace names)
    } else {
      t[i] = c;
    }
  }
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return l | (h << 16);
}

// x = hi + mid + lo exactly (bf16 parts, each residual exact in fp32)
__device__ __forceinline__ void split3(float x, float& hi, float& mid, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(x));
  const float r1 = x - hi;
  mid = __bfloat162float(__float2bfloat16_rn(r1));
  lo = r1 - mid;
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, float a, float b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(__float_as_uint(a)),
               "r"(__float_as_uint(b))
               : "memory");
}

// Sum over the 32 lanes of 8 per-lane values; afterwards lane L holds the
// total of value (L >> 2) & 7 (recursive halving: 9 shuffles for 8 values).
__device__ __forceinline__ float reduce8(float (&v)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const float send = hi ? v[i] : v[i + 4];
    v[i] = (hi ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const float send = hi ? v[i] : v[i + 2];
    v[i] = (hi ? v[i + 2] : v[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool hi = lane & 4;
    const float send = hi ? v[0] : v[1];
    v[0] = (hi ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// Block-wide exclusive scan of one value per thread (all threads call).
__device__ __noinline__ uint32_t block_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(v, lane);
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kNW ? scratch[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w, lane);
    if (lane < kNW) scratch[32 + lane] = wi - w;
    if (lane == 31) scratch[63] = wi;
  }
  __syncthreads();
  const uint32_t r = scratch[32 + warp] + inc - v;
  if (total) *total = scratch[63];
  __syncthreads();
  return r;
}

// The bin of a descending-ordered 4096-bin global histogram that holds the
// kk-th largest key: count(bins > b) < kk <= count(bins >= b). Returns b, the
// count above it and its own count; every CTA computes the same answer.
__device__ __noinline__ void find_bin(const uint32_t* gh, uint32_t kk, uint32_t* scratch, uint32_t* work,
                                      uint32_t* bin_out, uint32_t* above_out, uint32_t* count_out) {
  const int t = threadIdx.x, lane = t & 31;
  uint32_t* coarse = work + kRadixBins;
  if (t < 512) {
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(gh) + 2 * t);
    const uint4 b = __ldcg(reinterpret_cast<const uint4*>(gh) + 2 * t + 1);
    reinterpret_cast<uint4*>(work)[2 * t] = a;
    reinterpret_cast<uint4*>(work)[2 * t + 1] = b;
    uint32_t sum = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    if ((t & 7) == 0) coarse[t >> 3] = sum;
  }
  __syncthreads();
  if (t < 32) {
    uint32_t base = 0, bin = 0, cnt = 0;
#pragma unroll 1
    for (int level = 0; level < 2; ++level) {
      const uint32_t* src = level == 0 ? coarse : work + bin * 64;
      const uint32_t c0 = src[63 - 2 * lane], c1 = src[62 - 2 * lane];
      const uint32_t sum = c0 + c1;
      const uint32_t incl = warp_incl_scan(sum, lane);
      const uint32_t excl = incl - sum;
      const uint32_t need = kk - base;
      const bool here = excl < need && incl >= need;
      const int src_lane = __ffs(__ballot_sync(0xffffffffu, here)) - 1;
      uint32_t b = 0, ab = 0, c = 0;
      if (here) {
        if (excl + c0 >= need) {
          b = 63 - 2 * lane;
          ab = excl;
          c = c0;
        } else {
          b = 62 - 2 * lane;
          ab = excl + c0;
          c = c1;
        }
      }
      b = __shfl_sync(0xffffffffu, b, src_lane);
      ab = __shfl_sync(0xffffffffu, ab, src_lane);
      c = __shfl_sync(0xffffffffu, c, src_lane);
      base += ab;
      bin = level == 0 ? b : bin * 64 + b;
      cnt = c;
    }
    if (lane == 0) {
      scratch[64] = bin;
      scratch[65] = base;
      scratch[66] = cnt;
    }
  }
  __syncthreads();
  *bin_out = scratch[64];
  *above_out = scratch[65];
  *count_out = scratch[66];
  __syncthreads();
}

// One key into the shared histogram (digit at `shift`), aggregated over the
// warp's lanes hitting the same bin.
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t key, bool act, int shift) {
  const unsigned am = __ballot_sync(0xffffffffu, act);
  if (act) {
    const uint32_t bin = (key >> shift) & (kRadixBins - 1);
    const unsigned peers = __match_any_sync(am, bin);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], static_cast<uint32_t>(__popc(peers)));
  }
}

__device__ __noinline__ void hist_merge(const uint32_t* hist, uint32_t* gh) {
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) {
    const uint32_t c = hist[i];
    if (c) atomicAdd(gh + i, c);
  }
}

// fp64 cosine decision (tensor.cpp:92-113, selection_cache.cpp:29-35): every
// CTA reduces the same values in the same order -> bit-identical result.
// Returns kOwnMiss / kOwnHit / kOwnZero.
__device__ __noinline__ int decide(const float* __restrict__ q, const float* __restrict__ cq, int width,
                                   const float (&qa)[8], const float (&qb)[8], int first_flag, double theta,
                                   double* sd, double* cos_out) {
  double dot = 0.0, nu = 0.0, nv = 0.0;
  int nonzero = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double a = qa[u], b = qb[u];
    nonzero |= qa[u] != 0.0f;
    dot = fma(a, b, dot);
    nu = fma(a, a, nu);
    nv = fma(b, b, nv);
  }
  for (int i = threadIdx.x + 8 * blockDim.x; i < width; i += blockDim.x) {
    const float fa = __ldg(q + i), fb = __ldcg(cq + i);
    nonzero |= fa != 0.0f;
    dot = fma(static_cast<double>(fa), static_cast<double>(fb), dot);
    nu = fma(static_cast<double>(fa), static_cast<double>(fa), nu);
    nv = fma(static_cast<double>(fb), static_cast<double>(fb), nv);
  }
  dot = warp_sum_d(dot);
  nu = warp_sum_d(nu);
  nv = warp_sum_d(nv);
  nonzero = __any_sync(0xffffffffu, nonzero);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sd[warp * 4 + 0] = dot;
    sd[warp * 4 + 1] = nu;
    sd[warp * 4 + 2] = nv;
    sd[warp * 4 + 3] = nonzero ? 1.0 : 0.0;
  }
  __syncthreads();
  double D = lane < kNW ? sd[lane * 4 + 0] : 0.0;
  double U = lane < kNW ? sd[lane * 4 + 1] : 0.0;
  double V = lane < kNW ? sd[lane * 4 + 2] : 0.0;
  const int nz = __any_sync(0xffffffffu, lane < kNW && sd[lane * 4 + 3] != 0.0);
  D = warp_sum_d(D);
  U = warp_sum_d(U);
  V = warp_sum_d(V);
  __syncthreads();
  if (!nz) return kOwnZero;
  *cos_out = NAN;
  if (first_flag || U == 0.0 || V == 0.0) return kOwnMiss;
  double c;
  if (D * D >= U * V) c = D >= 0.0 ? 1.0 : -1.0;  // exact +-1 clamp
  else c = D / sqrt(U * V);
  *cos_out = c;
  return c < theta ? kOwnMiss : kOwnHit;  // strict <
}

struct Grid {
  unsigned int* ctr;
  unsigned int n, target;
  __device__ __forceinline__ void sync() {
    __syncthreads();
    target += n;
    if (threadIdx.x == 0) {
      red_release_add_u32(ctr, 1u);
      while (ld_acquire_u32(ctr) < target) {
      }
    }
    __syncthreads();
  }
};

template <int G>
__global__ void __launch_bounds__(kStepThreads, 1) step_kernel(const StepParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int CPS = G <= 4 ? 2 : 4;  // TMEM columns per stage per warp
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int H = p.H, Hkv = p.H_kv, nph = kCons / Hkv;
  const int row_bytes = Hkv * kD * 2;
  const int rstride = row_bytes + 16;
  const int sbytes = 16 * rstride;
  const int tpc = p.tpc, MS = p.stages_per_warp;
  // ---- shared memory carve (step_smem_bytes mirrors it)
  uint8_t* ring = smem;
  const size_t ring_bytes = align_up(static_cast<size_t>(p.ring_stages) * sbytes, 1024);
  float* mrec = reinterpret_cast<float*>(smem + ring_bytes);                 // [16][MS][G]
  size_t o = ring_bytes + align_up(static_cast<size_t>(kCons) * MS * G * 4, 128);
  int32_t* frames = reinterpret_cast<int32_t*>(smem + o);                    // [tpc]
  o += align_up(static_cast<size_t>(tpc) * 4, 128);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + o);                 // [256]
  o += 1024;
  float2* wst = reinterpret_cast<float2*>(smem + o);                         // [16][8] per-warp (m_ref, z)
  o += kCons * 8 * 8;
  float* mlog = reinterpret_cast<float*>(smem + o);                          // [H] M log2e + log2 Z
  o += 64 * 4;
  float* st_m = reinterpret_cast<float*>(smem + o);                          // [H] attention running max
  o += 64 * 4;
  float* st_l = reinterpret_cast<float*>(smem + o);                          // [H] running sum
  o += 64 * 4;
  float* st_c = reinterpret_cast<float*>(smem + o);                          // [H] batch rescale factor
  o += 64 * 4;
  int32_t* hrow = reinterpret_cast<int32_t*>(smem + o);                      // [kMaxHitSlice] hit rows
  o += kMaxHitSlice * 4;
  int32_t* wrow = reinterpret_cast<int32_t*>(smem + o);                      // [kMaxWinSlice] window rows
  o += kMaxWinSlice * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + o);                    // [kMaxBarPairs]
  uint64_t* empty = full + kMaxBarPairs;                                     // [kMaxBarPairs]
  uint64_t* abar = empty + kMaxBarPairs;                                     // attention staging
  // post-scan aliases of the ring
  uint32_t* hist = reinterpret_cast<uint32_t*>(ring);                        // [4096 + 64]
  float* cpart = reinterpret_cast<float*>(ring + 17 * 1024);                 // [Hkv][tpc]
  uint32_t* keys = reinterpret_cast<uint32_t*>(ring + 17 * 1024 + static_cast<size_t>(Hkv) * tpc * 4);  // [tpc]
  uint32_t* sl_tok = reinterpret_cast<uint32_t*>(ring + ring_bytes - static_cast<size_t>(3) * tpc * 4);  // [tpc]
  int32_t* sl_row = reinterpret_cast<int32_t*>(sl_tok + tpc);
  uint32_t* sl_key = sl_tok + 2 * tpc;
  uint16_t* att_k = reinterpret_cast<uint16_t*>(ring);                       // [kRB][Hkv*d]
  uint16_t* att_v = reinterpret_cast<uint16_t*>(ring + static_cast<size_t>(kRB) * row_bytes);
  float* scores = reinterpret_cast<float*>(ring + static_cast<size_t>(2) * kRB * row_bytes);  // [kRB + 1][H]
  float* red = scores + (kRB + 1) * 64;                                      // [nph][H][d]

  trace_at(p, 0);
  // ---------------------------------------------------------------- phase 0
  // the decision's operands first: they head the critical path
  const int width = H * kD;
  float qa[8], qb[8];
  int first_flag = 0;
  double theta = 0.0;
  if (p.select) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = tid + u * kStepThreads;
      qa[u] = i < width ? __ldg(p.q + i) : 0.f;
      qb[u] = i < width ? __ldcg(p.cached_q + i) : 0.f;
    }
    first_flag = __ldcg(&p.cache->first_flag);
    theta = __ldcg(&p.cache->theta);
  }
  if (tid < 2 * kMaxBarPairs + 1) {
    if (tid < kMaxBarPairs) mbar_init(&full[tid], 1);
    else if (tid < 2 * kMaxBarPairs) mbar_init(&empty[tid - kMaxBarPairs], Hkv);
    else mbar_init(abar, 1);
  }
  fence_mbar_init();
  Grid gs{p.bar + p.bar_slot, static_cast<unsigned int>(ncta), 0u};
  if (cta == 0 && tid == 0) p.bar[p.bar_slot ^ 32] = 0u;  // the next launch's barrier counter
  // the scan's slab rows (page_size 1: one page-table entry per token)
  const int T = p.T;
  const int j0 = min(T, cta * tpc);
  const int nloc = max(0, min(T, j0 + tpc) - j0);
  int32_t fr[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = tid + u * kStepThreads;
    fr[u] = (p.select && j < nloc) ? __ldcg(p.page_table + p.cand_begin + j0 + j) : 0;
  }
  // this CTA's slice of the cached selection (a hit attends it) and of the
  // windows init U local U current: loaded with the decision's operands
  const int ks = (p.k + ncta - 1) / ncta;  // <= kMaxHitSlice (host-checked)
  const int hi0 = cta * ks;
  int n_sel_c = 0;
  uint32_t h_tok = 0xffffffffu;
  int32_t h_row = 0;
  if (p.select) {
    n_sel_c = __ldcg(&p.cache->n_sel);
    if (tid < ks && hi0 + tid < p.k) {
      h_tok = __ldcg(p.sel + hi0 + tid);
      h_row = __ldcg(p.sel_rows + hi0 + tid);
    }
  }
  const int W = p.init_end + (p.N - p.lb) + 1;  // + the current token
  const int wc = (W + ncta - 1) / ncta;
  const int w0 = min(W, cta * wc), w1 = min(W, w0 + wc);
  const bool has_cur = w1 == W && w1 > w0;
  const int n_win = w1 - w0 - (has_cur ? 1 : 0);  // slab rows of the slice
  int32_t w_row = 0;
  if (tid < n_win) {
    const int i = w0 + tid;
    w_row = __ldcg(p.page_table + (i < p.init_end ? i : p.lb + (i - p.init_end)));
  }
  // the radix histograms are added to after B1 only
  for (int i = cta * kStepThreads + tid; i < 2 * kRadixBins; i += ncta * kStepThreads) p.ws_hist[i] = 0u;
  int own = kOwnNone;
  double cosv = NAN;
  trace_at(p, 24);
  if (p.select) own = decide(p.q, p.cached_q, width, qa, qb, first_flag, theta, reinterpret_cast<double*>(scratch), &cosv);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = tid + u * kStepThreads;
    if (j < nloc) frames[j] = fr[u];
  }
  for (int j = tid + 4 * kStepThreads; j < nloc; j += kStepThreads) frames[j] = __ldcg(p.page_table + p.cand_begin + j0 + j);
  if (cta == 0 && tid == 0 && p.select) p.cache->error = own == kOwnZero ? 1 : 0;
  if (own == kOwnZero) return;  // grid-uniform: nothing is mutated (selection_cache.cpp:18-27)
  if (cta == 0 && p.append_frame >= 0) {
    // append (kv_pool.cpp:55-85); this step never reads row N
    const size_t off = static_cast<size_t>(p.append_frame) * Hkv * kD;
    for (int i = tid; i < Hkv * kD; i += kStepThreads) {
      p.k_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(p.k_new[i]));
      p.v_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(p.v_new[i]));
    }
    if (tid == 0) p.page_table[p.N] = p.append_frame;
  }
  trace_at(p, 25);
  const bool miss = own == kOwnMiss;
  if (tid < n_win) {
    wrow[tid] = w_row;
    if (miss) {
      // attended after the scan: keep them in L2 across the K stream (evict_last)
      const uint64_t pol = policy_evict_last();
      bulk_prefetch_l2(reinterpret_cast<const char*>(p.k_slab) + static_cast<size_t>(w_row) * row_bytes, row_bytes, pol);
      bulk_prefetch_l2(reinterpret_cast<const char*>(p.v_slab) + static_cast<size_t>(w_row) * row_bytes, row_bytes, pol);
    }
  }
  int n_sel_part = 0;  // rows of the selected part (miss: set after the selection)
  if (own == kOwnHit) {
    // cached entries now inside the local window are attended there (make_windows)
    const bool in = tid < ks && hi0 + tid < n_sel_c && h_tok < static_cast<uint32_t>(p.lb);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0 && warp < 2) scratch[90 + warp] = __popc(bal);
    __syncthreads();
    if (in) hrow[(warp == 1 ? static_cast<int>(scratch[90]) : 0) + __popc(bal & ((1u << lane) - 1u))] = h_row;
    n_sel_part = static_cast<int>(scratch[90] + scratch[91]);
  }
  uint32_t tbase = 0;
  if (miss && warp == 1) tmem_alloc512(&scratch[250]);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  if (miss) tbase = scratch[250];
  trace_at(p, 1);

  // ---------------------------------------------------------------- phase 1
  const int nit = (nloc + 15) >> 4;
  const int cw = warp - 1, kvh = cw % Hkv, ph = cw / Hkv;
  const int nr = (warp >= 1 && nit > ph) ? (nit - ph + nph - 1) / nph : 0;  // stages of this consumer warp
  const uint32_t tw = tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                      static_cast<uint32_t>(((warp - 1) >> 2) * 128);
  uint32_t n_own = 0;  // this CTA's selected candidates (miss)
  if (miss) {
    const int kStages = p.ring_stages;
    if (warp == 0) {
      // producer: one bulk copy per 2 KB row, lane = row, evict_first
      const uint64_t pol = policy_evict_first();
      const char* kbase = reinterpret_cast<const char*>(p.k_slab);
      uint64_t eparity = 0;
      int s = 0, phs = 0, ph_prev = 0;
      for (int it = 0; it < nit; ++it) {
        const int rbase = it * 16;
        const int nrows = min(16, nloc - rbase);
        if (it >= kStages) {
          const int k = ph_prev * kStages + s;
          mbar_wait(&empty[k], static_cast<uint32_t>(eparity >> k) & 1u);
          eparity ^= 1ull << k;
          ph_prev = ph_prev + 1 == nph ? 0 : ph_prev + 1;
        }
        uint64_t* fb = &full[phs * kStages + s];
        if (lane == 0) mbar_arrive_expect_tx(fb, static_cast<uint32_t>(nrows * row_bytes));
        __syncwarp();
        if (lane < nrows)
          bulk_g2s(ring + static_cast<size_t>(s) * sbytes + static_cast<size_t>(lane) * rstride,
                   kbase + static_cast<size_t>(frames[rbase + lane]) * row_bytes, row_bytes, fb, pol);
        s = s + 1 == kStages ? 0 : s + 1;
        phs = phs + 1 == nph ? 0 : phs + 1;
      }
    } else {
      // consumers: warp (kv head kvh, phase ph) takes every nph-th stage
      uint32_t bq[8][3][2];
      {
        const int gq = lane >> 2;
        const float* qh = p.q + static_cast<size_t>(gq * Hkv + kvh) * kD;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
          float v[4], hi[4], mi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int dd = kc * 16 + (lane & 3) * 2 + (e & 1) + (e >> 1) * 8;
            v[e] = gq < G ? __ldg(qh + dd) : 0.f;
            split3(v[e], hi[e], mi[e], lo[e]);
          }
          bq[kc][0][0] = pack_bf16(hi[0], hi[1]);
          bq[kc][0][1] = pack_bf16(hi[2], hi[3]);
          bq[kc][1][0] = pack_bf16(mi[0], mi[1]);
          bq[kc][1][1] = pack_bf16(mi[2], mi[3]);
          bq[kc][2][0] = pack_bf16(lo[0], lo[1]);
          bq[kc][2][1] = pack_bf16(lo[2], lo[3]);
        }
      }
      const int g0 = (lane & 3) * 2;
      const bool v0 = g0 < G, v1 = g0 + 1 < G;
      float mref0 = -INFINITY, mref1 = -INFINITY, z0 = 0.f, z1 = 0.f;
      const uint32_t lrow = static_cast<uint32_t>((lane & 7) + ((lane >> 3) & 1) * 8);
      const uint32_t lcol = static_cast<uint32_t>((lane >> 4) * 16 + kvh * kD * 2);
      const uint32_t rbase_addr = smem_u32(ring) + lrow * rstride + lcol;
      float* mr = mrec + static_cast<size_t>(cw) * MS * G;
      uint32_t fparity = 0;
      int s = ph % kStages, r = 0;
      for (int it = ph; it < nit; it += nph, ++r) {
        mbar_wait(&full[ph * kStages + s], (fparity >> s) & 1u);
        fparity ^= 1u << s;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t abase = rbase_addr + static_cast<uint32_t>(s * sbytes);
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
          uint32_t a[4];
          ldsm_x4(a, abase + kc * 32);
          mma_bf16(c, a, bq[kc][0][0], bq[kc][0][1]);
          mma_bf16(c, a, bq[kc][1][0], bq[kc][1][1]);
          mma_bf16(c, a, bq[kc][2][0], bq[kc][2][1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[ph * kStages + s]);
        s += nph;
        while (s >= kStages) s -= kStages;
        // online softmax statistics, warp-uniform reference max per head
        const int rowA = it * 16 + (lane >> 2);
        const bool okA = rowA < nloc, okB = rowA + 8 < nloc;
        float x0 = fmaxf(okA ? c[0] : -INFINITY, okB ? c[2] : -INFINITY);
        float x1 = fmaxf(okA ? c[1] : -INFINITY, okB ? c[3] : -INFINITY);
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
          x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, o2));
          x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o2));
        }
        if (x0 > mref0) {
          z0 = mref0 == -INFINITY ? 0.f : z0 * ex2_approx((mref0 - x0) * kL2E);
          mref0 = x0;
        }
        if (x1 > mref1) {
          z1 = mref1 == -INFINITY ? 0.f : z1 * ex2_approx((mref1 - x1) * kL2E);
          mref1 = x1;
        }
        const float ml0 = mref0 * kL2E, ml1 = mref1 * kL2E;
        const float e0 = (v0 && okA) ? ex2_approx(fmaf(c[0], kL2E, -ml0)) : 0.f;
        const float e1 = (v1 && okA) ? ex2_approx(fmaf(c[1], kL2E, -ml1)) : 0.f;
        const float e2 = (v0 && okB) ? ex2_approx(fmaf(c[2], kL2E, -ml0)) : 0.f;
        const float e3 = (v1 && okB) ? ex2_approx(fmaf(c[3], kL2E, -ml1)) : 0.f;
        z0 += e0 + e2;
        z1 += e1 + e3;
        if (lane < 4) {
          if (v0) mr[r * G + g0] = mref0;
          if (v1) mr[r * G + g0 + 1] = mref1;
        }
        if constexpr (CPS == 2) {
          // heads >= 4 are empty: lanes l ^ 2 take the row-B values of lane l
          const float s0 = __shfl_xor_sync(0xffffffffu, e2, 2);
          const float s1 = __shfl_xor_sync(0xffffffffu, e3, 2);
          const bool b = lane & 2;
          tmem_st2(tw + static_cast<uint32_t>(r * 2), b ? s0 : e0, b ? s1 : e1);
        } else {
          tmem_st4(tw + static_cast<uint32_t>(r * 4), e0, e1, e2, e3);
        }
      }
      tmem_wait_st();
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) {
        z0 += __shfl_xor_sync(0xffffffffu, z0, o2);
        z1 += __shfl_xor_sync(0xffffffffu, z1, o2);
      }
      if (lane < 4) {
        wst[cw * 8 + g0] = make_float2(mref0, z0);
        wst[cw * 8 + g0 + 1] = make_float2(mref1, z1);
      }
    }
    __syncthreads();
    trace_at(p, 2);
    // CTA (m, z) per head from its nph warps (fixed order); the shared
    // histogram of the soft vote is zeroed meanwhile
    const int ncp = (ncta + 3) & ~3;
    if (tid < H) {
      const int h = tid, kv = h % Hkv, g = h / Hkv;
      float m = -INFINITY;
      for (int q2 = 0; q2 < nph; ++q2) m = fmaxf(m, wst[(kv + q2 * Hkv) * 8 + g].x);
      float z = 0.f;
      if (m > -INFINITY)
        for (int q2 = 0; q2 < nph; ++q2) {
          const float2 w = wst[(kv + q2 * Hkv) * 8 + g];
          if (w.x > -INFINITY) z += w.y * ex2_approx((w.x - m) * kL2E);
        }
      p.ws_mz[static_cast<size_t>(h) * ncp + cta] = make_float2(m, z);
    }
    for (int i = tid; i < kRadixBins; i += kStepThreads) hist[i] = 0u;
    trace_at(p, 3);
    gs.sync();  // B1
    trace_at(p, 4);

    // ------------------------------------------------------------ phase 2
    // the new cached query (every CTA read the old one before B1)
    for (int i = cta * kStepThreads + tid; i < width; i += ncta * kStepThreads) p.cached_q[i] = __ldg(p.q + i);
    // global M_h, Z_h: warp per head, lanes strided over the CTAs (fixed order)
    for (int h = warp; h < H; h += kNW) {
      const float2* row = p.ws_mz + static_cast<size_t>(h) * ncp;
      float2 v[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int c = lane + 32 * j;
        v[j] = c < ncta ? __ldcg(row + c) : make_float2(-INFINITY, 0.f);
      }
      float M = -INFINITY;
#pragma unroll
      for (int j = 0; j < 5; ++j) M = fmaxf(M, v[j].x);
      for (int c = lane + 160; c < ncta; c += 32) M = fmaxf(M, __ldcg(row + c).x);
      M = warp_max(M);
      float Z = 0.f;
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (v[j].x > -INFINITY) Z += v[j].y * ex2_approx((v[j].x - M) * kL2E);
      for (int c = lane + 160; c < ncta; c += 32) {
        const float2 w = __ldcg(row + c);
        if (w.x > -INFINITY) Z += w.y * ex2_approx((w.x - M) * kL2E);
      }
      Z = warp_sum(Z);
      if (lane == 0) mlog[h] = M * kL2E + __log2f(Z);
    }
    __syncthreads();
    trace_at(p, 13);
    if (warp >= 1) {
      // per (stage, head) factor e^(m_ref - M_h) / Z_h, in place
      float* mr = mrec + static_cast<size_t>(cw) * MS * G;
      for (int i = lane; i < nr * G; i += 32) {
        const int g = i % G;
        mr[i] = ex2_approx(mr[i] * kL2E - mlog[g * Hkv + kvh]);
      }
      __syncwarp();
      // this warp's rows: partial criticality over its kv head's G heads
      float* cp = cpart + static_cast<size_t>(kvh) * tpc;
#pragma unroll 1
      for (int r0 = 0; r0 < nr; r0 += 16 / CPS) {
        float v[16];
        tmem_ld16(tw + static_cast<uint32_t>(r0 * CPS), v);
        if constexpr (CPS == 2) {
          const int hp = (lane & 1) * 2;
          const int roff = (lane >> 2) + ((lane & 2) ? 8 : 0);
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) {
            const int r = r0 + q2;
            float part = 0.f;
            if (r < nr) {
              const float f0 = hp < G ? mr[r * G + hp] : 0.f;
              const float f1 = hp + 1 < G ? mr[r * G + hp + 1] : 0.f;
              part = fmaf(v[2 * q2 + 1], f1, v[2 * q2] * f0);
            }
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            const int row = (ph + r * nph) * 16 + roff;
            if (r < nr && (lane & 1) == 0 && row < nloc) cp[row] = part;
          }
        } else {
          const int g0 = (lane & 3) * 2;
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            const int r = r0 + q2;
            float pa = 0.f, pb = 0.f;
            if (r < nr) {
              const float f0 = g0 < G ? mr[r * G + g0] : 0.f;
              const float f1 = g0 + 1 < G ? mr[r * G + g0 + 1] : 0.f;
              pa = fmaf(v[4 * q2 + 1], f1, v[4 * q2] * f0);
              pb = fmaf(v[4 * q2 + 3], f1, v[4 * q2 + 2] * f0);
            }
            pa += __shfl_xor_sync(0xffffffffu, pa, 1);
            pb += __shfl_xor_sync(0xffffffffu, pb, 1);
            pa += __shfl_xor_sync(0xffffffffu, pa, 2);
            pb += __shfl_xor_sync(0xffffffffu, pb, 2);
            const int row = (ph + r * nph) * 16 + (lane >> 2);
            if (r < nr && (lane & 3) == 0) {
              if (row < nloc) cp[row] = pa;
              if (row + 8 < nloc) cp[row + 8] = pb;
            }
          }
        }
      }
    }
    tmem_fence_before_sync();
    __syncthreads();
    if (warp == 1) {
      tmem_fence_after_sync();
      tmem_dealloc512(tbase);
    }
    trace_at(p, 14);
    // crit[j] = sum over the kv heads (fixed order) -> key -> pass-1 histogram
    const bool radix = T > p.k;
    for (int b0 = 0; b0 < nloc; b0 += kStepThreads) {
      const int j = b0 + tid;
      float cr = 0.f;
      if (j < nloc)
        for (int g = 0; g < Hkv; ++g) cr += cpart[g * tpc + j];
      const uint32_t key = float_key(cr);
      if (j < nloc) keys[j] = key;
      if (radix) hist_add(hist, key, j < nloc, 20);
    }
    __syncthreads();
    trace_at(p, 5);

    // ------------------------------------------------------------ top-k
    // larger criticality first; keys equal in their top 24 bits rank as ties
    // (relative difference < 2^-15, inside the 1e-4 tie tolerance), which go
    // to the smaller position (tensor.cpp:81-88)
    uint32_t tau = 0, kk = static_cast<uint32_t>(p.k), take_all_eq = 1;
    int shift = 20;
    uint32_t pre_eq = 0;
    if (radix) {
      hist_merge(hist, p.ws_hist);
      gs.sync();  // B2
      trace_at(p, 6);
      uint32_t b1, above, cnt;
      find_bin(p.ws_hist, kk, scratch, hist, &b1, &above, &cnt);
      trace_at(p, 16);
      kk -= above;
      tau = b1;
      uint32_t eq_total = cnt;
      if (cnt > kk) {
        // the boundary bin is split: next 12 bits of its keys
        for (int i = tid; i < kRadixBins; i += kStepThreads) hist[i] = 0u;
        __syncthreads();
        for (int b0 = 0; b0 < nloc; b0 += kStepThreads) {
          const int j = b0 + tid;
          const uint32_t key = j < nloc ? keys[j] : 0u;
          hist_add(hist, key, j < nloc && (key >> 20) == b1, 8);
        }
        __syncthreads();
        hist_merge(hist, p.ws_hist + kRadixBins);
        trace_at(p, 17);
        gs.sync();  // B3
        trace_at(p, 18);
        uint32_t b2;
        find_bin(p.ws_hist + kRadixBins, kk, scratch, hist, &b2, &above, &eq_total);
        kk -= above;
        tau = (b1 << 12) | b2;
        shift = 8;
      }
      trace_at(p, 7);
      if (eq_total > kk) {
        // ties straddle the budget: the lowest positions win (every CTA's count)
        uint32_t neq = 0;
        for (int j = tid; j < nloc; j += kStepThreads) neq += (keys[j] >> shift) == tau;
        uint32_t tot;
        block_scan(neq, scratch, &tot);
        if (tid == 0) p.ws_cnt[cta] = tot;
        gs.sync();  // B3b
        if (tid < 32) {
          uint32_t s2 = 0;
#pragma unroll 1
          for (int c = tid; c < cta; c += 32) s2 += __ldcg(p.ws_cnt + c);
          s2 = __reduce_add_sync(0xffffffffu, s2);
          if (tid == 0) scratch[70] = s2;
        }
        __syncthreads();
        pre_eq = scratch[70];
        __syncthreads();
        take_all_eq = 0;
      }
    }
    // ascending compaction of this CTA's selected candidates
    uint32_t eq_seen = 0;
    for (int b0 = 0; b0 < nloc; b0 += kStepThreads) {
      const int j = b0 + tid;
      const uint32_t key = j < nloc ? keys[j] : 0u;
      bool take = j < nloc;
      if (radix && take) {
        const uint32_t kd = key >> shift;
        take = kd > tau || (kd == tau && take_all_eq);
      }
      if (radix && !take_all_eq) {
        const uint32_t is_eq = (j < nloc && (key >> shift) == tau) ? 1u : 0u;
        uint32_t eq_tot;
        const uint32_t rk = pre_eq + eq_seen + block_scan(is_eq, scratch, &eq_tot);
        if (is_eq && rk < kk) take = true;
        eq_seen += eq_tot;
      }
      uint32_t tot;
      const uint32_t pos = n_own + block_scan(take ? 1u : 0u, scratch, &tot);
      if (take) {
        sl_tok[pos] = static_cast<uint32_t>(p.cand_begin + j0 + j);
        sl_row[pos] = frames[j];
        sl_key[pos] = key;
        // attended right below: start the HBM reads now
        const uint64_t pol = policy_evict_last();
        bulk_prefetch_l2(reinterpret_cast<const char*>(p.k_slab) + static_cast<size_t>(frames[j]) * row_bytes, row_bytes, pol);
        bulk_prefetch_l2(reinterpret_cast<const char*>(p.v_slab) + static_cast<size_t>(frames[j]) * row_bytes, row_bytes, pol);
      }
      n_own += tot;
    }
    if (tid == 0) p.ws_nsel[cta] = n_own;
  }
  trace_at(p, 8);

  // ---------------------------------------------------------------- phase 3
  // rows of this CTA: [selected part | window slice]
  if (miss) n_sel_part = static_cast<int>(n_own);
#ifdef STEP_TWICE
  for (int twice = 0; twice < 2; ++twice) {
    __syncthreads();
#endif
  if (tid < H) {
    st_m[tid] = -INFINITY;
    st_l[tid] = 0.f;
  }
  // q of this warp's kv head in registers: lane holds d = 4 lane .. 4 lane + 3
  float qr[G][4];
  const int akv = (warp - 1) % Hkv, aph = (warp - 1) / Hkv;  // attention warp = (kv head, row phase)
  if (warp >= 1) {
#pragma unroll
    for (int m = 0; m < G; ++m) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(p.q + static_cast<size_t>(m * Hkv + akv) * kD) + lane);
      qr[m][0] = x.x * p.attn_scale;
      qr[m][1] = x.y * p.attn_scale;
      qr[m][2] = x.z * p.attn_scale;
      qr[m][3] = x.w * p.attn_scale;
    }
  }
  float acc[G][4];
#pragma unroll
  for (int m = 0; m < G; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
  __syncthreads();
  const int R = n_sel_part + n_win;
  const int nbatch = max(1, (R + kRB - 1) / kRB);
  uint32_t aparity = 0;
  for (int bt = 0; bt < nbatch; ++bt) {
    const int r0 = bt * kRB, nb = min(kRB, R - r0);
    const bool cur_here = has_cur && bt == nbatch - 1;
    if (nb > 0) {
      if (tid == 0) mbar_arrive_expect_tx(abar, static_cast<uint32_t>(2 * nb * row_bytes));
      __syncthreads();
      if (tid < nb) {
        const int i = r0 + tid;
        const int32_t row = i < n_sel_part ? (miss ? sl_row[i] : hrow[i]) : wrow[i - n_sel_part];
        const size_t off = static_cast<size_t>(row) * row_bytes;
        bulk_g2s_nohint(att_k + static_cast<size_t>(tid) * Hkv * kD, reinterpret_cast<const char*>(p.k_slab) + off,
                        row_bytes, abar);
        bulk_g2s_nohint(att_v + static_cast<size_t>(tid) * Hkv * kD, reinterpret_cast<const char*>(p.v_slab) + off,
                        row_bytes, abar);
      }
      mbar_wait(abar, aparity);
      aparity ^= 1u;
    }
    trace_at(p, 9);
    // scores s[i][h] = q_h . k_i / sqrt(d) (attention.cpp:72-86)
    if (warp >= 1) {
      for (int i = aph; i < nb + (cur_here ? 1 : 0); i += nph) {
        float kv[4];
        if (i < nb) {
          const uint2 x = *reinterpret_cast<const uint2*>(att_k + static_cast<size_t>(i) * Hkv * kD + akv * kD + 4 * lane);
          const float2 a = bf16x2_to_f2(x.x), b = bf16x2_to_f2(x.y);
          kv[0] = a.x, kv[1] = a.y, kv[2] = b.x, kv[3] = b.y;
        } else {
          const float4 x = __ldg(reinterpret_cast<const float4*>(p.k_new + akv * kD) + lane);
          kv[0] = x.x, kv[1] = x.y, kv[2] = x.z, kv[3] = x.w;
        }
        float sv[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          sv[m] = 0.f;
          if (m < G) sv[m] = fmaf(qr[m][3], kv[3], fmaf(qr[m][2], kv[2], fmaf(qr[m][1], kv[1], qr[m][0] * kv[0])));
        }
        const float tot = reduce8(sv, lane);
        const int m = (lane >> 2) & 7;
        if ((lane & 3) == 0 && m < G) scores[i * 64 + m * Hkv + akv] = tot;
      }
    }
    __syncthreads();
    trace_at(p, 19);
    // online softmax per head over this batch (attention.cpp:88-110)
    // warp per head, lane per row (n <= kRB + 1 <= 32)
    for (int h = warp; h < H; h += kNW) {
      const int n = nb + (cur_here ? 1 : 0);
      const float s = lane < n ? scores[lane * 64 + h] : -INFINITY;
      const float mo = st_m[h], mn = fmaxf(mo, warp_max(s));
      const float e = lane < n ? ex2_approx((s - mn) * kL2E) : 0.f;
      if (lane < n) scores[lane * 64 + h] = e;
      const float ls = warp_sum(e);
      if (lane == 0) {
        const float corr = mo == -INFINITY ? 0.f : ex2_approx((mo - mn) * kL2E);
        st_m[h] = mn;
        st_l[h] = st_l[h] * corr + ls;
        st_c[h] = corr;
      }
    }
    __syncthreads();
    trace_at(p, 20);
    // P.V
    if (warp >= 1) {
#pragma unroll
      for (int m = 0; m < G; ++m) {
        const float cf = st_c[m * Hkv + akv];
        acc[m][0] *= cf, acc[m][1] *= cf, acc[m][2] *= cf, acc[m][3] *= cf;
      }
      for (int i = aph; i < nb + (cur_here ? 1 : 0); i += nph) {
        float vv[4];
        if (i < nb) {
          const uint2 x = *reinterpret_cast<const uint2*>(att_v + static_cast<size_t>(i) * Hkv * kD + akv * kD + 4 * lane);
          const float2 a = bf16x2_to_f2(x.x), b = bf16x2_to_f2(x.y);
          vv[0] = a.x, vv[1] = a.y, vv[2] = b.x, vv[3] = b.y;
        } else {
          const float4 x = __ldg(reinterpret_cast<const float4*>(p.v_new + akv * kD) + lane);
          vv[0] = x.x, vv[1] = x.y, vv[2] = x.z, vv[3] = x.w;
        }
#pragma unroll
        for (int m = 0; m < G; ++m) {
          const float pm = scores[i * 64 + m * Hkv + akv];
          acc[m][0] = fmaf(pm, vv[0], acc[m][0]);
          acc[m][1] = fmaf(pm, vv[1], acc[m][1]);
          acc[m][2] = fmaf(pm, vv[2], acc[m][2]);
          acc[m][3] = fmaf(pm, vv[3], acc[m][3]);
        }
      }
    }
    __syncthreads();  // staging and scores free for the next batch
    trace_at(p, 21);
  }
  // the nph row phases of each kv head meet in shared memory (fixed order)
  if (warp >= 1) {
#pragma unroll
    for (int m = 0; m < G; ++m)
      *reinterpret_cast<float4*>(red + (static_cast<size_t>(aph) * H + m * Hkv + akv) * kD + 4 * lane) =
          make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
  }
  __syncthreads();
  float* po = p.ws_o + static_cast<size_t>(cta) * width;
  for (int i = tid; i < width / 4; i += kStepThreads) {
    float4 a = reinterpret_cast<const float4*>(red)[i];
    for (int q2 = 1; q2 < nph; ++q2) {
      const float4 b = reinterpret_cast<const float4*>(red + static_cast<size_t>(q2) * width)[i];
      a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    }
    reinterpret_cast<float4*>(po)[i] = a;
  }
  if (tid < H) p.ws_ml[static_cast<size_t>(cta) * H + tid] = make_float2(st_m[tid], st_l[tid]);
  trace_at(p, 10);
#ifdef STEP_TWICE
  }
#endif
  gs.sync();  // B4: every CTA's partial is in
  trace_at(p, 11);

  // ---------------------------------------------------------------- merge
  // outputs [o0, o0 + per) of the H*d, log-sum-exp over all CTAs' partials
  {
    const int per = (width + ncta - 1) / ncta;
    const int o0 = min(width, cta * per), no = min(width, o0 + per) - o0;
    float* mbuf = reinterpret_cast<float*>(ring);          // [2][ncta] weights (m, then e^(m - M))
    float* lbuf = mbuf + 2 * ncta;                          // [2][ncta] l
    float* obuf = lbuf + 2 * ncta;                          // [ncta][no]
    float* hdr = obuf + static_cast<size_t>(ncta) * per;    // [2] L
    const int hA = o0 / kD;
    // every load in flight at once (one L2 round trip), then into shared memory
    constexpr int kU = 8;
    float ov[kU];
    float2 mlv = make_float2(-INFINITY, 0.f);
    const int nld = ncta * no;
    if (tid < 2 * ncta) {
      const int hh = tid / ncta, c = tid - hh * ncta;
      if (hA + hh < H) mlv = __ldcg(p.ws_ml + static_cast<size_t>(c) * H + hA + hh);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = tid + u * kStepThreads;
      const int nq = max(no, 1);
      const int c = i / nq, oo = i - (i / nq) * nq;
      ov[u] = i < nld ? __ldcg(p.ws_o + static_cast<size_t>(c) * width + o0 + oo) : 0.f;
    }
    if (tid < 2 * ncta) {
      mbuf[tid] = mlv.x;
      lbuf[tid] = mlv.y;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = tid + u * kStepThreads;
      if (i < nld) obuf[i] = ov[u];
    }
    for (int i = tid + kU * kStepThreads; i < nld; i += kStepThreads) {
      const int c = i / no, oo = i - c * no;
      obuf[i] = __ldcg(p.ws_o + static_cast<size_t>(c) * width + o0 + oo);
    }
    __syncthreads();
    trace_at(p, 22);
    if (warp < 2) {
      const int hh = warp;
      float M = -INFINITY;
      for (int c = lane; c < ncta; c += 32) M = fmaxf(M, mbuf[hh * ncta + c]);
      M = warp_max(M);
      float L = 0.f;
      for (int c = lane; c < ncta; c += 32) {
        const float mc = mbuf[hh * ncta + c];
        const float w = (mc == -INFINITY) ? 0.f : ex2_approx((mc - M) * kL2E);
        mbuf[hh * ncta + c] = w;
        L = fmaf(w, lbuf[hh * ncta + c], L);
      }
      L = warp_sum(L);
      if (lane == 0) hdr[hh] = L;
    }
    __syncthreads();
    trace_at(p, 23);
    // warp per output, lanes strided over the CTAs (fixed order: lane sums,
    // then the butterfly)
    for (int oo = warp; oo < no; oo += kNW) {
      const int hh = (o0 + oo) / kD - hA;
      float a = 0.f;
      for (int c = lane; c < ncta; c += 32) a = fmaf(mbuf[hh * ncta + c], obuf[c * no + oo], a);
      a = warp_sum(a);
      if (lane == 0) {
        const float L = hdr[hh];
        p.out[o0 + oo] = L > 0.f ? a / L : 0.f;
      }
    }
  }
  // ---------------------------------------------------------------- cache entry
  if (miss) {
    // the SelectionResult, ascending: this CTA's list at the prefix of the counts
    // (one count per thread, all loads in flight: ncta <= kStepThreads)
    const uint32_t v = tid < ncta ? __ldcg(p.ws_nsel + tid) : 0u;
    const uint32_t s2 = __reduce_add_sync(0xffffffffu, tid < cta ? v : 0u);
    const uint32_t t2 = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) {
      scratch[100 + warp] = s2;
      scratch[120 + warp] = t2;
    }
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int w = 0; w < kNW; ++w) {
      off += scratch[100 + w];
      tot += scratch[120 + w];
    }
    const uint64_t pol = policy_evict_last();
    for (int i = tid; i < static_cast<int>(n_own); i += kStepThreads) {
      st_hint_u32(p.sel + off + i, sl_tok[i], pol);
      st_hint_u32(p.sel_crit + off + i, __float_as_uint(key_float(sl_key[i])), pol);
      st_hint_u32(p.sel_rows + off + i, static_cast<uint32_t>(sl_row[i]), pol);
    }
    if (cta == 0 && tid == 0) p.cache->n_sel = static_cast<int>(tot);
  }
  if (cta == 0 && tid == 0 && (own == kOwnMiss || own == kOwnHit)) {
    CacheState* c = p.cache;
    c->lookups += 1;
    if (own == kOwnHit) c->hits += 1;
    else c->first_flag = 0;
    c->last_hit = own == kOwnHit ? 1 : 0;
    c->last_cos = cosv;
  }
  trace_at(p, 12);
}

}  // namespace

const void* step_kernel_ptr(int G) {
  switch (G) {
    case 1: return reinterpret_cast<const void*>(&step_kernel<1>);
    case 2: return reinterpret_cast<const void*>(&step_kernel<2>);
    case 3: return reinterpret_cast<const void*>(&step_kernel<3>);
    case 4: return reinterpret_cast<const void*>(&step_kernel<4>);
    case 5: return reinterpret_cast<const void*>(&step_kernel<5>);
    case 6: return reinterpret_cast<const void*>(&step_kernel<6>);
    case 7: return reinterpret_cast<const void*>(&step_kernel<7>);
    case 8: return reinterpret_cast<const void*>(&step_kernel<8>);
  }
  return nullptr;
}

size_t step_smem_bytes(int H, int H_kv, int tpc, int stages_per_warp, int ring_stages) {
  const int G = H / H_kv;
  const size_t row_bytes = static_cast<size_t>(H_kv) * kD * 2;
  const size_t sbytes = 16 * (row_bytes + 16);
  const size_t ring = align_up(static_cast<size_t>(ring_stages) * sbytes, 1024);
  size_t o = ring + align_up(static_cast<size_t>(kCons) * stages_per_warp * G * 4, 128);
  o += align_up(static_cast<size_t>(tpc) * 4, 128);
  o += 1024 + kCons * 8 * 8 + 4 * 64 * 4 + (kMaxHitSlice + kMaxWinSlice) * 4;
  o += (2 * kMaxBarPairs + 1) * 8;
  return align_up(o, 128);
}

}  // namespace tsb

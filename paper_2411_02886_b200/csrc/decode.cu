// Fused persistent decode-step kernel (sm_100a).
//
// One cooperative launch runs the whole TokenSelect decode step of
// decode_step (reference attention.cpp:172-200) for one or more sequences:
//
//   phase 0  K1 append of the current token's K/V row (kv_pool.cpp:55-85)
//            K2 Selection Cache test, fp64 cosine vs. the cached query
//               (selection_cache.cpp:16-44, tensor.cpp:92-113)
//   phase 1  K3 paged dot-product scan S = q.K over the candidates
//               (selector.cpp:26-68, Alg. 2): K rows streamed by the TMA engine
//               (cp.async.bulk, evict_first) through an mbarrier ring, GQA
//               group sharing each row, FFMA2 + shuffle reduce-scatter;
//               per-CTA head max tracked on the fly, S kept on chip.
//   phase 2  K4 soft vote (softmax_rows + select_head_soft_vote,
//               tensor.cpp:31-52, selector.cpp:113-126): per-CTA (m, z),
//               one grid exchange, crit[j] = sum_h exp(S-M_h)/Z_h
//   phase 3  K5 radix select (11/11/10-bit digits) with the reference's tie
//               rule (larger score first, smaller index on ties, output
//               ascending; tensor.cpp:68-90, selector.cpp:72-85)
//   phase 4  K7 split-K sparse flash-decoding over init U selected U local U
//               current (make_windows attention.cpp:35-52, sdpa_full :54-112)
//   phase 5  K8 log-sum-exp merge of the per-CTA partials.
//
// Sequences of a batch are given disjoint CTA groups; phases are separated
// by grid barriers (all CTAs co-resident: cudaLaunchCooperativeKernel).
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "decode.h"
#include "params.h"

namespace tsb {

namespace {

constexpr int kBins = 2048;

struct Smem {
  uint8_t* ring;
  float* S;        // [H][tpc] (when on chip)
  uint32_t* keys;  // [tpc]
  uint32_t* hist;  // [kBins]
  int* headmax;    // [H] ordered-int max
  float* f;        // [H]
  uint32_t* scratch;  // [64]
  int32_t* frames; // [tpc] slab row of each local candidate
  uint64_t* full;  // [kMaxStages]
  uint64_t* empty; // [kMaxStages]
  uint64_t* att;   // attention staging barrier
  uint64_t* aux;   // bulk staging barrier (stats, partials)
};

__device__ __forceinline__ Smem carve(uint8_t* base, const DecodeParams& p) {
  SmemLayout L = smem_layout(p.H, p.H_kv * p.d * 2, p.tpc, p.s_in_smem, p.ring_bytes);
  Smem s;
  s.ring = base + L.ring;
  s.S = reinterpret_cast<float*>(base + L.s);
  s.keys = reinterpret_cast<uint32_t*>(base + L.keys);
  s.hist = reinterpret_cast<uint32_t*>(base + L.hist);
  s.headmax = reinterpret_cast<int*>(base + L.headmax);
  s.f = reinterpret_cast<float*>(base + L.f);
  s.scratch = reinterpret_cast<uint32_t*>(base + L.scratch);
  s.full = reinterpret_cast<uint64_t*>(base + L.bars);
  s.empty = s.full + kMaxStages;
  s.att = s.full + 2 * kMaxStages;
  s.aux = s.att + 1;
  s.frames = reinterpret_cast<int32_t*>(base + L.frames);
  return s;
}

__device__ __forceinline__ uint32_t cand_at(const SeqDesc& sd, int j) {
  return sd.cand ? sd.cand[j] : static_cast<uint32_t>(sd.cand_begin + j);
}

__device__ __forceinline__ size_t row_index(const SeqDesc& sd, uint32_t tok, int page_size) {
  if (page_size == 1) return static_cast<size_t>(sd.page_table[tok]);
  return static_cast<size_t>(sd.page_table[tok / page_size]) * page_size + tok % page_size;
}

// Phase trace: CTA 0 records %globaltimer at phase boundaries when enabled.
__device__ __forceinline__ void trace_pt(const DecodeParams& p, int i) {
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[i] = t;
  }
}

// Block-wide exclusive scan of one value per thread (all threads call).
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(v, lane);
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kDecodeWarps ? scratch[lane] : 0u;
    uint32_t wi = warp_incl_scan(w, lane);
    if (lane < kDecodeWarps) scratch[32 + lane] = wi - w;
    if (lane == 31) scratch[63] = wi;
  }
  __syncthreads();
  const uint32_t r = scratch[32 + warp] + inc - v;
  if (total) *total = scratch[63];
  __syncthreads();
  return r;
}

// Finds, in a histogram whose bins are ordered by key, the bin b such that
// count(bins > b) < kk <= count(bins >= b). Returns b and count(bins > b).
// All threads call; every CTA computes the same answer from the same data.
__device__ void find_bin(const uint32_t* gh, int nbins, uint32_t kk, uint32_t* scratch,
                         int* bin_out, uint32_t* above_out) {
  // thread t covers bins [nbins - (t+1)*per, nbins - t*per) in descending order
  const int per = (nbins + 511) / 512;
  const int t = threadIdx.x;
  uint32_t sum = 0;
  if (t < 512) {
    for (int i = 0; i < per; ++i) {
      const int b = nbins - 1 - (t * per + i);
      if (b >= 0) sum += __ldcg(gh + b);
    }
  }
  uint32_t tot;
  const uint32_t ex = block_excl_scan(t < 512 ? sum : 0u, scratch, &tot);
  if (t < 512 && ex < kk && ex + sum >= kk) {
    uint32_t acc = ex;
    for (int i = 0; i < per; ++i) {
      const int b = nbins - 1 - (t * per + i);
      const uint32_t c = __ldcg(gh + b);
      if (acc + c >= kk) {
        scratch[64] = static_cast<uint32_t>(b);
        scratch[65] = acc;
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
  *bin_out = static_cast<int>(scratch[64]);
  *above_out = scratch[65];
  __syncthreads();
}

// fp64 cosine Selection Cache decision (tensor.cpp:92-113,
// selection_cache.cpp:29-35). Deterministic block reduction: every CTA that
// evaluates it for the same sequence gets a bit-identical result.
// Returns 1 = miss, 0 = hit, 2 = zero query (error).
__device__ int cache_decision(const SeqDesc& sd, int width, double* scratch_d, double* cos_out) {
  const CacheState* cs = sd.cache;
  double dot = 0.0, nu = 0.0, nv = 0.0;
  int nonzero = 0;
  constexpr int kU = 8;  // loads in flight per thread
  for (int base = threadIdx.x; base < width; base += kU * blockDim.x) {
    float qa[kU], qb[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * blockDim.x;
      qa[u] = i < width ? __ldg(sd.q + i) : 0.f;
      qb[u] = i < width ? __ldcg(sd.cached_q + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const double a = static_cast<double>(qa[u]);
      const double b = static_cast<double>(qb[u]);
      nonzero |= (qa[u] != 0.0f);
      dot = fma(a, b, dot);
      nu = fma(a, a, nu);
      nv = fma(b, b, nv);
    }
  }
  nonzero = __syncthreads_or(nonzero);
  dot = warp_sum_d(dot);
  nu = warp_sum_d(nu);
  nv = warp_sum_d(nv);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    scratch_d[warp * 3 + 0] = dot;
    scratch_d[warp * 3 + 1] = nu;
    scratch_d[warp * 3 + 2] = nv;
  }
  __syncthreads();
  // every warp reduces the per-warp partials in the same fixed tree order
  double D = lane < kDecodeWarps ? scratch_d[lane * 3 + 0] : 0.0;
  double U = lane < kDecodeWarps ? scratch_d[lane * 3 + 1] : 0.0;
  double V = lane < kDecodeWarps ? scratch_d[lane * 3 + 2] : 0.0;
  D = warp_sum_d(D);
  U = warp_sum_d(U);
  V = warp_sum_d(V);
  __syncthreads();
  if (!nonzero) return 2;
  *cos_out = NAN;
  if (cs->first_flag) return 1;
  if (U == 0.0 || V == 0.0) return 1;  // unreachable: cached query is never zero
  double c;
  if (D * D >= U * V) c = D >= 0.0 ? 1.0 : -1.0;  // exact +-1 clamp
  else c = D / sqrt(U * V);
  *cos_out = c;
  return c < cs->theta ? 1 : 0;  // strict <
}

// --------------------------------------------------------------- the scan
// Fast path (sm_100a tensor cores, mma.sync bf16 -> fp32). The K rows of a
// stage (16 tokens, padded stride so ldmatrix is bank-conflict free) are the
// M x K operand; the query, exactly split into three bf16 parts
// (q = q_hi + q_mid + q_lo, 8+8+8 mantissa bits), is the K x N operand with
// one column per query head of the GQA group (h = g*H_kv + kvh, the
// reference's h mod H_kv map, selector.cpp:51). bf16 x bf16 products are
// exact in fp32, so S = sum_d q*k is formed from exact products with fp32
// accumulation. Consumer warp c owns kv head c % H_kv and every
// (16/H_kv)-th stage; one warp task = 16 tokens x one kv head.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
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

template <int D, int G>
__device__ void scan_fast(const DecodeParams& p, const SeqDesc& sd, const Smem& sm, int j0,
                          int nloc, float* Sbuf, int sstride, float* s_out_row0) {
  constexpr int KC = D / 16;  // k-chunks of 16 along d
  const int Hkv = p.H_kv;
  const int row_bytes = Hkv * D * 2;
  const int rstride = row_bytes + 16;  // padded ring row (ldmatrix conflict-free)
  const ScanGeom geom = scan_geom(p.H, p.H_kv, D, p.ring_bytes);
  const int R = geom.rows;  // 16 tokens per stage
  const int kStages = geom.stages;
  const int nit = (nloc + R - 1) / R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    // slab rows of all local candidates were staged in smem (sm.frames), so
    // issuing a stage is latency-free; rows land at a padded stride.
    const uint64_t pol = policy_evict_first();
    const char* kbase = reinterpret_cast<const char*>(p.k_slab);
    for (int it = 0; it < nit; ++it) {
      const int s = it % kStages;
      const int rbase = it * R;
      const int nrows = min(R, nloc - rbase);
      if (it >= kStages) mbar_wait(&sm.empty[s], ((it / kStages) & 1) ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[s], static_cast<uint32_t>(nrows * row_bytes));
      __syncwarp();
      if (lane < nrows)
        bulk_g2s(sm.ring + static_cast<size_t>(s * R + lane) * rstride,
                 kbase + static_cast<size_t>(sm.frames[rbase + lane]) * row_bytes, row_bytes, &sm.full[s], pol);
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = warp - 1;
  const int nphase = kDecodeConsumers / Hkv;
  const int kvh = cw % Hkv, phase = cw / Hkv;
  // B fragments: lane holds q[head g = lane/4][d = kc*16 + (lane%4)*2 + {0,1,8,9}]
  uint32_t bq[KC][3][2];
  {
    const int g = lane >> 2;
    const float* qh = sd.q + static_cast<size_t>(g * Hkv + kvh) * D;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int dd = kc * 16 + (lane & 3) * 2 + (e & 1) + (e >> 1) * 8;
        v[e] = g < G ? qh[dd] : 0.f;
      }
      float hi[4], mi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) split3(v[e], hi[e], mi[e], lo[e]);
      bq[kc][0][0] = pack_bf16x2(hi[0], hi[1]);
      bq[kc][0][1] = pack_bf16x2(hi[2], hi[3]);
      bq[kc][1][0] = pack_bf16x2(mi[0], mi[1]);
      bq[kc][1][1] = pack_bf16x2(mi[2], mi[3]);
      bq[kc][2][0] = pack_bf16x2(lo[0], lo[1]);
      bq[kc][2][1] = pack_bf16x2(lo[2], lo[3]);
    }
  }
  // this lane's C fragment: rows lane/4 (+8), columns (heads) 2*(lane%4) + {0,1}
  const int g0 = (lane & 3) * 2;
  float runmax0 = -INFINITY, runmax1 = -INFINITY;
  // ldmatrix row address: matrix lane/8 -> rows +8 for odd, cols +8 for >= 16
  const uint32_t lrow = static_cast<uint32_t>((lane & 7) + ((lane >> 3) & 1) * 8);
  const uint32_t lcol = static_cast<uint32_t>((lane >> 4) * 16 + kvh * D * 2);
  const uint32_t ring_base = smem_u32(sm.ring) + lrow * rstride + lcol;
  for (int it = phase; it < nit; it += nphase) {
    const int s = it % kStages;
    mbar_wait(&sm.full[s], (it / kStages) & 1);
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    if (!(p.debug_flags & 1)) {
      const uint32_t abase = ring_base + static_cast<uint32_t>(s * R * rstride);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t a[4];
        ldmatrix_x4(a, abase + kc * 32);
        mma_bf16_16816(c, a, bq[kc][0][0], bq[kc][0][1]);
        mma_bf16_16816(c, a, bq[kc][1][0], bq[kc][1][1]);
        mma_bf16_16816(c, a, bq[kc][2][0], bq[kc][2][1]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);  // operands consumed
    const int rbase = it * R + (lane >> 2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int g = g0 + (e & 1);
      const int row = rbase + (e >> 1) * 8;
      if (g < G && row < nloc) {
        const int h = g * Hkv + kvh;
        Sbuf[static_cast<size_t>(h) * sstride + row] = c[e];
        if (s_out_row0) s_out_row0[static_cast<size_t>(h) * sd.n_cand + row] = c[e];
        if (e & 1) runmax1 = fmaxf(runmax1, c[e]);
        else runmax0 = fmaxf(runmax0, c[e]);
      }
    }
  }
  if (g0 < G && runmax0 > -INFINITY) atomicMax(&sm.headmax[g0 * Hkv + kvh], float_ord(runmax0));
  if (g0 + 1 < G && runmax1 > -INFINITY) atomicMax(&sm.headmax[(g0 + 1) * Hkv + kvh], float_ord(runmax1));
}

// Generic path (any H, H_kv, d, page_size): one thread per (head, token),
// fp64 accumulation in the reference's d order, rounded to fp32 — this
// reproduces score_paged's S bit for bit (bf16 x fp32 products are exact in
// fp64, so the fused multiply-add equals the reference's multiply-then-add).
__device__ void scan_generic(const DecodeParams& p, const SeqDesc& sd, const Smem& sm, int j0,
                             int nloc, float* Sbuf, int sstride, float* s_out_row0) {
  const int d = p.d, row = p.H_kv * d;
  const int total = p.H * nloc;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int h = idx / nloc, jl = idx - (idx / nloc) * nloc;
    const uint16_t* key = p.k_slab + static_cast<size_t>(sm.frames[jl]) * row + (h % p.H_kv) * d;
    const float* qh = sd.q + static_cast<size_t>(h) * d;
    double acc = 0.0;
    for (int t = 0; t < d; ++t) acc = fma(static_cast<double>(qh[t]), static_cast<double>(bf16_bits_to_f(key[t])), acc);
    const float s = static_cast<float>(acc);
    Sbuf[static_cast<size_t>(h) * sstride + jl] = s;
    if (s_out_row0) s_out_row0[static_cast<size_t>(h) * sd.n_cand + jl] = s;
    atomicMax(&sm.headmax[h], float_ord(s));
  }
}

// ---------------------------------------------------------- attention rows
struct AttView {
  int n_rows;      // cached attended rows (excl. current)
  int init_end, lo1, n1, lb2;
};

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t att_token(const SeqDesc& sd, const AttView& v, int i) {
  if (sd.att_list) return sd.att_list[i];
  if (i < v.init_end) return static_cast<uint32_t>(i);
  i -= v.init_end;
  if (i < v.n1) return sd.sel[v.lo1 + i];
  i -= v.n1;
  return static_cast<uint32_t>(v.lb2 + i);
}

// split-K flash-decoding partial over rows [r0, r1) of the merged window
// list, plus the current token when `with_cur`; writes (o[d], m, l) per head.
// Rows are staged in smem (bulk copies, padded stride); per head a warp
// scores all staged rows at once (lane = row, q broadcast from smem), then
// does one online-softmax update and the P.V accumulation (lane = d slice).
__device__ void attend_partial(const DecodeParams& p, const SeqDesc& sd, const AttView& av,
                               const Smem& sm, int r0, int r1, bool with_cur, float* part) {
  const int H = p.H, Hkv = p.H_kv, d = p.d;
  const int row_elems = Hkv * d;
  const int row_bytes = row_elems * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kMaxDL = 8;            // d <= 256
  constexpr int kMaxHeadsPerWarp = 4;  // H <= 64
  const bool vec = (row_bytes % 16) == 0 && (d % 8) == 0;
  const int rstride = vec ? row_elems + 8 : row_elems;  // bf16 elements; +16 B breaks bank aliasing
  const bool d128 = vec && d == 128;                   // vectorised P.V layout (see below)
  // carve the ring: q (fp32, H*d) then K rows then V rows
  float* qs = reinterpret_cast<float*>(sm.ring);
  uint16_t* kbuf = reinterpret_cast<uint16_t*>(sm.ring + align_up(static_cast<size_t>(H) * d * 4, 128));
  const size_t avail = kRingBudget - align_up(static_cast<size_t>(H) * d * 4, 128);
  int cap = static_cast<int>(avail / (2 * static_cast<size_t>(rstride) * 2));
  if (cap > 32) cap = 32;
  uint16_t* vbuf = kbuf + static_cast<size_t>(cap) * rstride;
  for (int base = threadIdx.x; base < H * d; base += 8 * blockDim.x) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * blockDim.x;
      v[u] = i < H * d ? __ldg(sd.q + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * blockDim.x;
      if (i < H * d) qs[i] = v[u];
    }
  }
  float m_run[kMaxHeadsPerWarp], l_run[kMaxHeadsPerWarp], o_run[kMaxHeadsPerWarp][kMaxDL];
#pragma unroll
  for (int hs = 0; hs < kMaxHeadsPerWarp; ++hs) {
    m_run[hs] = -INFINITY;
    l_run[hs] = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxDL; ++i) o_run[hs][i] = 0.f;
  }
  uint32_t att_phase = 0;
  for (int c0 = r0; c0 < r1; c0 += cap) {
    const int nr = min(cap, r1 - c0);
    __syncthreads();  // previous sub-chunk consumed; qs visible
    if (vec) {
      if (threadIdx.x == 0) mbar_arrive_expect_tx(sm.att, static_cast<uint32_t>(nr * 2 * row_bytes));
      __syncthreads();
      if (static_cast<int>(threadIdx.x) < nr) {
        const int r = threadIdx.x;
        const size_t ri = row_index(sd, att_token(sd, av, c0 + r), p.page_size);
        bulk_g2s_nohint(kbuf + static_cast<size_t>(r) * rstride, p.k_slab + ri * row_elems, row_bytes, sm.att);
        bulk_g2s_nohint(vbuf + static_cast<size_t>(r) * rstride, p.v_slab + ri * row_elems, row_bytes, sm.att);
      }
      mbar_wait(sm.att, att_phase);
      att_phase ^= 1u;
    } else {
      for (int idx = threadIdx.x; idx < nr * row_elems * 2; idx += blockDim.x) {
        const int which = idx / (nr * row_elems);
        const int rem = idx - which * nr * row_elems;
        const int r = rem / row_elems, c = rem - (rem / row_elems) * row_elems;
        const uint32_t tok = att_token(sd, av, c0 + r);
        const uint16_t* src = (which ? p.v_slab : p.k_slab) + row_index(sd, tok, p.page_size) * row_elems;
        ((which ? vbuf : kbuf) + static_cast<size_t>(r) * rstride)[c] = src[c];
      }
      __syncthreads();
    }
#pragma unroll
    for (int hs = 0; hs < kMaxHeadsPerWarp; ++hs) {
      const int h = warp + hs * kDecodeWarps;
      if (h >= H) break;
      const int kvo = (h % Hkv) * d;
      const float* qh = qs + static_cast<size_t>(h) * d;
      // scores: lane r owns row r
      float s = -INFINITY;
      if (lane < nr) {
        const uint16_t* kr = kbuf + static_cast<size_t>(lane) * rstride + kvo;
        float2 acc = make_float2(0.f, 0.f);
        if (vec) {
          for (int t = 0; t < d; t += 8) {
            const uint4 kx = *reinterpret_cast<const uint4*>(kr + t);
            const float4 qa = *reinterpret_cast<const float4*>(qh + t);
            const float4 qb = *reinterpret_cast<const float4*>(qh + t + 4);
            ffma2(acc, bf16x2_to_f2(kx.x), make_float2(qa.x, qa.y));
            ffma2(acc, bf16x2_to_f2(kx.y), make_float2(qa.z, qa.w));
            ffma2(acc, bf16x2_to_f2(kx.z), make_float2(qb.x, qb.y));
            ffma2(acc, bf16x2_to_f2(kx.w), make_float2(qb.z, qb.w));
          }
        } else {
          for (int t = 0; t < d; ++t) acc.x = fmaf(qh[t], bf16_bits_to_f(kr[t]), acc.x);
        }
        s = (acc.x + acc.y) * p.attn_scale;
      }
      const float mt = warp_max(s);
      const float m_new = fmaxf(m_run[hs], mt);
      const float corr = expf(m_run[hs] - m_new);
      const float w = lane < nr ? expf(s - m_new) : 0.f;
      l_run[hs] = l_run[hs] * corr + warp_sum(w);
#pragma unroll
      for (int i = 0; i < kMaxDL; ++i) o_run[hs][i] *= corr;
      if (d == 128 && vec) {
        // lane owns d-elements [4*lane, 4*lane+4): one 8-byte smem load per row
        for (int r = 0; r < nr; ++r) {
          const float wr = __shfl_sync(0xffffffffu, w, r);
          const uint2 vv = *reinterpret_cast<const uint2*>(vbuf + static_cast<size_t>(r) * rstride + kvo + 4 * lane);
          const float2 v01 = bf16x2_to_f2(vv.x), v23 = bf16x2_to_f2(vv.y);
          o_run[hs][0] = fmaf(wr, v01.x, o_run[hs][0]);
          o_run[hs][1] = fmaf(wr, v01.y, o_run[hs][1]);
          o_run[hs][2] = fmaf(wr, v23.x, o_run[hs][2]);
          o_run[hs][3] = fmaf(wr, v23.y, o_run[hs][3]);
        }
      } else {
        for (int r = 0; r < nr; ++r) {
          const float wr = __shfl_sync(0xffffffffu, w, r);
          const uint16_t* vr = vbuf + static_cast<size_t>(r) * rstride + kvo;
#pragma unroll
          for (int i = 0; i < kMaxDL; ++i) {
            const int t = lane + 32 * i;
            if (t < d) o_run[hs][i] = fmaf(wr, bf16_bits_to_f(vr[t]), o_run[hs][i]);
          }
        }
      }
      m_run[hs] = m_new;
    }
  }
  if (with_cur) {
#pragma unroll
    for (int hs = 0; hs < kMaxHeadsPerWarp; ++hs) {
      const int h = warp + hs * kDecodeWarps;
      if (h >= H) break;
      const int kvo = (h % Hkv) * d;
      float part_dot = 0.f;
#pragma unroll
      for (int i = 0; i < kMaxDL; ++i) {
        const int t = lane + 32 * i;
        if (t < d) part_dot = fmaf(sd.q[static_cast<size_t>(h) * d + t], sd.k_new[kvo + t], part_dot);
      }
      const float s = warp_sum(part_dot) * p.attn_scale;
      const float m_new = fmaxf(m_run[hs], s);
      const float corr = expf(m_run[hs] - m_new);
      const float w = expf(s - m_new);
      l_run[hs] = l_run[hs] * corr + w;
#pragma unroll
      for (int i = 0; i < kMaxDL; ++i) {
        const int t = d128 ? 4 * lane + i : lane + 32 * i;
        if ((d128 ? i < 4 : t < d)) o_run[hs][i] = fmaf(w, sd.v_new[kvo + t], o_run[hs][i] * corr);
      }
      m_run[hs] = m_new;
    }
  }
  const int stride = att_stride(d);
#pragma unroll
  for (int hs = 0; hs < kMaxHeadsPerWarp; ++hs) {
    const int h = warp + hs * kDecodeWarps;
    if (h >= H) break;
    float* ph = part + static_cast<size_t>(h) * stride;
#pragma unroll
    for (int i = 0; i < kMaxDL; ++i) {
      const int t = d128 ? 4 * lane + i : lane + 32 * i;
      if ((d128 ? i < 4 : t < d)) ph[t] = o_run[hs][i];
    }
    if (lane == 0) {
      ph[d] = m_run[hs];
      ph[d + 1] = l_run[hs];
    }
  }
}

template <int D, int G, bool FAST>
__global__ void __launch_bounds__(kDecodeThreads, 1) decode_kernel(const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem sm = carve(smem_raw, p);
  const int cta = blockIdx.x;
  const int nblocks = gridDim.x;
  const int seq_id = cta / p.ctas_per_seq;
  const int cs = cta - seq_id * p.ctas_per_seq;
  const SeqDesc sd = p.seqs[seq_id];
  const int H = p.H;
  const int width = H * p.d;
  const int tid = threadIdx.x;
  const bool do_select = (p.mode & kModeSelect) != 0;

  if (FAST && tid < kMaxStages) {
    mbar_init(&sm.full[tid], 1);
    mbar_init(&sm.empty[tid], p.H_kv);  // the H_kv consumer warps of a stage
  }
  if (tid == 0) {
    mbar_init(sm.att, 1);
    mbar_init(sm.aux, 1);
  }
  uint32_t aux_phase = 0;
  for (int h = tid; h < H; h += blockDim.x) sm.headmax[h] = float_ord(-INFINITY);
  fence_mbar_init();
  GridBarrier* gbar = reinterpret_cast<GridBarrier*>(p.bar);
  unsigned int bar_gen = 0;
  if (tid == 0) bar_gen = grid_sync_begin(gbar);  // only thread 0 uses it
  __syncthreads();

  trace_pt(p, 0);
  // ---- phase 0: append + cache decision + histogram reset
  if ((p.mode & kModeAppend) && cs == 0 && sd.append_frame >= 0) {
    const int row = p.H_kv * p.d;
    const size_t off = (static_cast<size_t>(sd.append_frame) * p.page_size + sd.append_slot) * row;
    for (int i = tid; i < row; i += blockDim.x) {
      p.k_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(sd.k_new[i]));
      p.v_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(sd.v_new[i]));
    }
    if (tid == 0 && sd.append_page >= 0) sd.page_table[sd.append_page] = sd.append_frame;
  }
  // every CTA evaluates every sequence's decision so that the grid agrees on
  // whether any selection (and its barriers) runs this step
  double* scratch_d = reinterpret_cast<double*>(sm.hist);  // hist is free until phase 2
  int own = 0;        // 0 none, 1 miss (select), 2 hit
  int any_select = 0, any_radix = 0;
  double own_cos = NAN;
  for (int b = 0; b < p.n_seq; ++b) {
    const SeqDesc& s2 = (b == seq_id) ? sd : p.seqs[b];
    int st = 0;
    double c = NAN;
    if (s2.select) {
      if (p.mode & kModeCache) {
        const int dec = cache_decision(s2, width, scratch_d, &c);
        st = dec == 1 ? 1 : dec == 0 ? 2 : 3;
      } else {
        st = 1;
      }
    }
    if (st == 1) {
      any_select = 1;
      if (do_select && s2.n_cand > p.k) any_radix = 1;
    }
    if (b == seq_id) {
      own = st;
      own_cos = c;
    }
  }
  if (do_select && own == 1) {
    uint32_t* gh = p.ws_hist + static_cast<size_t>(seq_id) * 3 * kBins;
    for (int i = cs * blockDim.x + tid; i < 3 * kBins; i += p.ctas_per_seq * blockDim.x) gh[i] = 0u;
  }
  if (cs == 0 && tid == 0 && own == 3) sd.cache->error = 1;

  trace_pt(p, 1);
  // ---- phase 1: scan
  const int T = sd.n_cand;
  const int j0 = min(T, cs * p.tpc);
  const int nloc = max(0, min(T, j0 + p.tpc) - j0);
  float* Sbuf = p.s_in_smem ? sm.S : p.ws_s + static_cast<size_t>(cta) * H * p.tpc;
  uint32_t* keys = p.s_in_smem ? sm.keys : p.ws_keys + static_cast<size_t>(cta) * p.tpc;
  const int sstride = p.tpc;
  const bool scanning = (own == 1) && ((p.mode & (kModeScore | kModeSIn)) != 0);
  if (scanning) {
    if (p.mode & kModeSIn) {
      for (int idx = tid; idx < H * nloc; idx += blockDim.x) {
        const int h = idx / nloc, jl = idx - (idx / nloc) * nloc;
        const float s = sd.s_in[static_cast<size_t>(h) * T + j0 + jl];
        Sbuf[static_cast<size_t>(h) * sstride + jl] = s;
        atomicMax(&sm.headmax[h], float_ord(s));
      }
    } else {
      float* so = (p.mode & kModeSOut) ? sd.s_out + j0 : nullptr;
      for (int base = tid; base < nloc; base += 4 * blockDim.x) {
        int32_t fr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jl = base + u * blockDim.x;
          fr[u] = jl < nloc ? static_cast<int32_t>(row_index(sd, cand_at(sd, j0 + jl), p.page_size)) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (base + u * static_cast<int>(blockDim.x) < nloc) sm.frames[base + u * blockDim.x] = fr[u];
      }
      __syncthreads();
      if constexpr (FAST) scan_fast<D, G>(p, sd, sm, j0, nloc, Sbuf, sstride, so);
      else scan_generic(p, sd, sm, j0, nloc, Sbuf, sstride, so);
    }
  }
  __syncthreads();
  trace_pt(p, 2);

  if (do_select && own == 1 && p.method == 2) {
    // per-CTA softmax partials: m = max_j S, z = sum_j exp(S - m); S <- exp(S - m)
    const int warp = tid >> 5, lane = tid & 31;
    for (int h = warp; h < H; h += kDecodeWarps) {
      const float m = ord_float(sm.headmax[h]);
      float z = 0.f;
      float* sr = Sbuf + static_cast<size_t>(h) * sstride;
      if (m > -INFINITY) {
        float z1 = 0.f, z2 = 0.f, z3 = 0.f;
        int jl = lane;
        for (; jl + 96 < nloc; jl += 128) {
          const float e0 = expf(sr[jl] - m), e1 = expf(sr[jl + 32] - m);
          const float e2 = expf(sr[jl + 64] - m), e3 = expf(sr[jl + 96] - m);
          sr[jl] = e0;
          sr[jl + 32] = e1;
          sr[jl + 64] = e2;
          sr[jl + 96] = e3;
          z += e0;
          z1 += e1;
          z2 += e2;
          z3 += e3;
        }
        for (; jl < nloc; jl += 32) {
          const float e = expf(sr[jl] - m);
          sr[jl] = e;
          z += e;
        }
        z = (z + z1) + (z2 + z3);
      }
      z = warp_sum(z);
      if (lane == 0) {
        const size_t o = (static_cast<size_t>(seq_id) * H + h) * stats_stride(p.ctas_per_seq) + cs;
        p.ws_m[o] = m;
        p.ws_z[o] = z;
      }
    }
  }
  trace_pt(p, 3);
  if (any_select) grid_sync(gbar, nblocks, bar_gen);  // #1
  trace_pt(p, 4);

  // ---- phase 2: crit + cache bookkeeping
  if (own == 1 && cs == 0 && tid == 0 && (p.mode & kModeCache)) {
    CacheState* c = sd.cache;
    c->lookups += 1;
    c->first_flag = 0;
    c->last_hit = 0;
    c->last_cos = own_cos;
  }
  if (own == 2 && cs == 0 && tid == 0) {
    CacheState* c = sd.cache;
    c->lookups += 1;
    c->hits += 1;
    c->last_hit = 1;
    c->last_cos = own_cos;
  }
  if (own == 1 && (p.mode & kModeCache)) {
    // the new cached query (every CTA finished reading the old one before #1)
    for (int i = cs * blockDim.x + tid; i < width; i += p.ctas_per_seq * blockDim.x) sd.cached_q[i] = sd.q[i];
  }
  const int kk_total = p.k;
  uint32_t tau = 0, kk = 0;
  const bool radix_own = do_select && own == 1 && T > kk_total;
  if (do_select && own == 1) {
    if (p.method == 2) {
      const int warp = tid >> 5, lane = tid & 31;
      const int c0 = seq_id * p.ctas_per_seq;
      // stage every CTA's (m, z) of this sequence in smem with one coalesced pass
      float* pm = reinterpret_cast<float*>(sm.ring);
      float* pz = pm;
      const int nc = p.ctas_per_seq;
      const int ncp = stats_stride(nc);
      // the sequence's [h][cta] stats are two contiguous rows blocks: 2 bulk copies
      const size_t sbytes = static_cast<size_t>(H) * ncp * 4;
      if (tid == 0) {
        mbar_arrive_expect_tx(sm.aux, static_cast<uint32_t>(2 * sbytes));
        bulk_g2s_nohint(pm, p.ws_m + static_cast<size_t>(seq_id) * H * ncp, static_cast<uint32_t>(sbytes), sm.aux);
        bulk_g2s_nohint(pm + H * ncp, p.ws_z + static_cast<size_t>(seq_id) * H * ncp, static_cast<uint32_t>(sbytes), sm.aux);
      }
      pz = pm + H * ncp;
      mbar_wait(sm.aux, aux_phase);
      aux_phase ^= 1u;
      trace_pt(p, 15);
      for (int h = warp; h < H; h += kDecodeWarps) {
        float M = -INFINITY;
        for (int c = lane; c < nc; c += 32) M = fmaxf(M, pm[h * ncp + c]);
        M = warp_max(M);
        float Z = 0.f;
        for (int c = lane; c < nc; c += 32) {
          const float mc = pm[h * ncp + c];
          if (mc > -INFINITY) Z += pz[h * ncp + c] * expf(mc - M);
        }
        Z = warp_sum(Z);
        if (lane == 0) {
          const float ms = ord_float(sm.headmax[h]);
          sm.f[h] = (ms > -INFINITY) ? expf(ms - M) / Z : 0.f;
        }
      }
      trace_pt(p, 16);
      __syncthreads();
      for (int jl = tid; jl < nloc; jl += blockDim.x) {
        float c = 0.f;
        for (int h = 0; h < H; ++h) c = fmaf(Sbuf[static_cast<size_t>(h) * sstride + jl], sm.f[h], c);
        keys[jl] = float_key(c);
      }
    } else {
      for (int jl = tid; jl < nloc; jl += blockDim.x) {
        float c = 0.f;
        for (int h = 0; h < H; ++h) c += Sbuf[static_cast<size_t>(h) * sstride + jl];
        keys[jl] = float_key(c);
      }
    }
    __syncthreads();
  }

  trace_pt(p, 5);
  // ---- phase 3: radix select (3 passes, 11/11/10 bits)
  if (any_radix) {
    uint32_t prefix = 0;
    uint32_t* gh = p.ws_hist + static_cast<size_t>(seq_id) * 3 * kBins;
    kk = static_cast<uint32_t>(kk_total);
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
      const int sh = shifts[pass], wd = widths[pass];
      const int nb = 1 << wd;
      if (radix_own) {
        for (int i = tid; i < nb; i += blockDim.x) sm.hist[i] = 0u;
        __syncthreads();
        const int hs = sh + wd;  // bits above this digit must match the prefix
        for (int jl = tid; jl < nloc; jl += blockDim.x) {
          const uint32_t key = keys[jl];
          if (hs >= 32 || (key >> hs) == prefix) atomicAdd(&sm.hist[(key >> sh) & (nb - 1)], 1u);
        }
        __syncthreads();
        for (int i = tid; i < nb; i += blockDim.x) {
          const uint32_t c = sm.hist[i];
          if (c) atomicAdd(gh + pass * kBins + i, c);
        }
      }
      grid_sync(gbar, nblocks, bar_gen);  // #2..#4
      trace_pt(p, 6 + pass);
      if (radix_own) {
        int b;
        uint32_t above;
        find_bin(gh + pass * kBins, nb, kk, sm.scratch, &b, &above);
        kk -= above;
        prefix = (prefix << wd) | static_cast<uint32_t>(b);
      }
    }
    tau = prefix;
    // per-CTA (n_gt, n_eq)
    if (radix_own) {
      uint32_t ngt = 0, neq = 0;
      for (int jl = tid; jl < nloc; jl += blockDim.x) {
        const uint32_t key = keys[jl];
        ngt += key > tau;
        neq += key == tau;
      }
      uint32_t tg, te;
      block_excl_scan(ngt, sm.scratch, &tg);
      block_excl_scan(neq, sm.scratch, &te);
      if (tid == 0) {
        p.ws_cnt[static_cast<size_t>(cta) * 2 + 0] = tg;
        p.ws_cnt[static_cast<size_t>(cta) * 2 + 1] = te;
      }
    }
    grid_sync(gbar, nblocks, bar_gen);  // #5
    trace_pt(p, 9);
  }

  // ---- phase 3b: ascending compaction of the selection
  if (do_select && own == 1) {
    if (!radix_own) {
      // T <= k: every candidate is selected (pick() with take = T)
      for (int jl = tid; jl < nloc; jl += blockDim.x) {
        sd.sel[j0 + jl] = cand_at(sd, j0 + jl);
        sd.sel_crit[j0 + jl] = key_float(keys[jl]);
      }
      if (cs == 0 && tid == 0) sd.cache->n_sel = T;
    } else {
      uint32_t pgt = 0, peq = 0;
      const int c0 = seq_id * p.ctas_per_seq;
      if (tid < 32) {
        for (int c = tid; c < cs; c += 32) {
          pgt += __ldcg(p.ws_cnt + static_cast<size_t>(c0 + c) * 2 + 0);
          peq += __ldcg(p.ws_cnt + static_cast<size_t>(c0 + c) * 2 + 1);
        }
        pgt = __reduce_add_sync(0xffffffffu, pgt);
        peq = __reduce_add_sync(0xffffffffu, peq);
        if (tid == 0) {
          sm.scratch[66] = pgt;
          sm.scratch[67] = peq;
        }
      }
      __syncthreads();
      pgt = sm.scratch[66];
      peq = sm.scratch[67];
      __syncthreads();
      const uint32_t take_eq = kk > peq ? kk - peq : 0u;  // ties still available to this CTA
      uint32_t out_base = pgt + min(peq, kk);
      uint32_t eq_seen = 0;
      for (int t0 = 0; t0 < nloc; t0 += blockDim.x) {
        const int jl = t0 + tid;
        const uint32_t key = jl < nloc ? keys[jl] : 0u;
        const uint32_t is_eq = (jl < nloc && key == tau) ? 1u : 0u;
        uint32_t eq_tot;
        const uint32_t eq_rank = eq_seen + block_excl_scan(is_eq, sm.scratch, &eq_tot);
        const uint32_t take = (jl < nloc) && (key > tau || (is_eq && eq_rank < take_eq)) ? 1u : 0u;
        uint32_t take_tot;
        const uint32_t pos = block_excl_scan(take, sm.scratch, &take_tot);
        if (take) {
          sd.sel[out_base + pos] = cand_at(sd, j0 + jl);
          sd.sel_crit[out_base + pos] = key_float(key);
        }
        out_base += take_tot;
        eq_seen += eq_tot;
      }
      if (cs == 0 && tid == 0) sd.cache->n_sel = kk_total;
    }
  }
  trace_pt(p, 10);
  if (!(p.mode & kModeAttend)) return;
  if (any_select) grid_sync(gbar, nblocks, bar_gen);  // #6 selection visible
  trace_pt(p, 11);

  // ---- phase 4: split-K sparse flash-decoding partials
  AttView av{};
  if (!sd.att_list) {
    const int n_sel = (sd.select && own != 3) ? __ldcg(&sd.cache->n_sel) : 0;
    av.init_end = sd.init_end;
    const uint32_t ie = static_cast<uint32_t>(sd.init_end);
    const uint32_t lb = static_cast<uint32_t>(max(sd.local_begin, sd.init_end));
    // sorted selection: lower_bound(x) == count(sel < x), counted in parallel
    const uint32_t lbs = lb < ie ? ie : static_cast<uint32_t>(sd.local_begin);
    uint32_t cie = 0, clb = 0;
    for (int base = tid; base < n_sel; base += 4 * blockDim.x) {
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        v[u] = i < n_sel ? __ldcg(sd.sel + i) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cie += v[u] < ie;
        clb += v[u] < lbs;
      }
    }
    uint32_t tot_ie, tot_lb;
    block_excl_scan(cie, sm.scratch, &tot_ie);
    block_excl_scan(clb, sm.scratch, &tot_lb);
    const int lo1 = static_cast<int>(tot_ie), hi1 = static_cast<int>(tot_lb);
    trace_pt(p, 17);
    av.lo1 = lo1;
    av.n1 = max(0, hi1 - lo1);
    av.lb2 = static_cast<int>(lb);
    av.n_rows = sd.init_end + av.n1 + (sd.n_cached - av.lb2);
  } else {
    av.n_rows = sd.n_att;
  }
  const int total_rows = av.n_rows + 1;  // + current token
  const int per = (total_rows + p.ctas_per_seq - 1) / p.ctas_per_seq;
  const int r0 = min(total_rows, cs * per);
  const int r1 = min(total_rows, r0 + per);
  const bool with_cur = (r0 < r1) && (r1 == total_rows);
  float* part = p.ws_att + static_cast<size_t>(cta) * H * att_stride(p.d);
  attend_partial(p, sd, av, sm, r0, min(r1, av.n_rows), with_cur, part);
  trace_pt(p, 12);
  grid_sync(gbar, nblocks, bar_gen);  // #7
  trace_pt(p, 13);

  // ---- phase 5: LSE merge (attention.cpp:88-110 semantics)
  // Per head: weights w_c = exp(m_c - M) for all partials in parallel, then
  // the d output columns are summed by blockDim/d thread groups over
  // interleaved partials (independent loads, no serial L2 chain).
  {
    const int d = p.d, stride = att_stride(d);
    const int c0 = seq_id * p.ctas_per_seq;
    const int nparts = min(p.ctas_per_seq, (total_rows + per - 1) / per);
    float* wsm = reinterpret_cast<float*>(sm.hist);        // [nparts] weights (<= 2048)
    float* red = reinterpret_cast<float*>(sm.ring);        // [groups][d] partial sums
    float* bred = reinterpret_cast<float*>(sm.scratch);    // block reduction slots
    const int warp = tid >> 5, lane = tid & 31;
    const int groups = max(1, static_cast<int>(blockDim.x) / d);
    // partials are staged in smem chunk by chunk (one parallel load each) and
    // merged online, so every global read is independent
    float* stg = reinterpret_cast<float*>(sm.ring + 4096);
    const int pc = max(1, min(nparts, static_cast<int>((kRingBudget - 4096) / 4) / stride));
    for (int h = cs; h < H; h += p.ctas_per_seq) {
      const float* base = p.ws_att + (static_cast<size_t>(c0) * H + h) * stride;
      const size_t cstride = static_cast<size_t>(H) * stride;
      const int g = tid / d, t = tid - (tid / d) * d;
      float acc = 0.f, Mrun = -INFINITY, Lrun = 0.f;
      for (int cb = 0; cb < nparts; cb += pc) {
        const int n = min(pc, nparts - cb);
        // one bulk copy per partial record (16-byte padded), one barrier wait
        if (tid == 0) mbar_arrive_expect_tx(sm.aux, static_cast<uint32_t>(n * stride * 4));
        __syncthreads();
        for (int c = tid; c < n; c += blockDim.x)
          bulk_g2s_nohint(stg + c * stride, base + (cb + c) * cstride, static_cast<uint32_t>(stride * 4), sm.aux);
        mbar_wait(sm.aux, aux_phase);
        aux_phase ^= 1u;
        __syncthreads();
        float mloc = -INFINITY;
        for (int c = tid; c < n; c += blockDim.x) mloc = fmaxf(mloc, stg[c * stride + d]);
        mloc = warp_max(mloc);
        if (lane == 0) bred[warp] = mloc;
        __syncthreads();
        float Mc = lane < kDecodeWarps ? bred[lane] : -INFINITY;
        Mc = warp_max(Mc);
        const float Mnew = fmaxf(Mrun, Mc);
        const float scale = (Mrun == -INFINITY) ? 0.f : expf(Mrun - Mnew);
        __syncthreads();
        float lsum = 0.f;
        for (int c = tid; c < n; c += blockDim.x) {
          const float mc = stg[c * stride + d];
          const float w = (mc == -INFINITY) ? 0.f : expf(mc - Mnew);
          wsm[c] = w;
          lsum += w * stg[c * stride + d + 1];
        }
        lsum = warp_sum(lsum);
        if (lane == 0) bred[warp] = lsum;
        __syncthreads();
        float Lc = lane < kDecodeWarps ? bred[lane] : 0.f;
        Lc = warp_sum(Lc);
        Lrun = Lrun * scale + Lc;
        if (g < groups) {
          float a = 0.f;
          for (int c = g; c < n; c += groups) a = fmaf(wsm[c], stg[c * stride + t], a);
          acc = acc * scale + a;
        }
        Mrun = Mnew;
        __syncthreads();
      }
      if (g < groups) red[g * d + t] = acc;
      __syncthreads();
      for (int tt = tid; tt < d; tt += blockDim.x) {
        float O = 0.f;
        for (int gg = 0; gg < groups; ++gg) O += red[gg * d + tt];
        sd.out[static_cast<size_t>(h) * d + tt] = O / Lrun;
      }
      __syncthreads();
    }
  }
  trace_pt(p, 14);
}

}  // namespace

const void* decode_kernel_ptr(int D, int G, bool fast) {
  if (fast) {
    if (D == 128) {
      switch (G) {
        case 1: return reinterpret_cast<const void*>(&decode_kernel<128, 1, true>);
        case 2: return reinterpret_cast<const void*>(&decode_kernel<128, 2, true>);
        case 4: return reinterpret_cast<const void*>(&decode_kernel<128, 4, true>);
        case 7: return reinterpret_cast<const void*>(&decode_kernel<128, 7, true>);
        case 8: return reinterpret_cast<const void*>(&decode_kernel<128, 8, true>);
      }
    }
    if (D == 64) {
      switch (G) {
        case 1: return reinterpret_cast<const void*>(&decode_kernel<64, 1, true>);
        case 2: return reinterpret_cast<const void*>(&decode_kernel<64, 2, true>);
        case 4: return reinterpret_cast<const void*>(&decode_kernel<64, 4, true>);
        case 8: return reinterpret_cast<const void*>(&decode_kernel<64, 8, true>);
      }
    }
    return nullptr;
  }
  return reinterpret_cast<const void*>(&decode_kernel<0, 0, false>);
}

}  // namespace tsb

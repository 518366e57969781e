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


struct Smem {
  uint8_t* ring;
  float* S;        // [H][tpc] (when on chip)
  uint32_t* keys;  // [tpc]
  uint32_t* hist;  // [kRadixBins]
  int* prefix;     // [kMaxPrefix] per-CTA selection offsets of this sequence
  int* headmax;    // [H] ordered-int max
  float* f;        // [H]
  uint32_t* scratch;  // [256]
  int32_t* frames; // [tpc] slab row of each local candidate
  uint64_t* full;  // [nphase][kStages] (kMaxBarPairs)
  uint64_t* empty; // [nphase][kStages]
  uint64_t* att;   // [2] attention staging barriers (double buffer)
  uint64_t* aux;   // bulk staging barrier (stats)
};

__device__ __forceinline__ Smem carve(uint8_t* base, const DecodeParams& p) {
  SmemLayout L = smem_layout(p.H, p.H_kv * p.d * 2, p.tpc, p.s_in_smem, p.ring_bytes);
  Smem s;
  s.ring = base + L.ring;
  s.S = reinterpret_cast<float*>(base + L.s);
  s.keys = reinterpret_cast<uint32_t*>(base + L.keys);
  s.hist = reinterpret_cast<uint32_t*>(base + L.hist);
  s.prefix = reinterpret_cast<int*>(base + L.prefix);
  s.headmax = reinterpret_cast<int*>(base + L.headmax);
  s.f = reinterpret_cast<float*>(base + L.f);
  s.scratch = reinterpret_cast<uint32_t*>(base + L.scratch);
  s.full = reinterpret_cast<uint64_t*>(base + L.bars);
  s.empty = s.full + kMaxBarPairs;
  s.att = s.full + 2 * kMaxBarPairs;
  s.aux = s.att + 2;
  s.frames = reinterpret_cast<int32_t*>(base + L.frames);
  return s;
}

// LEAN launches have implicit candidates and power-of-two pages (abi.cpp).
template <bool LEAN = false>
__device__ __forceinline__ uint32_t cand_at(const SeqDesc& sd, int j) {
  if (LEAN) return static_cast<uint32_t>(sd.cand_begin + j);
  return sd.cand ? sd.cand[j] : static_cast<uint32_t>(sd.cand_begin + j);
}

// Slab row of token `tok` through the page table. Power-of-two pages take
// the shift path inline; any other page size goes through one out-of-line
// copy (integer division is long code, and the post-scan phases run from a
// cold instruction cache).
__device__ __noinline__ size_t row_index_div(const int32_t* page_table, uint32_t tok, int page_size) {
  return static_cast<size_t>(page_table[tok / page_size]) * page_size + tok % page_size;
}
template <bool LEAN = false>
__device__ __forceinline__ size_t row_index(const SeqDesc& sd, uint32_t tok, int page_size) {
  if (LEAN || (page_size & (page_size - 1)) == 0) {
    const int sh = __ffs(page_size) - 1;
    return (static_cast<size_t>(sd.page_table[tok >> sh]) << sh) | (tok & (page_size - 1));
  }
  return row_index_div(sd.page_table, tok, page_size);
}

// Phase trace (thread 0 of every CTA, trace[cta][kTraceStride] when enabled):
// SM clock64 stamps at the phase boundaries. The start (slot 0) and the end
// (slot 12) also record %globaltimer (slots 0 / 30, ns; the start clock goes
// to slot 29) so the host aligns the CTAs and converts cycles to ns.
__device__ __forceinline__ void trace_pt(const DecodeParams& p, int i) {
#ifdef TSB_NO_TRACE
  return;
#endif
  if (p.trace && threadIdx.x == 0) {
    unsigned long long* t = p.trace + blockIdx.x * kTraceStride;
    const unsigned long long c = clock64();
    if (i == 0 || i == 12) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      t[i == 0 ? 0 : 30] = g;
      t[i == 0 ? 29 : 12] = c;
    } else {
      t[i] = c;
    }
  }
}

// Sub-phase stamp into a CTA's trace row (nullptr: off); thread 0 only.
__device__ __forceinline__ void stamp(unsigned long long* tr, int i) {
#ifdef TSB_NO_TRACE
  return;
#endif
  if (tr && threadIdx.x == 0) tr[i] = clock64();
}

// Dev timing: TS_DEBUG_FLAGS = n << 8 ends the launch at stop point n
// (uniform over the grid, so no barrier is left waiting).
#ifndef TSB_LEAN_DEV
#define TSB_LEAN_DEV 1
#endif
#define TSB_STOP_AT(n) \
  if ((!LEAN || TSB_LEAN_DEV) && (p.debug_flags >> 8) == (n)) return

// Block-wide exclusive scan of one value per thread (all threads call).
// Out of line (like find_bin / radix_hist): the fused kernel's one-shot phases
// are instruction-fetch bound, so shared helpers are kept as single copies.
__device__ __noinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
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

// Finds, in a global histogram whose bins are ordered by key, the bin b such that
// count(bins > b) < kk <= count(bins >= b). Returns b and count(bins > b).
// All threads call; every CTA computes the same answer from the same data.
// Finds, in a pass histogram, the bin holding the kk-th largest key: 512
// threads load 8 bins each (one parallel pass over the 16 KB) into shared
// memory with 64-bin coarse sums, then warp 0 searches coarse then fine bins
// with shuffles. Returns the bin, the count in higher bins and the bin's own
// count. All threads call; `work` is >= 4096 + 64 words of shared memory.
__device__ __noinline__ void find_bin(const uint32_t* gh, uint32_t kk, uint32_t* scratch, uint32_t* work,
                                      int* bin_out, uint32_t* above_out, uint32_t* count_out,
                                      unsigned long long* tr, int ts) {
  const int t = threadIdx.x, lane = t & 31;
  uint32_t* coarse = work + kRadixBins;
  if (t < 512) {
    uint4 a = __ldcg(reinterpret_cast<const uint4*>(gh) + 2 * t);
    uint4 b = __ldcg(reinterpret_cast<const uint4*>(gh) + 2 * t + 1);
    reinterpret_cast<uint4*>(work)[2 * t] = a;
    reinterpret_cast<uint4*>(work)[2 * t + 1] = b;
    uint32_t sum = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    if ((t & 7) == 0) coarse[t >> 3] = sum;
  }
  __syncthreads();
  stamp(tr, ts);
  if (t < 32) {
    uint32_t base = 0, bin = 0, cnt = 0;
#pragma unroll
    for (int level = 0; level < 2; ++level) {
      // lane l covers bins (63 - 2l, 62 - 2l) of this level, descending
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
  *bin_out = static_cast<int>(scratch[64]);
  *above_out = scratch[65];
  *count_out = scratch[66];
  __syncthreads();
}

// fp64 cosine Selection Cache decision (tensor.cpp:92-113,
// selection_cache.cpp:29-35). The first kDecU * blockDim elements of q and
// the cached query arrive preloaded in registers (issued together with the
// other phase-0 loads); any rest is loaded here. Deterministic block
// reduction: every CTA that evaluates it for the same sequence gets a
// bit-identical result. Returns 1 = miss, 0 = hit, 2 = zero query (error).
constexpr int kDecU = 8;

struct DecisionLoads {
  float qa[kDecU], qb[kDecU];
  int first_flag;
  double theta;
};

__device__ __forceinline__ void decision_issue(const SeqDesc& sd, int width, DecisionLoads& L) {
#pragma unroll
  for (int u = 0; u < kDecU; ++u) {
    const int i = threadIdx.x + u * blockDim.x;
    L.qa[u] = i < width ? __ldg(sd.q + i) : 0.f;
    L.qb[u] = i < width ? __ldcg(sd.cached_q + i) : 0.f;
  }
  L.first_flag = __ldcg(&sd.cache->first_flag);
  L.theta = __ldcg(&sd.cache->theta);
}

__device__ int cache_decision(const SeqDesc& sd, int width, const DecisionLoads& L, double* scratch_d,
                              double* cos_out) {
  double dot = 0.0, nu = 0.0, nv = 0.0;
  int nonzero = 0;
#pragma unroll
  for (int u = 0; u < kDecU; ++u) {
    const double a = static_cast<double>(L.qa[u]);
    const double b = static_cast<double>(L.qb[u]);
    nonzero |= (L.qa[u] != 0.0f);
    dot = fma(a, b, dot);
    nu = fma(a, a, nu);
    nv = fma(b, b, nv);
  }
  for (int i = threadIdx.x + kDecU * blockDim.x; i < width; i += blockDim.x) {
    const float fa = __ldg(sd.q + i), fb = __ldcg(sd.cached_q + i);
    const double a = static_cast<double>(fa), b = static_cast<double>(fb);
    nonzero |= (fa != 0.0f);
    dot = fma(a, b, dot);
    nu = fma(a, a, nu);
    nv = fma(b, b, nv);
  }
  dot = warp_sum_d(dot);
  nu = warp_sum_d(nu);
  nv = warp_sum_d(nv);
  nonzero = __any_sync(0xffffffffu, nonzero);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    scratch_d[warp * 4 + 0] = dot;
    scratch_d[warp * 4 + 1] = nu;
    scratch_d[warp * 4 + 2] = nv;
    scratch_d[warp * 4 + 3] = nonzero ? 1.0 : 0.0;
  }
  __syncthreads();
  // every warp reduces the per-warp partials in the same fixed tree order
  const int nw = blockDim.x >> 5;
  double D = lane < nw ? scratch_d[lane * 4 + 0] : 0.0;
  double U = lane < nw ? scratch_d[lane * 4 + 1] : 0.0;
  double V = lane < nw ? scratch_d[lane * 4 + 2] : 0.0;
  const int nz = __any_sync(0xffffffffu, lane < nw && scratch_d[lane * 4 + 3] != 0.0);
  D = warp_sum_d(D);
  U = warp_sum_d(U);
  V = warp_sum_d(V);
  __syncthreads();
  if (!nz) return 2;
  *cos_out = NAN;
  if (L.first_flag) return 1;
  if (U == 0.0 || V == 0.0) return 1;  // unreachable: cached query is never zero
  double c;
  if (D * D >= U * V) c = D >= 0.0 ? 1.0 : -1.0;  // exact +-1 clamp
  else c = D / sqrt(U * V);
  *cos_out = c;
  return c < L.theta ? 1 : 0;  // strict <
}

// --------------------------------------------------------------- the scan
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kScratchTmem = 250;  // sm.scratch word holding the TMEM base address
constexpr int kScratchStageMode = 200;  // sm.scratch words [200, 216): the scan ring's per-slot layout
constexpr size_t kCritPartOffset = 64 * 1024;  // TMEM mode: per-kv-head criticality partials in the ring
constexpr int kLeanMode = kModeSelect | kModeScore | kModeCache | kModeAttend | kModeAppend;
constexpr int kLeanSelMode = kModeSelect | kModeScore;  // select_for_chunk's launch (prefill)
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

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
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


// TM: the S fragments stay in tensor memory (tbase: the CTA's allocation);
// consumer warp w keeps its r-th stage at columns r*4 .. r*4+3 of lane
// quarter w % 4, column block (w - 1) / 4 (decode.h, kTmemColsPerWarp).
__device__ __forceinline__ uint32_t tmem_warp_base(uint32_t tbase, int warp) {
  return tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(((warp - 1) >> 2) * kTmemColsPerWarp);
}

// zw (S spilled to global memory, soft vote): each consumer lane also keeps
// the softmax partial (m, z) of its two heads online -- log2-domain reference
// moved lazily (by > 8), z = sum 2^(S log2e - m) -- and the warps leave them
// in zw[phase][H] (the idle radix histogram), so phase 2 does not stream the
// spilled S through HBM twice (a read and an e^(S - m) write back).
template <int D, int G, bool TM>
__device__ void scan_fast(const DecodeParams& p, const SeqDesc& sd, const Smem& sm, int j0,
                          int nloc, float* Sbuf, int sstride, float* s_out_row0, int pre, uint32_t tbase,
                          float2* zw = nullptr) {
  constexpr int KC = D / 16;  // k-chunks of 16 along d
  const int Hkv = p.H_kv;
  const int row_bytes = Hkv * D * 2;
  const int rstride = row_bytes + 16;  // padded ring row (ldmatrix conflict-free)
  // whole stages through the tensor map where a stage's 16 rows are
  // consecutive slab rows, ascending or descending (page_size 1 pools hand
  // out frames downwards), else row copies; the general kernel only (TM /
  // LEAN keeps the row copies, whose code is smaller). Slots are 1024-B
  // aligned (swizzle atoms) and hold either layout; smode[slot] says which.
  const bool tma = !TM && p.scan_tma != 0 && (smem_u32(sm.ring) & 1023u) == 0;
  const ScanGeom geom = scan_geom(p.H, p.H_kv, D, p.ring_bytes, tma);
  const int sbytes = static_cast<int>(scan_stage_bytes(row_bytes, tma));
  volatile uint32_t* smode = sm.scratch + kScratchStageMode;  // [kMaxStages]: 0 rows, 1 ascending, 2 descending
  const int R = geom.rows;  // 16 tokens per stage
  const int kStages = geom.stages;
  const int nit = (nloc + R - 1) / R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    // slab rows of all local candidates were staged in smem (sm.frames), so
    // issuing a stage is latency-free; rows land at a padded stride.
    // Stage it: slot it % kStages, consumed by phase it % nphase; its
    // barrier pair is used every lcm(nphase, kStages) stages, so the use
    // index it / lcm gives the parity.
    // (running slot / phase counters and per-pair parity bits: no divisions
    // in the issue loop)
    const uint64_t pol = policy_evict_first();
    const char* kbase = reinterpret_cast<const char*>(p.k_slab);
    const int nph = kDecodeConsumers / Hkv;
    uint64_t eparity = 0;  // bit k: parity of the next completion of empty[k] to wait for
    int s = 0, ph = 0, ph_prev = 0;
    for (int it = 0; it < nit; ++it) {
      const int rbase = it * R;
      const int nrows = min(R, nloc - rbase);
      if (it >= kStages) {  // the slot's previous stage (consumed by phase ph_prev) is free
        const int k = ph_prev * kStages + s;
        mbar_wait(&sm.empty[k], static_cast<uint32_t>(eparity >> k) & 1u);
        eparity ^= 1ull << k;
        ph_prev = ph_prev + 1 == nph ? 0 : ph_prev + 1;
      }
      uint64_t* fb = &sm.full[ph * kStages + s];
      int mode = 0;
      if (tma) {
        const int32_t f0 = sm.frames[rbase];
        const int32_t fl = lane < nrows ? sm.frames[rbase + lane] : f0;
        mode = __all_sync(0xffffffffu, lane >= nrows || fl == f0 + lane) ? 1
               : __all_sync(0xffffffffu, lane >= nrows || fl == f0 - lane) ? 2 : 0;
      }
      if (mode) {
        // one op for the 16 rows (a partial stage loads its neighbours, or
        // zero fill outside the slab, unused)
        if (lane == 0) {
          smode[s] = static_cast<uint32_t>(mode);
          mbar_arrive_expect_tx(fb, static_cast<uint32_t>(R * row_bytes));
          const int32_t f0 = sm.frames[rbase];
          tma_load_3d(sm.ring + static_cast<size_t>(s) * sbytes, p.k_tmap, 0, mode == 1 ? f0 : f0 - (R - 1), 0, fb, pol);
        }
      } else {
        if (lane == 0) {
          smode[s] = 0u;
          mbar_arrive_expect_tx(fb, static_cast<uint32_t>(nrows * row_bytes));
        }
        __syncwarp();
        if (lane < nrows)
          bulk_g2s(sm.ring + static_cast<size_t>(s) * sbytes + static_cast<size_t>(lane) * rstride,
                   kbase + static_cast<size_t>(sm.frames[rbase + lane]) * row_bytes, row_bytes, fb, pol);
      }
      s = s + 1 == kStages ? 0 : s + 1;
      ph = ph + 1 == nph ? 0 : ph + 1;
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int cw = warp - 1;
  const int nphase = kDecodeConsumers / Hkv;
  const int kvh = cw % Hkv, phase = cw / Hkv;
  uint32_t fparity = 0;  // bit s: parity of the next completion of full[phase][s]
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
  // running max of this lane's two heads (the consumers stay lean: they
  // gate the ring's refill, so the scan's speed is theirs)
  float runmax0 = -INFINITY, runmax1 = -INFINITY;
  float zm0 = -INFINITY, zm1 = -INFINITY, zz0 = 0.f, zz1 = 0.f;  // online (m, z), log2 domain (zw)
  auto zadd = [](float& zm, float& zz, float a, float b) {  // a, b: logits (-inf: none)
    const float x = a * kLog2e, y = b * kLog2e, mx = fmaxf(x, y);
    if (mx > -INFINITY) {
      if (mx > zm + 8.f) {
        zz = zm > -INFINITY ? zz * ex2_approx(zm - mx) : 0.f;
        zm = mx;
      }
      zz += ex2_approx(x - zm) + ex2_approx(y - zm);
    }
  };
  // ldmatrix row address: matrix lane/8 -> rows +8 for odd, cols +8 for >= 16
  const uint32_t lrow = static_cast<uint32_t>((lane & 7) + ((lane >> 3) & 1) * 8);
  const uint32_t lcol = static_cast<uint32_t>((lane >> 4) * 16 + kvh * D * 2);
  const uint32_t ring_base = smem_u32(sm.ring) + lrow * rstride + lcol;
  // tensor-map layout: line z*16 + box row holds 128-B chunk z of that
  // row, its 16-B units XOR-swizzled with (box row & 7); this lane's ldmatrix
  // row is token lrow (box row lrow, or 15 - lrow for a descending stage),
  // k half lane / 16 of each 16-wide k chunk
  const int e0 = kvh * D + (lane >> 4) * 8;  // element of the row at kc = 0
  int s = phase % kStages, r = 0;  // this warp's slot and stage count
  for (int it = phase; it < nit; it += nphase, ++r) {
    mbar_wait(&sm.full[phase * kStages + s], (fparity >> s) & 1u);
    fparity ^= 1u << s;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const uint32_t abase = ring_base + static_cast<uint32_t>(s * sbytes);
      const uint32_t tbase_s = smem_u32(sm.ring) + static_cast<uint32_t>(s * sbytes);
      const uint32_t mode = tma ? smode[s] : 0u;
      const int br = mode == 2 ? 15 - static_cast<int>(lrow) : static_cast<int>(lrow);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t a[4];
        const int e = e0 + kc * 16;
        ldmatrix_x4(a, mode ? tbase_s + static_cast<uint32_t>(((e >> 6) * 16 + br) * 128 + ((((e >> 3) & 7) ^ (br & 7)) << 4))
                            : abase + kc * 32);
        mma_bf16_16816(c, a, bq[kc][0][0], bq[kc][0][1]);
        mma_bf16_16816(c, a, bq[kc][1][0], bq[kc][1][1]);
        mma_bf16_16816(c, a, bq[kc][2][0], bq[kc][2][1]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[phase * kStages + s]);  // operands consumed
    s += nphase;
    while (s >= kStages) s -= kStages;
    const int rbase = it * R + (lane >> 2);
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int g = g0 + (e & 1);
      const int row = rbase + (e >> 1) * 8;
      v[e] = -INFINITY;
      if (g < G && row < nloc) {
        const int h = g * Hkv + kvh;
        if constexpr (!TM) Sbuf[static_cast<size_t>(h) * sstride + row] = c[e];
        if (s_out_row0) s_out_row0[static_cast<size_t>(h) * sd.n_cand + row] = c[e];
        v[e] = c[e];
      }
    }
    runmax0 = fmaxf(runmax0, fmaxf(v[0], v[2]));
    runmax1 = fmaxf(runmax1, fmaxf(v[1], v[3]));
    if constexpr (TM) tmem_st4(tmem_warp_base(tbase, warp) + static_cast<uint32_t>(r * 4), c[0], c[1], c[2], c[3]);
    else if (zw) {
      zadd(zm0, zz0, v[0], v[2]);
      zadd(zm1, zz1, v[1], v[3]);
    }
  }
  if (!TM && zw) {
    // this warp's (m, z) per head: the eight lanes of a head pair, merged
    auto zmerge = [](float& zm, float& zz, int o) {
      const float om = __shfl_xor_sync(0xffffffffu, zm, o), oz = __shfl_xor_sync(0xffffffffu, zz, o);
      const float mx = fmaxf(zm, om);
      if (mx > -INFINITY) {
        zz = (zm > -INFINITY ? zz * ex2_approx(zm - mx) : 0.f) + (om > -INFINITY ? oz * ex2_approx(om - mx) : 0.f);
        zm = mx;
      }
    };
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      zmerge(zm0, zz0, o);
      zmerge(zm1, zz1, o);
    }
    if (lane < 4) {
      if (g0 < G) zw[phase * p.H + g0 * Hkv + kvh] = make_float2(zm0, zz0);
      if (g0 + 1 < G) zw[phase * p.H + (g0 + 1) * Hkv + kvh] = make_float2(zm1, zz1);
    }
  }
  if constexpr (TM) tmem_wait_st();
  runmax0 = fmaxf(runmax0, __shfl_xor_sync(0xffffffffu, runmax0, 4));
  runmax1 = fmaxf(runmax1, __shfl_xor_sync(0xffffffffu, runmax1, 4));
  runmax0 = fmaxf(runmax0, __shfl_xor_sync(0xffffffffu, runmax0, 8));
  runmax1 = fmaxf(runmax1, __shfl_xor_sync(0xffffffffu, runmax1, 8));
  runmax0 = fmaxf(runmax0, __shfl_xor_sync(0xffffffffu, runmax0, 16));
  runmax1 = fmaxf(runmax1, __shfl_xor_sync(0xffffffffu, runmax1, 16));
  if (lane < 4) {
    if (g0 < G && runmax0 > -INFINITY) atomicMax(&sm.headmax[g0 * Hkv + kvh], float_ord(runmax0));
    if (g0 + 1 < G && runmax1 > -INFINITY) atomicMax(&sm.headmax[(g0 + 1) * Hkv + kvh], float_ord(runmax1));
  }
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

// ------------------------------------------------------------ radix select
// Adds this CTA's non-empty shared-histogram bins into the global one.
__device__ __noinline__ void hist_merge(const uint32_t* hist, uint32_t* gh) {
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) {
    const uint32_t c = hist[i];
    if (c) atomicAdd(gh + i, c);
  }
}

// Local 12-bit digit histogram of this CTA's keys (optionally only keys whose
// bits above `pshift` equal `prefix`), aggregated per warp with match.any so a
// crowded bin costs one shared atomic per warp, then merged into the
// sequence's global histogram `gh`. All threads call.
__device__ __noinline__ void radix_hist(const uint32_t* keys, int nloc, int shift, int pshift, uint32_t prefix,
                                        uint32_t* hist, uint32_t* gh, unsigned long long* tr) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kRadixBins; i += blockDim.x) hist[i] = 0u;
  __syncthreads();
  stamp(tr, 38);
  for (int base = 0; base < nloc; base += blockDim.x) {
    const int jl = base + tid;
    uint32_t key = 0;
    bool act = false;
    if (jl < nloc) {
      key = keys[jl];
      act = pshift >= 32 || (key >> pshift) == prefix;
    }
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (act) {
      const uint32_t bin = (key >> shift) & (kRadixBins - 1);
      const unsigned peers = __match_any_sync(am, bin);
      if (lane == __ffs(peers) - 1) atomicAdd(&hist[bin], static_cast<uint32_t>(__popc(peers)));
    }
  }
  __syncthreads();
  stamp(tr, 39);
  hist_merge(hist, gh);
}


// One key into the shared histogram, aggregated over the warp's lanes that
// hit the same bin (all lanes call; `act` marks the lanes with a key).
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t key, bool act, int shift) {
  const unsigned am = __ballot_sync(0xffffffffu, act);
  if (act) {
    const uint32_t bin = (key >> shift) & (kRadixBins - 1);
    const unsigned peers = __match_any_sync(am, bin);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], static_cast<uint32_t>(__popc(peers)));
  }
}

// ---------------------------------------------------------- attention rows
// The attended rows of one sequence, in merged (ascending) order:
//   [0, init_end) ++ selection part ++ [lb, n_cached) ++ current token
// (make_windows + merged(), attention.cpp:21-52). The selection part is the
// cached SelectionResult filtered to [init_end, lb) on a hit (sel[lo1 + i]),
// or this step's fresh selection (already inside that range) held as
// per-CTA ascending lists located through the CTA prefix offsets.
struct AttView {
  int n_rows;      // cached attended rows (excl. current)
  int init_end, n1, lb;
  int lo1;         // hit: offset of the filtered range in sel[]
  int fresh;       // 1: selection part = per-CTA lists of this launch
  int ncta;        // fresh: CTAs of the sequence (prefix has ncta + 1 entries)
  int cta0;        // fresh: first CTA of the sequence
};

// Sum over the 32 lanes of P per-lane values v[0..P) (P a power of two <= 8)
// by recursive halving: after it, lane L holds the total of value index
// idx(L) = sum_s bit(L, 4 - s) * (P >> (s + 1)) -- log2(P) + 5 - log2(P)
// shuffles per P values instead of 5 per value.
template <int P>
__device__ __forceinline__ float transpose_reduce(float (&v)[8], int lane, int* idx) {
  int id = 0;
  int size = P;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (size > 1) {
      const int half = size >> 1;
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < half) {
          const float keep = hi ? v[i + half] : v[i];
          const float send = hi ? v[i] : v[i + half];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      if (hi) id += half;
      size = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  *idx = id;
  return v[0];
}

constexpr int kAttIdx = 1024;  // slab rows resolved per index window

// Slab row of merged row i: the selection part comes with its slab rows
// (published by the selecting CTAs, or cached with the SelectionResult),
// only the windows go through the page table.
template <bool LEAN>
__device__ __forceinline__ int32_t att_row(const DecodeParams& p, const SeqDesc& sd, const AttView& v,
                                           const int* prefix, int i) {
  if (!LEAN && sd.att_list) return static_cast<int32_t>(row_index(sd, sd.att_list[i], p.page_size));
  if (i < v.init_end) return static_cast<int32_t>(row_index<LEAN>(sd, static_cast<uint32_t>(i), p.page_size));
  i -= v.init_end;
  if (i < v.n1) {
    if (!v.fresh) {
      if (LEAN || sd.sel_rows) return __ldcg(sd.sel_rows + v.lo1 + i);
      return static_cast<int32_t>(row_index(sd, __ldcg(sd.sel + v.lo1 + i), p.page_size));
    }
    int lo = 0, hi = v.ncta - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    return __ldcg(p.ws_sel_row + static_cast<size_t>(v.cta0 + lo) * p.tpc + (i - prefix[lo]));
  }
  i -= v.n1;
  return static_cast<int32_t>(row_index<LEAN>(sd, static_cast<uint32_t>(v.lb + i), p.page_size));
}

// Tensor-core split-K flash-decoding partial (D = 64 / 128, G <= 8) of the
// query heads {g + m*H_kv} sharing KV head g over merged rows [r0, r1), plus
// the current token (fp32 k_t / v_t, CUDA cores) when `with_cur`.
//   * q staging and the slab-row pass issue their loads together, then the
//     K/V slices (d wide, this KV head only) are gathered with 16-byte
//     cp.async into padded rows (ldmatrix conflict-free), double-buffered;
//   * scores: S[16 rows x 8 heads] per m16n8k16 tile, K rows as A (ldmatrix),
//     q split exactly into three bf16 parts as B (bf16 x bf16 products are
//     exact in fp32) -- one warp per 16-row tile;
//   * P.V: O^T[16 d x 8 heads] += V^T (ldmatrix.trans) x P^T (P split into
//     three bf16 parts) -- warp = (d tile, row group);
//   * online softmax per head between them, fp32 (attention.cpp:88-110).
template <int D, bool LEAN>
__device__ void attend_group_mma(const DecodeParams& p, const SeqDesc& sd, const AttView& av, const Smem& sm,
                                 int g, int r0, int r1, bool with_cur, float* part) {
  constexpr int KC = D / 16;                 // k-chunks of the score MMA
  constexpr int DT = D / 16;                 // d tiles of the P.V MMA
  constexpr int RS = D + 8;                  // padded smem row stride (bf16 elements)
  const int H_kv = p.H_kv, G = p.H / p.H_kv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int RGP = max(1, (nwarps - (nwarps % DT)) / DT);  // row groups of the P.V warps
  const int row_elems = H_kv * D;
  // ---- carve the staging area
  uint8_t* base = sm.ring;
  float* qs = reinterpret_cast<float*>(base);                 // [8][D] (heads >= G zero)
  size_t o = static_cast<size_t>(8) * D * 4;
  float* ck = reinterpret_cast<float*>(base + o);             // [D] current K (fp32)
  float* cv = ck + D;                                         // [D] current V
  o += static_cast<size_t>(2) * D * 4;
  float* red = reinterpret_cast<float*>(base + o);            // [RGP][8][D]
  o += align_up(static_cast<size_t>(RGP) * 8 * D * 4, 128);
  float* stat = reinterpret_cast<float*>(base + o);           // [8][4] m_run, l_run
  int* hmax = reinterpret_cast<int*>(stat + 32);              // [2][8] sub-chunk score max (ordered ints)
  float* lpart = stat + 48;                                   // [kAttMaxRows / 16][8] row-slice sums of P
  o += align_up(static_cast<size_t>(48 + kAttMaxRows / 16 * 8) * 4, 128);
  int32_t* ridx = reinterpret_cast<int32_t*>(base + o);       // [kAttIdx] slab rows
  o += static_cast<size_t>(kAttIdx) * 4;
  uint2* qf = reinterpret_cast<uint2*>(base + o);             // [KC][3][32] B fragments of q (hi/mid/lo)
  o += static_cast<size_t>(KC) * 3 * 32 * 8;
  const size_t rest = static_cast<size_t>(p.att_bytes) > o ? static_cast<size_t>(p.att_bytes) - o : 0;
  // per row: 2 buffers x (K + V) padded slices + 8 probs + P fragments
  int cap = static_cast<int>(rest / (4 * RS * 2 + 32 + 32 + 48)) & ~15;
  cap = max(16, min(cap, kAttMaxRows));
  float* probs = reinterpret_cast<float*>(base + o);          // [cap + 16][8]
  o += align_up(static_cast<size_t>(cap + 16) * 32, 128);
  uint2* pf = reinterpret_cast<uint2*>(base + o);             // [cap / 16][3][32] B fragments of P^T
  o += align_up(static_cast<size_t>(cap / 16) * 3 * 32 * 8, 128);
  uint16_t* kb[2];
  uint16_t* vb[2];
  for (int b = 0; b < 2; ++b) {
    kb[b] = reinterpret_cast<uint16_t*>(base + o);
    o += static_cast<size_t>(cap) * RS * 2;
    vb[b] = reinterpret_cast<uint16_t*>(base + o);
    o += static_cast<size_t>(cap) * RS * 2;
  }
  const int nrows = max(0, r1 - r0);
  // ---- q (one element per thread, loads issued with the first slab-row pass)
  float qv = 0.f;
  {
    const int m = tid / D, t = tid - (tid / D) * D;
    if (tid < 8 * D) qv = m < G ? __ldg(sd.q + static_cast<size_t>(g + m * H_kv) * D + t) : 0.f;
    for (int i = tid + blockDim.x; i < 8 * D; i += blockDim.x) {
      const int m2 = i / D, t2 = i - (i / D) * D;
      qs[i] = m2 < G ? __ldg(sd.q + static_cast<size_t>(g + m2 * H_kv) * D + t2) : 0.f;
    }
  }
  if (with_cur)
    for (int t = tid; t < D; t += blockDim.x) {
      ck[t] = __ldg(sd.k_new + static_cast<size_t>(g) * D + t);
      cv[t] = __ldg(sd.v_new + static_cast<size_t>(g) * D + t);
    }
  if (tid < 8) {
    stat[tid * 4 + 0] = -INFINITY;
    stat[tid * 4 + 1] = 0.f;
    stat[tid * 4 + 2] = 1.f;
    hmax[tid] = hmax[8 + tid] = float_ord(-INFINITY);
  }
  // P.V accumulators: warp (d tile dt, row group rgp)
  const int dt = warp % DT, rgp = warp / DT;
  const bool pv_warp = rgp < RGP;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  // gather the slices of index-window rows [c0, c0 + nr) into buffer b
  constexpr int CPR = D * 2 / 16;  // 16-byte chunks per slice
  auto issue = [&](int c0, int nr, int b) {
    for (int idx = tid; idx < nr * CPR; idx += blockDim.x) {
      const int r = idx / CPR, q = idx - (idx / CPR) * CPR;
      const int64_t off = static_cast<int64_t>(ridx[c0 + r]) * row_elems + static_cast<int64_t>(g) * D + q * 8;
      cp_async16(kb[b] + static_cast<size_t>(r) * RS + q * 8, p.k_slab + off);
      cp_async16(vb[b] + static_cast<size_t>(r) * RS + q * 8, p.v_slab + off);
    }
    cp_async_commit();
  };
  int w0 = 0, sub = 0;
  bool first = true;
  for (;;) {
    const int nw = min(kAttIdx, nrows - w0);
    for (int r = tid; r < nw; r += blockDim.x) ridx[r] = att_row<LEAN>(p, sd, av, sm.prefix, r0 + w0 + r);
    const bool build_qf = first;
    if (first && tid < 8 * D) qs[tid] = qv;
    first = false;
    __syncthreads();
    trace_pt(p, 20);
    if (build_qf && tid < KC * 32) {
      // q^T as the score MMA's B operand, split exactly into three bf16 parts:
      // lane l holds q[head l/4][kc*16 + 2(l%4) + {0,1,8,9}]
      const int kc = tid >> 5, l = tid & 31;
      const int n = l >> 2, dd = kc * 16 + (l & 3) * 2;
      float h[4], m[4], lo[4];
      split3(qs[n * D + dd], h[0], m[0], lo[0]);
      split3(qs[n * D + dd + 1], h[1], m[1], lo[1]);
      split3(qs[n * D + dd + 8], h[2], m[2], lo[2]);
      split3(qs[n * D + dd + 9], h[3], m[3], lo[3]);
      qf[(kc * 3 + 0) * 32 + l] = make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
      qf[(kc * 3 + 1) * 32 + l] = make_uint2(pack_bf16x2(m[0], m[1]), pack_bf16x2(m[2], m[3]));
      qf[(kc * 3 + 2) * 32 + l] = make_uint2(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]));
    }
    const bool last_w = w0 + nw >= nrows;
    const int nsub = max(1, (nw + cap - 1) / cap);
    issue(0, min(cap, nw), sub & 1);
    for (int c = 0; c < nsub; ++c, ++sub) {
      const int c0 = c * cap;
      const int nr = max(0, min(cap, nw - c0));
      const int nr16 = (nr + 15) & ~15;
      const bool last = last_w && c == nsub - 1;
      const bool cur_here = last && with_cur;
      if (c + 1 < nsub) {
        issue(c0 + cap, min(cap, nw - c0 - cap), (sub + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      if (sub == 0) trace_pt(p, 21);
      const uint16_t* K = kb[sub & 1];
      uint16_t* V = vb[sub & 1];
      // zero the padding rows of V (P is zero there; keep 0 * garbage finite)
      for (int i = tid; i < (nr16 - nr) * (D / 8); i += blockDim.x) {
        const int r = nr + i / (D / 8), q = i - (i / (D / 8)) * (D / 8);
        *reinterpret_cast<uint4*>(V + static_cast<size_t>(r) * RS + q * 8) = make_uint4(0u, 0u, 0u, 0u);
      }
      // ---- scores: warp w -> rows [16w, 16w + 16)
      for (int mt = warp; mt * 16 < nr; mt += nwarps) {
        float ch[4] = {0.f, 0.f, 0.f, 0.f}, cm[4] = {0.f, 0.f, 0.f, 0.f}, cl[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t abase = smem_u32(K) +
                               static_cast<uint32_t>(((mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * RS + (lane >> 4) * 8) * 2);
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
          uint32_t a[4];
          ldmatrix_x4(a, abase + kc * 32);
          const uint2 bh = qf[(kc * 3 + 0) * 32 + lane], bm = qf[(kc * 3 + 1) * 32 + lane];
          const uint2 bl = qf[(kc * 3 + 2) * 32 + lane];
          mma_bf16_16816(ch, a, bh.x, bh.y);
          mma_bf16_16816(cm, a, bm.x, bm.y);
          mma_bf16_16816(cl, a, bl.x, bl.y);
        }
        float cacc[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) cacc[e] = ch[e] + (cm[e] + cl[e]);
        float tmax[2] = {-INFINITY, -INFINITY};  // this lane's two heads over its two rows
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = mt * 16 + (lane >> 2) + (e >> 1) * 8;
          const int col = (lane & 3) * 2 + (e & 1);
          const float sc = cacc[e] * p.attn_scale;
          if (row < nr) {
            probs[row * 8 + col] = sc;
            if (col < G) tmax[e & 1] = fmaxf(tmax[e & 1], sc);
          }
        }
        // the tile's max per head (lanes with equal lane % 4 share the heads)
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
          tmax[0] = fmaxf(tmax[0], __shfl_xor_sync(0xffffffffu, tmax[0], o2));
          tmax[1] = fmaxf(tmax[1], __shfl_xor_sync(0xffffffffu, tmax[1], o2));
        }
        if (lane < 4) {
          if (2 * lane < G) atomicMax(&hmax[(sub & 1) * 8 + 2 * lane], float_ord(tmax[0]));
          if (2 * lane + 1 < G) atomicMax(&hmax[(sub & 1) * 8 + 2 * lane + 1], float_ord(tmax[1]));
        }
      }
      if (cur_here && warp == nwarps - 1) {
        // current token row (fp32 K): one warp, G dot products
        for (int m = 0; m < G; ++m) {
          float a = 0.f;
          for (int t = lane; t < D; t += 32) a = fmaf(qs[m * D + t], ck[t], a);
          a = warp_sum(a) * p.attn_scale;
          if (lane == 0) {
            probs[cap * 8 + m] = a;  // slot past the tiles
            atomicMax(&hmax[(sub & 1) * 8 + m], float_ord(a));
          }
        }
      }
      __syncthreads();
      if (sub == 0) trace_pt(p, 22);
      // ---- online softmax fused into the P^T build (P.V's B operand, three
      // exact bf16 parts): P = e^(s - m_new) with m_new = max(m_run, this
      // sub-chunk's max); rows >= nr and heads >= G get P = 0. Row-slice sums
      // go to lpart (summed in a fixed order below: deterministic).
      const int nk = nr16 / 16;
      if (tid < nk * 32) {
        const int ks = tid >> 5, l = tid & 31;
        const int n = l >> 2, k0 = ks * 16 + (l & 3) * 2;
        const float m_new = fmaxf(stat[n * 4 + 0], ord_float(hmax[(sub & 1) * 8 + n]));
        const bool live = n < G && m_new > -INFINITY;
        float w[4];
        const int rr[4] = {k0, k0 + 1, k0 + 8, k0 + 9};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] = (live && rr[e] < nr) ? ex2_approx((probs[rr[e] * 8 + n] - m_new) * kLog2e) : 0.f;
        float h[4], m[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split3(w[e], h[e], m[e], lo[e]);
        pf[(ks * 3 + 0) * 32 + l] = make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
        pf[(ks * 3 + 1) * 32 + l] = make_uint2(pack_bf16x2(m[0], m[1]), pack_bf16x2(m[2], m[3]));
        pf[(ks * 3 + 2) * 32 + l] = make_uint2(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]));
        float ls = (w[0] + w[1]) + (w[2] + w[3]);
        ls += __shfl_xor_sync(0xffffffffu, ls, 1);
        ls += __shfl_xor_sync(0xffffffffu, ls, 2);
        if ((l & 3) == 0) lpart[ks * 8 + n] = ls;
      }
      if (tid < 8) hmax[((sub + 1) & 1) * 8 + tid] = float_ord(-INFINITY);  // the next sub-chunk's
      if (cur_here && tid >= 32 * 16 && tid < 32 * 16 + G) {
        const int m = tid - 32 * 16;
        const float m_new = fmaxf(stat[m * 4 + 0], ord_float(hmax[(sub & 1) * 8 + m]));
        probs[cap * 8 + m] = ex2_approx((probs[cap * 8 + m] - m_new) * kLog2e);
      }
      __syncthreads();
      if (sub == 0) trace_pt(p, 23);
      // ---- P.V on tensor cores
      if (pv_warp) {
        const int n0 = (lane & 3) * 2;
        // rescale by e^(m_run - m_new) (0 while m_run = -inf)
        const float mo0 = stat[n0 * 4 + 0], mo1 = stat[(n0 + 1) * 4 + 0];
        const float mn0 = fmaxf(mo0, ord_float(hmax[(sub & 1) * 8 + n0]));
        const float mn1 = fmaxf(mo1, ord_float(hmax[(sub & 1) * 8 + n0 + 1]));
        const float c0f = mo0 == -INFINITY ? 0.f : ex2_approx((mo0 - mn0) * kLog2e);
        const float c1f = mo1 == -INFINITY ? 0.f : ex2_approx((mo1 - mn1) * kLog2e);
        acc[0] *= c0f;
        acc[1] *= c1f;
        acc[2] *= c0f;
        acc[3] *= c1f;
        const int jm = lane >> 3, im = lane & 7;
        const uint32_t vbase = smem_u32(V) +
                               static_cast<uint32_t>((((jm >> 1) * 8 + im) * RS + dt * 16 + (jm & 1) * 8) * 2);
        for (int ks = rgp; ks < nk; ks += RGP) {
          uint32_t a[4];
          ldmatrix_x4_trans(a, vbase + static_cast<uint32_t>(ks * 16 * RS * 2));
          const uint2 bh = pf[(ks * 3 + 0) * 32 + lane], bm = pf[(ks * 3 + 1) * 32 + lane];
          const uint2 bl = pf[(ks * 3 + 2) * 32 + lane];
          mma_bf16_16816(acc, a, bh.x, bh.y);
          mma_bf16_16816(acc, a, bm.x, bm.y);
          mma_bf16_16816(acc, a, bl.x, bl.y);
        }
      }
      if (cur_here) {
        // the current token's P.V term, added once by row group 0
        if (pv_warp && rgp == 0) {
          const int n0 = (lane & 3) * 2, d0 = dt * 16 + (lane >> 2);
          acc[0] = fmaf(probs[cap * 8 + n0], cv[d0], acc[0]);
          acc[1] = fmaf(probs[cap * 8 + n0 + 1], cv[d0], acc[1]);
          acc[2] = fmaf(probs[cap * 8 + n0], cv[d0 + 8], acc[2]);
          acc[3] = fmaf(probs[cap * 8 + n0 + 1], cv[d0 + 8], acc[3]);
        }
      }
      __syncthreads();  // buffer and probs free for the next sub-chunk
      if (tid < G) {
        // running (m, l) of head tid; read by the next sub-chunk after its first barrier
        const float mo = stat[tid * 4 + 0];
        const float mn = fmaxf(mo, ord_float(hmax[(sub & 1) * 8 + tid]));
        float ls = cur_here ? probs[cap * 8 + tid] : 0.f;
        for (int ks = 0; ks < nk; ++ks) ls += lpart[ks * 8 + tid];
        const float corr = mo == -INFINITY ? 0.f : ex2_approx((mo - mn) * kLog2e);
        stat[tid * 4 + 0] = mn;
        stat[tid * 4 + 1] = stat[tid * 4 + 1] * corr + ls;
      }
      if (sub == 0) trace_pt(p, 24);
    }
    w0 += nw;
    if (last_w) break;
  }
  trace_pt(p, 25);
  // ---- reduce the row groups, write the partial record per head
  if (pv_warp) {
    const int n0 = (lane & 3) * 2, d0 = dt * 16 + (lane >> 2);
    float* rr = red + static_cast<size_t>(rgp) * 8 * D;
    rr[n0 * D + d0] = acc[0];
    rr[(n0 + 1) * D + d0] = acc[1];
    rr[n0 * D + d0 + 8] = acc[2];
    rr[(n0 + 1) * D + d0 + 8] = acc[3];
  }
  __syncthreads();
  const int stride = att_stride(D);
  for (int i = tid; i < G * D; i += blockDim.x) {
    const int m = i / D, t = i - (i / D) * D;
    float sacc = 0.f;
    for (int q = 0; q < RGP; ++q) sacc += red[(static_cast<size_t>(q) * 8 + m) * D + t];
    part[static_cast<size_t>(m) * stride + t] = sacc;
  }
  if (tid < G) {
    part[static_cast<size_t>(tid) * stride + D] = stat[tid * 4 + 0];
    part[static_cast<size_t>(tid) * stride + D + 1] = stat[tid * 4 + 1];
  }
}

// Split-K flash-decoding partial of the G query heads {g + m*H_kv} that share
// KV head g (the reference's h mod H_kv map, attention.cpp:78) over rows
// [r0, r1) of the merged list, plus the current token (fp32 k_t / v_t) when
// `with_cur`. Slab rows of up to kAttIdx rows are resolved first (one
// parallel pass over the page table), then only this KV head's d-wide K/V
// slices are gathered with 16-byte cp.async into a double buffer of `cap`
// rows. Scores: one warp per row, lane = d/32 contiguous elements, q held in
// registers, FFMA2 + transposed shuffle reduction. P.V: (row group, d pair)
// threads with FFMA2. Writes (o[d], m, l) per head (attention.cpp:88-110
// semantics, fp32). DT/GT = 0: runtime shapes (any d, G <= 8).

template <int DT, int GT>
__device__ void attend_group(const DecodeParams& p, const SeqDesc& sd, const AttView& av, const Smem& sm,
                             int g, int r0, int r1, bool with_cur, float* part) {
  constexpr bool kFast = DT > 0;
  const int H_kv = p.H_kv;
  const int d = kFast ? DT : p.d;
  const int G = kFast ? GT : p.H / p.H_kv;
  constexpr int E = kFast ? DT / 32 : 1;           // elements per lane (fast path)
  constexpr int P = GT <= 1 ? 1 : GT <= 2 ? 2 : GT <= 4 ? 4 : 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const bool even = (d & 1) == 0;
  const bool vec = (d % 8) == 0;          // 16-byte gathers
  const int ew = even ? 2 : 1;            // elements per P.V thread
  const int npt = d / ew;                 // P.V threads per row group
  const int RG = max(1, min(static_cast<int>(blockDim.x) / npt, 16));
  const int row_elems = H_kv * d;
  const size_t slice = static_cast<size_t>(d) * 2;  // bytes of one K (or V) slice
  // ---- carve the staging area (ring + the dead S/keys region)
  uint8_t* base = sm.ring;
  float* qs = reinterpret_cast<float*>(base);                       // [G][d]
  size_t o = align_up(static_cast<size_t>(G) * d * 4, 128);
  float* ck = reinterpret_cast<float*>(base + o);                   // [d] current K (fp32)
  float* cv = ck + d;                                               // [d] current V
  o += align_up(static_cast<size_t>(2) * d * 4, 128);
  float* red = reinterpret_cast<float*>(base + o);                  // [RG][G][d]
  o += align_up(static_cast<size_t>(RG) * G * d * 4, 128);
  float* stat = reinterpret_cast<float*>(base + o);                 // [8][4] m_run, l_run, corr
  o += 128;
  int32_t* ridx = reinterpret_cast<int32_t*>(base + o);             // [kAttIdx] slab rows
  o += static_cast<size_t>(kAttIdx) * 4;
  const size_t rest = static_cast<size_t>(p.att_bytes) > o ? static_cast<size_t>(p.att_bytes) - o : 0;
  // per row: 2 buffers x (K + V) slices + 8 probs
  int cap = static_cast<int>(rest / (4 * slice + 32 + 64));
  cap = max(1, min(cap, kAttMaxRows));
  float* probs = reinterpret_cast<float*>(base + o);                // [cap + 1][8]
  o += align_up(static_cast<size_t>(cap + 1) * 32, 128);
  uint16_t* kb[2];
  uint16_t* vb[2];
  for (int b = 0; b < 2; ++b) {
    kb[b] = reinterpret_cast<uint16_t*>(base + o);
    o += align_up(static_cast<size_t>(cap) * slice, 128);
    vb[b] = reinterpret_cast<uint16_t*>(base + o);
    o += align_up(static_cast<size_t>(cap) * slice, 128);
  }
  // ---- q heads of this KV head, current token K/V slices, running stats
  for (int i = tid; i < G * d; i += blockDim.x) {
    const int m = i / d, t = i - (i / d) * d;
    qs[i] = __ldg(sd.q + static_cast<size_t>(g + m * H_kv) * d + t);
  }
  if (with_cur)
    for (int t = tid; t < d; t += blockDim.x) {
      ck[t] = __ldg(sd.k_new + static_cast<size_t>(g) * d + t);
      cv[t] = __ldg(sd.v_new + static_cast<size_t>(g) * d + t);
    }
  if (tid < 8) {
    stat[tid * 4 + 0] = -INFINITY;
    stat[tid * 4 + 1] = 0.f;
    stat[tid * 4 + 2] = 1.f;
  }
  float2 acc[kAttMaxG];
#pragma unroll
  for (int m = 0; m < kAttMaxG; ++m) acc[m] = make_float2(0.f, 0.f);
  const int rg = tid / npt, pi = tid - (tid / npt) * npt;
  const int nrows = max(0, r1 - r0);
  const int cpr = static_cast<int>(slice / 16);  // 16-byte chunks per slice
  // gather the slices of rows [c0, c0 + nr) of the current index window into buffer b
  auto issue = [&](int c0, int nr, int b) {
    if (vec) {
      for (int idx = tid; idx < nr * cpr; idx += blockDim.x) {
        const int r = idx / cpr, q = idx - (idx / cpr) * cpr;
        const int64_t off = static_cast<int64_t>(ridx[c0 + r]) * row_elems + static_cast<int64_t>(g) * d + q * 8;
        cp_async16(kb[b] + static_cast<size_t>(r) * d + q * 8, p.k_slab + off);
        cp_async16(vb[b] + static_cast<size_t>(r) * d + q * 8, p.v_slab + off);
      }
    } else {
      for (int idx = tid; idx < nr * d; idx += blockDim.x) {
        const int r = idx / d, t = idx - (idx / d) * d;
        const int64_t off = static_cast<int64_t>(ridx[c0 + r]) * row_elems + static_cast<int64_t>(g) * d + t;
        kb[b][static_cast<size_t>(r) * d + t] = p.k_slab[off];
        vb[b][static_cast<size_t>(r) * d + t] = p.v_slab[off];
      }
    }
    cp_async_commit();
  };
  __syncthreads();  // qs / ck / stat visible
  // q slice of this lane in registers (fast path)
  float qr[kFast ? GT : 1][E];
  if constexpr (kFast) {
#pragma unroll
    for (int m = 0; m < GT; ++m)
#pragma unroll
      for (int e = 0; e < E; ++e) qr[m][e] = qs[m * DT + lane * E + e];
  }
  int w0 = 0;  // index window [w0, w0 + nw) of rows whose slab rows are in ridx
  int sub = 0;
  for (;;) {
    const int nw = min(kAttIdx, nrows - w0);
    for (int r = tid; r < nw; r += blockDim.x)
      ridx[r] = att_row<false>(p, sd, av, sm.prefix, r0 + w0 + r);
    __syncthreads();
    trace_pt(p, 20);
    const bool last_w = w0 + nw >= nrows;
    const int nsub = max(1, (nw + cap - 1) / cap);
    issue(0, min(cap, nw), sub & 1);
    for (int c = 0; c < nsub; ++c, ++sub) {
      const int c0 = c * cap;
      const int nr = max(0, min(cap, nw - c0));
      const bool last = last_w && c == nsub - 1;
      const int nrt = nr + ((last && with_cur) ? 1 : 0);  // + current token row
      if (c + 1 < nsub) {
        issue(c0 + cap, min(cap, nw - c0 - cap), (sub + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const uint16_t* K = kb[sub & 1];
      const uint16_t* V = vb[sub & 1];
      if (sub == 0) trace_pt(p, 21);
      // ---- scores s[r][m] = q_m . k_r / sqrt(d)
      for (int r = warp; r < nrt; r += nwarps) {
        if constexpr (kFast) {
          float kx[E];
          if (r < nr) {
            const uint16_t* kr = K + static_cast<size_t>(r) * DT + lane * E;
            if constexpr (E == 4) {
              const uint2 u = *reinterpret_cast<const uint2*>(kr);
              const float2 a = bf16x2_to_f2(u.x), b = bf16x2_to_f2(u.y);
              kx[0] = a.x; kx[1] = a.y; kx[2] = b.x; kx[3] = b.y;
            } else {
              const float2 a = bf16x2_to_f2(*reinterpret_cast<const uint32_t*>(kr));
              kx[0] = a.x; kx[1] = a.y;
            }
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e) kx[e] = ck[lane * E + e];
          }
          float v[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) v[m] = 0.f;
#pragma unroll
          for (int m = 0; m < GT; ++m) {
            float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int e = 0; e < E; e += 2) ffma2(a2, make_float2(qr[m][e], qr[m][e + 1]), make_float2(kx[e], kx[e + 1]));
            v[m] = a2.x + a2.y;
          }
          int hid;
          const float s = transpose_reduce<P>(v, lane, &hid);
          const int lowmask = (32 / P) - 1;  // lanes that share one head total
          if ((lane & lowmask) == 0 && hid < GT) probs[r * 8 + hid] = s * p.attn_scale;
        } else {
          float a[kAttMaxG];
#pragma unroll
          for (int m = 0; m < kAttMaxG; ++m) a[m] = 0.f;
          for (int t = lane; t < d; t += 32) {
            const float kk = r < nr ? bf16_bits_to_f(K[static_cast<size_t>(r) * d + t]) : ck[t];
#pragma unroll
            for (int m = 0; m < kAttMaxG; ++m)
              if (m < G) a[m] = fmaf(qs[m * d + t], kk, a[m]);
          }
#pragma unroll
          for (int m = 0; m < kAttMaxG; ++m)
            if (m < G) {
              const float s = warp_sum(a[m]);
              if (lane == 0) probs[r * 8 + m] = s * p.attn_scale;
            }
        }
      }
      __syncthreads();
      if (sub == 0) trace_pt(p, 22);
      // ---- online softmax per head (warp m owns head m)
      for (int m = warp; m < G; m += nwarps) {
        float mx = -INFINITY;
        for (int r = lane; r < nrt; r += 32) mx = fmaxf(mx, probs[r * 8 + m]);
        mx = warp_max(mx);
        const float m_old = stat[m * 4 + 0];
        const float m_new = fmaxf(m_old, mx);
        float l = 0.f;
        for (int r = lane; r < nrt; r += 32) {
          const float w = m_new == -INFINITY ? 0.f : expf(probs[r * 8 + m] - m_new);
          probs[r * 8 + m] = w;
          l += w;
        }
        l = warp_sum(l);
        if (lane == 0) {
          const float corr = m_old == -INFINITY ? 0.f : expf(m_old - m_new);
          stat[m * 4 + 0] = m_new;
          stat[m * 4 + 1] = stat[m * 4 + 1] * corr + l;
          stat[m * 4 + 2] = corr;
        }
      }
      __syncthreads();
      if (sub == 0) trace_pt(p, 23);
      // ---- P.V: thread (row group rg, element pair pi) over rows rg, rg + RG, ...
      if (rg < RG) {
#pragma unroll
        for (int m = 0; m < kAttMaxG; ++m)
          if (m < G) {
            const float corr = stat[m * 4 + 2];
            acc[m].x *= corr;
            acc[m].y *= corr;
          }
        for (int r = rg; r < nrt; r += RG) {
          float2 v2;
          if (r < nr) {
            if (even) {
              v2 = bf16x2_to_f2(*reinterpret_cast<const uint32_t*>(V + static_cast<size_t>(r) * d + 2 * pi));
            } else {
              v2 = make_float2(bf16_bits_to_f(V[static_cast<size_t>(r) * d + pi]), 0.f);
            }
          } else {
            v2 = even ? make_float2(cv[2 * pi], cv[2 * pi + 1]) : make_float2(cv[pi], 0.f);
          }
          const float4 w0v = *reinterpret_cast<const float4*>(probs + r * 8);
          const float4 w1v = *reinterpret_cast<const float4*>(probs + r * 8 + 4);
          const float w[8] = {w0v.x, w0v.y, w0v.z, w0v.w, w1v.x, w1v.y, w1v.z, w1v.w};
#pragma unroll
          for (int m = 0; m < kAttMaxG; ++m)
            if (m < G) ffma2(acc[m], make_float2(w[m], w[m]), v2);
        }
      }
      __syncthreads();  // buffer and probs free for the next sub-chunk
      if (sub == 0) trace_pt(p, 24);
    }
    w0 += nw;
    if (last_w) break;
  }
  trace_pt(p, 25);
  // ---- reduce the row groups, write the partial record per head
  if (rg < RG) {
#pragma unroll
    for (int m = 0; m < kAttMaxG; ++m)
      if (m < G) {
        red[(static_cast<size_t>(rg) * G + m) * d + ew * pi] = acc[m].x;
        if (even) red[(static_cast<size_t>(rg) * G + m) * d + 2 * pi + 1] = acc[m].y;
      }
  }
  __syncthreads();
  const int stride = att_stride(d);
  for (int i = tid; i < G * d; i += blockDim.x) {
    const int m = i / d, t = i - (i / d) * d;
    float s = 0.f;
    for (int q = 0; q < RG; ++q) s += red[(static_cast<size_t>(q) * G + m) * d + t];
    part[static_cast<size_t>(m) * stride + t] = s;
  }
  if (tid < G) {
    part[static_cast<size_t>(tid) * stride + d] = stat[tid * 4 + 0];
    part[static_cast<size_t>(tid) * stride + d + 1] = stat[tid * 4 + 1];
  }
}

// Log-sum-exp merge of the row-chunk partials of KV head g (attention.cpp
// :88-110 semantics): out[h] = sum_c e^(m_c - M) o_c / sum_c e^(m_c - M) l_c.
// Outputs [o0, o0 + nout) of the group's G*d, once all partials are in. One
// L2 round trip: the (m, l) of every chunk and these outputs' o values are
// loaded together into shared memory (`buf`, free staging), then warp per
// head forms M, L and the chunk weights, and thread per output sums its
// chunks.
template <bool LEAN>
__device__ void merge_outputs(const DecodeParams& p, const SeqDesc& sd, int g, const float* parts, int chunks,
                              int o0, int nout, float* buf) {
  const int d = p.d, G = p.H / p.H_kv, stride = att_stride(d);
  const size_t rec = static_cast<size_t>(G) * stride;  // floats per chunk
  if (nout <= 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  float* hdr = buf;                                // [G][2] M, L
  float* wts = buf + 2 * kAttMaxG;                 // [G][chunks] (m_c, then the weight e^(m_c - M))
  float* lcs = wts + G * chunks;                   // [G][chunks] l_c
  float* ov = lcs + G * chunks;                    // [chunks][nout]
  #pragma unroll 1
  for (int i = tid; i < G * chunks; i += blockDim.x) {
    const int m = i / chunks, c = i - (i / chunks) * chunks;
    const float* r = parts + c * rec + static_cast<size_t>(m) * stride + d;
    wts[i] = __ldcg(r);
    lcs[i] = __ldcg(r + 1);
  }
  // (a slice is about one element per thread; the loop is kept rolled: the
  // merge runs once per launch, from a cold instruction cache)
#pragma unroll 1
  for (int i = tid; i < nout * chunks; i += blockDim.x) {
    const int c = i / nout, oo = i - c * nout;
    const int o = o0 + oo, m = o / d, t = o - m * d;
    ov[i] = __ldcg(parts + c * rec + static_cast<size_t>(m) * stride + t);
  }
  __syncthreads();
  unsigned long long* const trc = p.trace ? p.trace + blockIdx.x * kTraceStride : nullptr;
  stamp(trc, 42);
  for (int m = warp; m < G; m += nwarps) {
    float M = -INFINITY;
    #pragma unroll 1
    for (int c = lane; c < chunks; c += 32) M = fmaxf(M, wts[m * chunks + c]);
    M = warp_max(M);
    float L = 0.f;
    #pragma unroll 1
    for (int c = lane; c < chunks; c += 32) {
      const float mc = wts[m * chunks + c];
      const float w = (M == -INFINITY || mc == -INFINITY) ? 0.f : fast_exp(mc - M);
      wts[m * chunks + c] = w;
      L = fmaf(w, lcs[m * chunks + c], L);
    }
    L = warp_sum(L);
    if (lane == 0) {
      hdr[m * 2 + 0] = M;
      hdr[m * 2 + 1] = L;
    }
  }
  __syncthreads();
  stamp(trc, 43);
  #pragma unroll 1
  for (int oo = tid; oo < nout; oo += blockDim.x) {
    const int o = o0 + oo, m = o / d, t = o - (o / d) * d;
    const float* wm = wts + m * chunks;
    float acc = 0.f;
    #pragma unroll 1
    for (int c = 0; c < chunks; ++c) acc = fmaf(wm[c], ov[c * nout + oo], acc);
    const float L = hdr[m * 2 + 1];
    sd.out[static_cast<size_t>(g + m * p.H_kv) * d + t] = L > 0.f ? acc / L : 0.f;  // empty shard: 0
    if (!LEAN && sd.ml_out && t == 0) {
      sd.ml_out[(g + m * p.H_kv) * 2 + 0] = hdr[m * 2 + 0];
      sd.ml_out[(g + m * p.H_kv) * 2 + 1] = L;
    }
  }
  __syncthreads();  // buf is the next group's attention staging
}

// Per-CTA softmax partials m = max_j S, z = sum_j e^(S - m) per head
// (softmax_rows, tensor.cpp:31-52), S <- e^(S - m) in place: warp per head,
// float4 rows, four independent SFU chains per lane.
__device__ __noinline__ void softmax_partials(float* Sbuf, int sstride, int nloc, int H, const int* headmax,
                                              float* m_out, float* z_out, size_t sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n4 = (nloc + 3) >> 2;
  for (int h = warp; h < H; h += kDecodeWarps) {
    const float m = ord_float(headmax[h]);
    const float ml = m * kLog2e;
    float4* sr = reinterpret_cast<float4*>(Sbuf + static_cast<size_t>(h) * sstride);
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    if (m > -INFINITY) {
      // S <- e^(S - m) in place (the soft vote then needs FMAs only); eight
      // float4 per lane in flight (S may be spilled to global memory: each
      // round of loads is an L2 / HBM round trip)
      for (int q0 = lane; q0 < n4; q0 += 8 * 32) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u * 32 < n4) v[u] = sr[q0 + u * 32];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u * 32 < n4) {
            v[u].x = ex2_approx(fmaf(v[u].x, kLog2e, -ml));
            v[u].y = ex2_approx(fmaf(v[u].y, kLog2e, -ml));
            v[u].z = ex2_approx(fmaf(v[u].z, kLog2e, -ml));
            v[u].w = ex2_approx(fmaf(v[u].w, kLog2e, -ml));
            sr[q0 + u * 32] = v[u];
            z0 += v[u].x;
            z1 += v[u].y;
            z2 += v[u].z;
            z3 += v[u].w;
          }
      }
    }
    const float z = warp_sum((z0 + z1) + (z2 + z3));
    if (lane == 0) {
      m_out[h * sh] = m;
      z_out[h * sh] = z;
    }
  }
}

// LEAN: the engine's single-sequence decode step (mode kLeanMode, soft vote,
// S on chip, no shard / explicit-list / S-in options). Those settings fold to
// constants, so the instantiation carries no code for the other modes: the
// one-shot phases run from a cold instruction cache, and their code size and
// branch count are their latency.
template <int D, int G, bool FAST, int LM>
__global__ void __launch_bounds__(kDecodeThreads, 1) decode_kernel(const DecodeParams p) {
  constexpr bool LEAN = LM != 0;  // LM: the specialisation's fixed mode (kLeanMode / kLeanSelMode), 0: p.mode
  extern __shared__ __align__(1024) uint8_t smem_raw[];  // TMA 128B-swizzle atoms (checked: else row copies)
  const Smem sm = carve(smem_raw, p);
  const int cta = blockIdx.x;
  const int nblocks = gridDim.x;
  const int pmode = LEAN ? LM : p.mode;
  const int n_seq = LEAN ? 1 : p.n_seq;
  const int s_in_smem = LEAN ? kSTmem : p.s_in_smem;
  const int method = LEAN ? 2 : p.method;
  const int seq_id = LEAN ? 0 : cta / p.ctas_per_seq;
  const int cs = cta - seq_id * p.ctas_per_seq;
  const int c0 = seq_id * p.ctas_per_seq;
  const SeqDesc sd = p.seqs[seq_id];
  const int H = p.H;
  const int width = H * p.d;
  const int tid = threadIdx.x;
  const bool do_select = (pmode & kModeSelect) != 0;
  // a launch queued programmatically behind this one (the prefill's prep
  // kernel after the selection launch) may be scheduled now; it waits for
  // this grid's completion before reading anything it writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (FAST && tid < kMaxBarPairs) {
    mbar_init(&sm.full[tid], 1);
    mbar_init(&sm.empty[tid], p.H_kv);  // the H_kv consumer warps of a phase
  }
  if (tid == 0) {
    mbar_init(&sm.att[0], 1);
    mbar_init(&sm.att[1], 1);
    mbar_init(sm.aux, 1);
  }
  uint32_t aux_phase = 0;
  for (int h = tid; h < H; h += blockDim.x) sm.headmax[h] = float_ord(-INFINITY);
  fence_mbar_init();
  GridSync gs{p.bar + p.bar_slot, static_cast<unsigned int>(nblocks), 0u};
  if (cta == 0) {  // the next launch's grid-barrier and merge counters
    if (tid == 0) p.bar[p.bar_slot ^ 32] = 0u;
    unsigned int* nxt = p.ws_acnt + (p.bar_slot ? 0 : kMaxSeqPerLaunch * p.H_kv);
    for (int i = tid; i < kMaxSeqPerLaunch * p.H_kv; i += blockDim.x) nxt[i] = 0u;
  }

  trace_pt(p, 0);
  unsigned long long* const trc = p.trace ? p.trace + blockIdx.x * kTraceStride : nullptr;
  TSB_STOP_AT(15);  // launch + prologue only
  // ---- phase 0: append, scan frames, Selection Cache decision(s), hit prep
  // the decision's loads first: they head the critical path
  DecisionLoads dl{};
  const bool dec_early = sd.select && !(pmode & kModeShardSelect) && (pmode & kModeCache);
  if (dec_early) decision_issue(sd, width, dl);
  // a possible hit's row indices (the cached selection's slab rows, 4 B each)
  // and the windows' page-table entries into L2 now, so the attention's
  // index pass after the decision reads them from L2 (tiny: one bulk
  // prefetch per CTA, 256 B, on the first CTAs)
  if (LEAN && tid == 0 && sd.select && (pmode & kModeAttend)) {
    const uint64_t pol = policy_evict_last();
    // [first, first + n) of a 4-byte array, 16-byte aligned whole pieces only
    auto pf = [&](const void* base, int first, int n) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(base) + static_cast<uintptr_t>(first) * 4;
      const uint32_t bytes = static_cast<uint32_t>(n * 4) & ~15u;
      if ((a & 15) == 0 && bytes) bulk_prefetch_l2(reinterpret_cast<const void*>(a), bytes, pol);
    };
    const int nsl = (p.k + 63) / 64;  // 256-B blocks of sel_rows
    const int n_pages = (sd.n_cached + p.page_size - 1) / p.page_size;
    if (cs < nsl) {
      pf(sd.sel_rows, cs * 64, min(64, p.k - cs * 64));
    } else if (cs == nsl) {
      pf(sd.page_table, 0, min(64, n_pages));  // the init window's pages
    } else if (cs == nsl + 1) {
      const int pg = (max(0, sd.local_begin) / p.page_size) & ~3;  // the local window's pages
      pf(sd.page_table, pg, min(64, n_pages - pg));
    }
  }
  stamp(trc, 45);
  const int T = sd.n_cand;
  const int j0 = min(T, cs * p.tpc);
  const int nloc = max(0, min(T, j0 + p.tpc) - j0);
  const bool may_scan = sd.select && (pmode & kModeScore) && !(pmode & kModeSIn);
  // slab rows of the scan candidates: issue the (page-table) loads now, store
  // after the decision so their latency overlaps it. Long CTA ranges
  // (batched / sharded contexts) load each page entry once instead (parked in
  // sm.prefix, idle until phase 6): per-token loads would be a chain of
  // round trips.
  int32_t fr_pre[4];
  const int psh = (p.page_size & (p.page_size - 1)) == 0 ? __ffs(p.page_size) - 1 : -1;
  const int pg0 = psh >= 0 ? (sd.cand_begin + j0) >> psh : 0;
  const int npg = (may_scan && nloc > 4 * static_cast<int>(blockDim.x) && psh >= 0 && !sd.cand)
                      ? ((sd.cand_begin + j0 + nloc - 1) >> psh) - pg0 + 1 : 0;
  const bool by_page = npg > 0 && npg <= kMaxPrefix;
  int32_t pg_pre = 0;
  if (by_page) {
    if (tid < npg) pg_pre = __ldcg(sd.page_table + pg0 + tid);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jl = tid + u * blockDim.x;
      fr_pre[u] = (may_scan && jl < nloc)
                      ? static_cast<int32_t>(row_index<LEAN>(sd, cand_at<LEAN>(sd, j0 + jl), p.page_size)) : 0;
    }
  }
  stamp(trc, 46);
  // hit prep: the cached selection (counted below init_end / local_begin after the decision)
  const bool hit_prep = (LEAN || !sd.att_list) && sd.select && (pmode & (kModeCache | kModeUseCached)) &&
                        (pmode & kModeAttend);
  const uint32_t ie = static_cast<uint32_t>(sd.init_end);
  const uint32_t lbs = static_cast<uint32_t>(max(sd.local_begin, sd.init_end));
  uint32_t selv[4];
  int n_sel_prev = 0;
  const bool sel_small = p.k <= 4 * static_cast<int>(blockDim.x);
  if (hit_prep) {
    n_sel_prev = __ldcg(&sd.cache->n_sel);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + u * blockDim.x;
      selv[u] = i < p.k ? __ldcg(sd.sel + i) : 0xffffffffu;
    }
  }
  stamp(trc, 47);
  const int pre = 0;  // ring stages issued before the decision (none)
  // Selection Cache decisions. A single sequence: every CTA evaluates it
  // (bit-identical) so the grid agrees on whether selection (and its
  // barriers) runs. Several sequences: each CTA evaluates its own and the
  // barriers run unconditionally.
  double* scratch_d = reinterpret_cast<double*>(sm.scratch);  // the ring may be filling (speculative scan)
  int own = 0;  // 0 no selection, 1 miss (select), 2 hit, 3 zero query
  double own_cos = NAN;
  const bool shard_sel = (pmode & kModeShardSelect) != 0;
  if (sd.select && shard_sel) {
    // decided by the kModeShardStats launch (a zero query there: nothing to select)
    own = __ldcg(&sd.cache->error) ? 3 : __ldcg(&sd.cache->last_hit) == 1 ? 2 : 1;
  } else if (sd.select && (pmode & kModeUseCached)) {
    // the selection was made (or kept) by earlier launches of this step; a
    // query they rejected (zero) appends nothing
    own = __ldcg(&sd.cache->error) ? 3 : 2;
  } else if (sd.select) {
    if (pmode & kModeCache) {
      trace_pt(p, 26);
      const int dec = cache_decision(sd, width, dl, scratch_d, &own_cos);
      own = dec == 1 ? 1 : dec == 0 ? 2 : 3;
    } else {
      own = 1;
    }
  }
  trace_pt(p, 27);
  uint32_t cie = 0, clb = 0;
  if (hit_prep && own == 2) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = tid + u * blockDim.x;
      const bool in = i < n_sel_prev;
      cie += in && selv[u] < ie;
      clb += in && selv[u] < lbs;
    }
    if (!sel_small)
      for (int i = tid + 4 * blockDim.x; i < n_sel_prev; i += blockDim.x) {
        const uint32_t v = __ldcg(sd.sel + i);
        cie += v < ie;
        clb += v < lbs;
      }
  }
  int any_select = 0, any_radix = 0;
  if (n_seq == 1) {
    any_select = own == 1;
    any_radix = do_select && own == 1 && T > p.k;
  } else {
    // (host-computed: a loop over the sequences' descriptors would be a chain
    // of dynamically indexed constant-bank loads)
    any_select = p.any_select;
    any_radix = do_select && p.any_radix;
  }
  if (by_page) {
    if (tid < npg) sm.prefix[tid] = pg_pre;
    __syncthreads();
    const int pm = p.page_size - 1;
    for (int jl = tid; jl < nloc; jl += blockDim.x) {
      const int tok = sd.cand_begin + j0 + jl;
      sm.frames[jl] = (sm.prefix[(tok >> psh) - pg0] << psh) | (tok & pm);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jl = tid + u * blockDim.x;
      if (may_scan && jl < nloc) sm.frames[jl] = fr_pre[u];
    }
    // long ranges (page size 1, > 4 candidates per thread): sixteen page-table
    // loads in flight per thread
    for (int jb = tid + 4 * blockDim.x; may_scan && jb < nloc; jb += 16 * blockDim.x) {
      int32_t fr[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int jl = jb + u * blockDim.x;
        fr[u] = jl < nloc ? static_cast<int32_t>(row_index<LEAN>(sd, cand_at<LEAN>(sd, j0 + jl), p.page_size)) : 0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (jb + u * static_cast<int>(blockDim.x) < nloc) sm.frames[jb + u * blockDim.x] = fr[u];
    }
  }
  if (do_select && own == 1 && T > p.k) {
    uint32_t* gh = p.ws_hist + static_cast<size_t>(seq_id) * 2 * kHistPass;
    for (int i = cs * blockDim.x + tid; i < 2 * kHistPass; i += p.ctas_per_seq * blockDim.x) gh[i] = 0u;
  }
  // zero query (lookup_or_select throws before any mutation,
  // selection_cache.cpp:18-27): the flag is per step, and the step appends
  // nothing and leaves the cache entry untouched
  if (cs == 0 && tid == 0 && sd.select && (pmode & kModeCache)) sd.cache->error = own == 3 ? 1 : 0;
  // append of the current token's row (kv_pool.cpp:55-85), after the decision.
  // This step never reads row N: the candidates end at N - n_local and the
  // current token is attended from k_new / v_new.
  // (an explicit-list attend launch of a sharded step whose stats launch
  // rejected the query appends nothing either)
  const bool rejected = !LEAN && sd.att_list && sd.cache && __ldcg(&sd.cache->error);
  if ((pmode & kModeAppend) && cs == 0 && sd.append_frame >= 0 && own != 3 && !rejected) {
    const int row = p.H_kv * p.d;
    const size_t off = (static_cast<size_t>(sd.append_frame) * p.page_size + sd.append_slot) * row;
    for (int i = tid; i < row; i += blockDim.x) {
      p.k_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(sd.k_new[i]));
      p.v_slab_w[off + i] = __bfloat16_as_ushort(__float2bfloat16_rn(sd.v_new[i]));
    }
    if (tid == 0 && sd.append_page >= 0) sd.page_table[sd.append_page] = sd.append_frame;
  }
  // LEAN miss: S goes to tensor memory (the whole 512 columns; one CTA per SM)
  const bool use_tmem = LEAN && own == 1;
  if (use_tmem && tid < 32) tmem_alloc512(&sm.scratch[kScratchTmem]);
  if (use_tmem) tmem_fence_before_sync();
  __syncthreads();
  uint32_t tbase = 0;
  if (use_tmem) {
    tmem_fence_after_sync();
    tbase = sm.scratch[kScratchTmem];
  }
  // releases the tensor memory (all threads call; uniform)
  bool tmem_held = use_tmem;
  auto tmem_release = [&]() {
    if (!tmem_held) return;
    tmem_fence_before_sync();
    __syncthreads();
    if (tid < 32) {
      tmem_fence_after_sync();
      tmem_dealloc512(tbase);
    }
    tmem_held = false;
  };
#undef TSB_STOP_AT
#define TSB_STOP_AT(n)                                                       \
  if ((!LEAN || TSB_LEAN_DEV) && (p.debug_flags >> 8) == (n)) {              \
    tmem_release();                                                          \
    return;                                                                  \
  }

  TSB_STOP_AT(1);
  trace_pt(p, 1);
  // ---- phase 1: scan (Alg. 2)
  float* Sbuf = s_in_smem == kSSmem ? sm.S : p.ws_s + static_cast<size_t>(cta) * H * p.tpc;  // unused for kSTmem
  uint32_t* keys = s_in_smem != kSGlobal ? sm.keys : p.ws_keys + static_cast<size_t>(cta) * p.tpc;
  const int sstride = p.tpc;
  const bool scanning = (own == 1) && ((pmode & (kModeScore | kModeSIn)) != 0);
  // S spilled to global memory with the soft vote: the scan forms the
  // softmax partials online and the criticality pass reads S once (raw)
  const bool online_z = FAST && !LEAN && s_in_smem == kSGlobal && method == 2 && do_select &&
                        !(pmode & (kModeShardStats | kModeShardSelect | kModeSIn));
  if (scanning) {
    if (pmode & kModeSIn) {
      for (int idx = tid; idx < H * nloc; idx += blockDim.x) {
        const int h = idx / nloc, jl = idx - (idx / nloc) * nloc;
        const float s = sd.s_in[static_cast<size_t>(h) * T + j0 + jl];
        Sbuf[static_cast<size_t>(h) * sstride + jl] = s;
        atomicMax(&sm.headmax[h], float_ord(s));
      }
    } else {
      float* so = (pmode & kModeSOut) ? sd.s_out + j0 : nullptr;
      if (online_z) {  // partials of phases that get no stage stay empty
        float2* zw = reinterpret_cast<float2*>(sm.hist);
        for (int i = tid; i < (kDecodeConsumers / p.H_kv) * H; i += blockDim.x) zw[i] = make_float2(-INFINITY, 0.f);
        __syncthreads();
      }
      if constexpr (FAST)
        scan_fast<D, G, LEAN>(p, sd, sm, j0, nloc, Sbuf, sstride, so, pre, tbase,
                              online_z ? reinterpret_cast<float2*>(sm.hist) : nullptr);
      else scan_generic(p, sd, sm, j0, nloc, Sbuf, sstride, so);
    }
  }
  // S rows are read four candidates at a time: pad each row to a multiple
  // of 4 with -inf (exp -> 0, never selected)
  if (!LEAN && scanning && (nloc & 3))
    for (int i = tid; i < H * 4; i += blockDim.x) {
      const int h = i >> 2, jl = nloc + (i & 3);
      if (jl < ((nloc + 3) & ~3)) Sbuf[static_cast<size_t>(h) * sstride + jl] = -INFINITY;
    }
  __syncthreads();
  trace_pt(p, 2);
  TSB_STOP_AT(2);

  // ---- phase 2: per-CTA softmax partials m = max_j S, z = sum_j e^(S - m) per
  // head (softmax_rows, tensor.cpp:31-52): warp per head, float4 rows, four
  // independent SFU chains per lane
  if (LEAN && own == 1) {
    // S in TMEM: each consumer warp turns its own fragments into e^(S - m_h)
    // (m_h: the CTA's head max from the scan) and sums them per head; the
    // (phase, head) sums meet in shared memory (the idle ring)
    float* wz = reinterpret_cast<float*>(sm.ring);  // [nphase][H]
    const int nph = kDecodeConsumers / p.H_kv;
    const int warp = tid >> 5, lane = tid & 31;
    if (warp >= 1) {
      const int cw = warp - 1, kvh = cw % p.H_kv, ph = cw / p.H_kv;
      const int g0 = (lane & 3) * 2;
      const int h0 = g0 * p.H_kv + kvh, h1 = (g0 + 1) * p.H_kv + kvh;
      const float ml0 = g0 < G ? ord_float(sm.headmax[h0]) * kLog2e : 0.f;
      const float ml1 = g0 + 1 < G ? ord_float(sm.headmax[h1]) * kLog2e : 0.f;
      const int nit = (nloc + 15) >> 4, nr = nit > ph ? (nit - ph + nph - 1) / nph : 0;
      const uint32_t tw = tmem_warp_base(tbase, warp);
      float z0 = 0.f, z1 = 0.f;
      // eight stages per TMEM round trip (the loads' latency, not the math,
      // is this loop's cost)
      if constexpr (G == 4) {
        // four query heads per KV head: the lanes of heads 4..7 (lane & 2)
        // hold no scores, so each takes the upper four stages of its partner
        // lane (lane ^ 2) -- half the exponentials per lane -- and hands the
        // results back for the store (the SFU issue, not the loads, bounds
        // this loop)
        const bool helper = (lane & 2) != 0;
        const float pl0 = __shfl_xor_sync(0xffffffffu, ml0, 2), pl1 = __shfl_xor_sync(0xffffffffu, ml1, 2);
        const float m0 = helper ? pl0 : ml0, m1 = helper ? pl1 : ml1;
#pragma unroll 1
        for (int r0 = 0; r0 < nr; r0 += 8) {
          float v[32];
          tmem_ld32(tw + static_cast<uint32_t>(r0 * 4), v);
          float u[16];  // owner: its stages 0..3; helper: the owner's stages 4..7
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float up = __shfl_xor_sync(0xffffffffu, v[16 + i], 2);
            u[i] = helper ? up : v[i];
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int q = (helper ? 4 : 0) + (i >> 2), e = i & 3;
            const int row = (ph + (r0 + q) * nph) * 16 + (lane >> 2) + (e >> 1) * 8;
            const bool ok = r0 + q < nr && row < nloc;
            const float w = ok ? ex2_approx(fmaf(u[i], kLog2e, -((e & 1) ? m1 : m0))) : 0.f;
            u[i] = w;
            if (e & 1) z1 += w;
            else z0 += w;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float back = __shfl_xor_sync(0xffffffffu, u[i], 2);
            v[i] = helper ? 0.f : u[i];
            v[16 + i] = helper ? 0.f : back;
          }
          tmem_st32(tw + static_cast<uint32_t>(r0 * 4), v);
        }
        // the helpers' sums belong to their owners' heads
        const float hz0 = __shfl_xor_sync(0xffffffffu, z0, 2), hz1 = __shfl_xor_sync(0xffffffffu, z1, 2);
        if (!helper) {
          z0 += hz0;
          z1 += hz1;
        } else {
          z0 = 0.f;
          z1 = 0.f;
        }
      } else {
#pragma unroll 1
        for (int r0 = 0; r0 < nr; r0 += 8) {
          float v[32];
          tmem_ld32(tw + static_cast<uint32_t>(r0 * 4), v);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int rbase = (ph + (r0 + q) * nph) * 16 + (lane >> 2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int g = g0 + (e & 1), row = rbase + (e >> 1) * 8;
              const bool ok = r0 + q < nr && g < G && row < nloc;
              const float w = ok ? ex2_approx(fmaf(v[q * 4 + e], kLog2e, -((e & 1) ? ml1 : ml0))) : 0.f;
              v[q * 4 + e] = w;
              if (e & 1) z1 += w;
              else z0 += w;
            }
          }
          tmem_st32(tw + static_cast<uint32_t>(r0 * 4), v);
        }
      }
      tmem_wait_st();
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        z0 += __shfl_xor_sync(0xffffffffu, z0, o);
        z1 += __shfl_xor_sync(0xffffffffu, z1, o);
      }
      if (lane < 4) {
        if (g0 < G) wz[ph * H + h0] = z0;
        if (g0 + 1 < G) wz[ph * H + h1] = z1;
      }
    }
    __syncthreads();
    const size_t sh = stats_stride(p.ctas_per_seq);
    const size_t so = static_cast<size_t>(seq_id) * H * sh + cs;
    for (int h = tid; h < H; h += blockDim.x) {
      float z = 0.f;
      for (int q = 0; q < nph; ++q) z += wz[q * H + h];  // fixed order
      p.ws_m[so + h * sh] = ord_float(sm.headmax[h]);
      p.ws_z[so + h * sh] = z;
    }
  } else if (do_select && own == 1 && method == 2 && !shard_sel) {
    const size_t sh = stats_stride(p.ctas_per_seq);
    const size_t so = static_cast<size_t>(seq_id) * H * sh + cs;
    if (online_z) {
      // the consumer warps' (m, z) per head, merged in phase order
      __syncthreads();
      const float2* zw = reinterpret_cast<const float2*>(sm.hist);
      const int nph = kDecodeConsumers / p.H_kv;
      for (int h = tid; h < H; h += blockDim.x) {
        float zm = -INFINITY, zz = 0.f;
        for (int q = 0; q < nph; ++q) {
          const float2 w = zw[q * H + h];
          const float mx = fmaxf(zm, w.x);
          if (mx > -INFINITY) {
            zz = (zm > -INFINITY ? zz * ex2_approx(zm - mx) : 0.f) + (w.x > -INFINITY ? w.y * ex2_approx(w.x - mx) : 0.f);
            zm = mx;
          }
        }
        p.ws_m[so + h * sh] = zm * kLn2;  // natural-log domain, like the other paths
        p.ws_z[so + h * sh] = zz;
      }
    } else {
      softmax_partials(Sbuf, sstride, nloc, H, sm.headmax, p.ws_m + so, p.ws_z + so, sh);
    }
  }
  TSB_STOP_AT(3);
  trace_pt(p, 3);
  if (any_select) gs.sync();  // B1: softmax partials of every CTA visible
  TSB_STOP_AT(4);
  trace_pt(p, 4);


  // ---- phase 3: criticality (soft vote / raw sum) + cache bookkeeping
  if (cs == 0 && tid == 0 && (pmode & kModeCache) && (own == 1 || own == 2)) {
    CacheState* c = sd.cache;
    c->lookups += 1;
    if (own == 2) c->hits += 1;
    else c->first_flag = 0;
    c->last_hit = own == 2 ? 1 : 0;
    c->last_cos = own_cos;
  }
  if (own == 1 && (pmode & kModeCache)) {
    // the new cached query (every CTA read the old one before B1)
    const uint64_t pol = policy_evict_last();
    for (int i = cs * blockDim.x + tid; i < width; i += p.ctas_per_seq * blockDim.x)
      st_hint_u32(sd.cached_q + i, __float_as_uint(sd.q[i]), pol);
  }
  if (pmode & kModeShardStats) {
    // this shard's per-head (m, z) from its CTAs' partials (every CTA
    // finished phase 2 at B1); S = e^(S - m_c) stays in the spill buffer
    // One warp per head, the CTAs' partials strided over the lanes (all loads
    // in flight; a thread walking them one by one spent ~130 us in L2
    // round trips). Fixed order: lane-ordered partial sums, then a butterfly.
    if (own == 1 && cs == 0 && method == 2) {
      const size_t sh = stats_stride(p.ctas_per_seq);
      const int lane = tid & 31, nw = static_cast<int>(blockDim.x >> 5);
      for (int h = tid >> 5; h < H; h += nw) {
        const float* mr = p.ws_m + (static_cast<size_t>(seq_id) * H + h) * sh;
        const float* zr = p.ws_z + (static_cast<size_t>(seq_id) * H + h) * sh;
        constexpr int kPer = (kMaxPrefix + 31) / 32;
        float mv[kPer], zv[kPer];
        float M = -INFINITY;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int c = lane + 32 * j;
          const bool ok = c < p.ctas_per_seq;
          mv[j] = ok ? __ldcg(mr + c) : -INFINITY;
          zv[j] = ok ? __ldcg(zr + c) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) M = fmaxf(M, mv[j]);
        M = warp_max(M);
        float Z = 0.f;
        if (M > -INFINITY) {
#pragma unroll
          for (int j = 0; j < kPer; ++j)
            if (mv[j] > -INFINITY) Z += zv[j] * expf(mv[j] - M);
        }
        Z = warp_sum(Z);
        if (lane == 0) {
          sd.shard_stats[h * 2 + 0] = M;
          sd.shard_stats[h * 2 + 1] = Z;
        }
      }
    } else if (cs == 0) {
      // no fresh statistics this step (a hit, or another method): all-ones
      // bits (NaN) mark them unset for the other ranks
      for (int i = tid; i < 2 * H; i += blockDim.x) reinterpret_cast<uint32_t*>(sd.shard_stats)[i] = 0xffffffffu;
    }
    return;
  }
  const bool radix_own = do_select && own == 1 && T > p.k;
  if (do_select && own == 1) {
    float* ml = sm.f;                                   // [H] f_h = e^(m_c - M_h) / Z_h
    if (method == 2 && shard_sel) {
      // global softmax stats from every shard's (m, z) (rank order); m_c of
      // this CTA from its partial of the stats launch
      const size_t sh = stats_stride(p.ctas_per_seq);
      for (int h = tid; h < H; h += blockDim.x) {
        const float mc = __ldcg(p.ws_m + (static_cast<size_t>(seq_id) * H + h) * sh + cs);
        // ranks' (m, z) pairs 8 at a time (loads in flight), merged in rank order
        constexpr int kR = 8;
        const float2* all = reinterpret_cast<const float2*>(sd.shard_all);
        float M = -INFINITY, Z = 0.f;
#pragma unroll 1
        for (int r0 = 0; r0 < sd.shard_world; r0 += kR) {
          float2 v[kR];
#pragma unroll
          for (int j = 0; j < kR; ++j)
            v[j] = r0 + j < sd.shard_world ? __ldcg(all + (r0 + j) * H + h) : make_float2(-INFINITY, 0.f);
          float Mn = M;
#pragma unroll
          for (int j = 0; j < kR; ++j) Mn = fmaxf(Mn, v[j].x);
          if (Mn > -INFINITY) {
            Z = M > -INFINITY ? Z * expf(M - Mn) : 0.f;
#pragma unroll
            for (int j = 0; j < kR; ++j)
              if (v[j].x > -INFINITY) Z += v[j].y * expf(v[j].x - Mn);
          }
          M = Mn;
        }
        ml[h] = mc > -INFINITY ? fast_exp(mc - M) / Z : 0.f;
      }
      __syncthreads();
    } else if (method == 2) {
      float* pm = reinterpret_cast<float*>(sm.ring);
      const int nc = p.ctas_per_seq;
      const int ncp = stats_stride(nc);
      const size_t sbytes = static_cast<size_t>(H) * ncp * 4;
      if (tid == 0) {
        mbar_arrive_expect_tx(sm.aux, static_cast<uint32_t>(2 * sbytes));
        bulk_g2s_nohint(pm, p.ws_m + static_cast<size_t>(seq_id) * H * ncp, static_cast<uint32_t>(sbytes), sm.aux);
        bulk_g2s_nohint(pm + H * ncp, p.ws_z + static_cast<size_t>(seq_id) * H * ncp, static_cast<uint32_t>(sbytes), sm.aux);
      }
      const float* pz = pm + H * ncp;
      mbar_wait(sm.aux, aux_phase);
      aux_phase ^= 1u;
      trace_pt(p, 13);
      // M_h = max_c m_c, Z_h = sum_c z_c e^(m_c - M_h): 16 threads per head,
      // a thread's partials (c = sub, sub + 16, ...) loaded together
      const int sub = tid & 15;
      constexpr int kPerS = kMaxPrefix / 16;
      for (int h0 = 0; h0 < H; h0 += blockDim.x >> 4) {  // warp-uniform trip count
        const int h = h0 + (tid >> 4);
        const bool hv = h < H;
        float M = -INFINITY, Z = 0.f;
        if constexpr (LEAN) {  // (a whole-GPU launch: ~10 partials per thread)
          float mv[kPerS], zv[kPerS];
#pragma unroll
          for (int j = 0; j < kPerS; ++j) {
            const int c = sub + 16 * j;
            const bool ok = hv && c < nc;
            mv[j] = ok ? pm[h * ncp + c] : -INFINITY;
            zv[j] = ok ? pz[h * ncp + c] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < kPerS; ++j) M = fmaxf(M, mv[j]);
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
#pragma unroll
          for (int j = 0; j < kPerS; ++j)
            if (mv[j] > -INFINITY) Z += zv[j] * fast_exp(mv[j] - M);
        } else {  // (batched launches: a few CTAs per sequence)
          if (hv)
            #pragma unroll 1
            for (int c = sub; c < nc; c += 16) M = fmaxf(M, pm[h * ncp + c]);
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
          if (hv)
            #pragma unroll 1
            for (int c = sub; c < nc; c += 16) {
              const float mc = pm[h * ncp + c];
              if (mc > -INFINITY) Z += pz[h * ncp + c] * fast_exp(mc - M);
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
        if (hv && sub == 0) {
          if (online_z) {
            // raw S: softmax_h(S) = 2^(S log2e - M_h log2e) / Z_h (the shift
            // kept in the head-max slot, which nothing reads past this point)
            ml[h] = Z > 0.f ? 1.f / Z : 0.f;
            reinterpret_cast<float*>(sm.headmax)[h] = M > -INFINITY ? M * kLog2e : 0.f;
          } else {
            const float mc = ord_float(sm.headmax[h]);
            ml[h] = mc > -INFINITY ? fast_exp(mc - M) / Z : 0.f;  // f_h: local e^(S - m_c) -> softmax
          }
        }
      }
      __syncthreads();
      trace_pt(p, 14);
    }
    if (radix_own) {
      for (int i = tid; i < kRadixBins; i += blockDim.x) sm.hist[i] = 0u;
      __syncthreads();
    }
    stamp(trc, 32);
    // crit[j] = sum_h softmax_h(S)[j] (select_head_soft_vote, selector.cpp:113-126)
    // = sum_h e^(S - m_c) f_h, or the raw logit sum (select_topk,
    // selector.cpp:89-99); two candidates per thread, keys straight into the
    // pass-1 histogram
    if constexpr (LEAN) {
      // S in TMEM: each consumer warp forms its rows' partial over its kv
      // head's query heads (sum_g e f_h), the four lanes of a row add up, and
      // the H_kv partials meet in shared memory (after the radix histogram
      // in the idle ring); then one pass per candidate in a fixed order
      float* cpart = reinterpret_cast<float*>(sm.ring + kCritPartOffset);  // [H_kv][tpc]
      const int nph = kDecodeConsumers / p.H_kv;
      const int warp = tid >> 5, lane = tid & 31;
      if (warp >= 1) {
        const int cw = warp - 1, kvh = cw % p.H_kv, ph = cw / p.H_kv;
        const int g0 = (lane & 3) * 2;
        const float f0 = g0 < G ? ml[g0 * p.H_kv + kvh] : 0.f;
        const float f1 = g0 + 1 < G ? ml[(g0 + 1) * p.H_kv + kvh] : 0.f;
        const int nit = (nloc + 15) >> 4, nr = nit > ph ? (nit - ph + nph - 1) / nph : 0;
        const uint32_t tw = tmem_warp_base(tbase, warp);
        float* cp = cpart + kvh * p.tpc;
        // eight stages per TMEM round trip; the 16 (stage, row half) sums of
        // a row quad meet by a transposing reduction over lanes ^1 and ^2
        // (12 shuffles), after which lane b + 2c of the quad holds the sums
        // of x[8b + 4c .. 8b + 4c + 3]
        const int b1 = lane & 1, c1 = (lane >> 1) & 1;
#pragma unroll 1
        for (int r0 = 0; r0 < nr; r0 += 8) {
          float v[32];
          tmem_ld32(tw + static_cast<uint32_t>(r0 * 4), v);
          float x[16];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            x[2 * q] = fmaf(v[q * 4 + 1], f1, v[q * 4 + 0] * f0);      // row lane/4
            x[2 * q + 1] = fmaf(v[q * 4 + 3], f1, v[q * 4 + 2] * f0);  // row lane/4 + 8
          }
          float y[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float send = b1 ? x[i] : x[i + 8];
            y[i] = (b1 ? x[i + 8] : x[i]) + __shfl_xor_sync(0xffffffffu, send, 1);
          }
          float z[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float send = c1 ? y[i] : y[i + 4];
            z[i] = (c1 ? y[i + 4] : y[i]) + __shfl_xor_sync(0xffffffffu, send, 2);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int idx = 8 * b1 + 4 * c1 + i, q = idx >> 1;
            const int row = (ph + (r0 + q) * nph) * 16 + (lane >> 2) + (idx & 1) * 8;
            if (r0 + q < nr && row < nloc) cp[row] = z[i];
          }
        }
      }
      tmem_release();  // (its barrier also publishes cpart)
      stamp(trc, 48);
      for (int base = 0; base < nloc; base += blockDim.x) {
        const int jl = base + tid;
        float c = 0.f;
        if (jl < nloc)
          for (int g = 0; g < p.H_kv; ++g) c += cpart[g * p.tpc + jl];
        const uint32_t key = float_key(c);
        if (jl < nloc) keys[jl] = key;
        if (radix_own) hist_add(sm.hist, key, jl < nloc, 20);
      }
      stamp(trc, 49);
    } else if (online_z) {
      // raw S (spilled): crit_j = sum_h 2^(S_hj log2e - M_h log2e) / Z_h, even
      // heads then odd into separate sums, each in head order
      const float* shift = reinterpret_cast<const float*>(sm.headmax);
      const int n2 = (nloc + 1) >> 1;
      const int hp = H & ~1;
      for (int base = 0; base < n2; base += blockDim.x) {
        const int q = base + tid;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        if (q < n2) {
          const float* s2 = Sbuf + 2 * q;
          int h = 0;
          for (; h < hp; h += 16) {
            float2 a[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
              if (h + u < hp) a[u] = *reinterpret_cast<const float2*>(s2 + static_cast<size_t>(h + u) * sstride);
#pragma unroll
            for (int u = 0; u < 16; u += 2)
              if (h + u < hp) {
                const float sa = shift[h + u], sb = shift[h + u + 1], fa = ml[h + u], fb = ml[h + u + 1];
                c0 = fmaf(ex2_approx(fmaf(a[u].x, kLog2e, -sa)), fa, c0);
                c1 = fmaf(ex2_approx(fmaf(a[u].y, kLog2e, -sa)), fa, c1);
                c2 = fmaf(ex2_approx(fmaf(a[u + 1].x, kLog2e, -sb)), fb, c2);
                c3 = fmaf(ex2_approx(fmaf(a[u + 1].y, kLog2e, -sb)), fb, c3);
              }
          }
          h = hp;
          if (h < H) {
            const float2 a = *reinterpret_cast<const float2*>(s2 + static_cast<size_t>(h) * sstride);
            c0 = fmaf(ex2_approx(fmaf(a.x, kLog2e, -shift[h])), ml[h], c0);
            c1 = fmaf(ex2_approx(fmaf(a.y, kLog2e, -shift[h])), ml[h], c1);
          }
        }
        const uint32_t k0 = float_key(c0 + c2), k1 = float_key(c1 + c3);
        if (q < n2) *reinterpret_cast<uint2*>(keys + 2 * q) = make_uint2(k0, k1);
        if (radix_own) {
          hist_add(sm.hist, k0, q < n2 && 2 * q < nloc, 20);
          hist_add(sm.hist, k1, q < n2 && 2 * q + 1 < nloc, 20);
        }
      }
    } else {
      const int n2 = (nloc + 1) >> 1;
      const bool soft = method == 2;
      for (int base = 0; base < n2; base += blockDim.x) {
        const int q = base + tid;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        if (q < n2) {
          const float* s2 = Sbuf + 2 * q;
          int h = 0;
          // sixteen heads' loads in flight (S may be spilled to global
          // memory: each round is an L2 / HBM round trip); even heads into
          // c0 / c1, odd heads into c2 / c3, each in head order
          const int hp = H & ~1;  // the heads taken in pairs
          for (; h < hp; h += 16) {
            float2 a[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
              if (h + u < hp) a[u] = *reinterpret_cast<const float2*>(s2 + static_cast<size_t>(h + u) * sstride);
#pragma unroll
            for (int u = 0; u < 16; u += 2)
              if (h + u < hp) {
                const float fa = soft ? ml[h + u] : 1.f, fb = soft ? ml[h + u + 1] : 1.f;
                c0 = fmaf(a[u].x, fa, c0);
                c1 = fmaf(a[u].y, fa, c1);
                c2 = fmaf(a[u + 1].x, fb, c2);
                c3 = fmaf(a[u + 1].y, fb, c3);
              }
          }
          h = hp;
          if (h < H) {
            const float2 a = *reinterpret_cast<const float2*>(s2 + static_cast<size_t>(h) * sstride);
            const float fa = soft ? ml[h] : 1.f;
            c0 = fmaf(a.x, fa, c0);
            c1 = fmaf(a.y, fa, c1);
          }
        }
        const uint32_t k0 = float_key(c0 + c2), k1 = float_key(c1 + c3);
        if (q < n2) *reinterpret_cast<uint2*>(keys + 2 * q) = make_uint2(k0, k1);
        if (radix_own) {
          hist_add(sm.hist, k0, q < n2 && 2 * q < nloc, 20);
          hist_add(sm.hist, k1, q < n2 && 2 * q + 1 < nloc, 20);
        }
      }
      }
    __syncthreads();
  }
  TSB_STOP_AT(5);
  trace_pt(p, 5);

  // ---- phase 4: radix select over 24-bit key prefixes (two 12-bit passes).
  // Larger criticality first; keys equal in their top 24 bits (relative
  // difference < 2^-15) rank as ties, which go to the smaller position
  // (tensor.cpp:81-88).
  uint32_t tau = 0, take_eq_all = 1;
  uint32_t kk = static_cast<uint32_t>(p.k);
  if (any_radix) {
    uint32_t* gh = p.ws_hist + static_cast<size_t>(seq_id) * 2 * kHistPass;
    if (radix_own) hist_merge(sm.hist, gh);
    trace_pt(p, 15);
    gs.sync();  // B2
    TSB_STOP_AT(6);
    trace_pt(p, 6);
    uint32_t b1 = 0;
    if (radix_own) {
      int b;
      uint32_t above;
      uint32_t cnt;
      find_bin(gh, kk, sm.scratch, sm.hist, &b, &above, &cnt, trc, 33);
      kk -= above;
      b1 = static_cast<uint32_t>(b);
      trace_pt(p, 16);
      radix_hist(keys, nloc, 8, 20, b1, sm.hist, gh + kHistPass, trc);
    }
    TSB_STOP_AT(7);
    trace_pt(p, 17);
    gs.sync();  // B3
    TSB_STOP_AT(8);
    trace_pt(p, 7);

    uint32_t eq_total = 0;
    if (radix_own) {
      int b;
      uint32_t above;
      find_bin(gh + kHistPass, kk, sm.scratch, sm.hist, &b, &above, &eq_total, trc, 36);
      kk -= above;
      tau = (b1 << 12) | static_cast<uint32_t>(b);
    }
    trace_pt(p, 18);
    // ties straddling the budget: the taken ones are the lowest positions,
    // which needs every CTA's tie count (one more exchange)
    int need_tie = 0;
    if (n_seq == 1) need_tie = radix_own && eq_total > kk;
    else need_tie = 1;
    if (need_tie) {
      if (radix_own) {
        uint32_t neq = 0;
        for (int jl = tid; jl < nloc; jl += blockDim.x) neq += (keys[jl] >> 8) == tau;
        uint32_t tot;
        block_excl_scan(neq, sm.scratch, &tot);
        if (tid == 0) p.ws_cnt[cta] = tot;
      }
      gs.sync();  // B3b
      if (radix_own && eq_total > kk) {
        uint32_t pre = 0;
        if (tid < 32) {
#pragma unroll 1
          for (int c = tid; c < cs; c += 32) pre += __ldcg(p.ws_cnt + c0 + c);
          pre = __reduce_add_sync(0xffffffffu, pre);
          if (tid == 0) sm.scratch[70] = pre;
        }
        __syncthreads();
        pre = sm.scratch[70];
        __syncthreads();
        take_eq_all = 0;
        kk = kk > pre ? kk - pre : 0u;  // ties this CTA may still take
      }
    }
  }

  trace_pt(p, 19);
  // ---- phase 5: ascending compaction of this CTA's selected candidates
  // up to two compacted entries per thread stay in registers for the
  // SelectionResult write after the offsets are known (no read back)
  const bool pub_regs = nloc <= 2 * static_cast<int>(blockDim.x);
  uint32_t pub_pos[2] = {0xffffffffu, 0xffffffffu}, pub_tok[2] = {0u, 0u};
  float pub_crit[2] = {0.f, 0.f};
  int32_t pub_row[2] = {-1, -1};
  if (do_select && own == 1) {
    uint32_t out_n = 0, eq_seen = 0;
    uint32_t* lt = p.ws_sel_tok + static_cast<size_t>(cta) * p.tpc;
    float* lc = p.ws_sel_crit + static_cast<size_t>(cta) * p.tpc;
    int32_t* lr = p.ws_sel_row + static_cast<size_t>(cta) * p.tpc;
    for (int base = 0; base < nloc; base += blockDim.x) {
      const int jl = base + tid;
      const uint32_t key = jl < nloc ? keys[jl] : 0u;
      bool take = jl < nloc;
      if (radix_own && take) {
        const uint32_t k24 = key >> 8;
        take = k24 > tau || (k24 == tau && take_eq_all);
      }
      if (radix_own && !take_eq_all) {
        const uint32_t is_eq = (jl < nloc && (key >> 8) == tau) ? 1u : 0u;
        uint32_t eq_tot;
        const uint32_t r = eq_seen + block_excl_scan(is_eq, sm.scratch, &eq_tot);
        if (is_eq && r < kk) take = true;
        eq_seen += eq_tot;
      }
      uint32_t tot;
      const uint32_t pos = out_n + block_excl_scan(take ? 1u : 0u, sm.scratch, &tot);
      if (take) {
        const int32_t row = may_scan ? sm.frames[jl] : -1;
        const uint32_t tok = cand_at<LEAN>(sd, j0 + jl) + (LEAN ? 0u : static_cast<uint32_t>(sd.shard_base));
        const float cr = key_float(key);
        lt[pos] = tok;
        lc[pos] = cr;
        lr[pos] = row;
        if (pub_regs) {
          const int u = base == 0 ? 0 : 1;
          pub_pos[u] = pos;
          pub_tok[u] = tok;
          pub_crit[u] = cr;
          pub_row[u] = row;
        }
        if (FAST && (pmode & kModeAttend) && row >= 0) {
          // the attention CTAs gather this row after B4: pull it into L2 now
          const uint32_t rb = static_cast<uint32_t>(p.H_kv * p.d * 2);
          const uint64_t pol = policy_evict_last();
          bulk_prefetch_l2(reinterpret_cast<const char*>(p.k_slab) + static_cast<size_t>(row) * rb, rb, pol);
          bulk_prefetch_l2(reinterpret_cast<const char*>(p.v_slab) + static_cast<size_t>(row) * rb, rb, pol);
        }
      }
      out_n += tot;
      stamp(trc, 40);
    }
    if (tid == 0) p.ws_nsel[cta] = out_n;
  }
  TSB_STOP_AT(9);
  trace_pt(p, 8);
  if (any_select) gs.sync();  // B4: per-CTA selections published
  TSB_STOP_AT(10);
  trace_pt(p, 9);

  // ---- phase 6: selection offsets; the SelectionResult (ascending) out
  if (do_select && own == 1) {
    const int nc = p.ctas_per_seq;
    const uint32_t v = tid < nc ? __ldcg(p.ws_nsel + c0 + tid) : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, sm.scratch, &tot);
    if (tid <= nc) sm.prefix[tid] = static_cast<int>(tid < nc ? ex : tot);
    __syncthreads();
    stamp(trc, 41);
    const int my0 = sm.prefix[cs], myn = sm.prefix[cs + 1] - my0;
    const uint32_t* lt = p.ws_sel_tok + static_cast<size_t>(cta) * p.tpc;
    const float* lc = p.ws_sel_crit + static_cast<size_t>(cta) * p.tpc;
    if (cs == 0 && tid == 0) sd.cache->n_sel = static_cast<int>(tot);
    if (shard_sel) {
      for (int i = tid; i < myn; i += blockDim.x) {
        sd.shard_cands[my0 + i] = __ldcg(lt + i);
        sd.shard_cands[p.k + my0 + i] = float_key(__ldcg(lc + i));
      }
      if (cs == 0 && tid == 0) sd.shard_cands[2 * p.k] = tot;
    }
  }
  if (shard_sel && own == 2 && cs == 0) {
    // Selection Cache hit: this shard's cached candidates, with their keys
    const int n = __ldcg(&sd.cache->n_sel);
    for (int i = tid; i < n; i += blockDim.x) {
      sd.shard_cands[i] = __ldcg(sd.sel + i);
      sd.shard_cands[p.k + i] = float_key(__ldcg(sd.sel_crit + i));
    }
    if (tid == 0) sd.shard_cands[2 * p.k] = static_cast<uint32_t>(n);
  }
  TSB_STOP_AT(11);
  trace_pt(p, 10);
  // the SelectionResult (ascending) into the cache entry, evict_last: the
  // next launch stages it. Nobody reads it in this launch, so the stores are
  // fire-and-forget (from registers; read back only for large CTA lists).
  if (do_select && own == 1) {
    const int my0 = sm.prefix[cs];
    const uint64_t pol = policy_evict_last();
    if (pub_regs) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (pub_pos[u] != 0xffffffffu) {
          const int i = my0 + static_cast<int>(pub_pos[u]);
          st_hint_u32(sd.sel + i, pub_tok[u], pol);
          st_hint_u32(sd.sel_crit + i, __float_as_uint(pub_crit[u]), pol);
          if (LEAN || sd.sel_rows) st_hint_u32(sd.sel_rows + i, static_cast<uint32_t>(pub_row[u]), pol);
        }
    } else {
      const int myn = sm.prefix[cs + 1] - my0;
      const uint32_t* lt = p.ws_sel_tok + static_cast<size_t>(cta) * p.tpc;
      const float* lc = p.ws_sel_crit + static_cast<size_t>(cta) * p.tpc;
      const int32_t* lr = p.ws_sel_row + static_cast<size_t>(cta) * p.tpc;
      for (int i = tid; i < myn; i += blockDim.x) {
        st_hint_u32(sd.sel + my0 + i, __ldcg(lt + i), pol);
        st_hint_u32(sd.sel_crit + my0 + i, __float_as_uint(__ldcg(lc + i)), pol);
        if (LEAN || sd.sel_rows) st_hint_u32(sd.sel_rows + my0 + i, static_cast<uint32_t>(__ldcg(lr + i)), pol);
      }
    }
  }
  if (!(pmode & kModeAttend)) return;

  // ---- phase 7: split-K sparse flash-decoding (KV head x row chunk)
  AttView av{};
  if (!LEAN && sd.att_list) {
    av.n_rows = sd.n_att_dev ? __ldcg(sd.n_att_dev) : sd.n_att;
  } else {
    av.init_end = sd.init_end;
    av.lb = static_cast<int>(lbs);
    if (own == 1) {
      av.fresh = 1;
      av.n1 = sm.prefix[p.ctas_per_seq];
      av.ncta = p.ctas_per_seq;
      av.cta0 = c0;
    } else if (own == 2) {
      uint32_t tie, tlb;
      if (p.k < 65536) {  // both counts in one reduction
        uint32_t tot;
        block_excl_scan(cie | (clb << 16), sm.scratch, &tot);
        tie = tot & 0xffffu;
        tlb = tot >> 16;
      } else {
        block_excl_scan(cie, sm.scratch, &tie);
        block_excl_scan(clb, sm.scratch, &tlb);
      }
      av.lo1 = static_cast<int>(tie);
      av.n1 = max(0, static_cast<int>(tlb) - static_cast<int>(tie));
    }

    av.n_rows = sd.init_end + av.n1 + (sd.n_cached - av.lb);
  }
  const AttSplit split = att_split(p.H_kv, p.ctas_per_seq);
  const int gi = cs % split.groups, ci = cs / split.groups;
  if (ci < split.chunks) {
    const int total_rows = av.n_rows + ((!LEAN && sd.no_cur) ? 0 : 1);  // + current token
    const int per = max(1, (total_rows + split.chunks - 1) / split.chunks);
    const int r0 = min(total_rows, ci * per);
    const int r1 = min(total_rows, r0 + per);
    const bool with_cur = !(!LEAN && sd.no_cur) && (r0 < r1) && (r1 == total_rows);
    const int Gq = p.H / p.H_kv;
    const int stride = att_stride(p.d);
    for (int g = gi; g < p.H_kv; g += split.groups) {
      float* parts = p.ws_att + (static_cast<size_t>(seq_id) * p.H_kv + g) * split.chunks * Gq * stride;
      if constexpr (FAST) {
        attend_group_mma<D, LEAN>(p, sd, av, sm, g, r0, min(r1, av.n_rows), with_cur,
                            parts + static_cast<size_t>(ci) * Gq * stride);
      }
      else
        attend_group<0, 0>(p, sd, av, sm, g, r0, min(r1, av.n_rows), with_cur,
                           parts + static_cast<size_t>(ci) * Gq * stride);
      TSB_STOP_AT(12);
      trace_pt(p, 11);
      // the group's chunks wait for each other (all co-resident), then each
      // merges its slice of the outputs (no grid barrier). Measured: this
      // beats the last chunk merging all G*d outputs alone by ~5 us.
      __syncthreads();
      if (tid == 0) {
        unsigned int* ctr = p.ws_acnt + (p.bar_slot ? kMaxSeqPerLaunch * p.H_kv : 0) + seq_id * p.H_kv + g;
        red_release_add_u32(ctr, 1u);
        while (ld_acquire_u32(ctr) < static_cast<unsigned int>(split.chunks)) {
        }
      }
      __syncthreads();
      TSB_STOP_AT(13);
      trace_pt(p, 28);
      {
        const int n_out = Gq * p.d, per = (n_out + split.chunks - 1) / split.chunks;
        const int o0 = min(n_out, ci * per);
        merge_outputs<LEAN>(p, sd, g, parts, split.chunks, o0, min(n_out, o0 + per) - o0,
                      reinterpret_cast<float*>(sm.ring));
      }
      trace_pt(p, 31);
    }
  }
  // the cache entry for the host (every field this launch changes was written
  // by this thread: error, the lookup bookkeeping, n_sel)
  if (sd.cache_mirror && cs == 0 && tid == 0) *sd.cache_mirror = *sd.cache;
  trace_pt(p, 12);
}

}  // namespace

const void* decode_kernel_ptr(int D, int G, bool fast, int variant) {
#define TSB_K(d, g)                                                                                 \
  return variant == 1   ? reinterpret_cast<const void*>(&decode_kernel<d, g, true, kLeanMode>)     \
         : variant == 2 ? reinterpret_cast<const void*>(&decode_kernel<d, g, true, kLeanSelMode>)  \
                        : reinterpret_cast<const void*>(&decode_kernel<d, g, true, 0>)
  if (fast) {
    if (D == 128) {
      switch (G) {
        case 1: TSB_K(128, 1);
        case 2: TSB_K(128, 2);
        case 4: TSB_K(128, 4);
        case 7: TSB_K(128, 7);
        case 8: TSB_K(128, 8);
      }
    }
    if (D == 64) {
      switch (G) {
        case 1: TSB_K(64, 1);
        case 2: TSB_K(64, 2);
        case 4: TSB_K(64, 4);
        case 8: TSB_K(64, 8);
      }
    }
    return nullptr;
  }
#undef TSB_K
  if (variant) return nullptr;  // the LEAN specialisations exist for the tensor-core path only
  return reinterpret_cast<const void*>(&decode_kernel<0, 0, false, 0>);
}

}  // namespace tsb

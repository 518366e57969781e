// Chunked-prefill sparse attention on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in tensor memory): the C-row case of
// sparse_attend (attention.cpp:114-123 -> sdpa_full :54-112) for head_dim
// 128 and G = H / H_kv in {1, 2, 4, 8}.
//
// One CTA = 128 query rows = the G query heads of KV head g (h mod H_kv,
// :78) x 128 / G chunk rows; grid = (C / (128 / G), H_kv). Keys come in
// tiles of 64: the merged cached rows (init U selected U local, gathered
// through the page table) and then the chunk's own rows, causal (:83).
//
//   S = Q K^T     tcgen05.mma kind::f16, M = 128, N = 64, K = 128 (8 steps),
//                 A = Q (smem, K-major SW128), B = K (smem, K-major SW128),
//                 D = S in TMEM (64 columns). Q (fp32) is split exactly into
//                 three bf16 parts; cached K is bf16 (exact); the chunk's own
//                 K (fp32 in the reference) is split into three parts as well
//                 (loaded one part at a time), so every product is exact and
//                 only the fp32 summation order differs from the reference.
//   softmax       thread = query row = TMEM lane: tcgen05.ld of its 64 scores,
//                 mask, online softmax in the exp2 domain with a lazily moved
//                 reference max (O and l are rescaled only when the max grows
//                 by more than 2^8), P split into three bf16 parts -> smem
//   O += P V      tcgen05.mma M = 128, N = 128, K = 64 (4 steps),
//                 A = P (smem, K-major SW128), B = V (smem, MN-major SW128),
//                 D = O in TMEM (128 columns)
//
// The tile's K/V rows arrive by 16-byte cp.async written straight into the
// 128B-swizzled layouts the UMMA descriptors describe; the next cached tile's
// gather is in flight while the current one is computed. Thread 0 issues
// every MMA (tcgen05.commit -> mbarrier).
#include <cfloat>
#include <cmath>

#include "aux.h"
#include "common.cuh"

namespace tsb {

namespace {

constexpr int kD = 128;
constexpr int kM = 128;          // query rows per CTA (UMMA M)
constexpr int kKT = 64;          // keys per tile (UMMA N of S, K of P.V)
constexpr int kThr = 384;        // 8 softmax warps, 1 MMA warp, 3 producer warps
constexpr int kSmThr = 256;      // softmax threads (two per query row)
constexpr int kProdThr = 96;     // producer threads (warps 9-11)
constexpr int kRowsUpFront = 4096;
constexpr float kLog2e = 1.4426950408889634f;

// shared memory (bytes), every operand region 1024-B aligned
constexpr int kQPart = kM * kD * 2;    // 32 KB per Q part: [2 atoms][128 rows][128 B]
constexpr int kKVTile = kKT * kD * 2;  // 16 KB: [2 atoms][64 rows][128 B]
constexpr int kPPart = kM * kKT * 2;   // 16 KB per P part: [128 rows][128 B]
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + 3 * kQPart;        // 2 buffers of K
constexpr int kOffV = kOffK + 2 * kKVTile;       // 2 buffers of V
constexpr int kOffP = kOffV + 2 * kKVTile;       // 3 P parts
constexpr int kOffRows = kOffP + 3 * kPPart;     // slab rows of the cached keys
constexpr int kOffBar = kOffRows + kRowsUpFront * 4;
constexpr int kOffRed = kOffBar + 256;              // [2 tiles][2 halves][128] row-max / row-sum exchange
constexpr int kSmem = kOffRed + 4 * kM * 4;

__device__ __forceinline__ uint16_t bfb(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
// x = h + m + l exactly: h = x truncated to bf16 (8 significant bits), the
// residual r = x - h is exact in fp32 and has at most 16 significant bits,
// m = r truncated, l = r - m has at most 8 -- every part is a bf16 value
// (its fp32 bits end in 16 zeros). Bit masks and two FADDs: no conversion
// instructions on the quarter-rate pipe.
__device__ __forceinline__ void sp3(float x, float& h, float& m, float& l) {
  h = __uint_as_float(__float_as_uint(x) & 0xFFFF0000u);
  const float r = x - h;
  m = __uint_as_float(__float_as_uint(r) & 0xFFFF0000u);
  l = r - m;
}
// two bf16 values (fp32 with zero low halves) -> one packed word
__device__ __forceinline__ uint32_t pk2(float lo, float hi) {
  return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x7632);
}

// byte offset of 16-byte chunk c (0..15 along d) of row r in a K-major
// SW128 tile of R rows: [atom c / 8][row][chunk (c % 8) ^ (r % 8)]
__device__ __forceinline__ uint32_t sw_off(int R, int r, int c) {
  return static_cast<uint32_t>((c >> 3) * R * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// UMMA shared-memory descriptor (sm_100, version 1): 128B swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor, kind::f16: bf16 x bf16 -> fp32, K-major A
__device__ __forceinline__ uint32_t idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(b_mn_major) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

// S (K part pk of the tile) += Q parts x K: the part pairs whose products
// matter at fp32 resolution (q_lo x k_mid / k_lo fall below it)
__device__ __forceinline__ void issue_qk(uint32_t q_base, uint32_t k_base, uint32_t s_tmem, int pk, bool first) {
  const uint32_t id = idesc(kM, kKT, 0);
  const int nq = pk == 0 ? 3 : 2;
  bool acc = !first;
  for (int pq = 0; pq < nq; ++pq)
#pragma unroll
    for (int kk = 0; kk < kD / 16; ++kk) {
      const uint32_t qa = q_base + pq * kQPart + (kk >> 2) * (kM * 128) + (kk & 3) * 32;
      const uint32_t ka = k_base + (kk >> 2) * (kKT * 128) + (kk & 3) * 32;
      umma(s_tmem, sdesc(qa, 16, 1024), sdesc(ka, 16, 1024), id, acc ? 1u : 0u);
      acc = true;
    }
}

// O += P parts x V (V part pv): B = V as MN-major (d contiguous per key)
__device__ __forceinline__ void issue_pv(uint32_t p_base, uint32_t v_base, uint32_t o_tmem, int pv, bool first) {
  const uint32_t id = idesc(kM, kD, 1);
  const int np = pv == 0 ? 3 : 2;
  bool acc = !first;
  for (int pp = 0; pp < np; ++pp)
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      const uint32_t pa = p_base + pp * kPPart + kk * 32;
      const uint32_t va = v_base + kk * 2048;  // 16 keys = two 8-key groups of 1024 B
      umma(o_tmem, sdesc(pa, 16, 1024), sdesc(va, kKT * 128, 1024), id, acc ? 1u : 0u);
      acc = true;
    }
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Warp roles in the cached-key loop (the chunk's own rows follow with every
// thread on one serialised path):
//   warps 0-7   softmax: two threads per query row (TMEM lane quarter w % 4,
//               key / d column half w / 4)
//   warp 8      MMA issue (lane 0): QK(t) as soon as K(t) landed and S[t % 2]
//               was read, then P.V(t - 1) -- the tensor core runs QK(t) while
//               the softmax warps work on tile t - 1
//   warps 9-11  producers: cp.async gathers of K(t) / V(t) into the double
//               buffers, each signalled by its own mbarrier
// Every hand-off is an mbarrier per buffer, so no waiter can fall two phases
// behind: s_full[b] (QK done), pv_done[b] (P.V done), kvk_full[b] / kvv_full[b]
// (K / V landed), s_free[b] (S read), p_full (P written).
__global__ void __launch_bounds__(kThr, 1) prefill_tc_kernel(PrefillAttendParams p, const uint16_t* kc3,
                                                             const uint16_t* vc3) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int G = p.H / p.H_kv;
  const int rows_per_head = kM / G;  // chunk rows per CTA
  const int g = blockIdx.y;
  const int i0 = blockIdx.x * rows_per_head;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row_elems = p.H_kv * kD;
  const int n_cached = p.n_att_ptr ? *p.n_att_ptr : p.n_att;
  const int n_cur = min(p.C, i0 + rows_per_head);  // chunk rows any row here can see
  const int nct = (n_cached + kKT - 1) / kKT;
  const int n_tiles = nct + (n_cur + kKT - 1) / kKT;
  const uint32_t sbase = smem_u32(smem);
  int32_t* rows_all = reinterpret_cast<int32_t*>(smem + kOffRows);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* s_full = bars + 0;    // [2]
  uint64_t* pv_done = bars + 2;   // [2]
  uint64_t* kvk_full = bars + 4;  // [2]
  uint64_t* kvv_full = bars + 6;  // [2]
  uint64_t* s_free = bars + 8;    // [2]
  uint64_t* p_full = bars + 10;   // [1]
  uint64_t* c_done = bars + 11;   // [1] the serialised chunk path's MMAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 128);
  float* red = reinterpret_cast<float*>(smem + kOffRed);  // [2][2][kM]
  const bool rows_up_front = n_cached <= kRowsUpFront;
  unsigned long long* trc = (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) ? p.trace : nullptr;
  auto stamp = [&](int i) {
    if (trc && i < 512) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      trc[i] = gt;
    }
  };
  stamp(0);
  auto lookup = [&](int key) -> int32_t {
    const uint32_t tok = p.att[key];
    return p.page_size == 1 ? p.page_table[tok]
                            : p.page_table[tok / p.page_size] * p.page_size + static_cast<int32_t>(tok % p.page_size);
  };

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&pv_done[i], 1);
      mbar_init(&kvk_full[i], kProdThr);
      mbar_init(&kvv_full[i], kProdThr);
      mbar_init(&s_free[i], kSmThr);
    }
    mbar_init(p_full, kSmThr);
    mbar_init(c_done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  stamp(5);
  // ---- Q parts: row m = (head m / rows_per_head, chunk row i0 + m % rows_per_head)
  for (int idx = tid; idx < kM * (kD / 8); idx += kThr) {
    const int m = idx >> 4, c = idx & 15;
    const int hm = m / rows_per_head, i = i0 + (m - hm * rows_per_head);
    float x[8];
    if (i < p.C) {
      const float4* src = reinterpret_cast<const float4*>(p.q + static_cast<size_t>(i) * p.H * kD +
                                                          static_cast<size_t>(g + hm * p.H_kv) * kD + c * 8);
      const float4 a = src[0], b = src[1];
      x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = 0.f;
    }
    uint32_t hw[4], mw[4], lw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float h0, m0, l0, h1, m1, l1;
      sp3(x[2 * u], h0, m0, l0);
      sp3(x[2 * u + 1], h1, m1, l1);
      hw[u] = pk2(h0, h1);
      mw[u] = pk2(m0, m1);
      lw[u] = pk2(l0, l1);
    }
    const uint32_t off = sw_off(kM, m, c);
    *reinterpret_cast<uint4*>(smem + kOffQ + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(smem + kOffQ + kQPart + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    *reinterpret_cast<uint4*>(smem + kOffQ + 2 * kQPart + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  if (rows_up_front) {
    // all of this thread's list loads in flight, then all its page-table loads
    constexpr int kPer = (kRowsUpFront + kThr - 1) / kThr;
    uint32_t tok[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int key = tid + u * kThr;
      tok[u] = key < n_cached ? __ldg(p.att + key) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int key = tid + u * kThr;
      if (key < n_cached)
        rows_all[key] = p.page_size == 1 ? __ldg(p.page_table + tok[u])
                                         : __ldg(p.page_table + tok[u] / p.page_size) * p.page_size +
                                               static_cast<int32_t>(tok[u] % p.page_size);
    }
  }
  fence_async_smem();  // Q parts -> the tensor core
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const uint32_t s_tmem = tbase;           // columns [0, 128): S[2] of 64 columns
  const uint32_t o_tmem = tbase + 128;     // columns [128, 256): one tile's P.V (fresh per tile)
  const uint32_t orun_tmem = tbase + 256;  // columns [256, 384): the running O, fp32 round-to-nearest adds

  // gather of a tile's K and/or V rows (part `part` of the chunk's split copy
  // for chunk tiles) into buffer b, swizzled, by threads gt of gn; padding
  // rows zeroed; one cp.async group
  auto gather = [&](int tile, int b, int part, bool k_on, bool v_on, int gt, int gn) {
    uint8_t* kb = smem + kOffK + b * kKVTile;
    uint8_t* vb = smem + kOffV + b * kKVTile;
    for (int idx = gt; idx < kKT * 16; idx += gn) {
      const int r = idx >> 4, c = idx & 15;
      const uint32_t off = sw_off(kKT, r, c);
      const uint16_t* ks = nullptr;
      const uint16_t* vs = nullptr;
      if (tile < nct) {
        const int key = tile * kKT + r;
        if (key < n_cached) {
          const int32_t ri = rows_up_front ? rows_all[key] : lookup(key);
          const size_t o = static_cast<size_t>(ri) * row_elems + static_cast<size_t>(g) * kD + c * 8;
          ks = p.k_slab + o;
          vs = p.v_slab + o;
        }
      } else {
        const int j = (tile - nct) * kKT + r;
        if (j < n_cur) {
          const size_t o = static_cast<size_t>(part) * p.C * row_elems + static_cast<size_t>(j) * row_elems +
                           static_cast<size_t>(g) * kD + c * 8;
          ks = kc3 + o;
          vs = vc3 + o;
        }
      }
      if (k_on) {
        if (ks) cp_async16(kb + off, ks);
        else *reinterpret_cast<uint4*>(kb + off) = make_uint4(0u, 0u, 0u, 0u);
      }
      if (v_on) {
        if (vs) cp_async16(vb + off, vs);
        else *reinterpret_cast<uint4*>(vb + off) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    cp_async_commit();
  };

  // ---- softmax state: thread (row m, half) of warps 0-7
  const bool is_sm = warp < 8;
  const int m = (warp & 3) * 32 + lane;  // TMEM lane = query row
  const int half = (warp >> 2) & 1;
  const uint32_t lane_sel = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const int hm = m / rows_per_head;
  const int i_row = i0 + (m - hm * rows_per_head);
  float m_ref = -INFINITY, l_run = 0.f;  // (l_run: this thread's half of the row)
  const float sl2 = p.scale * kLog2e;
  bool delta_pending = false;  // a completed tile P.V not yet added into O_run
  bool o_folded = false;       // O_run holds data
  constexpr int KH = kKT / 2;  // this thread's key columns
  float s[KH];
  // O_run (+)= delta, then * c: this thread's 64 of the row's 128 columns
  auto fold = [&](float c) {
    float a16[16], b16[16];
#pragma unroll 1
    for (int q = 0; q < kD / 32; ++q) {
      const uint32_t col = lane_sel + half * (kD / 2) + q * 16;
      tmem_ld16(o_tmem + col, a16);
      if (o_folded) {
        tmem_ld16(orun_tmem + col, b16);
#pragma unroll
        for (int u = 0; u < 16; ++u) a16[u] = (b16[u] + a16[u]) * c;
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) a16[u] *= c;
      }
      tmem_st16(orun_tmem + col, a16);
    }
    tmem_wait_st();
    o_folded = true;
  };
  auto fold_scale = [&](float c) {
    float a16[16];
#pragma unroll 1
    for (int q = 0; q < kD / 32; ++q) {
      const uint32_t col = lane_sel + half * (kD / 2) + q * 16;
      tmem_ld16(orun_tmem + col, a16);
#pragma unroll
      for (int u = 0; u < 16; ++u) a16[u] *= c;
      tmem_st16(orun_tmem + col, a16);
    }
    tmem_wait_st();
  };
  // (1) this thread's 32 scores of the tile -> s[], own max -> red[rb][half][m]
  auto sm_load = [&](uint32_t s_addr, int k0, bool chunk, int rb) {
    const int lim = chunk ? min(n_cur - 1, i_row) + 1 : n_cached;  // visible keys: [0, lim)
    const int kb0 = k0 + half * KH;
    float v16[16];
#pragma unroll
    for (int q = 0; q < KH / 16; ++q) {
      tmem_ld16(s_addr + lane_sel + half * KH + q * 16, v16);
#pragma unroll
      for (int u = 0; u < 16; ++u) s[q * 16 + u] = v16[u];
    }
    float mt = -INFINITY;
#pragma unroll
    for (int u = 0; u < KH; ++u) {
      const bool ok = i_row < p.C && kb0 + u < lim;
      s[u] = ok ? s[u] * sl2 : -INFINITY;  // log2-domain logits
      mt = fmaxf(mt, s[u]);
    }
    red[(rb * 2 + half) * kM + m] = mt;
  };
  // (2) after the max exchange and after the previous P.V completed: lazy
  // reference max (moved only when the max grows by > 8; the TMEM accesses
  // are warp-collective, so a warp rescales together), the previous tile's
  // P.V folded into O_run, P = 2^(s - m_ref) split into three bf16 parts -> smem
  auto sm_finish = [&](int rb) {
    const float mt = fmaxf(red[(rb * 2 + half) * kM + m], red[(rb * 2 + (half ^ 1)) * kM + m]);
    const bool need = mt > m_ref + 8.f;
    float corr = 1.f;
    if (need) {
      corr = m_ref == -INFINITY ? 0.f : ex2_approx(m_ref - mt);
      l_run *= corr;
      m_ref = mt;
    }
    if (delta_pending) {
      fold(corr);
      delta_pending = false;
    } else if (o_folded && __any_sync(0xffffffffu, need)) {
      fold_scale(corr);
    }
    float ls = 0.f;
#pragma unroll
    for (int c = 0; c < KH / 8; ++c) {
      uint32_t hw[4], mw[4], lw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float p0 = s[c * 8 + 2 * u] == -INFINITY ? 0.f : ex2_approx(s[c * 8 + 2 * u] - m_ref);
        const float p1 = s[c * 8 + 2 * u + 1] == -INFINITY ? 0.f : ex2_approx(s[c * 8 + 2 * u + 1] - m_ref);
        ls += p0 + p1;
        float h0, m0, l0, h1, m1, l1;
        sp3(p0, h0, m0, l0);
        sp3(p1, h1, m1, l1);
        hw[u] = pk2(h0, h1);
        mw[u] = pk2(m0, m1);
        lw[u] = pk2(l0, l1);
      }
      const int cc = half * (KH / 8) + c;  // 16-byte chunk of the row's 128 B of P
      const uint32_t off = static_cast<uint32_t>(m * 128 + ((cc ^ (m & 7)) << 4));
      *reinterpret_cast<uint4*>(smem + kOffP + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(smem + kOffP + kPPart + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
      *reinterpret_cast<uint4*>(smem + kOffP + 2 * kPPart + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    l_run += ls;
  };

  stamp(1);
  // ================================================ cached keys, specialised
  if (nct > 0) {
    if (is_sm) {
      for (int t = 0; t < nct; ++t) {
        const int b = t & 1;
        mbar_wait(&s_full[b], static_cast<uint32_t>(t >> 1) & 1u);  // QK(t) done
        tmem_fence_after_sync();
        sm_load(s_tmem + b * kKT, t * kKT, false, b);
        tmem_fence_before_sync();
        mbar_arrive(&s_free[b]);  // S[b] read: QK(t + 2) may overwrite it
        named_sync(1, kSmThr);    // row maxima exchanged
        if (t >= 1) {             // P.V(t - 1): its delta and the P buffer
          mbar_wait(&pv_done[(t - 1) & 1], static_cast<uint32_t>((t - 1) >> 1) & 1u);
          tmem_fence_after_sync();
        }
        sm_finish(b);
        fence_async_smem();  // P -> the tensor core
        tmem_fence_before_sync();
        mbar_arrive(p_full);
        delta_pending = true;  // P.V(t), once issued and completed
        if (t == 0) stamp(8);
      }
      // the last P.V
      mbar_wait(&pv_done[(nct - 1) & 1], static_cast<uint32_t>((nct - 1) >> 1) & 1u);
      tmem_fence_after_sync();
      stamp(2);
    } else if (warp == 8) {
      if (lane == 0) {
        for (int t = 0; t <= nct; ++t) {
          if (t < nct) {
            const int b = t & 1;
            mbar_wait(&kvk_full[b], static_cast<uint32_t>(t >> 1) & 1u);            // K(t) landed
            if (t >= 2) mbar_wait(&s_free[b], static_cast<uint32_t>((t - 2) >> 1) & 1u);  // S[b] read
            tmem_fence_after_sync();
            issue_qk(sbase + kOffQ, sbase + kOffK + b * kKVTile, s_tmem + b * kKT, 0, true);
            umma_commit(&s_full[b]);
          }
          if (t >= 1) {  // P.V(t - 1)
            const int pb = (t - 1) & 1;
            mbar_wait(p_full, static_cast<uint32_t>(t - 1) & 1u);                    // P(t - 1) written
            mbar_wait(&kvv_full[pb], static_cast<uint32_t>((t - 1) >> 1) & 1u);       // V(t - 1) landed
            tmem_fence_after_sync();
            issue_pv(sbase + kOffP, sbase + kOffV + pb * kKVTile, o_tmem, 0, true);
            umma_commit(&pv_done[pb]);
          }
        }
      }
      __syncwarp();
    } else {
      // producers: K(t) after QK(t - 2) freed buffer t % 2, V(t) after P.V(t - 2)
      const int pt = tid - 9 * 32;
      for (int t = 0; t < nct; ++t) {
        const int b = t & 1;
        if (t >= 2) mbar_wait(&s_full[b], static_cast<uint32_t>((t - 2) >> 1) & 1u);
        gather(t, b, 0, true, false, pt, kProdThr);
        if (t >= 2) mbar_wait(&pv_done[b], static_cast<uint32_t>((t - 2) >> 1) & 1u);
        gather(t, b, 0, false, true, pt, kProdThr);
        cp_async_wait<1>();  // K(t) landed
        fence_async_smem();
        mbar_arrive(&kvk_full[b]);
        cp_async_wait<0>();  // V(t) landed
        fence_async_smem();
        mbar_arrive(&kvv_full[b]);
      }
    }
  }
  __syncthreads();
  tmem_fence_after_sync();

  // ================================================ the chunk's own rows
  // fp32 K/V in three exact bf16 parts, one part at a time through buffer 0,
  // causal; every thread on one serialised path (at most a few tiles)
  uint32_t c_phase = 0;
  auto c_mma_wait = [&]() {
    mbar_wait(c_done, c_phase);
    c_phase ^= 1u;
    tmem_fence_after_sync();
  };
  auto publish = [&]() {
    cp_async_wait<0>();
    fence_async_smem();
    __syncthreads();
  };
  for (int t = nct; t < n_tiles; ++t) {
    for (int pk = 0; pk < 3; ++pk) {
      gather(t, 0, pk, true, pk == 0, tid, kThr);
      publish();
      if (tid == 0) {
        tmem_fence_after_sync();
        issue_qk(sbase + kOffQ, sbase + kOffK, s_tmem, pk, pk == 0);
        umma_commit(c_done);
      }
      c_mma_wait();
      __syncthreads();
    }
    if (is_sm) sm_load(s_tmem, (t - nct) * kKT, true, 0);
    __syncthreads();
    if (is_sm) sm_finish(0);
    if (is_sm) tmem_fence_before_sync();
    fence_async_smem();
    __syncthreads();
    for (int pv = 0; pv < 3; ++pv) {
      if (pv > 0) {
        gather(t, 0, pv, false, true, tid, kThr);
        publish();
      }
      if (tid == 0) {
        tmem_fence_after_sync();
        issue_pv(sbase + kOffP, sbase + kOffV, o_tmem, pv, pv == 0);
        umma_commit(c_done);
      }
      c_mma_wait();
      __syncthreads();
    }
    if (is_sm) delta_pending = true;
  }
  stamp(3);
  // ---- epilogue: O_run / l -> out row (i_row, head g + hm * H_kv), each
  // softmax thread its half of the d columns; l = the two halves' sums
  if (is_sm) red[half * kM + m] = l_run;
  __syncthreads();
  if (is_sm) {
    if (delta_pending) fold(1.f);  // (its P.V completed)
    const float l = l_run + red[(half ^ 1) * kM + m];
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const bool live = i_row < p.C;  // (warp-collective TMEM loads; rows past the chunk are not stored)
    float* orow = p.out + static_cast<size_t>(live ? i_row : 0) * p.H * kD + static_cast<size_t>(g + hm * p.H_kv) * kD +
                  half * (kD / 2);
    float v16[16];
#pragma unroll 1
    for (int q = 0; q < kD / 32; ++q) {
      tmem_ld16(orun_tmem + lane_sel + half * (kD / 2) + q * 16, v16);
      if (live)
#pragma unroll
        for (int u = 0; u < 16; u += 4)
          *reinterpret_cast<float4*>(orow + q * 16 + u) =
              make_float4(v16[u] * inv, v16[u + 1] * inv, v16[u + 2] * inv, v16[u + 3] * inv);
    }
  }
  stamp(4);
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, 512);
  }
}

__global__ void split3_tc_kernel(const float* __restrict__ x, int n, uint16_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float h, m, l;
    sp3(x[i], h, m, l);
    out[i] = static_cast<uint16_t>(__float_as_uint(h) >> 16);
    out[n + i] = static_cast<uint16_t>(__float_as_uint(m) >> 16);
    out[2 * static_cast<size_t>(n) + i] = static_cast<uint16_t>(__float_as_uint(l) >> 16);
  }
}

}  // namespace

cudaError_t launch_prefill_tc(const PrefillAttendParams& p, cudaStream_t st) {
  const int G = p.H / p.H_kv;
  if (p.d != kD || (G != 1 && G != 2 && G != 4 && G != 8) || p.page_size < 1 || !p.split_ws)
    return cudaErrorInvalidValue;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const int n = p.C * p.H_kv * kD;
  uint16_t* kc3 = p.split_ws;
  uint16_t* vc3 = p.split_ws + 3 * static_cast<size_t>(n);
  split3_tc_kernel<<<148, 512, 0, st>>>(p.k_cur, n, kc3);
  split3_tc_kernel<<<148, 512, 0, st>>>(p.v_cur, n, vc3);
  const int rph = kM / G;
  dim3 grid((p.C + rph - 1) / rph, p.H_kv);
  prefill_tc_kernel<<<grid, kThr, kSmem, st>>>(p, kc3, vc3);
  return cudaGetLastError();
}

}  // namespace tsb

// Chunked-prefill sparse attention on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in tensor memory): the C-row case of
// sparse_attend (attention.cpp:114-123 -> sdpa_full :54-112) for head_dim
// 128 and G = H / H_kv <= 16.
//
// One CTA = 128 query rows = the G query heads of KV head g (h mod H_kv,
// :78) x floor(128 / G) chunk rows (the rest padding when G does not divide
// 128, e.g. Qwen2's 7); grid = (C / floor(128 / G), H_kv). Keys come in
// tiles of 64: the merged cached rows (init U selected U local, gathered
// through the page table) and then the chunk's own rows, causal (:83).
//
//   S = Q K^T     tcgen05.mma kind::f16, M = 128, N = 64, K = 128 (8 steps),
//                 A = Q (tensor memory), B = K (smem, K-major SW128),
//                 D = S in TMEM (64 columns). Q (fp32) is split exactly into
//                 three bf16 parts; cached K is bf16 (exact); the chunk's own
//                 K (fp32 in the reference) is split into three parts as well
//                 (loaded one part at a time), so every product is exact and
//                 only the fp32 summation order differs from the reference.
//   softmax       thread = query row = TMEM lane (two threads per row, one per
//                 key half): tcgen05.ld of its 32 scores, mask, online
//                 softmax in the exp2 domain with a lazily moved reference
//                 max (O and l are rescaled only when the max grows by more
//                 than 2^8), P split into three bf16 parts -> TMEM, over S
//   O += P V      tcgen05.mma M = 128, N = 128, K = 64 (4 steps),
//                 A = P (tensor memory), B = V (smem, MN-major SW128),
//                 D = a fresh per-tile delta in TMEM (128 columns), added
//                 into the running O (registers) on the CUDA cores with
//                 round-to-nearest fp32 adds -- accumulating every tile in
//                 the tensor core's own adder lost precision
//
// K/V tiles arrive by TMA (two 64 x 64 boxes per 16 KB tile, 128B swizzle =
// the UMMA layout) from prep_tc_kernel's contiguous copies, two loads ahead of
// the tensor core; one elected lane of the MMA warp issues every MMA
// (tcgen05.commit -> mbarrier).
#include <cuda.h>

#include <cfloat>
#include <cmath>
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "aux.h"
#include "common.cuh"

namespace tsb {

namespace {

constexpr int kD = 128;
constexpr int kM = 128;          // query rows per CTA (UMMA M)
constexpr int kKT = 64;          // keys per tile (UMMA N of S, K of P.V)
constexpr int kThr = 352;        // 8 softmax warps, 1 MMA warp, a K and a V producer warp
constexpr int kSmThr = 256;      // softmax threads (two per query row)
constexpr float kLog2e = 1.4426950408889634f;

// shared memory (bytes), every operand region 1024-B aligned
constexpr int kKVTile = kKT * kD * 2;  // 16 KB: [2 atoms][64 rows][128 B]
constexpr int kOffK = 0;                         // 2 buffers of K
constexpr int kOffV = kOffK + 2 * kKVTile;       // 2 buffers of V
constexpr int kOffBar = kOffV + 2 * kKVTile;
constexpr int kOffRed = kOffBar + 256;              // [2 tiles][2 halves][128] row-max / row-sum exchange
constexpr int kOutStride = kD + 4;                  // staged output row (floats; 16-B aligned, conflict-light)
constexpr int kOffOut = kOffRed + 4 * kM * 4;       // [128 rows][kOutStride] output staging
constexpr int kSmem = kOffOut + kM * kOutStride * 4;

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
// two floats -> round-to-nearest bf16 pair (a in the low half)
__device__ __forceinline__ uint32_t bf2_rn(float a, float b) {
  uint32_t w;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(w) : "f"(a), "f"(b));
  return w;
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

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(id), "r"(acc));
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
// matter at fp32 resolution (q_lo x k_mid / k_lo fall below it). A = Q in
// tensor memory (64 columns per part); dk: the descriptor of the K slot -- a
// descriptor plus (byte offset >> 4) is the descriptor of the offset
// address, so every MMA's operands are one add of a constant away (the
// issue rate is the limit for these small MMAs).
__device__ __forceinline__ void issue_qk(uint32_t q_tmem, uint64_t dk, uint32_t s_tmem, int pk, bool first) {
  constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kKT >> 3) << 17) |
                          (static_cast<uint32_t>(kM >> 4) << 24);
#pragma unroll
  for (int pq = 0; pq < 3; ++pq) {
    if (pq == 2 && pk != 0) break;
#pragma unroll
    for (int kk = 0; kk < kD / 16; ++kk) {
      const uint32_t ko = ((kk >> 2) * (kKT * 128) + (kk & 3) * 32) >> 4;
      umma_ts(s_tmem, q_tmem + pq * (kD / 2) + kk * 8, dk + ko, id, (pq == 0 && kk == 0 && first) ? 0u : 1u);
    }
  }
}

// delta (+)= P parts x V (V part pv): A = P in tensor memory (two bf16 per
// 32-bit column, 32 columns per part), B = V as MN-major (d contiguous per key)
__device__ __forceinline__ void issue_pv(uint32_t p_tmem, uint64_t dv, uint32_t o_tmem, int pv, bool first, bool p3) {
  constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (static_cast<uint32_t>(kD >> 3) << 17) |
                          (static_cast<uint32_t>(kM >> 4) << 24);
#pragma unroll
  for (int pp = 0; pp < 3; ++pp) {
    if (pp == 2 && (pv != 0 || !p3)) break;
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      const uint32_t vo = (kk * 2048) >> 4;  // 16 keys = two 8-key groups of 1024 B
      umma_ts(o_tmem, p_tmem + pp * (kKT / 2) + kk * 8, dv + vo, id, (pp == 0 && kk == 0 && first) ? 0u : 1u);
    }
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// programmatic dependent launch: the attention kernel starts (TMEM, barriers,
// its Q) while prep_tc_kernel finishes, and waits here for prep's results
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// named barrier that also ORs a predicate over its participants
__device__ __forceinline__ bool bar_red_or(int id, int n, bool v) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %3, 0;\n\tbarrier.cta.red.or.pred q, %1, %2, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
               : "=r"(r)
               : "r"(id), "r"(n), "r"(v ? 1u : 0u)
               : "memory");
  return r != 0;
}

// TMA: one 64 x 64 box at (col, row) -> 8 KB at dst
__device__ __forceinline__ void tma_tile2d(void* dst, const CUtensorMap* tm, int col, int row, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}

// Work items. A unit is (row block x, KV head g): 128 query rows against its
// tiles -- the cached tiles [0, nct) (the same attended rows for every unit)
// then the chunk's own tiles, causal, so later row blocks have more of them.
// Units differ in cost by up to 40 %, so the host cuts the concatenated tile
// sequence of all units into one contiguous, equal-cost range per CTA; a
// range may end inside a unit (a piece). A unit cut into pieces leaves each
// piece's unnormalised O, log2 reference max and row sum in a partial slot,
// and the last of its pieces to finish merges them (log-sum-exp, piece order).
constexpr int kMaxPieces = 4;
struct TcPiece {
  int16_t x, g, t0, t1;  // unit and its tile range [t0, t1)
  int16_t slot;          // partial slot (-1: the whole unit, written directly)
  int16_t unit;
};
struct TcWork {
  int32_t n;
  TcPiece pc[kMaxPieces];
};
struct TcSplit {
  const TcWork* work;        // [grid]
  const int16_t* unit_slot0; // [units] first partial slot of a split unit
  const int16_t* unit_np;    // [units] its pieces
  float* part_o;             // [slots][128 rows][128]
  float* part_ml;            // [slots][128 rows][2]: log2 reference max, row sum
  unsigned* cnt;             // [units] pieces finished (zeroed by prep_tc_kernel)
  int nct;                   // cached tiles per unit (planned from n_att_max)
  int fold;                  // fold the P.V delta into O every `fold` tiles (1 or 2; see the softmax loop)
  int p3;                    // P in three truncated bf16 parts (1) or two rounded ones (0; see sm_p)
};

// Warp roles (cached tiles and the chunk's own tiles alike, over the CTA's
// pieces in order):
//   warps 0-7   softmax: two threads per query row (TMEM lane quarter w % 4,
//               key / d column half w / 4); P(t) goes over S(t) in TMEM; at
//               a piece start they stage its Q in TMEM (q_ready), at its end
//               they write the output rows or the partial (and merge)
//   warp 8      MMA issue (one elected lane): QK(t) as soon as its K loads
//               landed, then P.V(t - 1) once P(t - 1) is written -- the tensor
//               core runs QK(t) while the softmax warps work on tile t - 1,
//               and runs P.V(t - 2) before the QK(t) that overwrites its P; at
//               a piece start P.V(t - 1) goes first, then it waits for the Q
//   warp 9/10   TMA producers of the K / V loads into two slots each: one load
//               per cached tile, three (the split parts) per chunk tile
// Every hand-off is an mbarrier per buffer, so no waiter can fall two phases
// behind: s_full[b] (QK done), pv_done[b] (P.V done), kvk_full[s] / kvv_full[s]
// (K / V load landed in slot s), k_free[s] / v_free[s] (the MMAs reading slot
// s completed), p_full (P written and the previous delta folded), q_ready
// (a piece's Q staged). Tile-indexed barriers count the CTA's tiles across
// its pieces.
__global__ void __launch_bounds__(kThr, 1)
    prefill_tc_kernel(PrefillAttendParams p, TcSplit sp, const __grid_constant__ CUtensorMap tm_kg,
                      const __grid_constant__ CUtensorMap tm_vg, const __grid_constant__ CUtensorMap tm_kc,
                      const __grid_constant__ CUtensorMap tm_vc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  grid_dep_launch();  // (the chunk's append, launched after this grid, reads none of its inputs)
  const int G = p.H / p.H_kv;
  const int rows_per_head = kM / G;  // chunk rows per unit
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int n_cached = 0;  // (<= nct * 64; read after the programmatic-launch wait)
  const int nct = sp.nct;
  const TcWork wk = sp.work[blockIdx.x];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* s_full = bars + 0;    // [2]
  uint64_t* pv_done = bars + 2;   // [2]
  uint64_t* kvk_full = bars + 4;  // [2]
  uint64_t* kvv_full = bars + 6;  // [2]
  uint64_t* q_ready = bars + 8;   // [1]
  uint64_t* p_full = bars + 10;   // [1]
  uint64_t* k_free = bars + 11;   // [2] the MMAs reading a K slot completed
  uint64_t* v_free = bars + 13;   // [2] the MMAs reading a V slot completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 128);
  int* last_flag = reinterpret_cast<int*>(smem + kOffBar + 136);
  volatile int* fresh_flag = reinterpret_cast<volatile int*>(smem + kOffBar + 144);  // [2] P.V(t) starts a fresh delta
  float* red = reinterpret_cast<float*>(smem + kOffRed);  // [2][2][kM]
  // dev trace (TS_PREFILL_TRACE): %globaltimer at the CTA's start, each
  // piece's end and the CTA's end -> trace[cta * 8 + slot]
  auto mark = [&](int slot) {
    if (p.trace && blockIdx.x < 512) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.trace[blockIdx.x * 8 + slot] = gt;
    }
  };
  if (tid == 0) mark(0);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&pv_done[i], 1);
      mbar_init(&kvk_full[i], 1);  // (+ the TMA transaction bytes)
      mbar_init(&kvv_full[i], 1);
    }
    mbar_init(q_ready, kSmThr);
    mbar_init(p_full, kSmThr);
    mbar_init(&k_free[0], 1);
    mbar_init(&k_free[1], 1);
    mbar_init(&v_free[0], 1);
    mbar_init(&v_free[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  // tensor memory (512 columns x 128 lanes = query rows):
  const uint32_t sp_tmem = tbase;       // [0, 192): S/P[2], 96 columns each -- S (fp32, 64 columns),
                                        //   then P over it (3 bf16 parts x 32 columns)
  const uint32_t q_tmem = tbase + 192;  // [192, 384): Q, 3 bf16 parts x 64 columns
  const uint32_t o_tmem = tbase + 384;  // [384, 512): one tile's P.V (fresh per tile)
  constexpr int kSP = 3 * kKT / 2;      // columns per S/P buffer
  auto nk = [&](int t) { return t < nct ? 1 : 3; };  // loads per tile

  // TMA load of part `part` of unit-tile `tile` (KV head g)'s K or V rows
  // into the 16-KB slot at `dst`: two 64 x 64 boxes (the d halves; 128B
  // swizzle = the UMMA layout) of the gathered cached rows (tm_kg / tm_vg)
  // or of the chunk's split copy (tm_kc / tm_vc), completing on `bar`. Rows
  // past the attended count are zeros (prep_tc_kernel) or out of bounds
  // (zero-filled); rows of the chunk past the causal limit are masked in the
  // softmax.
  auto tma_tile = [&](int g, int tile, int part, bool is_k, uint8_t* dst, uint64_t* bar) {
    if (lane == 0) mbar_arrive_expect_tx(bar, kKVTile);
    __syncwarp();
    if (lane < 2) {
      const bool cached = tile < nct;
      const CUtensorMap* tm = cached ? (is_k ? &tm_kg : &tm_vg) : (is_k ? &tm_kc : &tm_vc);
      const int row = cached ? tile * kKT : part * p.C + (tile - nct) * kKT;
      tma_tile2d(dst + lane * (kKT * 128), tm, g * kD + lane * 64, row, bar);
    }
  };

  if (warp < 8) {
    // ================================================ softmax warps
    const int m = (warp & 3) * 32 + lane;  // TMEM lane = query row
    const int half = (warp >> 2) & 1;
    const uint32_t lane_sel = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int hm = m / rows_per_head;  // (G * rows_per_head <= 128: rows past it are padding)
    const float sl2 = p.scale * kLog2e;
    constexpr int KH = kKT / 2;  // this thread's key columns
    float s[KH];
    float orun[kD / 2];  // the running O: this thread's 64 of the row's 128 columns
    float m_ref, l_run;  // (l_run: this thread's half of the row)
    int i_row = 0, n_cur = 0;
    bool row_ok = false;
    // O_run = (O_run + delta) * c
    auto fold = [&](float c) {
      float a[32];
      const bool moved = __any_sync(0xffffffffu, c != 1.f);  // (rare: a reference move in the warp's rows)
#pragma unroll
      for (int q = 0; q < kD / 64; ++q) {
        tmem_ld32(o_tmem + lane_sel + half * (kD / 2) + q * 32, a);
        if (moved) {
#pragma unroll
          for (int u = 0; u < 32; ++u) orun[q * 32 + u] = (orun[q * 32 + u] + a[u]) * c;
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u) orun[q * 32 + u] += a[u];
        }
      }
    };
    // the normalised rows -> out, through shared memory so that a warp stores
    // whole 512-B rows (a thread's own 256 B of a row, 16 KB apart from its
    // neighbours', would scatter every store instruction over 32 lines)
    float* ostage = reinterpret_cast<float*>(smem + kOffOut);
    auto write_rows = [&](float inv, int g, int i0) {
#pragma unroll
      for (int u = 0; u < kD / 2; u += 4)
        *reinterpret_cast<float4*>(ostage + m * kOutStride + half * (kD / 2) + u) =
            make_float4(orun[u] * inv, orun[u + 1] * inv, orun[u + 2] * inv, orun[u + 3] * inv);
      named_sync(1, kSmThr);
      for (int r = warp; r < kM; r += kSmThr / 32) {  // warp per row, lane per 16 B
        const int hr = r / rows_per_head, ir = i0 + (r - hr * rows_per_head);
        if (hr < G && ir < p.C)
          *reinterpret_cast<float4*>(p.out + static_cast<size_t>(ir) * p.H * kD + static_cast<size_t>(g + hr * p.H_kv) * kD + lane * 4) =
              *reinterpret_cast<const float4*>(ostage + r * kOutStride + lane * 4);
      }
    };
    // (1) this thread's 32 scores of the tile -> s[], own max -> red[rb][half][m]
    auto sm_load = [&](uint32_t s_addr, int k0, bool chunk, int rb) -> bool {
      const int lim = chunk ? min(n_cur - 1, i_row) + 1 : n_cached;  // visible keys: [0, lim)
      const int kb0 = k0 + half * KH;
      tmem_ld32(s_addr + lane_sel + half * KH, s);
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      const int nv = row_ok ? lim - kb0 : 0;  // visible keys among this thread's 32
      // raw scores (the log2-domain scale sl2 > 0 is applied in sm_p's FMA);
      // keys past the visible limit -> -inf (only a boundary tile has them)
      if (__any_sync(0xffffffffu, nv < KH)) {
#pragma unroll
        for (int u = 0; u < KH; ++u) s[u] = u < nv ? s[u] : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < KH; ++u) mx[u & 3] = fmaxf(mx[u & 3], s[u]);
      const float mh = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;  // log2-domain max
      red[(rb * 2 + half) * kM + m] = mh;
      return mh > m_ref + 8.f;  // (the row moves its reference iff either half says so)
    };
    // (2) after the max exchange: lazy reference max (moved only when the max
    // grows by > 8), P = 2^(s - m_ref) split into three bf16 parts -> P[rb] in
    // tensor memory; returns the factor that moves O and l to the new reference
    // P3: three truncated parts (exact to 24 bits); else two round-to-nearest
    // parts, hi = rn(p), mid = rn(p - hi): |error| <= 2^-17 p, unbiased,
    // which keeps the output within the 1e-5 relative-Frobenius bar with a
    // third of the P.V products and of the P stores saved
    auto sm_p = [&](int rb, auto p3tag) -> float {
      constexpr bool P3 = decltype(p3tag)::value;
      const float mt = fmaxf(red[(rb * 2 + half) * kM + m], red[(rb * 2 + (half ^ 1)) * kM + m]);
      float corr = 1.f;
      if (mt > m_ref + 8.f) {
        corr = m_ref == -INFINITY ? 0.f : ex2_approx(m_ref - mt);
        l_run *= corr;
        m_ref = mt;
      }
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
      float hw[KH / 2], mw[KH / 2], lw[KH / 2];  // packed pairs (bit patterns)
      const float mu = m_ref == -INFINITY ? 0.f : m_ref;  // (a row with no visible key yet: every p = 2^-inf = 0)
#pragma unroll
      for (int c = 0; c < KH / 2; ++c) {
        const float p0 = ex2_approx(fmaf(s[2 * c], sl2, -mu));
        const float p1 = ex2_approx(fmaf(s[2 * c + 1], sl2, -mu));
        ls[c & 3] += p0 + p1;
        if constexpr (P3) {
          float h0, m0, l0, h1, m1, l1;
          sp3(p0, h0, m0, l0);
          sp3(p1, h1, m1, l1);
          hw[c] = __uint_as_float(pk2(h0, h1));
          mw[c] = __uint_as_float(pk2(m0, m1));
          lw[c] = __uint_as_float(pk2(l0, l1));
        } else {
          const uint32_t h = bf2_rn(p0, p1);
          hw[c] = __uint_as_float(h);
          mw[c] = __uint_as_float(bf2_rn(p0 - __uint_as_float(h << 16), p1 - __uint_as_float(h & 0xFFFF0000u)));
        }
      }
      l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      const uint32_t pa = sp_tmem + rb * kSP + lane_sel + half * (KH / 2);
      tmem_st16(pa, hw);
      tmem_st16(pa + kKT / 2, mw);
      if constexpr (P3) tmem_st16(pa + kKT, lw);
      return corr;
    };
    // ---- a unit's Q -> tensor memory: thread (row m, half) splits its 64 d
    // columns of the row's query (head g + hm * H_kv, chunk row ir) into
    // three exact bf16 parts, two per 32-bit column; then q_ready. (Called
    // for the next piece as soon as the current piece's last QK completed,
    // so the next piece's first QK overlaps this piece's drain.)
    auto stage_q = [&](const TcPiece& pc) {
      const int ir = pc.x * rows_per_head + (m - hm * rows_per_head);
      const bool ok = hm < G && ir < p.C;
      const float4* src = reinterpret_cast<const float4*>(p.q + static_cast<size_t>(ok ? ir : 0) * p.H * kD +
                                                          static_cast<size_t>(pc.g + (ok ? hm : 0) * p.H_kv) * kD +
                                                          half * (kD / 2));
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // 32 d columns -> 16 TMEM columns per part
        float hw[16], mw[16], lw[16];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float4 xv = ok ? src[c * 8 + u] : make_float4(0.f, 0.f, 0.f, 0.f);
          float h0, m0, l0, h1, m1, l1;
          sp3(xv.x, h0, m0, l0);
          sp3(xv.y, h1, m1, l1);
          hw[2 * u] = __uint_as_float(pk2(h0, h1));
          mw[2 * u] = __uint_as_float(pk2(m0, m1));
          lw[2 * u] = __uint_as_float(pk2(l0, l1));
          sp3(xv.z, h0, m0, l0);
          sp3(xv.w, h1, m1, l1);
          hw[2 * u + 1] = __uint_as_float(pk2(h0, h1));
          mw[2 * u + 1] = __uint_as_float(pk2(m0, m1));
          lw[2 * u + 1] = __uint_as_float(pk2(l0, l1));
        }
        const uint32_t qa = q_tmem + lane_sel + half * (kD / 4) + c * 16;
        tmem_st16(qa, hw);
        tmem_st16(qa + kD / 2, mw);
        tmem_st16(qa + kD, lw);
      }
      tmem_wait_st();
      tmem_fence_before_sync();
      mbar_arrive(q_ready);
    };
    int i = 0;    // the CTA's tile counter
    int unf = 0;  // tiles whose P.V the delta holds unfolded
    // a tile whose P.V completion was not waited for (the delta kept
    // accumulating): observed before the next wait on the other buffer's
    // barrier, so that with fold 2 every completion of pv_done is waited
    // for in order (never more than one phase ahead)
    int unwaited = -1;
    auto wait_pv = [&](int u) {
      if (unwaited >= 0 && unwaited == u - 1) mbar_wait(&pv_done[unwaited & 1], static_cast<uint32_t>(unwaited >> 1) & 1u);
      unwaited = -1;
      mbar_wait(&pv_done[u & 1], static_cast<uint32_t>(u >> 1) & 1u);
    };
    if (wk.n > 0) stage_q(wk.pc[0]);  // (the query is an input: before prep_tc_kernel's results)
    grid_dep_wait();
    n_cached = p.n_att_ptr ? *p.n_att_ptr : p.n_att;
    for (int pi = 0; pi < wk.n; ++pi) {
      const TcPiece pc = wk.pc[pi];
      const int g = pc.g, i0 = pc.x * rows_per_head;
      n_cur = min(p.C, i0 + rows_per_head);  // chunk rows any row here can see
      i_row = i0 + (m - hm * rows_per_head);
      row_ok = hm < G && i_row < p.C;
      m_ref = -INFINITY;
      l_run = 0.f;
#pragma unroll
      for (int u = 0; u < kD / 2; ++u) orun[u] = 0.f;
      for (int t = pc.t0; t < pc.t1; ++t, ++i) {
        const int b = i & 1;
        const bool chunk = t >= nct;
        mbar_wait(&s_full[b], static_cast<uint32_t>(i >> 1) & 1u);  // QK(i) done
        tmem_fence_after_sync();
        const bool need = sm_load(sp_tmem + b * kSP, chunk ? (t - nct) * kKT : t * kKT, chunk, b);
        // row maxima exchanged (every thread's S[b] loads done: P goes over
        // them), and whether any row of the CTA moves its reference max
        const bool any_need = bar_red_or(1, kSmThr, need);
        const float corr = sp.p3 ? sm_p(b, std::true_type{}) : sm_p(b, std::false_type{});
        // the delta holds the P.V of the `unf` tiles since the last fold; it
        // is folded every kFold tiles, and before any reference move (its
        // tiles and P(t) would otherwise mix two references)
        bool fresh = true;
        if (t > pc.t0) {
          if (unf >= sp.fold || any_need) {  // P.V(i - 1) completed: the delta into O_run
            wait_pv(i - 1);
            tmem_fence_after_sync();
            fold(corr);
            unf = 1;
          } else {
            fresh = false;  // P.V(t) accumulates onto the delta
            ++unf;
            unwaited = i - 1;
          }
        } else {
          unf = 1;
        }
        if (tid == 0) fresh_flag[b] = fresh ? 1 : 0;
        tmem_wait_st();  // P stored
        tmem_fence_before_sync();
        mbar_arrive(p_full);
        if (t == pc.t1 - 1 && pi + 1 < wk.n) stage_q(wk.pc[pi + 1]);  // (every QK of this piece completed)
      }
      // the piece's last P.V
      if (tid == 0 && pi == 0) mark(4);
      wait_pv(i - 1);
      tmem_fence_after_sync();
      if (tid == 0 && pi == 0) mark(3);
      fold(1.f);
      // ---- the piece's rows: l = the two halves' sums
      named_sync(1, kSmThr);  // (every thread past its last red[] read)
      red[half * kM + m] = l_run;
      named_sync(1, kSmThr);
      if (tid == 0 && pi == 0) mark(6);
      const float l = l_run + red[(half ^ 1) * kM + m];
      if (pc.slot < 0) {
        write_rows(l > 0.f ? 1.f / l : 0.f, g, pc.x * rows_per_head);
      } else {
        // partial: unnormalised O (log2 reference m_ref), the row sum
        // layout [slot][half][16 float4][128 rows]: a warp's lanes (rows)
        // store 512 contiguous bytes per float4
        float4* po = reinterpret_cast<float4*>(sp.part_o) + (static_cast<size_t>(pc.slot) * 2 + half) * (kD / 8) * kM + m;
#pragma unroll
        for (int u = 0; u < kD / 8; ++u) po[u * kM] = make_float4(orun[4 * u], orun[4 * u + 1], orun[4 * u + 2], orun[4 * u + 3]);
        if (half == 0)
          *reinterpret_cast<float2*>(sp.part_ml + (static_cast<size_t>(pc.slot) * kM + m) * 2) = make_float2(m_ref, l);
        named_sync(1, kSmThr);
        // release: the barrier orders every thread's partial stores before
        // thread 0's gpu-scope fence (cumulative), then the arrival
        if (tid == 0) {
          __threadfence();
          *last_flag = atomicAdd(sp.cnt + pc.unit, 1u) + 1u == static_cast<unsigned>(sp.unit_np[pc.unit]);
        }
        named_sync(1, kSmThr);
        if (tid == 0 && pi == 0) mark(5);
        if (*last_flag) {
          // the unit's last piece: log-sum-exp merge of its pieces in order
          // (acquire: thread 0's fenced atomic saw every other arrival)
          __threadfence();
          const int s0 = sp.unit_slot0[pc.unit], np = sp.unit_np[pc.unit];
          float M = -INFINITY;
          for (int k = 0; k < np; ++k) M = fmaxf(M, __ldcg(sp.part_ml + (static_cast<size_t>(s0 + k) * kM + m) * 2));
          float L = 0.f;
#pragma unroll
          for (int u = 0; u < kD / 2; ++u) orun[u] = 0.f;
          for (int k = 0; k < np; ++k) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(sp.part_ml + (static_cast<size_t>(s0 + k) * kM + m) * 2));
            const float w = ml.x == -INFINITY ? 0.f : ex2_approx(ml.x - M);
            L = fmaf(w, ml.y, L);
            const float4* pk = reinterpret_cast<const float4*>(sp.part_o) + (static_cast<size_t>(s0 + k) * 2 + half) * (kD / 8) * kM + m;
#pragma unroll
            for (int u = 0; u < kD / 8; ++u) {
              const float4 o = __ldcg(pk + u * kM);
              orun[4 * u] = fmaf(w, o.x, orun[4 * u]);
              orun[4 * u + 1] = fmaf(w, o.y, orun[4 * u + 1]);
              orun[4 * u + 2] = fmaf(w, o.z, orun[4 * u + 2]);
              orun[4 * u + 3] = fmaf(w, o.w, orun[4 * u + 3]);
            }
          }
          write_rows(L > 0.f ? 1.f / L : 0.f, g, pc.x * rows_per_head);
        }
      }
      named_sync(1, kSmThr);  // (red[] and last_flag reused by the next piece)
      if (tid == 0 && pi < 3) mark(1 + pi);
    }
  } else if (warp == 8) {
    grid_dep_wait();
    // ================================================ MMA issue
    // the whole warp runs the loop (warp-uniform operands stay in uniform
    // registers); one elected lane issues the MMAs and commits
    const uint64_t dk0 = sdesc(sbase + kOffK, 16, 1024);
    const uint64_t dv0 = sdesc(sbase + kOffV, kKT * 128, 1024);
    int i = 0, lk = 0, lv = 0;  // tile counter; next K / V load to consume
    int prev_i = -1, prev_nk = 0;
    auto do_pv = [&](int u, int nku) {  // P.V(u): its V loads in order, into the fresh delta
      mbar_wait(p_full, static_cast<uint32_t>(u) & 1u);  // P(u) written (and the delta folded, or kept)
      const bool fresh = fresh_flag[u & 1] != 0;
      for (int pv = 0; pv < nku; ++pv, ++lv) {
        const int vs = lv & 1;
        mbar_wait(&kvv_full[vs], static_cast<uint32_t>(lv >> 1) & 1u);
        tmem_fence_after_sync();
        if (elect_one()) {
          issue_pv(sp_tmem + (u & 1) * kSP, dv0 + vs * (kKVTile >> 4), o_tmem, pv, fresh && pv == 0, sp.p3 != 0);
          umma_commit(&v_free[vs]);
          if (pv == nku - 1) umma_commit(&pv_done[u & 1]);
        }
        __syncwarp();
      }
    };
    for (int pi = 0; pi < wk.n; ++pi) {
      const TcPiece pc = wk.pc[pi];
      for (int t = pc.t0; t < pc.t1; ++t, ++i) {
        if (t == pc.t0) {
          // a new piece: the previous piece's last P.V first (its softmax
          // finishes with it and then stages this piece's Q)
          if (prev_i >= 0) {
            do_pv(prev_i, prev_nk);
            prev_i = -1;
          }
          mbar_wait(q_ready, static_cast<uint32_t>(pi) & 1u);
          tmem_fence_after_sync();
        }
        // QK(i): its K loads in order, accumulated into S[i % 2] (S[b] =
        // P(i - 2): its P.V was issued before this QK; the tensor core runs
        // them in order)
        const int b = i & 1, nkt = nk(t);
        for (int pk = 0; pk < nkt; ++pk, ++lk) {
          const int ks = lk & 1;
          mbar_wait(&kvk_full[ks], static_cast<uint32_t>(lk >> 1) & 1u);  // this K load landed
          tmem_fence_after_sync();
          if (elect_one()) {
            issue_qk(q_tmem, dk0 + ks * (kKVTile >> 4), sp_tmem + b * kSP, pk, pk == 0);
            umma_commit(&k_free[ks]);
            if (pk == nkt - 1) umma_commit(&s_full[b]);
          }
          __syncwarp();
        }
        if (prev_i >= 0) do_pv(prev_i, prev_nk);
        prev_i = i;
        prev_nk = nkt;
      }
    }
    if (prev_i >= 0) do_pv(prev_i, prev_nk);
  } else {
    // ================================================ TMA producers
    // warp 9 streams the K loads, warp 10 the V loads, each into its slot
    // once the MMAs that read the slot's previous load completed. (The
    // streams are independent: a tile's last K part is needed before the
    // P.V that frees a V slot of the same tile.)
    grid_dep_wait();  // (the tiles come from prep_tc_kernel's copies)
    const bool is_k = warp == 9;
    uint64_t* freed = is_k ? k_free : v_free;
    uint64_t* full = is_k ? kvk_full : kvv_full;
    uint8_t* slots = smem + (is_k ? kOffK : kOffV);
    int li = 0;
    for (int pi = 0; pi < wk.n; ++pi) {
      const TcPiece pc = wk.pc[pi];
      for (int t = pc.t0; t < pc.t1; ++t)
        for (int part = 0; part < nk(t); ++part, ++li) {
          const int sl = li & 1;
          if (li >= 2) mbar_wait(&freed[sl], static_cast<uint32_t>((li - 2) >> 1) & 1u);
          tma_tile(pc.g, t, part, is_k, slots + sl * kKVTile, &full[sl]);
        }
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    tmem_dealloc(tbase, 512);
  }
  if (tid == 0) mark(7);
}

// Before the attention kernel, one launch: (1) the chunk's fp32 K and V split
// exactly into three bf16 parts ([3][C][H_kv * d] each), (2) the attended
// cached rows (init U selected U local, through the page table) gathered
// into contiguous [n_att_max][H_kv * d] copies, a warp per row, zeros from
// the attended count to n_att_max -- so every K/V tile
// of the attention kernel is two plain TMA boxes (a row gather per tile,
// TMA gather4 or cp.async, issues an order of magnitude slower).
__global__ void prep_tc_kernel(PrefillAttendParams p, uint16_t* __restrict__ kc3, uint16_t* __restrict__ vc3,
                               uint16_t* __restrict__ kg, uint16_t* __restrict__ vg, unsigned* __restrict__ cnt,
                               int n_units) {
  const int n = p.C * p.H_kv * kD;
  const int stride = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  grid_dep_launch();  // (the attention kernel waits for this grid's completion before reading its results)
  if (blockIdx.x == 0)
    for (int u = threadIdx.x; u < n_units; u += blockDim.x) cnt[u] = 0u;  // the split units' piece counters
  // (1) the chunk's K / V -> three exact bf16 parts, four elements per
  // thread (an input: this runs while the selection launch before it ends,
  // this kernel being launched programmatically after it)
  const int n4 = n >> 2;  // (n: a multiple of kD)
  for (int i = gtid; i < 2 * n4; i += stride) {
    const bool v = i >= n4;
    const int j = v ? i - n4 : i;
    const float4 x = __ldg(reinterpret_cast<const float4*>(v ? p.v_cur : p.k_cur) + j);
    float h[4], m[4], l[4];
    sp3(x.x, h[0], m[0], l[0]);
    sp3(x.y, h[1], m[1], l[1]);
    sp3(x.z, h[2], m[2], l[2]);
    sp3(x.w, h[3], m[3], l[3]);
    uint2* out = reinterpret_cast<uint2*>(v ? vc3 : kc3);
    out[j] = make_uint2(pk2(h[0], h[1]), pk2(h[2], h[3]));
    out[n4 + j] = make_uint2(pk2(m[0], m[1]), pk2(m[2], m[3]));
    out[2 * n4 + j] = make_uint2(pk2(l[0], l[1]), pk2(l[2], l[3]));
  }
  grid_dep_wait();  // the selection (and its count) complete
  // (2) the attended list: explicit (p.att), or the implicit windows around
  // the selection -- its split points by counting (one pass over the
  // selection per CTA: one L2 round trip; a binary search is a chain of them)
  int ie = 0, lb = 0, c_ie = 0, c_lb = 0;
  if (p.win_n_att) {
    const int n_sel = p.win_sel && p.win_n_sel ? *p.win_n_sel : 0;
    ie = p.win_init_end;
    lb = max(p.win_local_begin, ie);
    for (int i = threadIdx.x; i < n_sel; i += blockDim.x) {
      const uint32_t t = __ldcg(p.win_sel + i);
      c_ie += t < static_cast<uint32_t>(ie);
      c_lb += t < static_cast<uint32_t>(p.win_local_begin);
    }
  }
  int n_cached, lo1 = 0, n1 = 0;
  if (p.win_n_att) {
    __shared__ int red[2][32];
    for (int o = 16; o > 0; o >>= 1) {
      c_ie += __shfl_xor_sync(0xffffffffu, c_ie, o);
      c_lb += __shfl_xor_sync(0xffffffffu, c_lb, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = c_ie;
      red[1][threadIdx.x >> 5] = c_lb;
    }
    __syncthreads();
    int a = 0, b = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    lo1 = a;
    n1 = p.win_local_begin > ie ? max(0, b - a) : 0;
    n_cached = ie + n1 + max(0, p.win_cached - lb);
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.win_n_att = n_cached;
  } else {
    n_cached = p.n_att_ptr ? *p.n_att_ptr : p.n_att;
  }
  // (3) the attended rows, gathered: a warp per row, all of a lane's loads
  // in flight before its stores. Rows past the attended count, up to the
  // planned bound, are zeros (the attention kernel's tile grid follows the
  // bound)
  constexpr int kPerLane = 4;  // 16-byte vectors per lane and pass (a whole row for H_kv <= 8)
  const int n_rows = p.n_att_max;
  const int row_vec = p.H_kv * kD / 8;  // 16-byte vectors per row
  const int lane = threadIdx.x & 31;
  for (int key = gtid >> 5; key < n_rows; key += stride >> 5) {
    uint4* kd = reinterpret_cast<uint4*>(kg + static_cast<size_t>(key) * row_vec * 8);
    uint4* vd = reinterpret_cast<uint4*>(vg + static_cast<size_t>(key) * row_vec * 8);
    if (key < n_cached) {
      const uint32_t tok = !p.win_n_att ? p.att[key]
                                 : key < ie ? static_cast<uint32_t>(key)
                                 : key < ie + n1 ? __ldcg(p.win_sel + lo1 + key - ie)
                                                 : static_cast<uint32_t>(lb + key - ie - n1);
      const int32_t ri = p.page_size == 1 ? p.page_table[tok]
                                          : p.page_table[tok / p.page_size] * p.page_size + static_cast<int32_t>(tok % p.page_size);
      const uint4* ks = reinterpret_cast<const uint4*>(p.k_slab + static_cast<size_t>(ri) * row_vec * 8);
      const uint4* vs = reinterpret_cast<const uint4*>(p.v_slab + static_cast<size_t>(ri) * row_vec * 8);
      for (int c0 = 0; c0 < row_vec; c0 += 32 * kPerLane) {
        uint4 kb[kPerLane], vb[kPerLane];
#pragma unroll
        for (int u = 0; u < kPerLane; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c < row_vec) {
            kb[u] = __ldg(ks + c);
            vb[u] = __ldg(vs + c);
          }
        }
#pragma unroll
        for (int u = 0; u < kPerLane; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c < row_vec) {
            kd[c] = kb[u];
            vd[c] = vb[u];
          }
        }
      }
    } else {
      for (int c = lane; c < row_vec; c += 32) kd[c] = vd[c] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

}  // namespace

namespace {

using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D bf16 tensor map over [rows][width] (row pitch = width), box = 64 x 64,
// 128B swizzle; false when the encoder is unavailable
bool encode_2d(CUtensorMap* m, const void* base, size_t width, size_t rows) {
  static TmapEncodeFn enc = []() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<TmapEncodeFn>(nullptr);
    return reinterpret_cast<TmapEncodeFn>(f);
  }();
  if (!enc) return false;
  const cuuint64_t dims[2] = {width, rows};
  const cuuint64_t strides[1] = {width * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kKT)};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the maps of the last workspace layout seen, re-encoded when it changes
struct MapCache {
  std::mutex mu;
  const void* ws = nullptr;
  size_t rows = 0, width = 0, c = 0;
  alignas(64) CUtensorMap tkg, tvg, tkc, tvc;
};

}  // namespace

namespace {

// The work plan of one launch shape (host; cached with its device copy).
struct TcPlan {
  int grid = 0, nct = 0, n_units = 0, n_slots = 0;
  std::vector<TcWork> work;
  std::vector<int16_t> slot0, np;
  void* dev = nullptr;  // [work | slot0 | np]
};

// Equal-cost contiguous ranges of the units' concatenated tiles (KV-head
// major, so neighbouring pieces share K/V columns), one per SM. A chunk tile
// costs ~2.2 cached tiles (three K and three V parts; measured 3.6 vs 1.6 us).
// Falls back to one unit per CTA (no split) when a CTA would need more than
// kMaxPieces pieces or TS_PREFILL_NO_SPLIT is set.
TcPlan make_tc_plan(int C, int H, int H_kv, int n_att_max, int n_sms) {
  const int G = H / H_kv, rph = kM / G;
  const int nx = (C + rph - 1) / rph;
  TcPlan pl;
  pl.nct = (n_att_max + kKT - 1) / kKT;
  pl.n_units = nx * H_kv;
  auto tiles = [&](int x) { return pl.nct + (min(C, (x + 1) * rph) + kKT - 1) / kKT; };
  static const long chunk_cost = std::getenv("TS_PREFILL_CCOST") ? std::atol(std::getenv("TS_PREFILL_CCOST")) : 22L;
  auto cost = [&](int t) { return t < pl.nct ? 10L : chunk_cost; };
  long W = 0;
  for (int x = 0; x < nx; ++x)
    for (int t = 0; t < tiles(x); ++t) W += H_kv * cost(t);
  auto unsplit = [&]() {
    pl.grid = pl.n_units;
    pl.n_slots = 0;
    pl.work.assign(pl.grid, TcWork{});
    pl.slot0.assign(pl.n_units, -1);
    pl.np.assign(pl.n_units, 1);
    for (int g = 0; g < H_kv; ++g)
      for (int x = 0; x < nx; ++x) {
        const int u = g * nx + x;
        TcWork& w = pl.work[u];
        w.n = 1;
        w.pc[0] = TcPiece{static_cast<int16_t>(x), static_cast<int16_t>(g), 0, static_cast<int16_t>(tiles(x)), -1,
                          static_cast<int16_t>(u)};
      }
  };
  static const bool no_split = std::getenv("TS_PREFILL_NO_SPLIT") != nullptr;
  if (no_split || pl.n_units >= n_sms || pl.nct + nx > 30000) {
    unsplit();
    return pl;
  }
  pl.grid = n_sms;
  pl.work.assign(pl.grid, TcWork{});
  std::vector<int> pieces(pl.n_units, 0);
  int c = 0;
  long acc = 0;
  // no sliver pieces: a piece costs a pipeline drain and refill (and a merge
  // when its unit is split), so a unit that would start with less than kSliver
  // of a CTA's budget left starts on the next CTA, and a unit within kSliver
  // of its end is finished where it is
  constexpr long kSliver = 60;  // (6 cached tiles)
  for (int g = 0; g < H_kv; ++g)
    for (int x = 0; x < nx; ++x) {
      const int u = g * nx + x;
      long rem = 0;
      for (int t = 0; t < tiles(x); ++t) rem += cost(t);
      if (c < pl.grid - 1 && pl.work[c].n > 0 && W * (c + 1) / pl.grid - acc < kSliver) ++c;
      for (int t = 0; t < tiles(x); ++t) {
        if (acc >= W * (c + 1) / pl.grid && c < pl.grid - 1 && rem > kSliver) ++c;
        rem -= cost(t);
        TcWork& w = pl.work[c];
        if (w.n == 0 || w.pc[w.n - 1].unit != u) {
          if (w.n == kMaxPieces) {
            unsplit();
            return pl;
          }
          w.pc[w.n++] = TcPiece{static_cast<int16_t>(x), static_cast<int16_t>(g), static_cast<int16_t>(t),
                                static_cast<int16_t>(t + 1), -1, static_cast<int16_t>(u)};
          ++pieces[u];
        } else {
          w.pc[w.n - 1].t1 = static_cast<int16_t>(t + 1);
        }
        acc += cost(t);
      }
    }
  pl.slot0.assign(pl.n_units, -1);
  pl.np.assign(pl.n_units, 1);
  std::vector<int> next(pl.n_units, 0);
  for (int u = 0; u < pl.n_units; ++u)
    if (pieces[u] > 1) {
      pl.slot0[u] = static_cast<int16_t>(pl.n_slots);
      pl.np[u] = static_cast<int16_t>(pieces[u]);
      pl.n_slots += pieces[u];
    }
  for (TcWork& w : pl.work)  // CTA order = each unit's piece order
    for (int k = 0; k < w.n; ++k) {
      TcPiece& pc = w.pc[k];
      if (pieces[pc.unit] > 1) pc.slot = static_cast<int16_t>(pl.slot0[pc.unit] + next[pc.unit]++);
    }
  return pl;
}

// Plans by shape, kept for the process's lifetime: a plan depends on the
// cached tiles (ceil(n_att_max / 64)), not on n_att_max itself, so a growing
// context makes a few dozen at most; entries never move or free, so a
// concurrent launch from another thread never sees its plan released.
struct PlanCache {
  std::mutex mu;
  std::map<std::array<int, 5>, TcPlan> plans;
};

// the cached plan of this shape (made and uploaded on first use)
const TcPlan& tc_plan(const PrefillAttendParams& p, cudaStream_t st, cudaError_t* err) {
  static PlanCache pc;
  static int n_sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  (void)st;
  std::lock_guard<std::mutex> lk(pc.mu);
  const std::array<int, 5> key = {p.C, p.H, p.H_kv, (p.n_att_max + kKT - 1) / kKT, n_sms};
  *err = cudaSuccess;
  auto it = pc.plans.find(key);
  if (it != pc.plans.end() && it->second.dev) return it->second;
  TcPlan& pl = pc.plans[key];
  pl = make_tc_plan(p.C, p.H, p.H_kv, p.n_att_max, n_sms);
  const size_t wb = pl.work.size() * sizeof(TcWork), ub = pl.n_units * sizeof(int16_t);
  std::vector<uint8_t> h(wb + 2 * ub);
  std::memcpy(h.data(), pl.work.data(), wb);
  std::memcpy(h.data() + wb, pl.slot0.data(), ub);
  std::memcpy(h.data() + wb + ub, pl.np.data(), ub);
  void* d = nullptr;
  if ((*err = cudaMalloc(&d, h.size())) != cudaSuccess) return pl;
  if ((*err = cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
    cudaFree(d);
    return pl;
  }
  pl.dev = d;
  return pl;
}

size_t tc_split_bytes(const TcPlan& pl) {
  return (static_cast<size_t>(pl.n_slots) * kM * (kD + 2) * 4 + static_cast<size_t>(pl.n_units) * 4 + 255) / 256 * 256;
}

}  // namespace

size_t prefill_tc_extra_ws_bytes(const PrefillAttendParams& p, cudaStream_t st) {
  cudaError_t e;
  const TcPlan& pl = tc_plan(p, st, &e);
  return e == cudaSuccess ? tc_split_bytes(pl) : 0;
}

cudaError_t launch_prefill_tc(const PrefillAttendParams& p, cudaStream_t st) {
  const int G = p.H / p.H_kv;
  if (p.d != kD || p.H % p.H_kv != 0 || G < 1 || G > 16 || p.page_size < 1 || !p.split_ws || p.n_att_max < 0)
    return cudaErrorInvalidValue;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const size_t width = static_cast<size_t>(p.H_kv) * kD;
  const size_t n = static_cast<size_t>(p.C) * width;
  uint16_t* kc3 = p.split_ws;
  uint16_t* vc3 = kc3 + 3 * n;
  uint16_t* kg = vc3 + 3 * n;
  uint16_t* vg = kg + static_cast<size_t>(p.n_att_max) * width;
  cudaError_t perr;
  const TcPlan& pl = tc_plan(p, st, &perr);
  if (perr != cudaSuccess) return perr;
  // the split units' partials and piece counters, after the gathered rows
  uint8_t* xs = reinterpret_cast<uint8_t*>(vg + static_cast<size_t>(p.n_att_max) * width);
  xs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(xs) + 255) & ~static_cast<uintptr_t>(255));
  TcSplit sp{};
  sp.work = static_cast<const TcWork*>(pl.dev);
  sp.unit_slot0 = reinterpret_cast<const int16_t*>(static_cast<const uint8_t*>(pl.dev) + pl.work.size() * sizeof(TcWork));
  sp.unit_np = sp.unit_slot0 + pl.n_units;
  sp.part_o = reinterpret_cast<float*>(xs);
  sp.part_ml = sp.part_o + static_cast<size_t>(pl.n_slots) * kM * kD;
  sp.cnt = reinterpret_cast<unsigned*>(sp.part_ml + static_cast<size_t>(pl.n_slots) * kM * 2);
  sp.nct = pl.nct;
  static const int fold_every = std::getenv("TS_PREFILL_FOLD1") ? 1
                               : std::getenv("TS_PREFILL_FOLD") ? std::max(1, std::atoi(std::getenv("TS_PREFILL_FOLD")))
                                                                : 2;
  sp.fold = fold_every;
  static const bool p3 = std::getenv("TS_PREFILL_P3") != nullptr;  // (A/B: the exact three-part P)
  sp.p3 = p3 ? 1 : 0;
  const size_t g_rows = std::max(p.n_att_max, 1);
  static MapCache mc;
  alignas(64) CUtensorMap tkg, tvg, tkc, tvc;
  {
    std::lock_guard<std::mutex> lk(mc.mu);
    // (keyed on n_att_max itself: it also places vg, and a reallocated
    // workspace can come back at the same address)
    if (mc.ws != kc3 || mc.c != static_cast<size_t>(p.C) || mc.width != width || mc.rows != static_cast<size_t>(p.n_att_max)) {
      mc.ws = nullptr;
      if (!encode_2d(&mc.tkc, kc3, width, 3 * static_cast<size_t>(p.C)) || !encode_2d(&mc.tvc, vc3, width, 3 * static_cast<size_t>(p.C)) ||
          !encode_2d(&mc.tkg, kg, width, g_rows) || !encode_2d(&mc.tvg, vg, width, g_rows))
        return cudaErrorNotSupported;
      mc.ws = kc3, mc.c = p.C, mc.width = width, mc.rows = static_cast<size_t>(p.n_att_max);
    }
    tkg = mc.tkg, tvg = mc.tvg, tkc = mc.tkc, tvc = mc.tvc;
  }
  static const bool no_pdl = std::getenv("TS_NO_PDL") != nullptr;
  {
    // programmatic launch after the selection launch (its chunk split
    // overlaps the selection's end; it waits before reading the selection)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * 148);
    cfg.blockDim = dim3(512);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t pe = cudaLaunchKernelEx(&cfg, prep_tc_kernel, p, kc3, vc3, kg, vg, sp.cnt, pl.n_units);
    if (pe != cudaSuccess) return pe;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t le = cudaLaunchKernelEx(&cfg, prefill_tc_kernel, p, sp, tkg, tvg, tkc, tvc);
  if (le != cudaSuccess) return le;
  return cudaGetLastError();
}

}  // namespace tsb

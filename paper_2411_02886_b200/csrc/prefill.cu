// Chunked-prefill sparse attention on tensor cores (sm_100a): the C-row
// (C = chunk_size, 512 in BASELINE configs[4]) case of sparse_attend
// (attention.cpp:114-123 -> sdpa_full :54-112). Query row i of the chunk
// attends every merged cached row (init U selected U local windows, gathered
// through the page table) and the chunk's own rows j <= i (causal, :83).
//
// One CTA = 32 (or 16) chunk rows x the G query heads sharing KV head g
// (h mod H_kv, :78); one warp per (head, 16-row tile). Per key tile of 32 rows:
//   S = Q K^T   mma.sync m16n8k16 bf16 -> fp32; Q (fp32) split exactly into
//               three bf16 parts; cached K is bf16 (exact); the chunk's own K
//               (fp32 in the reference) is split into three parts as well, so
//               every product the reference forms is formed exactly here
//   online softmax per row (fp32), P = e^(S - m)
//   O += P V    P split into three bf16 parts (A from the S accumulators,
//               FA2 register reuse), V^T via ldmatrix.trans; chunk V split too
// Cached K/V slices (d wide, this KV head) arrive by 16-byte cp.async into
// padded rows (ldmatrix conflict-free), double-buffered (the next tile's
// gather is in flight while this one is computed), 32 keys per tile.
#include <cfloat>
#include <cmath>

#include "aux.h"
#include "common.cuh"

namespace tsb {

namespace {

constexpr int kPD = 128;          // head dim of the tensor-core path
constexpr int kPRS = kPD + 8;     // padded smem row (bf16 elements)
constexpr int kPKT = 32;          // keys per tile
constexpr int kPMaxG = 8;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
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
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t (&r)[2], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ uint16_t bf(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
__device__ __forceinline__ uint32_t pk(float lo, float hi) {
  return static_cast<uint32_t>(bf(lo)) | (static_cast<uint32_t>(bf(hi)) << 16);
}
// x = hi + mid + lo exactly (each a bf16)
__device__ __forceinline__ void sp3(float x, float& h, float& m, float& l) {
  h = __bfloat162float(__float2bfloat16_rn(x));
  const float r = x - h;
  m = __bfloat162float(__float2bfloat16_rn(r));
  l = r - m;
}

// One 32-key tile for this warp's 16 rows: S = Q K^T (KP parts of K), mask,
// online softmax, O += P V (KP parts of V). `key_of(c)` maps tile column c
// to its visibility for fragment row `i`.
template <int KP>
__device__ __forceinline__ void flash_tile(const uint32_t qbase, const uint32_t qpart, const uint16_t* kb,
                                           const uint16_t* vb, float scale, int lane, bool chunk_tile, int k0,
                                           int n_valid, int i_lo, float (&o)[kPD / 8][4], float (&mrow)[2],
                                           float (&lrow)[2]) {
  float s[kPKT / 8][4];
#pragma unroll
  for (int n = 0; n < kPKT / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll 2
  for (int kc = 0; kc < kPD / 16; ++kc) {
    uint32_t a[3][4];
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) ldsm_x4(a[pq], qbase + pq * qpart + kc * 32);
#pragma unroll
    for (int n = 0; n < kPKT / 8; ++n) {
#pragma unroll
      for (int pkk = 0; pkk < KP; ++pkk) {
        uint32_t bb[2];
        // B (K^T, "col"): rows = keys n*8 + (lane & 7), 16 B of d at kc*16 + (lane>>3 & 1)*8
        ldsm_x2(bb, smem_u32(kb) + static_cast<uint32_t>(((pkk * kPKT + n * 8 + (lane & 7)) * kPRS + kc * 16 +
                                                           ((lane >> 3) & 1) * 8) * 2));
        mma16816(s[n], a[0], bb[0], bb[1]);
        mma16816(s[n], a[1], bb[0], bb[1]);
        if (pkk == 0) mma16816(s[n], a[2], bb[0], bb[1]);  // q_lo x k_mid/lo fall below fp32 resolution
      }
    }
  }
  // mask: cached tile -> column valid if < n_valid; chunk tile -> row i sees chunk rows j <= i
  float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int n = 0; n < kPKT / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = k0 + n * 8 + (lane & 3) * 2 + (e & 1);
      const int i = i_lo + (e >> 1) * 8;
      const bool ok = c < n_valid && (!chunk_tile || c <= i);
      s[n][e] = ok ? s[n][e] * scale : -INFINITY;
      mt[e >> 1] = fmaxf(mt[e >> 1], s[n][e]);
    }
  float corr[2], mnew[2], ls[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mt[h] = fmaxf(mt[h], __shfl_xor_sync(0xffffffffu, mt[h], 1));
    mt[h] = fmaxf(mt[h], __shfl_xor_sync(0xffffffffu, mt[h], 2));
    mnew[h] = fmaxf(mrow[h], mt[h]);
    corr[h] = mrow[h] == -INFINITY ? 0.f : expf(mrow[h] - mnew[h]);
    mrow[h] = mnew[h];
  }
#pragma unroll
  for (int n = 0; n < kPKT / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = e >> 1;
      const float w = mnew[h] == -INFINITY ? 0.f : expf(s[n][e] - mnew[h]);
      s[n][e] = w;
      ls[h] += w;
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    ls[h] += __shfl_xor_sync(0xffffffffu, ls[h], 1);
    ls[h] += __shfl_xor_sync(0xffffffffu, ls[h], 2);
    lrow[h] = lrow[h] * corr[h] + ls[h];
  }
#pragma unroll
  for (int n = 0; n < kPD / 8; ++n) {
    o[n][0] *= corr[0];
    o[n][1] *= corr[0];
    o[n][2] *= corr[1];
    o[n][3] *= corr[1];
  }
  // O += P V over k-steps of 16 keys: A = P from the S accumulators (FA2 reuse)
#pragma unroll
  for (int ks = 0; ks < kPKT / 16; ++ks) {
    uint32_t pa[3][4];
    {
      const float x[8] = {s[2 * ks][0], s[2 * ks][1], s[2 * ks][2], s[2 * ks][3],
                          s[2 * ks + 1][0], s[2 * ks + 1][1], s[2 * ks + 1][2], s[2 * ks + 1][3]};
      float hh[8], mm[8], ll[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) sp3(x[u], hh[u], mm[u], ll[u]);
      // a0 = (row r, keys 2t..2t+1), a1 = (row r+8), a2 = (row r, keys 8+2t..), a3 = (row r+8)
      pa[0][0] = pk(hh[0], hh[1]); pa[0][1] = pk(hh[2], hh[3]); pa[0][2] = pk(hh[4], hh[5]); pa[0][3] = pk(hh[6], hh[7]);
      pa[1][0] = pk(mm[0], mm[1]); pa[1][1] = pk(mm[2], mm[3]); pa[1][2] = pk(mm[4], mm[5]); pa[1][3] = pk(mm[6], mm[7]);
      pa[2][0] = pk(ll[0], ll[1]); pa[2][1] = pk(ll[2], ll[3]); pa[2][2] = pk(ll[4], ll[5]); pa[2][3] = pk(ll[6], ll[7]);
    }
#pragma unroll
    for (int n = 0; n < kPD / 8; ++n) {
#pragma unroll
      for (int pv = 0; pv < KP; ++pv) {
        uint32_t bb[2];
        // B (V, k = keys x n = d): ldmatrix.trans of rows (keys) ks*16 + (lane & 15), d columns n*8..
        ldsm_x2_trans(bb, smem_u32(vb) + static_cast<uint32_t>(((pv * kPKT + ks * 16 + (lane & 15)) * kPRS + n * 8) * 2));
        mma16816(o[n], pa[0], bb[0], bb[1]);
        mma16816(o[n], pa[1], bb[0], bb[1]);
        if (pv == 0) mma16816(o[n], pa[2], bb[0], bb[1]);
      }
    }
  }
}

// Chunk K/V (fp32) -> three exact bf16 parts, [part][C][H_kv * d], once per
// chunk (every CTA of the attention then stages them with cp.async).
__global__ void split3_kernel(const float* __restrict__ x, int n, uint16_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float h, m, l;
    sp3(x[i], h, m, l);
    out[i] = bf(h);
    out[n + i] = bf(m);
    out[2 * static_cast<size_t>(n) + i] = bf(l);
  }
}

// One CTA = kPQ (32) chunk rows x the G query heads of KV head g; warp w
// takes head w % G and the 16-row tile w / G. The merged cached rows' slab
// rows are resolved once per CTA (att list -> page table) into shared memory,
// and the 32-key K/V tiles are double-buffered: tile t + 1's cp.async gather
// is in flight while tile t is computed.
constexpr int kPRowsMax = 4096;  // merged cached rows resolved up front (else per tile)

template <int kPQ>  // chunk rows per CTA: 32 (two m16 tiles) when the smem fits, else 16
__global__ void __launch_bounds__(256) prefill_flash_kernel(PrefillAttendParams p, const uint16_t* kc3,  // <= 8 warps (rq 32: G <= 4)
                                                                        const uint16_t* vc3) {
  extern __shared__ __align__(128) uint8_t psm_raw[];
  const int G = p.H / p.H_kv;
  const int g = blockIdx.y;
  const int i0 = blockIdx.x * kPQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % G, wt = warp / G;  // head, 16-row tile
  const int nthr = blockDim.x;
  const int row_elems = p.H_kv * kPD;
  const int n_cached = p.n_att_ptr ? *p.n_att_ptr : p.n_att;
  const int n_cur = min(p.C, i0 + kPQ);                  // chunk rows any row here can see
  const int nct = (n_cached + kPKT - 1) / kPKT;          // cached tiles, then chunk tiles
  const int n_tiles = nct + (n_cur + kPKT - 1) / kPKT;
  const size_t qbytes = static_cast<size_t>(3) * G * kPQ * kPRS * 2;
  const size_t tbytes = static_cast<size_t>(3) * kPKT * kPRS * 2;
  uint16_t* sq = reinterpret_cast<uint16_t*>(psm_raw);  // [3][G * kPQ][kPRS], row = head * kPQ + i
  uint16_t* kbuf[2] = {reinterpret_cast<uint16_t*>(psm_raw + qbytes), reinterpret_cast<uint16_t*>(psm_raw + qbytes + 2 * tbytes)};
  uint16_t* vbuf[2] = {reinterpret_cast<uint16_t*>(psm_raw + qbytes + tbytes),
                       reinterpret_cast<uint16_t*>(psm_raw + qbytes + 3 * tbytes)};
  int32_t* rows_all = reinterpret_cast<int32_t*>(psm_raw + qbytes + 4 * tbytes);  // [kPRowsMax]
  const bool rows_up_front = n_cached <= kPRowsMax;
  auto lookup = [&](int key) -> int32_t {
    const uint32_t tok = p.att[key];
    return p.page_size == 1 ? p.page_table[tok]
                            : p.page_table[tok / p.page_size] * p.page_size + static_cast<int32_t>(tok % p.page_size);
  };

  // ---- Q parts: row (m, i) = q[i0 + i][(g + m*H_kv) * d + :]; slab rows of the cached keys
  for (int idx = threadIdx.x; idx < G * kPQ * kPD; idx += nthr) {
    const int r = idx / kPD, t = idx - (idx / kPD) * kPD;
    const int m = r / kPQ, i = r - (r / kPQ) * kPQ;
    const float x = (i0 + i < p.C) ? p.q[static_cast<size_t>(i0 + i) * p.H * kPD + (g + m * p.H_kv) * kPD + t] : 0.f;
    float h, mm, l;
    sp3(x, h, mm, l);
    sq[(0 * G * kPQ + r) * kPRS + t] = bf(h);
    sq[(1 * G * kPQ + r) * kPRS + t] = bf(mm);
    sq[(2 * G * kPQ + r) * kPRS + t] = bf(l);
  }
  if (rows_up_front)
    for (int key = threadIdx.x; key < n_cached; key += nthr) rows_all[key] = lookup(key);
  __syncthreads();

  constexpr int CPR = kPD * 2 / 16;  // 16-byte chunks per row slice
  auto issue = [&](int tile, int b) {
    uint16_t* kb = kbuf[b];
    uint16_t* vb = vbuf[b];
    if (tile < nct) {
      const int k0 = tile * kPKT;
      for (int idx = threadIdx.x; idx < kPKT * CPR; idx += nthr) {
        const int r = idx / CPR, c = idx - (idx / CPR) * CPR;
        const int key = k0 + r;
        const int32_t ri = key < n_cached ? (rows_up_front ? rows_all[key] : lookup(key)) : -1;
        if (ri >= 0) {
          const int64_t off = static_cast<int64_t>(ri) * row_elems + static_cast<int64_t>(g) * kPD + c * 8;
          cp_async16(kb + r * kPRS + c * 8, p.k_slab + off);
          cp_async16(vb + r * kPRS + c * 8, p.v_slab + off);
        } else {  // padding row: zero (P is zero there; keep 0 * V finite)
          *reinterpret_cast<uint4*>(kb + r * kPRS + c * 8) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(vb + r * kPRS + c * 8) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    } else {
      const int j0 = (tile - nct) * kPKT;
      for (int idx = threadIdx.x; idx < 3 * kPKT * CPR; idx += nthr) {
        const int pp = idx / (kPKT * CPR), rem = idx - pp * (kPKT * CPR);
        const int r = rem / CPR, c = rem - (rem / CPR) * CPR;
        const int j = j0 + r;
        uint16_t* kd = kb + (pp * kPKT + r) * kPRS + c * 8;
        uint16_t* vd = vb + (pp * kPKT + r) * kPRS + c * 8;
        if (j < n_cur) {
          const size_t off = static_cast<size_t>(pp) * p.C * row_elems + static_cast<size_t>(j) * row_elems +
                             static_cast<size_t>(g) * kPD + c * 8;
          cp_async16(kd, kc3 + off);
          cp_async16(vd, vc3 + off);
        } else {
          *reinterpret_cast<uint4*>(kd) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(vd) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
    cp_async_commit();
  };

  float o[kPD / 8][4];
#pragma unroll
  for (int n = 0; n < kPD / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int r_lo = lane >> 2;  // fragment rows r_lo, r_lo + 8 of this warp's 16
  const uint32_t qbase = smem_u32(sq) + static_cast<uint32_t>(
                             ((wm * kPQ + wt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * kPRS + (lane >> 4) * 8) * 2);
  const uint32_t qpart = static_cast<uint32_t>(G * kPQ * kPRS * 2);
  const int i_lo = i0 + wt * 16 + r_lo;

  if (n_tiles > 0) issue(0, 0);
  for (int tile = 0; tile < n_tiles; ++tile) {
    if (tile + 1 < n_tiles) {
      issue(tile + 1, (tile + 1) & 1);  // that buffer's tile (tile - 1) was consumed before the last barrier
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int b = tile & 1;
    if (tile >= nct)
      flash_tile<3>(qbase, qpart, kbuf[b], vbuf[b], p.scale, lane, true, (tile - nct) * kPKT, n_cur, i_lo, o, mrow,
                    lrow);
    else
      flash_tile<1>(qbase, qpart, kbuf[b], vbuf[b], p.scale, lane, false, tile * kPKT, n_cached, 0, o, mrow, lrow);
    __syncthreads();  // buffer b is free for tile + 2
  }
  // ---- normalise and store rows r_lo, r_lo + 8 of head wm, tile wt
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = i_lo + h * 8;
    if (i >= p.C) continue;
    const float inv = 1.f / lrow[h];
    float* orow = p.out + static_cast<size_t>(i) * p.H * kPD + (g + wm * p.H_kv) * kPD;
#pragma unroll
    for (int n = 0; n < kPD / 8; ++n) {
      const int t = n * 8 + (lane & 3) * 2;
      *reinterpret_cast<float2*>(orow + t) = make_float2(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
    }
  }
}

}  // namespace

size_t prefill_flash_smem(int G, int rq) {
  return static_cast<size_t>(3) * G * rq * kPRS * 2 + static_cast<size_t>(4) * 3 * kPKT * kPRS * 2 + kPRowsMax * 4;
}

cudaError_t launch_prefill_flash(const PrefillAttendParams& p, cudaStream_t st) {
  const int G = p.H / p.H_kv;
  if (p.d != kPD || G > kPMaxG || p.page_size < 1 || !p.split_ws) return cudaErrorInvalidValue;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int rq = (G <= 4 && prefill_flash_smem(G, 32) <= static_cast<size_t>(optin)) ? 32 : 16;  // <= 8 warps
  const size_t smem = prefill_flash_smem(G, rq);
  const void* fn = rq == 32 ? reinterpret_cast<const void*>(&prefill_flash_kernel<32>)
                            : reinterpret_cast<const void*>(&prefill_flash_kernel<16>);
  static size_t set[2] = {0, 0};
  if (smem > set[rq == 32]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    set[rq == 32] = smem;
  }
  const int n = p.C * p.H_kv * kPD;
  uint16_t* kc3 = p.split_ws;
  uint16_t* vc3 = p.split_ws + 3 * static_cast<size_t>(n);
  split3_kernel<<<148, 512, 0, st>>>(p.k_cur, n, kc3);
  split3_kernel<<<148, 512, 0, st>>>(p.v_cur, n, vc3);
  dim3 grid((p.C + rq - 1) / rq, p.H_kv);
  if (rq == 32) prefill_flash_kernel<32><<<grid, G * 2 * 32, smem, st>>>(p, kc3, vc3);
  else prefill_flash_kernel<16><<<grid, G * 32, smem, st>>>(p, kc3, vc3);
  return cudaGetLastError();
}

}  // namespace tsb

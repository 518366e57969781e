// Auxiliary sm_100a kernels around the fused decode step:
//   K1  kv_append      PagedKvPool::append_kv row copy (kv_pool.cpp:55-85), fp32 -> bf16
//       kv_gather      PagedKvPool::gather (kv_pool.cpp:87-101), bf16 -> fp32
//   K9  chunk_mean     tensor.cpp:133-150 (fp64 column sums, x 1/c, round to fp32)
//   K6  windows        make_windows + merged() (attention.cpp:35-52), device list
//       prefill_attend sparse_attend for a C-row chunk (attention.cpp:114-123 with
//                      sdpa_full's causal mask :83), CUDA-core flash attention
//       max_index      bounds check for explicit index lists (kv_pool.cpp:92-95)
#include <cfloat>
#include <cmath>
#include <algorithm>

#include "aux.h"
#include "common.cuh"

namespace tsb {

namespace {

// Destination slab rows: dst_rows[r], or (dst_rows == nullptr) through the
// sequence's page table for logical positions pos0 + r.
__global__ void kv_append_kernel(uint16_t* k_slab, uint16_t* v_slab, const float* k, const float* v,
                                 const uint16_t* kb, const uint16_t* vb, const int64_t* dst_rows,
                                 const int32_t* pt, int64_t pos0, int page_size, int t, int row) {
  const int64_t total = static_cast<int64_t>(t) * row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row, c = i - (i / row) * row;
    const int64_t tok = pos0 + r;
    const int64_t dst = dst_rows ? dst_rows[r] : static_cast<int64_t>(pt[tok / page_size]) * page_size + tok % page_size;
    const int64_t off = dst * row + c;
    if (k) {
      k_slab[off] = __bfloat16_as_ushort(__float2bfloat16_rn(k[i]));
      v_slab[off] = __bfloat16_as_ushort(__float2bfloat16_rn(v[i]));
    } else {
      k_slab[off] = kb[i];
      v_slab[off] = vb[i];
    }
  }
  // launched programmatically after the prefill attention (which reads none
  // of these rows): done only once that grid is, so later work on the stream
  // sees both complete (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__global__ void kv_gather_kernel(const uint16_t* k_slab, const uint16_t* v_slab, const int64_t* src_rows,
                                 int n, int row, float* k_out, float* v_out) {
  const int64_t total = static_cast<int64_t>(n) * row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row, c = i - (i / row) * row;
    const int64_t off = src_rows[r] * row + c;
    if (k_out) k_out[i] = bf16_bits_to_f(k_slab[off]);
    if (v_out) v_out[i] = bf16_bits_to_f(v_slab[off]);
  }
}

// Sequential fp64 column sums in row order: bit-identical to chunk_mean
// (tensor.cpp:133-150). CTA = 16 columns (256 CTAs for a 4096-wide query);
// rows pass through shared memory in tiles of 256 by cp.async, two tiles in
// flight from the start (a 512-row chunk is loaded with one round trip), and
// a half warp adds each landed tile's rows in order (one dependent fp64 add
// per row and column -- the chain the reference's order imposes) while the
// next tile lands.
constexpr int kCmCols = 16, kCmTile = 256, kCmThr = 128;
__global__ void __launch_bounds__(kCmThr) chunk_mean_kernel(const float* q, int c, int width, float* out) {
  __shared__ __align__(16) float tile[2][kCmTile][kCmCols];
  constexpr int kVec = kCmCols / 4;                       // 16-byte pieces per row
  constexpr int kPer = kCmTile * kVec / kCmThr;           // pieces per thread per tile (8)
  const int tid = threadIdx.x;
  const int j0 = blockIdx.x * kCmCols;
  const int ntile = (c + kCmTile - 1) / kCmTile;
  const bool vec = (width & 3) == 0;  // rows 16-byte aligned
  auto issue = [&](int t) {
    const int r0 = t * kCmTile, nr = min(kCmTile, c - r0);
    float* buf = &tile[t & 1][0][0];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = tid + u * kCmThr, r = i / kVec, cv = (i % kVec) * 4;
      if (r >= nr) continue;
      const float* src = q + static_cast<size_t>(r0 + r) * width + j0 + cv;
      float* dst = buf + r * kCmCols + cv;
      if (vec && j0 + cv + 4 <= width) {
        cp_async16(dst, src);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e] = j0 + cv + e < width ? __ldg(src + e) : 0.f;
      }
    }
    cp_async_commit();
  };
  issue(0);
  if (ntile > 1) issue(1);
  else cp_async_commit();  // (an empty group: the wait below counts two)
  double acc = 0.0;
  for (int t = 0; t < ntile; ++t) {
    cp_async_wait<1>();  // tile t landed (tile t + 1 may still be in flight)
    __syncthreads();
    if (tid < kCmCols) {
      const int nr = min(kCmTile, c - t * kCmTile);
      const float* tc = &tile[t & 1][0][tid];
      int r = 0;
      for (; r + 8 <= nr; r += 8) {  // (the loads and conversions of 8 rows ahead of the add chain)
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = static_cast<double>(tc[(r + u) * kCmCols]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += x[u];
      }
      for (; r < nr; ++r) acc += static_cast<double>(tc[r * kCmCols]);
    }
    __syncthreads();  // (buffer t & 1 free)
    if (t + 2 < ntile) issue(t + 2);
    else cp_async_commit();
  }
  const int j = j0 + tid;
  if (tid < kCmCols && j < width) out[j] = static_cast<float>(acc * (1.0 / static_cast<double>(c)));
}

__global__ void max_index_kernel(const uint32_t* idx, int n, unsigned int* out) {
  unsigned int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = max(m, idx[i] + 1u);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__device__ __forceinline__ int lower_bound_dev(const uint32_t* a, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// make_windows + merged(): init [0,init_end) ++ sel filtered to
// [init_end, local_begin) ++ local [max(local_begin,init_end), cached).
// Selected indices >= cached are reported through *bad (gather would throw).
__global__ void windows_kernel(const uint32_t* sel, const int* n_sel_ptr, int n_sel_fixed,
                               int cached, int init_end, int local_begin, uint32_t* out,
                               int* n_out, unsigned int* bad) {
  const int n_sel = n_sel_ptr ? *n_sel_ptr : n_sel_fixed;
  const uint32_t ie = static_cast<uint32_t>(init_end);
  const uint32_t lb = static_cast<uint32_t>(local_begin > init_end ? local_begin : init_end);
  const int lo1 = lower_bound_dev(sel, n_sel, ie);
  const int hi1 = local_begin > init_end ? lower_bound_dev(sel, n_sel, static_cast<uint32_t>(local_begin)) : lo1;
  const int lo2 = lower_bound_dev(sel, n_sel, static_cast<uint32_t>(cached));
  const int n1 = hi1 > lo1 ? hi1 - lo1 : 0;
  const int nl = cached - static_cast<int>(lb);
  const int total = init_end + n1 + (nl > 0 ? nl : 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t t;
    if (i < init_end) t = static_cast<uint32_t>(i);
    else if (i < init_end + n1) t = sel[lo1 + i - init_end];
    else t = lb + static_cast<uint32_t>(i - init_end - n1);
    out[i] = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_out = total;
    if (lo2 < n_sel) atomicMax(bad, sel[lo2] + 1u);
  }
}

// ------------------------------------------------------------ prefill attn
// One CTA per (tile of QT query rows, kv head): the G query heads of the kv
// group share every staged K/V tile. Keys = the attended cached rows (via the
// page table) followed by the C current rows (fp32, causal).
constexpr int kQT = 4;      // query rows per CTA (one warp each)
constexpr int kKT = 32;     // keys per tile
constexpr int kMaxG = 8;
constexpr int kMaxDL = 8;   // d <= 256

__global__ void __launch_bounds__(kQT * 32) prefill_attend_kernel(PrefillAttendParams p) {
  extern __shared__ float psm[];
  const int d = p.d, G = p.H / p.H_kv;
  const int kvh = blockIdx.y;
  const int i0 = blockIdx.x * kQT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = i0 + warp;  // this warp's query row within the chunk
  const int ds = d + 1;     // padded fp32 row stride (conflict-free column reads)
  float* Ks = psm;
  float* Vs = Ks + kKT * ds;
  float* Qs = Vs + kKT * ds;  // [kQT][G][d]
  const int row = p.H_kv * d;
  // query rows of this warp into smem
  for (int idx = lane; idx < G * d; idx += 32) {
    const int g = idx / d, t = idx - (idx / d) * d;
    Qs[(warp * G + g) * d + t] = (i < p.C) ? p.q[static_cast<size_t>(i) * p.H * d + (g * p.H_kv + kvh) * d + t] : 0.f;
  }
  float m_run[kMaxG], l_run[kMaxG], o_run[kMaxG][kMaxDL];
#pragma unroll
  for (int g = 0; g < kMaxG; ++g) {
    m_run[g] = -INFINITY;
    l_run[g] = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxDL; ++u) o_run[g][u] = 0.f;
  }
  const int n_cached = p.n_att_ptr ? *p.n_att_ptr : p.n_att;
  const int last_q = min(p.C, i0 + kQT) - 1;
  const int n_keys = n_cached + last_q + 1;  // keys any row of this tile can see
  for (int k0 = 0; k0 < n_keys; k0 += kKT) {
    const int nk = min(kKT, n_keys - k0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nk * d; idx += blockDim.x) {
      const int r = idx / d, t = idx - (idx / d) * d;
      const int key = k0 + r;
      float kv, vv;
      if (key < n_cached) {
        const uint32_t tok = p.att[key];
        const int64_t rr = p.page_size == 1 ? static_cast<int64_t>(p.page_table[tok])
                                             : static_cast<int64_t>(p.page_table[tok / p.page_size]) * p.page_size + tok % p.page_size;
        kv = bf16_bits_to_f(p.k_slab[rr * row + kvh * d + t]);
        vv = bf16_bits_to_f(p.v_slab[rr * row + kvh * d + t]);
      } else {
        const int c = key - n_cached;
        kv = p.k_cur[static_cast<size_t>(c) * row + kvh * d + t];
        vv = p.v_cur[static_cast<size_t>(c) * row + kvh * d + t];
      }
      Ks[r * ds + t] = kv;
      Vs[r * ds + t] = vv;
    }
    __syncthreads();
    if (i >= p.C) continue;
    const int visible = n_cached + i + 1;  // causal bound for row i
    const int key = k0 + lane;
    const bool ok = lane < nk && key < visible;
    for (int g = 0; g < G; ++g) {
      const float* qg = Qs + (warp * G + g) * d;
      float s = -INFINITY;
      if (ok) {
        float acc = 0.f;
        for (int t = 0; t < d; ++t) acc = fmaf(qg[t], Ks[lane * ds + t], acc);
        s = acc * p.scale;
      }
      const float mt = warp_max(s);
      if (mt == -INFINITY) continue;
      const float m_new = fmaxf(m_run[g], mt);
      const float corr = expf(m_run[g] - m_new);
      const float w = ok ? expf(s - m_new) : 0.f;
      l_run[g] = l_run[g] * corr + warp_sum(w);
#pragma unroll
      for (int u = 0; u < kMaxDL; ++u) o_run[g][u] *= corr;
      for (int r = 0; r < nk; ++r) {
        const float wr = __shfl_sync(0xffffffffu, w, r);
        if (wr == 0.f) continue;
#pragma unroll
        for (int u = 0; u < kMaxDL; ++u) {
          const int t = lane + 32 * u;
          if (t < d) o_run[g][u] = fmaf(wr, Vs[r * ds + t], o_run[g][u]);
        }
      }
      m_run[g] = m_new;
    }
  }
  if (i >= p.C) return;
  for (int g = 0; g < G; ++g) {
    const float inv = 1.f / l_run[g];
    float* o = p.out + static_cast<size_t>(i) * p.H * d + (g * p.H_kv + kvh) * d;
#pragma unroll
    for (int u = 0; u < kMaxDL; ++u) {
      const int t = lane + 32 * u;
      if (t < d) o[t] = o_run[g][u] * inv;
    }
  }
}

// ------------------------------------------------------- sharded decode
// Global top-k over every shard's local top-k candidates:
// the global top-k under the total order (24-bit key prefix desc, position
// asc) is a subset of the union of the shards' local top-k under the same
// order, so selecting from the union is exact. Shards' lists are ascending
// and shards are ordered by position, so the concatenation is ascending and
// ties resolve by concatenation order. Then this shard's attended rows
// (local positions, ascending): its init rows, its selected rows filtered to
// the current windows (attention.cpp:35-52), its local-window rows.
constexpr int kMergeThreads = 1024;
constexpr int kMergeBins = 4096;

__device__ uint32_t block_scan_excl_1024(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = scratch[lane];
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    scratch[32 + lane] = wi - w;
    if (lane == 31) scratch[64] = wi;
  }
  __syncthreads();
  const uint32_t r = scratch[32 + warp] + inc - v;
  *total = scratch[64];
  __syncthreads();
  return r;
}

// bin b of `hist` (descending) holding the kk-th largest; above = count in higher bins
__device__ void merge_find_bin(const uint32_t* hist, uint32_t kk, uint32_t* scratch, int* bin, uint32_t* above) {
  constexpr int per = kMergeBins / kMergeThreads;
  const int t = threadIdx.x;
  uint32_t c[per], sum = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    c[i] = hist[kMergeBins - 1 - (t * per + i)];
    sum += c[i];
  }
  uint32_t tot;
  const uint32_t ex = block_scan_excl_1024(sum, scratch, &tot);
  if (ex < kk && ex + sum >= kk) {
    uint32_t acc = ex;
    for (int i = 0; i < per; ++i) {
      if (acc + c[i] >= kk) {
        scratch[80] = kMergeBins - 1 - (t * per + i);
        scratch[81] = acc;
        break;
      }
      acc += c[i];
    }
  }
  __syncthreads();
  *bin = static_cast<int>(scratch[80]);
  *above = scratch[81];
  __syncthreads();
}

__global__ void __launch_bounds__(kMergeThreads) shard_merge_kernel(const uint32_t* all, int world, int k,
                                                                   uint32_t ie, uint32_t lbs, uint32_t base,
                                                                   uint32_t n_r, uint32_t init_hi, uint32_t loc_lo,
                                                                   uint32_t* att, int* n_att) {
  __shared__ uint32_t hist[kMergeBins];
  __shared__ uint32_t scratch[128];
  __shared__ uint32_t offs[65];
  const int tid = threadIdx.x;
  const size_t stride = 2 * static_cast<size_t>(k) + 1;
  if (tid == 0) {
    uint32_t o = 0;
    for (int r = 0; r < world; ++r) {
      offs[r] = o;
      o += all[r * stride + 2 * k];
    }
    offs[world] = o;
  }
  __syncthreads();
  const uint32_t total = offs[world];
  auto entry = [&](uint32_t i, uint32_t* idx, uint32_t* key) {
    int r = 0;
    while (r + 1 < world && offs[r + 1] <= i) ++r;
    const uint32_t j = i - offs[r];
    *idx = all[r * stride + j];
    *key = all[r * stride + k + j] >> 8;  // 24-bit prefix, as the fused kernel ranks
  };
  uint32_t tau = 0, need_eq = 0xffffffffu;
  const bool radix = total > static_cast<uint32_t>(k);
  if (radix) {
    uint32_t kk = static_cast<uint32_t>(k), prefix = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int sh = pass == 0 ? 12 : 0;
      for (int i = tid; i < kMergeBins; i += kMergeThreads) hist[i] = 0u;
      __syncthreads();
      for (uint32_t i = tid; i < total; i += kMergeThreads) {
        uint32_t idx, key;
        entry(i, &idx, &key);
        if (pass == 0 || (key >> 12) == prefix) atomicAdd(&hist[(key >> sh) & (kMergeBins - 1)], 1u);
      }
      __syncthreads();
      int b;
      uint32_t above;
      merge_find_bin(hist, kk, scratch, &b, &above);
      kk -= above;
      prefix = pass == 0 ? static_cast<uint32_t>(b) : (prefix << 12) | static_cast<uint32_t>(b);
    }
    tau = prefix;
    need_eq = kk;  // ties at tau still to take, lowest positions first
  }
  // own init rows
  for (uint32_t i = tid; i < init_hi; i += kMergeThreads) att[i] = i;
  // own selected rows, ascending
  uint32_t out = init_hi, eq_seen = 0;
  for (uint32_t b0 = 0; b0 < total; b0 += kMergeThreads) {
    const uint32_t i = b0 + tid;
    uint32_t idx = 0, key = 0;
    if (i < total) entry(i, &idx, &key);
    const uint32_t is_eq = (radix && i < total && key == tau) ? 1u : 0u;
    uint32_t eq_tot;
    const uint32_t eq_rank = eq_seen + block_scan_excl_1024(is_eq, scratch, &eq_tot);
    eq_seen += eq_tot;
    bool take = i < total && (!radix || key > tau || (is_eq && eq_rank < need_eq));
    take = take && idx >= ie && idx < lbs && idx >= base && idx < base + n_r;
    uint32_t tot;
    const uint32_t pos = block_scan_excl_1024(take ? 1u : 0u, scratch, &tot);
    if (take) att[out + pos] = idx - base;
    out += tot;
  }
  // own local-window rows
  for (uint32_t i = loc_lo + tid; i < n_r; i += kMergeThreads) att[out + (i - loc_lo)] = i;
  if (tid == 0) *n_att = static_cast<int>(out + (n_r > loc_lo ? n_r - loc_lo : 0));
}

// Cross-shard log-sum-exp merge of normalised outputs o_r with (M_r, L_r):
// out = sum_r e^(M_r - M) L_r o_r / sum_r e^(M_r - M) L_r, shards in rank order.
// Rank r's o block starts at o_all + r * o_stride, its (M, L) pairs at
// ml_all + r * ml_stride (separate arrays, or one packed [H*d | H*2] block).
__global__ void shard_combine_kernel(const float* o_all, const float* ml_all, int world, int H, int d,
                                     size_t o_stride, size_t ml_stride, float* out) {
  const int h = blockIdx.x;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float M = -INFINITY;
    for (int r = 0; r < world; ++r) M = fmaxf(M, ml_all[r * ml_stride + h * 2]);
    float num = 0.f, den = 0.f;
    for (int r = 0; r < world; ++r) {
      const float mr = ml_all[r * ml_stride + h * 2];
      const float lr = ml_all[r * ml_stride + h * 2 + 1];
      if (mr == -INFINITY || lr == 0.f) continue;
      const float w = expf(mr - M) * lr;
      num = fmaf(w, o_all[r * o_stride + static_cast<size_t>(h) * d + t], num);
      den += w;
    }
    out[static_cast<size_t>(h) * d + t] = num / den;
  }
}

}  // namespace

cudaError_t launch_kv_append(uint16_t* k_slab, uint16_t* v_slab, const float* k, const float* v,
                             const uint16_t* kb, const uint16_t* vb, const int64_t* dst_rows, int t,
                             int row, cudaStream_t st, const int32_t* pt, int64_t pos0, int page_size, bool pdl) {
  if (t <= 0) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(t) * row;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (!pdl) {
    kv_append_kernel<<<blocks, 256, 0, st>>>(k_slab, v_slab, k, v, kb, vb, dst_rows, pt, pos0, page_size, t, row);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kv_append_kernel, k_slab, v_slab, k, v, kb, vb, dst_rows, pt, pos0, page_size, t, row);
}

cudaError_t launch_kv_gather(const uint16_t* k_slab, const uint16_t* v_slab, const int64_t* src_rows,
                             int n, int row, float* k_out, float* v_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(n) * row;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  kv_gather_kernel<<<blocks, 256, 0, st>>>(k_slab, v_slab, src_rows, n, row, k_out, v_out);
  return cudaGetLastError();
}

cudaError_t launch_chunk_mean(const float* q, int c, int width, float* out, cudaStream_t st) {
  chunk_mean_kernel<<<(width + kCmCols - 1) / kCmCols, kCmThr, 0, st>>>(q, c, width, out);
  return cudaGetLastError();
}

cudaError_t launch_max_index(const uint32_t* idx, int n, unsigned int* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = std::min((n + 255) / 256, 148 * 4);
  max_index_kernel<<<blocks, 256, 0, st>>>(idx, n, out);
  return cudaGetLastError();
}

cudaError_t launch_windows(const uint32_t* sel, const int* n_sel_ptr, int n_sel_fixed, int cached,
                           int init_end, int local_begin, uint32_t* out, int* n_out,
                           unsigned int* bad, cudaStream_t st) {
  windows_kernel<<<16, 256, 0, st>>>(sel, n_sel_ptr, n_sel_fixed, cached, init_end, local_begin, out,
                                     n_out, bad);
  return cudaGetLastError();
}

cudaError_t launch_prefill_attend(const PrefillAttendParams& p, cudaStream_t st) {
  const int G = p.H / p.H_kv;
  if (G > kMaxG || p.d > 32 * kMaxDL) return cudaErrorInvalidValue;
  const size_t smem = (2 * kKT * (p.d + 1) + kQT * G * p.d) * sizeof(float);
  dim3 grid((p.C + kQT - 1) / kQT, p.H_kv);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  prefill_attend_kernel<<<grid, kQT * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_shard_merge(const uint32_t* all, int world, int k, uint32_t ie, uint32_t lbs, uint32_t base,
                               uint32_t n_r, uint32_t init_hi, uint32_t loc_lo, uint32_t* att, int* n_att,
                               cudaStream_t st) {
  if (world > 64) return cudaErrorInvalidValue;
  shard_merge_kernel<<<1, kMergeThreads, 0, st>>>(all, world, k, ie, lbs, base, n_r, init_hi, loc_lo, att, n_att);
  return cudaGetLastError();
}

cudaError_t launch_shard_combine(const float* o_all, const float* ml_all, int world, int H, int d, float* out,
                                 cudaStream_t st, bool packed) {
  const size_t hd = static_cast<size_t>(H) * d;
  const size_t o_stride = packed ? hd + 2 * H : hd, ml_stride = packed ? hd + 2 * H : 2 * static_cast<size_t>(H);
  shard_combine_kernel<<<H, 128, 0, st>>>(o_all, ml_all, world, H, d, o_stride, ml_stride, out);
  return cudaGetLastError();
}

}  // namespace tsb

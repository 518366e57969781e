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

__global__ void kv_append_kernel(uint16_t* k_slab, uint16_t* v_slab, const float* k, const float* v,
                                 const uint16_t* kb, const uint16_t* vb, const int64_t* dst_rows,
                                 int t, int row) {
  const int64_t total = static_cast<int64_t>(t) * row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row, c = i - (i / row) * row;
    const int64_t off = dst_rows[r] * row + c;
    if (k) {
      k_slab[off] = __bfloat16_as_ushort(__float2bfloat16_rn(k[i]));
      v_slab[off] = __bfloat16_as_ushort(__float2bfloat16_rn(v[i]));
    } else {
      k_slab[off] = kb[i];
      v_slab[off] = vb[i];
    }
  }
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

// Sequential fp64 column sums in row order: bit-identical to chunk_mean.
__global__ void chunk_mean_kernel(const float* q, int c, int width, float* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= width) return;
  double acc = 0.0;
  for (int i = 0; i < c; ++i) acc += static_cast<double>(q[static_cast<size_t>(i) * width + j]);
  out[j] = static_cast<float>(acc * (1.0 / static_cast<double>(c)));
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

}  // namespace

cudaError_t launch_kv_append(uint16_t* k_slab, uint16_t* v_slab, const float* k, const float* v,
                             const uint16_t* kb, const uint16_t* vb, const int64_t* dst_rows, int t,
                             int row, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(t) * row;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  kv_append_kernel<<<blocks, 256, 0, st>>>(k_slab, v_slab, k, v, kb, vb, dst_rows, t, row);
  return cudaGetLastError();
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
  chunk_mean_kernel<<<(width + 127) / 128, 128, 0, st>>>(q, c, width, out);
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

}  // namespace tsb

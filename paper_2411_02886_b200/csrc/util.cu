// The reference's tensor utilities on the device (the free functions the
// pybind module exports, proj/python/bindings.cpp:60-116), fp64 like the
// reference so results match it to the last bits of fp32:
//
//   softmax_rows_kernel  softmax_rows (tensor.cpp:31-52): per row max, e in
//                        fp64 stored as fp32, fp64 sum over the unrounded e,
//                        p = fp32(fp32(e) * (1 / sum))
//   topk64_kernel        topk_indices (tensor.cpp:68-90) over fp64 scores:
//                        larger first, the smaller index on ties, output
//                        ascending (exact 64-bit radix select)
//   cosine_kernel        cosine (tensor.cpp:92-113): fp64 sums, dot^2 >= nu*nv
//                        clamps to exactly +-1
//   sdpa_full_kernel     sdpa_full (attention.cpp:54-112): C query rows over
//                        N key rows, query i sees keys [0, N - C + i]
//                        (causal within the current rows, :83), fp64 softmax
//                        and P.V, rounded to fp32
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "util.h"

namespace tsb {

namespace {

constexpr int kUT = 512;

__device__ double block_reduce_d(double v, double* sh, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, x) : v + x;
  }
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = lane < nw ? sh[lane] : (is_max ? -INFINITY : 0.0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, r, o);
    r = is_max ? fmax(r, x) : r + x;
  }
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kUT) softmax_rows_kernel(const float* __restrict__ m, int cols, float* out) {
  __shared__ double sh[32];
  const float* row = m + static_cast<size_t>(blockIdx.x) * cols;
  float* orow = out + static_cast<size_t>(blockIdx.x) * cols;
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) mx = fmax(mx, static_cast<double>(row[j]));
  mx = block_reduce_d(mx, sh, true);
  double s = 0.0;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) s += exp(static_cast<double>(row[j]) - mx);
  s = block_reduce_d(s, sh, false);
  const double inv = 1.0 / s;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) {
    const float e = static_cast<float>(exp(static_cast<double>(row[j]) - mx));
    orow[j] = static_cast<float>(static_cast<double>(e) * inv);
  }
}

// order-preserving double -> uint64 key (larger double => larger key; -0 == +0)
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  if ((b << 1) == 0ull) b = 0ull;
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

__device__ uint32_t uscan(uint32_t v, uint32_t* sh, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t inc = warp_incl_scan(v, lane);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < nw ? sh[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w, lane);
    sh[32 + lane] = wi - w;
    if (lane == 31) sh[64] = wi;
  }
  __syncthreads();
  const uint32_t r = sh[32 + warp] + inc - v;
  *total = sh[64];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kUT) topk64_kernel(const double* __restrict__ s, int n, int k, uint32_t* out,
                                                     int* n_out) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh[80];
  __shared__ unsigned long long thr_sh;
  const int tid = threadIdx.x;
  const uint32_t kk = static_cast<uint32_t>(min(k, n));
  unsigned long long prefix = 0ull;
  uint32_t need = kk;
  const bool all = kk >= static_cast<uint32_t>(n);
  if (!all) {
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0u;
      __syncthreads();
      for (int j = tid; j < n; j += blockDim.x) {
        const unsigned long long key = dkey(s[j]);
        if (pass == 0 || (key >> (shift + 8)) == prefix) atomicAdd(&hist[(key >> shift) & 255ull], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t acc = 0;
        int b = 255;
        for (; b > 0; --b) {
          if (acc + hist[b] >= need) break;
          acc += hist[b];
        }
        sh[70] = static_cast<uint32_t>(b);
        sh[71] = need - acc;
      }
      __syncthreads();
      prefix = (prefix << 8) | sh[70];
      need = sh[71];
      __syncthreads();
    }
  }
  if (tid == 0) thr_sh = prefix;
  __syncthreads();
  // ascending compaction: key > thr, or key == thr among the first `need` ties
  uint32_t pos0 = 0, eq_seen = 0;
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int j = b0 + tid;
    const unsigned long long key = j < n ? dkey(s[j]) : 0ull;
    const uint32_t eq = (!all && j < n && key == thr_sh) ? 1u : 0u;
    uint32_t eq_tot;
    const uint32_t r = eq_seen + uscan(eq, sh, &eq_tot);
    eq_seen += eq_tot;
    const uint32_t take = (j < n && (all || key > thr_sh || (eq && r < need))) ? 1u : 0u;
    uint32_t tot;
    const uint32_t pos = pos0 + uscan(take, sh, &tot);
    if (take) out[pos] = static_cast<uint32_t>(j);
    pos0 += tot;
  }
  if (tid == 0) *n_out = static_cast<int>(pos0);
}

__global__ void __launch_bounds__(kUT) cosine_kernel(const double* __restrict__ u, const double* __restrict__ v,
                                                     int n, double* out) {
  __shared__ double sh[32];
  double dot = 0.0, nu = 0.0, nv = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    dot = fma(u[i], v[i], dot);
    nu = fma(u[i], u[i], nu);
    nv = fma(v[i], v[i], nv);
  }
  dot = block_reduce_d(dot, sh, false);
  nu = block_reduce_d(nu, sh, false);
  nv = block_reduce_d(nv, sh, false);
  if (threadIdx.x == 0) {
    double c;
    if (nu == 0.0 || nv == 0.0) c = NAN;  // the host reports the error (tensor.cpp:100-103)
    else if (dot * dot >= nu * nv) c = dot >= 0.0 ? 1.0 : -1.0;
    else c = dot / sqrt(nu * nv);
    *out = c;
  }
}

// one CTA per (query row, head); keys of the head's KV group (h mod H_kv)
__global__ void __launch_bounds__(kUT) sdpa_full_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                        const float* __restrict__ v, int C, int N, int H, int H_kv,
                                                        int d, double scale, float* out, double* ws) {
  __shared__ double sh[32];
  const int i = blockIdx.x / H, h = blockIdx.x - (blockIdx.x / H) * H, g = h % H_kv;
  const int nk = N - C + i + 1;  // causal within the current rows
  const float* qh = q + static_cast<size_t>(i) * H * d + static_cast<size_t>(h) * d;
  double* lg = ws + static_cast<size_t>(blockIdx.x) * N;
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const float* kr = k + static_cast<size_t>(j) * H_kv * d + static_cast<size_t>(g) * d;
    double a = 0.0;
    for (int t = 0; t < d; ++t) a += static_cast<double>(qh[t]) * static_cast<double>(kr[t]);
    a *= scale;
    lg[j] = a;
    mx = fmax(mx, a);
  }
  mx = block_reduce_d(mx, sh, true);
  double den = 0.0;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const double e = exp(lg[j] - mx);
    lg[j] = e;
    den += e;
  }
  den = block_reduce_d(den, sh, false);  // (also orders the lg writes before the reads below)
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double a = 0.0;
    for (int j = 0; j < nk; ++j) a += lg[j] * static_cast<double>(v[static_cast<size_t>(j) * H_kv * d + static_cast<size_t>(g) * d + t]);
    out[static_cast<size_t>(i) * H * d + static_cast<size_t>(h) * d + t] = static_cast<float>(a / den);
  }
}

}  // namespace

cudaError_t launch_softmax_rows(const float* m, int rows, int cols, float* out, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  softmax_rows_kernel<<<rows, kUT, 0, st>>>(m, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_topk64(const double* s, int n, int k, uint32_t* out, int* n_out, cudaStream_t st) {
  topk64_kernel<<<1, kUT, 0, st>>>(s, n, k, out, n_out);
  return cudaGetLastError();
}

cudaError_t launch_cosine(const double* u, const double* v, int n, double* out, cudaStream_t st) {
  cosine_kernel<<<1, kUT, 0, st>>>(u, v, n, out);
  return cudaGetLastError();
}

cudaError_t launch_sdpa_full(const float* q, const float* k, const float* v, int C, int N, int H, int H_kv, int d,
                             float* out, double* ws, cudaStream_t st) {
  if (C <= 0) return cudaSuccess;
  sdpa_full_kernel<<<C * H, 128, 0, st>>>(q, k, v, C, N, H, H_kv, d, 1.0 / sqrt(static_cast<double>(d)), out, ws);
  return cudaGetLastError();
}

}  // namespace tsb

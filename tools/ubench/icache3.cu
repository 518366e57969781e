// Microbenchmark (dev tool): cost of K short one-shot code phases (distinct
// code, ~120 instructions each, separated by __syncthreads) vs the same phase
// code executed K times, at 148 x 544 threads, after an HBM streaming phase.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int ID>
__device__ __noinline__ float phase(float x, float* sm) {
  // ~100 instructions of distinct code per ID
#pragma unroll
  for (int i = 0; i < 24; ++i) x = fmaf(x, 1.0001f + ID * 1e-6f + i * 1e-7f, 0.5f * ID);
  sm[threadIdx.x] = x;
  __syncthreads();
  x += sm[(threadIdx.x + 1 + ID) % blockDim.x];
#pragma unroll
  for (int i = 0; i < 24; ++i) x = fmaf(x, 0.9999f - ID * 1e-6f, 0.25f + i * 1e-3f);
  __syncthreads();
  return x;
}

template <int... IDs>
__device__ float distinct(float x, float* sm) {
  ((x = phase<IDs>(x, sm)), ...);
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(544, 1) k(const float4* big, size_t n4, float* out, unsigned long long* ts) {
  __shared__ float sm[1024];
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(big + i);
    acc += v.x + v.y + v.z + v.w;
  }
  __syncthreads();
  unsigned long long t0 = gt();
  if (MODE == 0) {
    acc = distinct<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>(acc, sm);
  } else {
#pragma unroll 1
    for (int r = 0; r < 16; ++r) acc = phase<1>(acc, sm);
  }
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) ts[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  size_t bytes = 256ull << 20;
  float4* big;
  cudaMalloc(&big, bytes);
  cudaMemset(big, 0, bytes);
  float* out;
  cudaMalloc(&out, 148 * 544 * 4);
  unsigned long long* ts;
  cudaMalloc(&ts, 148 * 8);
  unsigned long long h[148];
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      if (mode == 0) k<0><<<148, 544>>>(big, bytes / 16, out, ts);
      else k<1><<<148, 544>>>(big, bytes / 16, out, ts);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("%s: 16 phases in %.2f us (mean over CTAs)\n", mode == 0 ? "distinct code" : "same code x16", s / 148 / 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

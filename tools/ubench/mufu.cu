// Microbenchmark (dev tool): MUFU.EX2 vs FFMA throughput per SM at 544 threads/SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int MODE>
__global__ void __launch_bounds__(544, 1) k(float* out, unsigned long long* ts, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  unsigned long long t0 = gt();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      else a[i] = fmaf(a[i], 0.999f, -0.0001f);
    }
  }
  __syncthreads();
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) ts[blockIdx.x] = t1 - t0;
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; unsigned long long* ts; cudaMalloc(&out, 148 * 544 * 4); cudaMalloc(&ts, 148 * 8);
  unsigned long long h[148];
  int iters = 1000;
  for (int m = 0; m < 2; ++m) {
    for (int r = 0; r < 3; ++r) { if (m == 0) k<0><<<148, 544>>>(out, ts, iters); else k<1><<<148, 544>>>(out, ts, iters); }
    cudaDeviceSynchronize();
    cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
    double ns = 0; for (int i = 0; i < 148; ++i) ns += h[i]; ns /= 148;
    double ops = 544.0 * 8 * iters;
    printf("%s: %.1f us, %.2f ops/ns per SM (%.1f per clk @1.965GHz)\n", m == 0 ? "ex2+fadd" : "ffma", ns / 1000, ops / ns, ops / ns / 1.965);
  }
  return 0;
}

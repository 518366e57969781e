// Microbenchmark (dev tool): cost of cold one-shot code after a memory-bound
// phase, at the fused decode kernel's launch shape. Phase B is N straight-line
// dependent-ish instructions, timed by %globaltimer on thread 0, run twice
// (cold, then warm) in the same launch.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define OP(i) a##i = fmaf(a##i, b, c);
#define OPS8 OP(0) OP(1) OP(2) OP(3) OP(4) OP(5) OP(6) OP(7)
#define OPS64 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8
#define OPS512 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64

template <int N512>
__device__ __noinline__ float phaseB(float b, float c) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll
  for (int i = 0; i < N512; ++i) {
    asm volatile("" ::: "memory");
    OPS512
  }
  return a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int N512>
__global__ void __launch_bounds__(544, 1) k(const float4* big, size_t n4, float* out, unsigned long long* ts, int stream) {
  float acc = 0.f;
  if (stream) {  // phase A: stream `big` once (HBM bound)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcs(big + i);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  __syncthreads();
  unsigned long long t0 = gt();
  acc += phaseB<N512>(1.0001f, 0.5f);
  __syncthreads();
  unsigned long long t1 = gt();
  acc += phaseB<N512>(1.0002f, 0.25f);
  __syncthreads();
  unsigned long long t2 = gt();
  if (threadIdx.x == 0) {
    ts[blockIdx.x * 2 + 0] = t1 - t0;
    ts[blockIdx.x * 2 + 1] = t2 - t1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int N512>
void run(const float4* big, size_t n4, float* out, unsigned long long* ts, int stream) {
  unsigned long long h[296];
  for (int rep = 0; rep < 3; ++rep) k<N512><<<148, 544>>>(big, n4, out, ts, stream);
  cudaDeviceSynchronize();
  cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0, w = 0;
  for (int i = 0; i < 148; ++i) { c += h[2 * i]; w += h[2 * i + 1]; }
  printf("N=%5d instr  stream=%d: cold %.2f us, warm %.2f us (mean over CTAs)\n", N512 * 512, stream, c / 148 / 1000,
         w / 148 / 1000);
}

int main() {
  size_t bytes = 256ull << 20;
  float4* big;
  cudaMalloc(&big, bytes);
  cudaMemset(big, 0, bytes);
  float* out;
  cudaMalloc(&out, 148 * 544 * 4);
  unsigned long long* ts;
  cudaMalloc(&ts, 296 * 8);
  size_t n4 = bytes / 16;
  for (int s = 0; s < 2; ++s) {
    run<1>(big, n4, out, ts, s);
    run<2>(big, n4, out, ts, s);
    run<4>(big, n4, out, ts, s);
    run<8>(big, n4, out, ts, s);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

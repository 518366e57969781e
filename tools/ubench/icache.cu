// Microbenchmark (dev tool): cost of executing straight-line code once per
// launch vs the same instruction count in a loop, at the fused decode
// kernel's launch shape (148 CTAs x 544 threads, 1 CTA/SM).
#include <cstdio>
#include <cuda_runtime.h>

#define OP(i) a##i = fmaf(a##i, b, c);
#define OPS8 OP(0) OP(1) OP(2) OP(3) OP(4) OP(5) OP(6) OP(7)
#define OPS64 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8 OPS8
#define OPS512 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64 OPS64

template <int N512>
__global__ void __launch_bounds__(544, 1) straight(float* out, float b, float c) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll
  for (int i = 0; i < N512; ++i) {
    asm volatile("" ::: "memory");
    OPS512
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void __launch_bounds__(544, 1) looped(float* out, float b, float c, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    OPS512
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void empty_k(float* out) {
  if (threadIdx.x == 0 && out == nullptr) out[0] = 1.f;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / 100.f;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 544 * 4);
  dim3 g(148), b(544);
  printf("empty: %.2f us\n", timeit([&] { empty_k<<<g, b>>>(out); }));
  printf("straight 512 instr: %.2f us\n", timeit([&] { straight<1><<<g, b>>>(out, 1.0001f, 0.5f); }));
  printf("straight 2048 instr: %.2f us\n", timeit([&] { straight<4><<<g, b>>>(out, 1.0001f, 0.5f); }));
  printf("straight 4096 instr: %.2f us\n", timeit([&] { straight<8><<<g, b>>>(out, 1.0001f, 0.5f); }));
  printf("straight 8192 instr: %.2f us\n", timeit([&] { straight<16><<<g, b>>>(out, 1.0001f, 0.5f); }));
  printf("looped 512 x1: %.2f us\n", timeit([&] { looped<<<g, b>>>(out, 1.0001f, 0.5f, 1); }));
  printf("looped 512 x4: %.2f us\n", timeit([&] { looped<<<g, b>>>(out, 1.0001f, 0.5f, 4); }));
  printf("looped 512 x8: %.2f us\n", timeit([&] { looped<<<g, b>>>(out, 1.0001f, 0.5f, 8); }));
  printf("looped 512 x16: %.2f us\n", timeit([&] { looped<<<g, b>>>(out, 1.0001f, 0.5f, 16); }));
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

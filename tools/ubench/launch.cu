// Microbenchmark (dev tool): host cost of launching the decode-shaped grid
// (148 x 544, 200 KB dynamic smem, 3 KB params) cooperatively vs normally.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

struct Big { char b[3000]; };

__global__ void __launch_bounds__(544, 1) k(Big p, int* out) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0 && p.b[blockIdx.x % 3000] == 42) out[blockIdx.x] = sm[0];
}

int main() {
  int* out;
  cudaMalloc(&out, 4096);
  Big p{};
  size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  void* args[] = {&p, &out};
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int mode = 0; mode < 3; ++mode) {
    for (int i = 0; i < 50; ++i) cudaLaunchCooperativeKernel((void*)k, 148, 544, args, smem, st);
    cudaStreamSynchronize(st);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) {
      if (mode == 0) cudaLaunchCooperativeKernel((void*)k, 148, 544, args, smem, st);
      else if (mode == 1) k<<<148, 544, smem, st>>>(p, out);
      else cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), k<<<148, 544, smem, st>>>(p, out);
    }
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    printf("mode %d (%s): host %.2f us/launch, total %.2f us/launch\n", mode,
           mode == 0 ? "cooperative" : mode == 1 ? "normal" : "normal+setattr",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / 2000);
  }
  return 0;
}

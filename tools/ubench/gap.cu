// Microbenchmark (dev tool): GPU-side gap between back-to-back launches of a
// decode-shaped grid (148 x 544, 220 KB smem) that runs a fixed 10 us:
// period - 10 us, cooperative vs normal launch, and with a stream of
// independent (non-cooperative) launches.
#include <cstdio>
#include <cuda_runtime.h>

struct Big { char b[3000]; };

__global__ void __launch_bounds__(544, 1) k(Big p, int* out, unsigned long long ns) {
  extern __shared__ char sm[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
  if (threadIdx.x == 0 && p.b[blockIdx.x % 3000] == 42) out[blockIdx.x] = sm[0];
}

int main() {
  int* out;
  cudaMalloc(&out, 4096);
  Big p{};
  size_t smem = 220 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long ns = 10000;
  void* args[] = {&p, &out, &ns};
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int i = 0; i < 10; ++i) cudaLaunchCooperativeKernel((void*)k, 148, 544, args, smem, st);
      cudaEventRecord(e0, st);
      for (int i = 0; i < 100; ++i) {
        if (mode == 0) cudaLaunchCooperativeKernel((void*)k, 148, 544, args, smem, st);
        else k<<<148, 544, smem, st>>>(p, out, ns);
      }
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %s: period %.2f us (kernel 10 us)\n", mode == 0 ? "cooperative" : "normal", ms * 1000 / 100);
    }
  }
  return 0;
}

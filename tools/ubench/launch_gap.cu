// Dev: back-to-back cost of an (almost) empty 148 x 544 kernel by launch kind
// and dynamic shared memory (the fused decode kernel's launch shape).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ubench/launch_gap.cu -o /tmp/lg
#include <cooperative_groups.h>
#include <cstdio>

__global__ void __launch_bounds__(544, 1) k_empty(int* x) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (x && sm[0] < 0) x[0] = 1;
}
__global__ void __launch_bounds__(544, 1) k_tmem(int* x) {
  extern __shared__ __align__(16) int sm[];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(sm))) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  const unsigned t = static_cast<unsigned>(sm[0]);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
  if (x && t == 0xffffffffu) x[0] = 1;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int R = 200;
  for (int kind = 0; kind < 2; ++kind)
    for (int tm = 0; tm < 2; ++tm)
      for (size_t smem : {size_t(1024), size_t(100 * 1024), size_t(231 * 1024)}) {
        void* fn = tm ? reinterpret_cast<void*>(k_tmem) : reinterpret_cast<void*>(k_empty);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int* nul = nullptr;
        void* args[] = {&nul};
        for (int w = 0; w < 10; ++w)
          kind ? cudaLaunchCooperativeKernel(fn, 148, 544, args, smem, 0) : cudaLaunchKernel(fn, 148, 544, args, smem, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < R; ++r)
          kind ? cudaLaunchCooperativeKernel(fn, 148, 544, args, smem, 0) : cudaLaunchKernel(fn, 148, 544, args, smem, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-11s %-5s smem %6zu: %.2f us per launch (%s)\n", kind ? "cooperative" : "normal", tm ? "tmem" : "plain", smem,
               ms * 1000 / R, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}

// Microbenchmark (dev tool): HBM -> smem streaming rate of cp.async.bulk as a
// function of the copy size (148 CTAs, 6-slot x 32 KB ring, one producer
// warp, one consumer warp that only waits / releases).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(n)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su(b)), "r"(par) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)),
               "l"(src), "r"(n), "r"(su(b)) : "memory");
}

constexpr int kSlots = 6, kSlot = 32768;
__global__ void k(const char* src, size_t per_cta, int csize) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlots * kSlot);
  uint64_t* empty = full + kSlots;
  if (threadIdx.x < kSlots) { init(&full[threadIdx.x], 1); init(&empty[threadIdx.x], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  const int nst = static_cast<int>(per_cta / kSlot);
  const int per = kSlot / csize;  // copies per slot
  if (threadIdx.x < 32) {
    for (int it = 0; it < nst; ++it) {
      const int s = it % kSlots;
      if (it >= kSlots) wait(&empty[s], ((it / kSlots) & 1) ^ 1);
      if (threadIdx.x == 0) expect(&full[s], kSlot);
      __syncwarp();
      for (int c = threadIdx.x; c < per; c += 32)
        bulk(sm + s * kSlot + c * csize, base + static_cast<size_t>(it) * kSlot + c * csize, csize, &full[s]);
    }
  } else if (threadIdx.x < 64) {
    for (int it = 0; it < nst; ++it) {
      const int s = it % kSlots;
      wait(&full[s], (it / kSlots) & 1);
      __syncwarp();
      if (threadIdx.x == 32) arrive(&empty[s]);
    }
  }
}

int main() {
  const size_t per_cta = 7ull << 20;  // 7 MB per CTA, 1 GB total
  char* src;
  cudaMalloc(&src, per_cta * 148);
  cudaMemset(src, 1, per_cta * 148);
  const int smem = kSlots * kSlot + 2 * kSlots * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int cs : {512, 1024, 2048, 4096, 8192, 16384, 32768}) {
    k<<<148, 64, smem>>>(src, per_cta, cs);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<148, 64, smem>>>(src, per_cta, cs);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("copy %6d B: %.0f GB/s\n", cs, 5.0 * per_cta * 148 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

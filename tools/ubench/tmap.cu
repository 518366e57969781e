// Microbenchmark (dev tool): can a 3-D tensor map view the K slab as
// [chunk (128 B)][token row][64 bf16] (non-monotone strides) so one TMA op
// brings 16 rows x 2 KB with the 128B swizzle keyed by the token row? And its
// streaming rate vs 1-D bulk copies.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

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
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(su(dst)), "l"(m), "r"(x), "r"(y), "r"(z), "r"(su(b)) : "memory");
}

constexpr int kSlots = 6, kSlot = 32768;
__global__ void layout(const __grid_constant__ CUtensorMap m, uint16_t* out) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlot);
  if (threadIdx.x == 0) init(full, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) { expect(full, kSlot); tma3(sm, &m, 0, 32, 0, full); }
  wait(full, 0);
  for (int i = threadIdx.x; i < kSlot / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

__global__ void stream(const __grid_constant__ CUtensorMap m, int rows_per_cta) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlots * kSlot);
  uint64_t* empty = full + kSlots;
  if (threadIdx.x < kSlots) { init(&full[threadIdx.x], 1); init(&empty[threadIdx.x], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int nst = rows_per_cta / 16, row0 = blockIdx.x * rows_per_cta;
  if (threadIdx.x == 0) {
    for (int it = 0; it < nst; ++it) {
      const int s = it % kSlots;
      if (it >= kSlots) wait(&empty[s], ((it / kSlots) & 1) ^ 1);
      expect(&full[s], kSlot);
      tma3(sm + s * kSlot, &m, 0, row0 + it * 16, 0, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < nst; ++it) {
      const int s = it % kSlots;
      wait(&full[s], (it / kSlots) & 1);
      arrive(&empty[s]);
    }
  }
}

int main() {
  const int rows = 148 * 3584;  // 148 CTAs x 3584 rows x 2 KB = 1.09 GB
  uint16_t* slab;
  cudaMalloc(&slab, static_cast<size_t>(rows) * 1024 * 2);
  // slab[row][e] = (row * 1024 + e) & 0xffff as a marker
  uint16_t* h = new uint16_t[64 * 1024];
  for (int r = 0; r < 64; ++r) for (int e = 0; e < 1024; ++e) h[r * 1024 + e] = static_cast<uint16_t>((r << 10) | e);
  cudaMemcpy(slab, h, 64 * 1024 * 2, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), 16};  // x: 64 el, y: token rows, z: 128-B chunk
  cuuint64_t strides[2] = {2048, 128};                             // y stride 2 KB, z stride 128 B
  cuuint32_t box[3] = {64, 16, 16};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, slab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", static_cast<int>(r));
  if (r != CUDA_SUCCESS) return 0;
  uint16_t* out;
  cudaMalloc(&out, kSlot);
  cudaFuncSetAttribute(layout, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlot + 1024);
  layout<<<1, 128, kSlot + 1024>>>(m, out);
  uint16_t* o = new uint16_t[kSlot / 2];
  cudaMemcpy(o, out, kSlot, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  // smem line L (128 B = 64 el) : print (row, elem) of its first element for lines 0..20
  for (int L = 0; L < 20; ++L) {
    const uint16_t v = o[L * 64];
    printf("line %2d: row %d elem %d | 2nd 16B chunk starts elem %d\n", L, v >> 10, v & 1023, o[L * 64 + 8] & 1023);
  }
  const int smem = kSlots * kSlot + 2 * kSlots * 8 + 1024;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  stream<<<148, 64, smem>>>(m, 3584);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stream<<<148, 64, smem>>>(m, 3584);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("tensor 32 KB ops: %.0f GB/s (%s)\n", 5.0 * rows * 2048 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

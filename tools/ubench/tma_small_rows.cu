// Dev: TMA gather4 / 2-D tile loads into the K-major SW128 tile layout the
// tcgen05 prefill reads ([2 atoms][64 rows][128 B], chunk c of row r at
// (c % 8) ^ (r % 8)), including gather4 destinations at 512-B offsets and
// out-of-bounds rows (expected zero-filled).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2411_02886_b200/csrc tools/ubench/tma_gather_test.cu -o /tmp/tg
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

using namespace tsb;

__global__ void k_gather(const __grid_constant__ CUtensorMap tm, const int* rows, int col0, uint16_t* out, int tile_mode,
                         int row0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(bar, 16384);
  __syncwarp();
  if (tile_mode) {
    if (lane < 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(sm + lane * 8192)),
          "l"(&tm), "r"(col0 + lane * 64), "r"(row0), "r"(smem_u32(bar))
          : "memory");
  } else if (lane < 16) {
    for (int a = 0; a < 2; ++a)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5, %6}], [%7];" ::"r"(smem_u32(sm + a * 8192 + lane * 512)),
          "l"(&tm), "r"(col0 + a * 64), "r"(rows[4 * lane]), "r"(rows[4 * lane + 1]), "r"(rows[4 * lane + 2]),
          "r"(rows[4 * lane + 3]), "r"(smem_u32(bar))
          : "memory");
  }
  mbar_wait(bar, 0);
  for (int i = lane; i < 8192; i += 32) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 1000, W = 1024;
  std::vector<uint16_t> h(static_cast<size_t>(R) * W);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < W; ++c) h[static_cast<size_t>(r) * W + c] = static_cast<uint16_t>((r * 7 + c * 13) & 0xFFFF) | 1;
  uint16_t *d, *dout;
  int* drows;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&dout, 16384);
  cudaMalloc(&drows, 64 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(f);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    alignas(64) CUtensorMap tm;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(R)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(W) * 2};
    const cuuint32_t box[2] = {64, mode ? 64u : 1u};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("mode %d encode %d\n", mode, int(r));
    std::vector<int> rows(64);
    const int row0 = 0;  // tile mode: rows 960..1023 (24 out of bounds)
    for (int i = 0; i < 64; ++i) rows[i] = mode ? row0 + i : (i == 5 || i == 62 ? R + 17 : (i * 389 + 11) % R);
    cudaMemcpy(drows, rows.data(), 64 * 4, cudaMemcpyHostToDevice);
    const int col0 = 3 * 128;
    cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 17408);
    k_gather<<<1, 32, 17408>>>(tm, drows, col0, dout, mode, row0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
    std::vector<uint16_t> o(8192);
    cudaMemcpy(o.data(), dout, 16384, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 64; ++rr)
      for (int c = 0; c < 16; ++c)
        for (int u = 0; u < 8; ++u) {
          const size_t off = ((c >> 3) * 64 * 128 + rr * 128 + (((c & 7) ^ (rr & 7)) << 4)) / 2 + u;
          const int src = rows[rr];
          const uint16_t want = src < R ? h[static_cast<size_t>(src) * W + col0 + c * 8 + u] : 0;
          if (o[off] != want && bad++ < 5) printf("  mismatch row %d chunk %d u %d: got %d want %d\n", rr, c, u, o[off], want);
        }
    printf("mode %d (%s): %d mismatches\n", mode, mode ? "tile 64x64" : "gather4", bad);
    fails += bad != 0 || e != cudaSuccess;
  }
  printf(fails ? "FAIL\n" : "PASS\n");
  return fails;
}

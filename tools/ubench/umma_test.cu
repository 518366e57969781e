// Dev: minimal tcgen05.mma checks of the descriptors prefill_tc.cu uses.
//   test 1: D[128 x 64] = A[128 x 128] . B[64 x 128]^T, A and B K-major SW128
//   test 2: D[128 x 128] = P[128 x 64] . V[64 x 128], P K-major, V MN-major SW128
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2411_02886_b200/csrc tools/ubench/umma_test.cu -o /tmp/umma_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"

using namespace tsb;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc(int M, int N, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ uint32_t sw_off(int R, int r, int c) {
  return static_cast<uint32_t>((c >> 3) * R * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// A: [128][128] bf16 row-major (K = 128), B: [64][128] (N rows, K), out D [128][64]
// test 2: P [128][64] (K = 64), V [64 keys][128 d], out O [128][128]
__global__ void k_test(const uint16_t* A, const uint16_t* B, const uint16_t* P, const uint16_t* V, float* D, float* O,
                       int* status) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;                 // 32 KB
  uint8_t* sb = sm + 32768;         // 16 KB
  uint8_t* sp = sm + 49152;         // 16 KB
  uint8_t* sv = sm + 65536;         // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 81920);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 81936);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int r = i >> 4, c = i & 15;
    *reinterpret_cast<uint4*>(sa + sw_off(128, r, c)) = *reinterpret_cast<const uint4*>(A + r * 128 + c * 8);
  }
  for (int i = tid; i < 64 * 16; i += blockDim.x) {
    const int r = i >> 4, c = i & 15;
    *reinterpret_cast<uint4*>(sb + sw_off(64, r, c)) = *reinterpret_cast<const uint4*>(B + r * 128 + c * 8);
    *reinterpret_cast<uint4*>(sv + sw_off(64, r, c)) = *reinterpret_cast<const uint4*>(V + r * 128 + c * 8);
  }
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(sp + r * 128 + ((c ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(P + r * 64 + c * 8);
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t t = *slot;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb), p0 = smem_u32(sp), v0 = smem_u32(sv);
    for (int kk = 0; kk < 8; ++kk)
      umma(t, sdesc(a0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), sdesc(b0 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
           idesc(128, 64, 0), kk > 0);
    for (int kk = 0; kk < 4; ++kk)
      umma(t + 128, sdesc(p0 + kk * 32, 16, 1024), sdesc(v0 + kk * 2048, 8192, 1024), idesc(128, 128, 1), kk > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  }
  // bounded wait: report a hang instead of hanging
  uint32_t done = 0;
  for (long it = 0; it < 20000000 && !done; ++it) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(0u)
                 : "memory");
  }
  if (!done) {
    if (tid == 0) *status = -1;
    return;  // (TMEM leaks: dev tool)
  }
  tmem_fence_after_sync();
  if (tid < 128) {
    float v[16];
    for (int q = 0; q < 4; ++q) {
      tmem_ld16(t + (static_cast<uint32_t>(warp * 32) << 16) + q * 16, v);
      for (int u = 0; u < 16; ++u) D[tid * 64 + q * 16 + u] = v[u];
    }
    for (int q = 0; q < 8; ++q) {
      tmem_ld16(t + 128 + (static_cast<uint32_t>(warp * 32) << 16) + q * 16, v);
      for (int u = 0; u < 16; ++u) O[tid * 128 + q * 16 + u] = v[u];
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(t) : "memory");
  }
  if (tid == 0) *status = 1;
}

static uint16_t f2bf(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return static_cast<uint16_t>((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf2f(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float x;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  std::vector<uint16_t> A(128 * 128), B(64 * 128), P(128 * 64), V(64 * 128);
  srand(1);
  auto rnd = [] { return static_cast<float>(rand()) / RAND_MAX * 2.f - 1.f; };
  for (auto& x : A) x = f2bf(rnd());
  for (auto& x : B) x = f2bf(rnd());
  for (auto& x : P) x = f2bf(rnd());
  for (auto& x : V) x = f2bf(rnd());
  uint16_t *dA, *dB, *dP, *dV;
  float *dD, *dO;
  int* ds;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaMalloc(&dO, 128 * 128 * 4);
  cudaMalloc(&ds, 4);
  cudaMemset(ds, 0, 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 90000);
  k_test<<<1, 256, 90000>>>(dA, dB, dP, dV, dD, dO, ds);
  cudaError_t e = cudaDeviceSynchronize();
  int st = 0;
  cudaMemcpy(&st, ds, 4, cudaMemcpyDeviceToHost);
  printf("kernel: %s, status %d\n", cudaGetErrorString(e), st);
  if (e != cudaSuccess || st != 1) return 1;
  std::vector<float> D(128 * 64), O(128 * 128);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 64; ++j) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += double(bf2f(A[i * 128 + k])) * bf2f(B[j * 128 + k]);
      e1 = fmax(e1, fabs(s - D[i * 64 + j]));
    }
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += double(bf2f(P[i * 64 + k])) * bf2f(V[k * 128 + j]);
      e2 = fmax(e2, fabs(s - O[i * 128 + j]));
    }
  printf("QK^T max abs err %.3e, PV max abs err %.3e (D[0]=%f O[0]=%f)\n", e1, e2, D[0], O[0]);
  return (e1 < 1e-3 && e2 < 1e-3) ? 0 : 2;
}

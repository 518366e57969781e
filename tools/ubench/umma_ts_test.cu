// Dev: tcgen05.mma with the A operand in tensor memory (the "ts" form), as a
// TMEM-resident Q / P would use it, and the MMA issue rate per shape:
//   test 1: D[128 x 64]  = A[128 x 128] (TMEM) . B[64 x 128]^T (smem, K-major SW128)
//   test 2: D[128 x 128] = P[128 x 64]  (TMEM) . V[64 x 128]   (smem, MN-major SW128)
//   timing: 240 back-to-back MMAs of each form, A in smem vs A in TMEM
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2411_02886_b200/csrc tools/ubench/umma_ts_test.cu -o /tmp/uts
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t sw_off(int R, int r, int c) {
  return static_cast<uint32_t>((c >> 3) * R * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}
__device__ bool bwait(uint64_t* bar, uint32_t ph) {
  uint32_t done = 0;
  for (long it = 0; it < 20000000 && !done; ++it)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
  return done;
}

constexpr uint32_t cD = 0, cD2 = 64, cA = 192, cP = 256;

// 240 MMAs of one form, straight-line in groups of 8 (descriptor + (byte offset >> 4) = the offset address's descriptor)
template <int F>
__device__ long long run(uint32_t t, uint64_t da, uint64_t db, uint64_t dp, uint64_t dv, uint32_t id, uint64_t* bar) {
  const long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 30; ++i) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      constexpr int dummy = 0;
      const uint32_t ao = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4, bo = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
      if constexpr (F == 0) umma_ss(t + 448, da + ao, db + bo, id, 1);
      if constexpr (F == 1) umma_ts(t + 448, t + cA + kk * 8, db + bo, id, 1);
      if constexpr (F == 2) umma_ss(t + 320, dp + (((kk & 3) * 32) >> 4), dv + (((kk & 3) * 2048) >> 4), id, 1);
      if constexpr (F == 3) umma_ts(t + 320, t + cP + (kk & 3) * 8, dv + (((kk & 3) * 2048) >> 4), id, 1);
      if constexpr (F == 4 || F == 6) umma_ss(t + 256, da + ao, db + bo, id, 1);  // (B rows past 64 read the next buffer)
      if constexpr (F == 5 || F == 7) umma_ts(t + 256, t + cA + kk * 8, db + bo, id, 1);
      (void)dummy;
    }
  }
  commit(&bar[1 + (F & 1)]);
  bwait(&bar[1 + (F & 1)], (F >> 1) & 1);
  return clock64() - c0;
}

__global__ void k_test(const uint16_t* A, const uint16_t* B, const uint16_t* P, const uint16_t* V, float* D, float* O,
                       int* status, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;            // 32 KB A (for the smem-A timing)
  uint8_t* sb = sm + 32768;    // 16 KB
  uint8_t* sp = sm + 49152;    // 16 KB
  uint8_t* sv = sm + 65536;    // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 81920);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 81952);
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
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t t = *slot;
  // A and P rows -> TMEM: thread = row = lane, two bf16 per 32-bit column (low half = even k)
  if (tid < 128) {
    const uint32_t lsel = static_cast<uint32_t>(warp * 32) << 16;
    float v[16];
    for (int q = 0; q < 4; ++q) {
      for (int u = 0; u < 16; ++u) {
        const uint32_t lo = A[tid * 128 + (q * 16 + u) * 2], hi = A[tid * 128 + (q * 16 + u) * 2 + 1];
        v[u] = __uint_as_float(lo | (hi << 16));
      }
      tmem_st16(t + lsel + cA + q * 16, v);
    }
    for (int q = 0; q < 2; ++q) {
      for (int u = 0; u < 16; ++u) {
        const uint32_t lo = P[tid * 64 + (q * 16 + u) * 2], hi = P[tid * 64 + (q * 16 + u) * 2 + 1];
        v[u] = __uint_as_float(lo | (hi << 16));
      }
      tmem_st16(t + lsel + cP + q * 16, v);
    }
    tmem_wait_st();
  }
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb), p0 = smem_u32(sp), v0 = smem_u32(sv);
    for (int kk = 0; kk < 8; ++kk)
      umma_ts(t + cD, t + cA + kk * 8, sdesc(b0 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idesc(128, 64, 0), kk > 0);
    for (int kk = 0; kk < 4; ++kk)
      umma_ts(t + cD2, t + cP + kk * 8, sdesc(v0 + kk * 2048, 8192, 1024), idesc(128, 128, 1), kk > 0);
    commit(&bar[0]);
    const bool ok = bwait(&bar[0], 0);
    if (!ok) *status = -1;
    // timing: 240 MMAs per form (results discarded), descriptors precomputed
    // (a descriptor + (byte offset >> 4) = the descriptor of the offset address)
    const uint64_t da = sdesc(a0, 16, 1024), db = sdesc(b0, 16, 1024), dp = sdesc(p0, 16, 1024), dv = sdesc(v0, 8192, 1024);
    const uint32_t iq = idesc(128, 64, 0), ipv = idesc(128, 128, 1), iq128 = idesc(128, 128, 0);
    const uint32_t iq256 = idesc(128, 256, 0);
    cyc[0] = run<0>(t, da, db, dp, dv, iq, bar);
    cyc[1] = run<1>(t, da, db, dp, dv, iq, bar);
    cyc[2] = run<2>(t, da, db, dp, dv, ipv, bar);
    cyc[3] = run<3>(t, da, db, dp, dv, ipv, bar);
    cyc[4] = run<4>(t, da, db, dp, dv, iq128, bar);
    cyc[5] = run<5>(t, da, db, dp, dv, iq128, bar);
    cyc[6] = run<6>(t, da, db, dp, dv, iq256, bar);
    cyc[7] = run<7>(t, da, db, dp, dv, iq256, bar);
  }
  __syncthreads();
  tmem_fence_after_sync();
  if (tid < 128) {
    float v[16];
    for (int q = 0; q < 4; ++q) {
      tmem_ld16(t + cD + (static_cast<uint32_t>(warp * 32) << 16) + q * 16, v);
      for (int u = 0; u < 16; ++u) D[tid * 64 + q * 16 + u] = v[u];
    }
    for (int q = 0; q < 8; ++q) {
      tmem_ld16(t + cD2 + (static_cast<uint32_t>(warp * 32) << 16) + q * 16, v);
      for (int u = 0; u < 16; ++u) O[tid * 128 + q * 16 + u] = v[u];
    }
  }
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
  }
  if (tid == 0 && *status == 0) *status = 1;
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
  long long* dc;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaMalloc(&dO, 128 * 128 * 4);
  cudaMalloc(&ds, 4);
  cudaMalloc(&dc, 64);
  cudaMemset(ds, 0, 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 90000);
  k_test<<<1, 128, 90000>>>(dA, dB, dP, dV, dD, dO, ds, dc);
  cudaError_t e = cudaDeviceSynchronize();
  int st = 0;
  cudaMemcpy(&st, ds, 4, cudaMemcpyDeviceToHost);
  printf("kernel: %s, status %d\n", cudaGetErrorString(e), st);
  if (e != cudaSuccess || st != 1) return 1;
  std::vector<float> D(128 * 64), O(128 * 128);
  long long cyc[8];
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 64, cudaMemcpyDeviceToHost);
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
  printf("A in TMEM: QK^T max abs err %.3e, PV max abs err %.3e\n", e1, e2);
  const char* nm[8] = {"QK 128x64x16, A smem", "QK 128x64x16, A tmem", "PV 128x128x16, A smem", "PV 128x128x16, A tmem",
                       "QK 128x128x16, A smem", "QK 128x128x16, A tmem", "QK 128x256x16, A smem", "QK 128x256x16, A tmem"};
  for (int f = 0; f < 8; ++f) printf("  %s: %.1f clk per MMA\n", nm[f], cyc[f] / 240.0);
  return (e1 < 1e-3 && e2 < 1e-3) ? 0 : 2;
}

// Microbenchmark: cost and resolution of clock64 / %globaltimer on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out) {
  unsigned long long c0 = clock64(), g0, g1, c1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long prev = g0, steps = 0, mind = ~0ull;
  for (int i = 0; i < 1000; ++i) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (g != prev) { steps++; if (g - prev < mind) mind = g - prev; prev = g; }
  }
  c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  // clock64 resolution
  unsigned long long a = clock64(), b = clock64(), cprev = b, cst = 0, cmin = ~0ull;
  for (int i = 0; i < 1000; ++i) { unsigned long long c = clock64(); if (c != cprev) { cst++; if (c - cprev < cmin) cmin = c - cprev; cprev = c; } }
  unsigned long long c2 = clock64();
  out[0] = c1 - c0; out[1] = g1 - g0; out[2] = steps; out[3] = mind; out[4] = b - a; out[5] = cst; out[6] = cmin; out[7] = c2 - b;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  unsigned long long h[8];
  for (int r = 0; r < 3; ++r) {
    k<<<1, 1>>>(d); cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("1000 globaltimer reads: %llu cycles, %llu ns, %llu changes, min step %llu ns | clock64: back-to-back %llu, 1000 reads %llu cycles, %llu changes, min step %llu\n",
           h[0], h[1], h[2], h[3], h[4], h[7], h[5], h[6]);
  }
}

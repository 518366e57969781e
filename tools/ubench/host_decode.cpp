// Host cost of ts_engine_decode_async without Python (dev tool).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#include "../../include/tokenselect.h"

int main(int argc, char** argv) {
  const int NC = argc > 2 ? atoi(argv[2]) : 100;
  const size_t N = argc > 1 ? atol(argv[1]) : 131072;
  ts_engine_config cfg;
  ts_engine_config_default(&cfg);
  cfg.num_heads = 32; cfg.num_kv_heads = 8; cfg.head_dim = 128;
  ts_engine* e;
  if (ts_engine_create(&cfg, N + 8192, 1, &e)) { printf("%s\n", ts_last_error()); return 1; }
  uint16_t* kv;
  const size_t chunk = 16384;
  cudaMalloc(&kv, chunk * 1024 * 2);
  cudaMemset(kv, 0x3f, chunk * 1024 * 2);
  for (size_t s = 0; s < N; s += chunk) ts_engine_append_bf16(e, 0, kv, kv, chunk);
  float *q, *k, *out;
  cudaMalloc(&q, 4096 * 4); cudaMalloc(&k, 1024 * 4); cudaMalloc(&out, 4096 * 4);
  std::vector<float> hq(4096, 0.5f);
  cudaMemcpy(q, hq.data(), 4096 * 4, cudaMemcpyHostToDevice);
  cudaMemset(k, 0, 1024 * 4);
  ts_engine_set_theta(e, 0, -2.0);
  for (int i = 0; i < 20; ++i) ts_engine_decode_async(e, q, k, k, out);
  ts_engine_sync(e);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < NC; ++i) ts_engine_decode_async(e, q, k, k, out);
  auto t1 = std::chrono::steady_clock::now();
  ts_engine_sync(e);
  auto t2 = std::chrono::steady_clock::now();
  printf("N=%zu host %.2f us/call, wall %.2f us/call\n", N, std::chrono::duration<double, std::micro>(t1 - t0).count() / NC,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / NC);
  ts_engine_destroy(e);
  return 0;
}

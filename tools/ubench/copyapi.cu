// Host-side API cost of the small copies a decode call makes (dev microbench):
// H2D of the 24 KB q|k|v block and D2H of the 16 KB output, pinned vs pageable,
// plus an empty kernel launch for scale. nvcc -O2 -arch=sm_100a copyapi.cu -o copyapi
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__global__ void empty_kernel() {}
struct BigParams {
  char b[3816];
};
struct SmallParams {
  char b[440];
};
__global__ void big_kernel(const __grid_constant__ BigParams p) {
  if (p.b[threadIdx.x] == 123) asm volatile("trap;");
}
__global__ void small_kernel(const __grid_constant__ SmallParams p) {
  if (p.b[threadIdx.x % 440] == 123) asm volatile("trap;");
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename F>
static void bench(const char* name, F f, cudaStream_t st) {
  for (int i = 0; i < 20; ++i) f();
  cudaStreamSynchronize(st);
  const int n = 500;
  double api = 0, tot = 0;
  for (int i = 0; i < n; ++i) {
    const double t0 = now_us();
    f();
    const double t1 = now_us();
    cudaStreamSynchronize(st);
    const double t2 = now_us();
    api += t1 - t0;
    tot += t2 - t0;
  }
  std::printf("%-40s api %6.2f us   api+sync %6.2f us\n", name, api / n, tot / n);
}

extern "C" int bench_main() {
  const size_t in_bytes = 24576, out_bytes = 16384 + 256;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  void *d_in, *d_out, *h_pin, *h_pin_out, *h_wc, *h_mapped, *d_mapped;
  cudaMalloc(&d_in, in_bytes);
  cudaMalloc(&d_out, out_bytes);
  cudaMallocHost(&h_pin, in_bytes);
  cudaMallocHost(&h_pin_out, out_bytes);
  cudaHostAlloc(&h_wc, in_bytes, cudaHostAllocWriteCombined);
  cudaHostAlloc(&h_mapped, in_bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&d_mapped, h_mapped, 0);
  std::vector<char> pageable(in_bytes), pageable_out(out_bytes);
  bench("empty kernel launch", [&] { empty_kernel<<<1, 32, 0, st>>>(); }, st);
  bench("empty kernel launch x148 CTAs", [&] { empty_kernel<<<148, 544, 0, st>>>(); }, st);
  bench("H2D 24KB pinned", [&] { cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st); }, st);
  bench("H2D 24KB write-combined", [&] { cudaMemcpyAsync(d_in, h_wc, in_bytes, cudaMemcpyHostToDevice, st); }, st);
  bench("H2D 24KB pageable", [&] { cudaMemcpyAsync(d_in, pageable.data(), in_bytes, cudaMemcpyHostToDevice, st); }, st);
  bench("H2D 4KB pinned", [&] { cudaMemcpyAsync(d_in, h_pin, 4096, cudaMemcpyHostToDevice, st); }, st);
  bench("H2D 24KB pinned, cudaMemcpyDefault", [&] { cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyDefault, st); }, st);
  bench("D2H 16KB pinned", [&] { cudaMemcpyAsync(h_pin_out, d_out, out_bytes, cudaMemcpyDeviceToHost, st); }, st);
  bench("D2H 16KB pageable", [&] { cudaMemcpyAsync(pageable_out.data(), d_out, out_bytes, cudaMemcpyDeviceToHost, st); }, st);
  bench("H2D pinned + launch + D2H pinned", [&] {
    cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st);
    empty_kernel<<<148, 544, 0, st>>>();
    cudaMemcpyAsync(h_pin_out, d_out, out_bytes, cudaMemcpyDeviceToHost, st);
  }, st);
  bench("H2D 24KB pinned (again)", [&] { cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st); }, st);
  bench("H2D 24KB pinned, Default (again)", [&] { cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyDefault, st); }, st);
  {
    // the library's pattern: pack into the pinned block, time only the copy call
    for (int i = 0; i < 20; ++i) cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    double api = 0;
    for (int i = 0; i < 500; ++i) {
      std::memcpy(h_pin, pageable.data(), in_bytes);
      const double t0 = now_us();
      cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st);
      api += now_us() - t0;
      cudaStreamSynchronize(st);
    }
    std::printf("%-40s api %6.2f us\n", "H2D 24KB pinned after host packing", api / 500);
  }
  for (int coop = 0; coop < 2; ++coop) {
    // H2D api time when each iteration is H2D, a (cooperative) 148x544 launch, D2H, sync
    double api_h2d = 0, api_launch = 0, api_d2h = 0;
    const int n = 300;
    for (int i = 0; i < n + 20; ++i) {
      const double t0 = now_us();
      cudaMemcpyAsync(d_in, h_pin, in_bytes, cudaMemcpyHostToDevice, st);
      const double t1 = now_us();
      if (coop) {
        void* args[] = {nullptr};
        cudaLaunchCooperativeKernel((const void*)empty_kernel, dim3(148), dim3(544), args, 0, st);
      } else {
        empty_kernel<<<148, 544, 0, st>>>();
      }
      const double t2 = now_us();
      cudaMemcpyAsync(h_pin_out, d_out, out_bytes, cudaMemcpyDeviceToHost, st);
      const double t3 = now_us();
      cudaStreamSynchronize(st);
      if (i >= 20) {
        api_h2d += t1 - t0;
        api_launch += t2 - t1;
        api_d2h += t3 - t2;
      }
    }
    std::printf("%s step: h2d api %.2f us, launch api %.2f us, d2h api %.2f us\n", coop ? "cooperative" : "plain",
                api_h2d / n, api_launch / n, api_d2h / n);
  }
  {
    BigParams bp{};
    SmallParams sp{};
    cudaFuncSetAttribute((const void*)big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute((const void*)small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    void* bargs[] = {&bp};
    void* sargs[] = {&sp};
    bench("coop launch, 3816-B params, 200KB smem", [&] {
      cudaLaunchCooperativeKernel((const void*)big_kernel, dim3(148), dim3(544), bargs, 200 * 1024, st);
    }, st);
    bench("coop launch, 440-B params, 200KB smem", [&] {
      cudaLaunchCooperativeKernel((const void*)small_kernel, dim3(148), dim3(544), sargs, 200 * 1024, st);
    }, st);
    bench("plain launch, 3816-B params, 200KB smem", [&] { big_kernel<<<148, 544, 200 * 1024, st>>>(bp); }, st);
    bench("plain launch, 440-B params, 200KB smem", [&] { small_kernel<<<148, 544, 200 * 1024, st>>>(sp); }, st);
  }
  bench("memcpy 24KB host->pinned", [&] { std::memcpy(h_pin, pageable.data(), in_bytes); }, st);
  bench("cudaPointerGetAttributes", [&] {
    cudaPointerAttributes a{};
    cudaPointerGetAttributes(&a, h_pin);
  }, st);
  bench("cudaStreamSynchronize (idle)", [&] {}, st);
  return 0;
}

#ifndef COPYAPI_LIB
int main() { return bench_main(); }
#endif

// Dev: end-to-end cost of one synchronous decode-like step -- H2D of a 24 KB
// pinned block, a cooperative 148 x 544 kernel with ~200 KB dynamic smem that
// spins ~T us, stream sync -- issued with direct API calls vs replayed as a
// CUDA graph (kernel params updated per step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ubench/graph_e2e.cu -o /tmp/ge
#include <chrono>
#include <cstdio>
#include <vector>

struct Params {
  const float* in;
  float* out;
  long long spin;
  int step;
  char pad[900];  // (a DecodeParams-sized argument)
};

__global__ void __launch_bounds__(544, 1) k_step(const Params p) {
  extern __shared__ float sm[];
  const long long t0 = clock64();
  if (threadIdx.x == 0) sm[0] = p.in[blockIdx.x];
  while (clock64() - t0 < p.spin) {
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) p.out[0] = sm[0] + p.step;
}

int main() {
  const size_t bytes = 24576, smem = 200 * 1024;
  float *h, *d, *o;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&d, bytes);
  cudaMallocHost(&o, 64);
  float* od;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&od), o, 0);
  cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Params p{};
  p.in = d;
  p.out = od;
  p.spin = 50 * 1900;  // ~50 us at 1.9 GHz
  const int R = 300;
  auto now = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  for (int mode = 0; mode < 2; ++mode) {
    cudaGraphExec_t ge = nullptr;
    cudaGraphNode_t kn = nullptr;
    cudaKernelNodeParams kp{};
    void* args[] = {&p};
    if (mode == 1) {
      cudaGraph_t g;
      cudaGraphCreate(&g, 0);
      cudaGraphNode_t mn;
      cudaMemcpy3DParms mp{};
      mp.srcPtr = make_cudaPitchedPtr(h, bytes, bytes, 1);
      mp.dstPtr = make_cudaPitchedPtr(d, bytes, bytes, 1);
      mp.extent = make_cudaExtent(bytes, 1, 1);
      mp.kind = cudaMemcpyHostToDevice;
      cudaGraphAddMemcpyNode(&mn, g, nullptr, 0, &mp);
      kp.func = reinterpret_cast<void*>(k_step);
      kp.gridDim = dim3(148);
      kp.blockDim = dim3(544);
      kp.sharedMemBytes = smem;
      kp.kernelParams = args;
      cudaGraphAddKernelNode(&kn, g, &mn, 1, &kp);
      cudaLaunchAttributeValue v{};
      v.cooperative = 1;
      printf("coop attr: %s\n", cudaGetErrorString(cudaGraphKernelNodeSetAttribute(kn, cudaLaunchAttributeCooperative, &v)));
      printf("instantiate: %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
    }
    std::vector<double> ts;
    for (int r = 0; r < R; ++r) {
      const double t0 = now();
      h[0] = static_cast<float>(r);
      p.step = r;
      if (mode == 0) {
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
        cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_step), dim3(148), dim3(544), args, smem, st);
      } else {
        cudaGraphExecKernelNodeSetParams(ge, kn, &kp);
        cudaGraphLaunch(ge, st);
      }
      cudaStreamSynchronize(st);
      ts.push_back(now() - t0);
      if (o[0] != static_cast<float>(r) + r) printf("wrong result %f at %d (%s)\n", o[0], r, cudaGetErrorString(cudaGetLastError()));
    }
    double s = 0;
    for (int r = 20; r < R; ++r) s += ts[r];
    printf("%s: %.2f us per step (kernel spin ~50 us) %s\n", mode ? "graph" : "direct", s / (R - 20), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

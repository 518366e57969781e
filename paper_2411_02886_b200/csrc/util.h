// Launchers of the reference's tensor utilities on the device (util.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tsb {

cudaError_t launch_softmax_rows(const float* m, int rows, int cols, float* out, cudaStream_t st);
cudaError_t launch_topk64(const double* s, int n, int k, uint32_t* out, int* n_out, cudaStream_t st);
cudaError_t launch_cosine(const double* u, const double* v, int n, double* out, cudaStream_t st);
// ws: C * H * N doubles (the logits of every (row, head))
cudaError_t launch_sdpa_full(const float* q, const float* k, const float* v, int C, int N, int H, int H_kv, int d,
                             float* out, double* ws, cudaStream_t st);

}  // namespace tsb

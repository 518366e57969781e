// Launchers for the auxiliary kernels (aux.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tsb {

struct PrefillAttendParams {
  const float* q;          // [C][H*d]
  const float* k_cur;      // [C][H_kv*d]
  const float* v_cur;
  const uint16_t* k_slab;  // bf16 bits
  const uint16_t* v_slab;
  const int32_t* page_table;
  int page_size;
  const uint32_t* att;     // attended cached rows (merged windows)
  int n_att;
  const int* n_att_ptr;    // device count (overrides n_att when set)
  int n_att_max;           // bound on the attended count (the tensor-core paths' gathered copy)
  // tcgen05 path, implicit windows (win_n_att set): the attended rows are
  // [0, win_init_end) ++ the selection inside [win_init_end, win_local_begin)
  // ++ [max(win_local_begin, win_init_end), win_cached) -- make_windows +
  // merged() (attention.cpp:21-52) formed inside prep_tc_kernel, which also
  // writes the count to win_n_att (then n_att_ptr)
  const uint32_t* win_sel;   // ascending selection (nullptr: none)
  const int* win_n_sel;      // its device count
  int win_init_end, win_local_begin, win_cached;
  int* win_n_att;
  int C, H, H_kv, d;
  float scale;
  float* out;              // [C][H*d]
  uint16_t* split_ws;      // tensor-core paths: [2][3][C][H_kv*d] bf16 parts of the chunk K/V, then
                           // (tcgen05) [2][n_att_max][H_kv*d] the attended cached K/V rows, gathered
  unsigned long long* trace;  // dev: %globaltimer stamps of CTA (0, 0) of the tcgen05 kernel (nullptr: off)
};

cudaError_t launch_kv_append(uint16_t* k_slab, uint16_t* v_slab, const float* k, const float* v,
                             const uint16_t* kb, const uint16_t* vb, const int64_t* dst_rows, int t,
                             int row, cudaStream_t st,
                             const int32_t* pt = nullptr, int64_t pos0 = 0, int page_size = 1, bool pdl = false);
cudaError_t launch_kv_gather(const uint16_t* k_slab, const uint16_t* v_slab, const int64_t* src_rows,
                             int n, int row, float* k_out, float* v_out, cudaStream_t st);
cudaError_t launch_chunk_mean(const float* q, int c, int width, float* out, cudaStream_t st);
cudaError_t launch_max_index(const uint32_t* idx, int n, unsigned int* out, cudaStream_t st);
cudaError_t launch_windows(const uint32_t* sel, const int* n_sel_ptr, int n_sel_fixed, int cached,
                           int init_end, int local_begin, uint32_t* out, int* n_out,
                           unsigned int* bad, cudaStream_t st);
cudaError_t launch_prefill_attend(const PrefillAttendParams& p, cudaStream_t st);
// tensor-core path (prefill.cu): d = 128, G <= 8; cudaErrorInvalidValue otherwise
cudaError_t launch_prefill_flash(const PrefillAttendParams& p, cudaStream_t st);
// tcgen05 path (prefill_tc.cu): d = 128, G <= 16; cudaErrorInvalidValue otherwise
cudaError_t launch_prefill_tc(const PrefillAttendParams& p, cudaStream_t st);
// extra bytes launch_prefill_tc needs in split_ws past the gathered rows (the
// balanced plan's partial slots and piece counters), + 256 for alignment
size_t prefill_tc_extra_ws_bytes(const PrefillAttendParams& p, cudaStream_t st);
cudaError_t launch_shard_merge(const uint32_t* all, int world, int k, uint32_t ie, uint32_t lbs, uint32_t base,
                               uint32_t n_r, uint32_t init_hi, uint32_t loc_lo, uint32_t* att, int* n_att,
                               cudaStream_t st);
// packed: rank blocks of [H*d outputs | H x (M, L)] (ml_all = o_all + H*d)
cudaError_t launch_shard_combine(const float* o_all, const float* ml_all, int world, int H, int d, float* out,
                                 cudaStream_t st, bool packed = false);

}  // namespace tsb

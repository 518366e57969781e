// select_head_vote on the device (vote.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "params.h"

namespace tsb {

struct VoteWorkspace {
  uint32_t* thr;    // [H] per-head k-th largest key
  int* cut;         // [H] index of the last tie taken per head
  uint32_t* votes;  // [T]
  uint32_t* vhist;  // [65]
};

// S: device [H][T] scores (row h = head h). Writes the SelectionResult
// (ascending candidates, votes as criticality, optional slab rows through a
// page-size-1 page table) and its size to *n_out (device). No-op when
// skip_if_hit is set and its last lookup hit.
cudaError_t launch_head_vote(const float* S, int H, int T, int k, const uint32_t* cand, int cand_begin,
                             const int32_t* page_table, uint32_t* sel, float* crit, int32_t* sel_rows, int* n_out,
                             VoteWorkspace ws, const CacheState* skip_if_hit, cudaStream_t st);

}  // namespace tsb

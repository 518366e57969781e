// The single-sequence decode step kernel (step.cu): launch descriptor shared
// by the host C-ABI layer (abi.cpp) and the kernel.
#pragma once

#include <cstddef>
#include <cstdint>

#include "decode.h"
#include "params.h"

namespace tsb {

constexpr int kStepThreads = kDecodeThreads;     // 1 TMA producer warp + 16 consumer warps
constexpr int kStepRowsPerBatch = 24;            // attended K/V rows staged per batch (96 KB)
constexpr int kStepMaxStagesPerWarp = 64;        // TMEM: 128 columns per consumer warp, 2 per stage (G <= 4)

struct StepParams {
  const uint16_t* k_slab;   // bf16 bits [frames][H_kv][d] (page_size 1)
  const uint16_t* v_slab;
  uint16_t* k_slab_w;
  uint16_t* v_slab_w;
  int32_t* page_table;      // frame per logical position
  int H, H_kv;              // d = 128
  int k;                    // selection budget
  int N;                    // cached tokens at step start
  int select;               // 1: the Selection Cache lookup / selection runs this step
  int cand_begin;           // candidates [cand_begin, cand_begin + T)
  int T;
  int init_end;             // windows: [0, init_end) and [lb, N) + the current token
  int lb;
  int tpc;                  // candidates per CTA (multiple of 16)
  int stages_per_warp;      // mrec rows per consumer warp
  int ring_stages;          // K ring depth
  float attn_scale;
  const float* q;           // [H * d]
  const float* k_new;       // [H_kv * d] fp32
  const float* v_new;
  float* out;               // [H * d]
  int32_t append_frame;     // slab row of position N (-1: none)
  CacheState* cache;
  float* cached_q;          // [H * d]
  uint32_t* sel;            // [k] cached SelectionResult (ascending)
  float* sel_crit;
  int32_t* sel_rows;
  // workspace
  float2* ws_mz;            // [H][stats_stride(ncta)] per-CTA (m, z)
  uint32_t* ws_hist;        // [2][kRadixBins]
  uint32_t* ws_cnt;         // [ncta] keys tied at the threshold
  uint32_t* ws_nsel;        // [ncta] selected candidates per CTA
  float* ws_o;              // [ncta][H * d] attention partials (unnormalised)
  float2* ws_ml;            // [ncta][H] (m, l) of the partials
  unsigned int* bar;        // grid barrier counters: bar[slot], the other slot is reset
  int bar_slot;
  unsigned long long* trace;  // [CTA][kTraceStride] clock64 stamps (nullptr: off)
};

const void* step_kernel_ptr(int G);
size_t step_smem_bytes(int H, int H_kv, int tpc, int stages_per_warp, int ring_stages);

}  // namespace tsb

// Host/device shared constants, scan geometry and shared-memory layout of
// the fused decode kernel (decode.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#if defined(__CUDACC__)
#define TSB_HD __host__ __device__
#else
#define TSB_HD
#endif

namespace tsb {

constexpr int kDecodeConsumers = 16;            // tensor-core consumer warps of the scan
constexpr int kDecodeWarps = kDecodeConsumers + 1;  // + warp 0: TMA producer
constexpr int kDecodeThreads = kDecodeWarps * 32;
constexpr int kMaxStages = 16;
// Ring barriers are per (consumer phase, slot): a consumer warp takes every
// nphase-th stage, so with kStages % nphase != 0 one barrier per slot would be
// shared by the phases and a warp's parity wait could alias a phase it skipped.
constexpr int kMaxBarPairs = 64;
constexpr size_t kRingBudget = 96 * 1024;        // minimum K-row ring (also attention staging)
constexpr int kRadixBins = 4096;                 // 12-bit radix digits (2 passes -> 24-bit keys)
constexpr int kHistPass = kRadixBins;            // global histogram words per pass
constexpr int kMaxPrefix = 256;                  // >= ctas_per_seq + 1
constexpr int kAttMaxG = 8;                      // query heads per KV head on the attention path
constexpr int kAttMaxRows = 256;                 // rows per attention sub-chunk (upper bound)
constexpr int kTraceStride = 64;                 // phase-trace slots per CTA

TSB_HD inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Fast-path geometry: stages of 16 tokens (one m16 MMA tile), rows at a
// 16-byte padded stride; consumer warp c takes kv head c % H_kv of every
// (16 / H_kv)-th stage.
struct ScanGeom {
  int fast;     // 1: tensor-core TMA path, 0: generic path
  int rows;     // R: tokens per stage
  int stages;   // ring depth
};

// Stage bytes: padded rows (row-by-row bulk copies), or with the tensor map a
// slot that takes either those or 16 dense swizzled rows.
TSB_HD inline size_t scan_stage_bytes(int row_bytes, bool tma) {
  // with the tensor map a slot holds either layout, at a 1024-B aligned stride
  return tma ? align_up(static_cast<size_t>(16) * (row_bytes + 16), 1024) : static_cast<size_t>(16) * (row_bytes + 16);
}

TSB_HD inline ScanGeom scan_geom(int H, int H_kv, int d, size_t ring_bytes = kRingBudget, bool tma = false) {
  ScanGeom g{0, 0, 0};
  if (H_kv <= 0 || H % H_kv != 0) return g;
  const int G = H / H_kv;
  if (!(d == 128 || d == 64) || G > 8 || G < 1) return g;
  if (H_kv > kDecodeConsumers || kDecodeConsumers % H_kv != 0) return g;
  const size_t stage = scan_stage_bytes(H_kv * d * 2, tma);
  int stages = static_cast<int>(ring_bytes / stage);
  if (stages > kMaxStages) stages = kMaxStages;
  const int nphase = kDecodeConsumers / H_kv;
  if (stages * nphase > kMaxBarPairs) stages = kMaxBarPairs / nphase;
  if (stages < 2) return g;
  g.fast = 1;
  g.rows = 16;
  g.stages = stages;
  return g;
}

struct SmemLayout {
  size_t ring, s, keys, frames, hist, prefix, headmax, f, scratch, bars, total;
};

// S storage modes (DecodeParams::s_in_smem): 0 spilled to global (ws_s),
// 1 shared memory, 2 tensor memory (the LEAN kernel; keys stay in smem).
constexpr int kSGlobal = 0, kSSmem = 1, kSTmem = 2;
// TMEM mode: every consumer warp keeps its own stages' S fragments in its lane
// quarter, 4 columns per stage, 128 columns per warp (4 warps per quarter).
constexpr int kTmemColsPerWarp = 128;
TSB_HD inline bool tmem_fits(int H_kv, int tpc) {
  if (H_kv <= 0 || H_kv > 8 || kDecodeConsumers % H_kv) return false;
  const int nphase = kDecodeConsumers / H_kv;
  const int nit = (tpc + 15) / 16;
  return (nit + nphase - 1) / nphase * 4 <= kTmemColsPerWarp;
}

TSB_HD inline SmemLayout smem_layout(int H, int row_bytes, int tpc, int s_in_smem,
                                     size_t ring_bytes = kRingBudget) {
  SmemLayout L{};
  size_t o = 0;
  L.ring = o;
  size_t ring = ring_bytes;
  const size_t att = static_cast<size_t>(2) * 8 * row_bytes;  // >= 8 attended K+V rows
  if (att > ring) ring = att;
  o += align_up(ring, 128);
  L.s = o;
  if (s_in_smem == kSSmem) o += align_up(static_cast<size_t>(H) * tpc * 4, 128);
  // criticality keys overwrite S row 0 in place (each thread writes the keys
  // of the candidates whose S column it has just read); with S in TMEM they
  // get their own array
  L.keys = L.s;
  if (s_in_smem == kSTmem) o += align_up(static_cast<size_t>(tpc) * 4, 128);
  L.frames = o;  // slab row of every candidate of the CTA (TMA producer lookahead)
  o += align_up(static_cast<size_t>(tpc) * 4, 128);
  L.hist = L.ring;  // radix histogram: the ring is idle between the scan and the attention
  L.prefix = o;
  o += kMaxPrefix * 4;
  L.headmax = o;
  o += align_up(static_cast<size_t>(H) * 4, 16);
  L.f = o;
  o += align_up(static_cast<size_t>(H) * 4, 16);
  L.scratch = o;
  o += 256 * 4;
  L.bars = o;
  o += (2 * kMaxBarPairs + 4) * 8;  // full/empty ring barriers + attention (x2) + aux
  L.total = align_up(o, 128);
  return L;
}

// Attention partial (o[d], m, l) record, padded to 16 bytes for bulk copies.
TSB_HD inline int att_stride(int d) { return (d + 2 + 3) & ~3; }
// Per-sequence stats rows [h][ctas], padded to 16 bytes for bulk copies.
TSB_HD inline int stats_stride(int ctas) { return (ctas + 3) & ~3; }

// Attention decomposition of one sequence's CTAs: (KV-head group, row chunk).
struct AttSplit {
  int groups;  // CTAs per row chunk (each owns KV heads g = gi, gi + groups, ...)
  int chunks;  // row chunks per KV head
};
TSB_HD inline AttSplit att_split(int H_kv, int ctas_per_seq) {
  AttSplit a;
  a.groups = H_kv < ctas_per_seq ? H_kv : ctas_per_seq;
  a.chunks = ctas_per_seq / a.groups;
  return a;
}

// variant 0: the general kernel; 1: LEAN, the engine's single-sequence decode
// step; 2: LEAN select-only (select_for_chunk)
const void* decode_kernel_ptr(int D, int G, bool fast, int variant);

}  // namespace tsb

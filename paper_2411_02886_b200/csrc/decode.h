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

constexpr int kDecodeWarps = 16;                 // warp 0: TMA producer, 1..15: consumers
constexpr int kDecodeThreads = kDecodeWarps * 32;
constexpr int kConsumerWarps = kDecodeWarps - 1;
constexpr int kMaxStages = 8;
constexpr size_t kRingBudget = 96 * 1024;        // K-row ring (also attention staging)

TSB_HD inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Fast-path geometry: a lane owns EPL contiguous elements of one kv head,
// WPR warps cover one K row (H_kv*d bf16), each consumer warp handles two
// rows per stage, so a stage holds R = 2*floor(15/WPR) rows.
struct ScanGeom {
  int fast;     // 1: templated TMA path, 0: generic path
  int epl;      // elements per lane (8 or 16)
  int wpr;      // warps per row
  int rows;     // R: rows per stage
  int stages;   // ring depth
};

TSB_HD inline int fast_group_ok(int G) { return G == 1 || G == 2 || G == 4 || G == 7 || G == 8; }

TSB_HD inline ScanGeom scan_geom(int H, int H_kv, int d) {
  ScanGeom g{0, 0, 0, 0, 0};
  if (H_kv <= 0 || H % H_kv != 0) return g;
  const int G = H / H_kv;
  if (!(d == 128 || d == 64) || !fast_group_ok(G)) return g;
  const int epl = G > 4 ? 8 : 16;
  const int E = H_kv * d;
  if (E % (32 * epl) != 0) return g;
  const int wpr = E / (32 * epl);
  if (wpr > kConsumerWarps) return g;
  const int rows = 2 * (kConsumerWarps / wpr);
  if (rows > 32) return g;  // one producer lane per row
  const size_t stage = static_cast<size_t>(rows) * E * 2;
  int stages = static_cast<int>(kRingBudget / stage);
  if (stages > kMaxStages) stages = kMaxStages;
  if (stages < 2) return g;
  g.fast = 1;
  g.epl = epl;
  g.wpr = wpr;
  g.rows = rows;
  g.stages = stages;
  return g;
}

struct SmemLayout {
  size_t ring, s, keys, frames, hist, headmax, f, scratch, bars, total;
};

TSB_HD inline SmemLayout smem_layout(int H, int row_bytes, int tpc, int s_in_smem) {
  SmemLayout L{};
  size_t o = 0;
  L.ring = o;
  size_t ring = kRingBudget;
  const size_t att = static_cast<size_t>(2) * 8 * row_bytes;  // >= 8 attended K+V rows
  if (att > ring) ring = att;
  o += align_up(ring, 128);
  L.s = o;
  if (s_in_smem) o += align_up(static_cast<size_t>(H) * tpc * 4, 128);
  L.keys = o;
  if (s_in_smem) o += align_up(static_cast<size_t>(tpc) * 4, 128);
  L.frames = o;  // slab row of every candidate of the CTA (TMA producer lookahead)
  o += align_up(static_cast<size_t>(tpc) * 4, 128);
  L.hist = o;
  o += 2048 * 4;
  L.headmax = o;
  o += align_up(static_cast<size_t>(H) * 4, 16);
  L.f = o;
  o += align_up(static_cast<size_t>(H) * 4, 16);
  L.scratch = o;
  o += 128 * 4;
  L.bars = o;
  o += (2 * kMaxStages + 2) * 8;  // full/empty ring barriers + attention barrier
  L.total = align_up(o, 128);
  return L;
}

// Attention partial (o[d], m, l) record, padded to 16 bytes for bulk copies.
TSB_HD inline int att_stride(int d) { return (d + 2 + 3) & ~3; }
// Per-sequence stats rows [h][ctas], padded to 16 bytes for bulk copies.
TSB_HD inline int stats_stride(int ctas) { return (ctas + 3) & ~3; }

const void* decode_kernel_ptr(int D, int G, bool fast);

}  // namespace tsb

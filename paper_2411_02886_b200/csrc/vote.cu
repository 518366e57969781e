// select_head_vote (Eq. 6, reference selector.cpp:101-111) on the device:
// every head votes for its own top-k tokens (topk_indices, tensor.cpp:68-90:
// larger score first, the smaller index on ties), the votes are summed and
// the k tokens with the most votes are picked (pick(), selector.cpp:72-85:
// the smaller index on equal votes), output ascending.
//
//   head_topk_kernel   one CTA per head: exact 32-bit radix select of the
//                      head's k-th largest score (four 8-bit passes over the
//                      order-preserving keys) and the index of the last tie
//                      it takes -> (threshold, cut) per head
//   vote_count_kernel  votes[j] = #heads with (key > thr) or (key == thr and
//                      j <= cut), histogram of the vote counts
//   vote_pick_kernel   one CTA: the vote threshold, ties by position, the
//                      ascending compaction -> SelectionResult
//
// All three kernels are no-ops when `skip_if_hit` points to a Selection Cache
// state whose last lookup hit (the engine's decode path launches them
// unconditionally after the decision launch).
#include "common.cuh"
#include "params.h"
#include "vote.h"

namespace tsb {

namespace {

constexpr int kVT = 1024;

// the engine's decode path: nothing to select on a hit or a rejected (zero) query
__device__ __forceinline__ bool skip(const CacheState* c) {
  return c && (__ldcg(&c->last_hit) == 1 || __ldcg(&c->error) != 0);
}

// Exclusive block scan (kVT threads) of one value per thread; *total = sum.
__device__ uint32_t vscan(uint32_t v, uint32_t* sh, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(v, lane);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = sh[lane];
    const uint32_t wi = warp_incl_scan(w, lane);
    sh[32 + lane] = wi - w;
    if (lane == 31) sh[64] = wi;
  }
  __syncthreads();
  const uint32_t r = sh[32 + warp] + inc - v;
  *total = sh[64];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kVT) head_topk_kernel(const float* __restrict__ S, int T, int k,
                                                        uint32_t* thr_out, int* cut_out, const CacheState* hit) {
  if (skip(hit)) return;
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh[80];
  const int h = blockIdx.x, tid = threadIdx.x;
  const float* row = S + static_cast<size_t>(h) * T;
  const uint32_t kk = static_cast<uint32_t>(min(k, T));
  if (kk >= static_cast<uint32_t>(T)) {  // every token is in the head's top-k
    if (tid == 0) {
      thr_out[h] = 0u;
      cut_out[h] = T - 1;
    }
    return;
  }
  uint32_t prefix = 0, need = kk;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += kVT) hist[i] = 0u;
    __syncthreads();
    for (int j = tid; j < T; j += kVT) {
      const uint32_t key = float_key(__ldg(row + j));
      if (pass == 0 || (key >> (shift + 8)) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // descending bins: lane l covers bins 255 - 8l .. 248 - 8l
      uint32_t c[8], s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = hist[255 - 8 * tid - i];
        s += c[i];
      }
      const uint32_t incl = warp_incl_scan(s, tid);
      const uint32_t excl = incl - s;
      const bool here = excl < need && incl >= need;
      if (here) {
        uint32_t acc = excl;
        int b = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (acc + c[i] >= need) {
            b = 255 - 8 * tid - i;
            break;
          }
          acc += c[i];
        }
        sh[70] = static_cast<uint32_t>(b);
        sh[71] = need - acc;  // still needed inside bin b
      }
    }
    __syncthreads();
    prefix = (prefix << 8) | sh[70];
    need = sh[71];
    __syncthreads();
  }
  // prefix = the k-th largest key; the first `need` keys equal to it (by index) are taken
  int cut = -1;
  uint32_t seen = 0;
  for (int b0 = 0; b0 < T; b0 += kVT) {
    const int j = b0 + tid;
    const uint32_t eq = (j < T && float_key(__ldg(row + j)) == prefix) ? 1u : 0u;
    uint32_t tot;
    const uint32_t r = seen + vscan(eq, sh, &tot);
    if (eq && r == need - 1) sh[72] = static_cast<uint32_t>(j);
    seen += tot;
    __syncthreads();
    if (seen >= need) {
      cut = static_cast<int>(sh[72]);
      break;
    }
  }
  if (tid == 0) {
    thr_out[h] = prefix;
    cut_out[h] = cut;
  }
}

__global__ void vote_count_kernel(const float* __restrict__ S, int H, int T, const uint32_t* __restrict__ thr,
                                  const int* __restrict__ cut, uint32_t* votes, uint32_t* vhist,
                                  const CacheState* hit) {
  if (skip(hit)) return;
  __shared__ uint32_t lh[65];
  for (int i = threadIdx.x; i <= H; i += blockDim.x) lh[i] = 0u;
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < T) {
    uint32_t v = 0;
    for (int h = 0; h < H; ++h) {
      const uint32_t key = float_key(__ldg(S + static_cast<size_t>(h) * T + j));
      const uint32_t t = __ldg(thr + h);
      v += (key > t || (key == t && j <= __ldg(cut + h))) ? 1u : 0u;
    }
    votes[j] = v;
    atomicAdd(&lh[v], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= H; i += blockDim.x)
    if (lh[i]) atomicAdd(vhist + i, lh[i]);
}

__global__ void __launch_bounds__(kVT) vote_pick_kernel(const uint32_t* __restrict__ votes, const uint32_t* vhist,
                                                        int H, int T, int k, const uint32_t* cand, int cand_begin,
                                                        const int32_t* page_table, uint32_t* sel, float* crit,
                                                        int32_t* sel_rows, int* n_out, const CacheState* hit) {
  if (skip(hit)) return;
  __shared__ uint32_t sh[80];
  const int tid = threadIdx.x;
  const uint32_t kk = static_cast<uint32_t>(min(k, T));
  if (tid == 0) {
    // vote threshold: count(votes > v) < kk <= count(votes >= v)
    uint32_t above = 0;
    int v = H;
    for (; v >= 0; --v) {
      const uint32_t c = __ldcg(vhist + v);
      if (above + c >= kk) break;
      above += c;
    }
    sh[70] = static_cast<uint32_t>(max(v, 0));
    sh[71] = kk - above;  // ties at the threshold taken, lowest positions first
  }
  __syncthreads();
  const uint32_t vt = sh[70], need = sh[71];
  uint32_t out = 0, eq_seen = 0;
  for (int b0 = 0; b0 < T; b0 += kVT) {
    const int j = b0 + tid;
    const uint32_t v = j < T ? __ldcg(votes + j) : 0u;
    const uint32_t eq = (j < T && v == vt) ? 1u : 0u;
    uint32_t eq_tot;
    const uint32_t r = eq_seen + vscan(eq, sh, &eq_tot);
    eq_seen += eq_tot;
    const uint32_t take = (j < T && (v > vt || (eq && r < need))) ? 1u : 0u;
    uint32_t tot;
    const uint32_t pos = out + vscan(take, sh, &tot);
    if (take) {
      const uint32_t tok = cand ? __ldg(cand + j) : static_cast<uint32_t>(cand_begin + j);
      sel[pos] = tok;
      crit[pos] = static_cast<float>(v);
      if (sel_rows) sel_rows[pos] = __ldg(page_table + tok);
    }
    out += tot;
  }
  if (tid == 0) *n_out = static_cast<int>(out);
}

}  // namespace

cudaError_t launch_head_vote(const float* S, int H, int T, int k, const uint32_t* cand, int cand_begin,
                             const int32_t* page_table, uint32_t* sel, float* crit, int32_t* sel_rows, int* n_out,
                             VoteWorkspace ws, const CacheState* skip_if_hit, cudaStream_t st) {
  if (H < 1 || H > 64 || T < 1 || k < 1) return cudaErrorInvalidValue;
  head_topk_kernel<<<H, kVT, 0, st>>>(S, T, k, ws.thr, ws.cut, skip_if_hit);
  cudaError_t e = cudaMemsetAsync(ws.vhist, 0, 65 * 4, st);
  if (e != cudaSuccess) return e;
  vote_count_kernel<<<(T + 255) / 256, 256, 0, st>>>(S, H, T, ws.thr, ws.cut, ws.votes, ws.vhist, skip_if_hit);
  vote_pick_kernel<<<1, kVT, 0, st>>>(ws.votes, ws.vhist, H, T, k, cand, cand_begin, page_table, sel, crit, sel_rows,
                                      n_out, skip_if_hit);
  return cudaGetLastError();
}

}  // namespace tsb

// C-ABI host layer (include/tokenselect.h): the paged KV pool with the
// reference's LIFO frame allocator, the AttentionEngine, and the standalone
// selection / attention entry points, all launching the sm_100a kernels in
// decode.cu and aux.cu. Validation happens before any device work and
// reports the reference's exception type + message (see tokenselect.h).
#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tokenselect.h"
#include "aux.h"
#include "decode.h"
#include "step.h"
#include "vote.h"
#include "util.h"
#include "comm.h"
#include "params.h"

using tsb::CacheState;
using tsb::DecodeParams;
using tsb::SeqDesc;

namespace {

thread_local std::string g_err;
const bool g_force_global_s = std::getenv("TS_FORCE_GLOBAL_S") != nullptr && std::getenv("TS_FORCE_GLOBAL_S")[0];
const int g_debug_flags = std::getenv("TS_DEBUG_FLAGS") ? std::atoi(std::getenv("TS_DEBUG_FLAGS")) : 0;
const bool g_force_cuda_core_prefill = std::getenv("TS_CUDA_CORE_PREFILL") != nullptr;
const bool g_prefill_mma_sync = std::getenv("TS_PREFILL_MMA_SYNC") != nullptr;  // dev: the mma.sync prefill kernel
const bool g_no_lean = std::getenv("TS_NO_LEAN") != nullptr;  // dev: always the general kernel
// the single-sequence step kernel (step.cu) is opt-in: TS_STEP=1. Measured on
// B200 (profiles/r02_step/): stream 54.1 vs 52.5 us/step for the fused kernel
const bool g_no_step = !(std::getenv("TS_STEP") && std::getenv("TS_STEP")[0] == '1');
const bool g_no_tma = std::getenv("TS_NO_TMA") != nullptr;      // dev: row-by-row scan copies
const bool g_no_h2d_primer = std::getenv("TS_NO_H2D_PRIMER") != nullptr;  // dev: see ts_engine_decode
const bool g_debug_tma = std::getenv("TS_DEBUG_TMA") != nullptr;
std::atomic<uint64_t> g_launches{0};
constexpr size_t kTraceSlots = tsb::kTraceStride * 1024;
// host-side profile of the decode launch path (TS_HOST_PROF=1): ns per stage
const bool g_host_prof = std::getenv("TS_HOST_PROF") != nullptr;
double g_prof[4] = {0, 0, 0, 0};
uint64_t g_prof_n = 0;
double g_prof_ld[2] = {0, 0};  // launch_decode: params fill, everything before the launch API
// ts_engine_decode (host buffers): pointer queries, stage+H2D, engine_step, D2H issue, sync wait, unpack
double g_e2e_prof[6] = {0, 0, 0, 0, 0, 0};
uint64_t g_e2e_n = 0;
double g_e2e_memcpy = 0;  // zero check + host packing part of stage+h2d
double g_e2e_h2dapi = 0;  // the cudaMemcpyAsync call
inline double now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch()).count();
}  // [cta][32] %globaltimer stamps (<= 1024 CTAs)

struct ts_error : std::runtime_error {
  ts_status code;
  ts_error(ts_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(ts_status c, const std::string& m) { throw ts_error(c, m); }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
ts_status guarded(Fn&& fn) {
  try {
    fn();
    return TS_OK;
  } catch (const ts_error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "allocation failed";
    return TS_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TS_INVALID_ARGUMENT;
  }
}

struct DeviceInfo {
  int device = -1;
  int num_sms = 0;
  int smem_optin = 0;
};

const DeviceInfo& device_info() {
  static DeviceInfo info = [] {
    DeviceInfo d;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return d;
    }
    cudaGetDevice(&d.device);
    cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, d.device);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d.device);
    return d;
  }();
  if (info.device < 0) fail(TS_CUDA_ERROR, "no CUDA device: the tokenselect library has no CPU path");
  return info;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Growable device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  // grows geometrically: workspaces track the context length step by step,
  // and every reallocation (cudaFree) synchronises the device
  void* ensure(size_t bytes) {
    if (bytes <= n) return p;
    static const bool dbg = std::getenv("TS_DEBUG_ALLOC") != nullptr;
    if (dbg) std::fprintf(stderr, "[tokenselect] DevBuf %p: %zu -> %zu bytes\n", static_cast<void*>(this), n, bytes);
    if (p) cudaFree(p);
    p = nullptr;
    const size_t want = std::max<size_t>({bytes, n + n / 2, 256});
    n = 0;
    ck(cudaMalloc(&p, want), "cudaMalloc");
    n = want;
    return p;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Host input -> device (staged); device input passes through.
template <typename T>
const T* dev_in(const T* p, size_t count, DevBuf& stage, cudaStream_t st) {
  if (!p || count == 0) return p;
  if (is_device_ptr(p)) return p;
  T* d = static_cast<T*>(stage.ensure(count * sizeof(T)));
  ck(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
  return d;
}

// Per-launch workspaces of the fused kernel + its grid barrier and the
// attention-merge arrival counters (both self-resetting across launches).
struct Workspace {
  DevBuf s, keys, m, z, hist, cnt, nsel, sel_tok, sel_crit, sel_row, att, acnt, bar;
  // select_head_vote (vote.cu): per-head thresholds, votes, and the scores it votes on
  DevBuf v_thr, v_cut, v_votes, v_hist, v_s;
  tsb::VoteWorkspace vote(int H, int T) {
    return tsb::VoteWorkspace{static_cast<uint32_t*>(v_thr.ensure(static_cast<size_t>(H) * 4)),
                              static_cast<int*>(v_cut.ensure(static_cast<size_t>(H) * 4)),
                              static_cast<uint32_t*>(v_votes.ensure(static_cast<size_t>(T) * 4)),
                              static_cast<uint32_t*>(v_hist.ensure(65 * 4))};
  }
  float* vote_scores(int n_seq, int H, int T) {
    return static_cast<float*>(v_s.ensure(static_cast<size_t>(n_seq) * H * T * 4));
  }
  size_t acnt_n = 0;
  unsigned launches = 0;
  void prepare(int n_ctas, int H, int H_kv, int d, int tpc, int s_in_smem, int n_seq, cudaStream_t st) {
    if (!s_in_smem) {
      s.ensure(static_cast<size_t>(n_ctas) * H * tpc * 4);
      keys.ensure(static_cast<size_t>(n_ctas) * tpc * 4);
    }
    const int cps = n_ctas / n_seq;
    m.ensure(static_cast<size_t>(n_seq) * H * tsb::stats_stride(cps) * 4);
    z.ensure(static_cast<size_t>(n_seq) * H * tsb::stats_stride(cps) * 4);
    hist.ensure(static_cast<size_t>(n_seq) * 2 * tsb::kHistPass * 4);
    cnt.ensure(static_cast<size_t>(n_ctas) * 4);
    nsel.ensure(static_cast<size_t>(n_ctas) * 4);
    sel_tok.ensure(static_cast<size_t>(n_ctas) * tpc * 4);
    sel_crit.ensure(static_cast<size_t>(n_ctas) * tpc * 4);
    sel_row.ensure(static_cast<size_t>(n_ctas) * tpc * 4);
    att.ensure(static_cast<size_t>(n_ctas) * H * tsb::att_stride(d) * 4);
    const size_t na = static_cast<size_t>(tsb::kMaxSeqPerLaunch) * H_kv * 2;  // two slots alternate per launch
    if (na > acnt_n) {
      acnt.ensure(na * 4);
      ck(cudaMemsetAsync(acnt.p, 0, acnt.n, st), "memset counters");
      acnt_n = na;
    }
    if (!bar.p) {
      bar.ensure(256);
      ck(cudaMemsetAsync(bar.p, 0, 256, st), "memset barrier");
    }
  }
};

// TMA tensor map of a K slab for the scan: the slab viewed as
// [128-B chunk][slab row][64 bf16] (strides: the row, 128 B per chunk), box =
// 16 rows x the whole row, 128B swizzle keyed by the row
// (tools/ubench/tmap.cu). nullptr when the row is not a whole number of 128-B
// chunks or the encoder is unavailable.
using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
void* encode_k_tmap(uint16_t* slab, size_t rows, size_t row_bytes, cudaStream_t st) {
  if (row_bytes % 128 || row_bytes / 128 > 256 || rows < 16 || rows >= (1ull << 32) || g_no_tma) return nullptr;
  static TmapEncodeFn enc = []() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (g_debug_tma) std::fprintf(stderr, "[tokenselect] cuTensorMapEncodeTiled entry point: %d / %d\n", int(e), int(q));
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess) return static_cast<TmapEncodeFn>(nullptr);
    return reinterpret_cast<TmapEncodeFn>(f);
  }();
  if (!enc) return nullptr;
  alignas(64) CUtensorMap m;
  const cuuint64_t dims[3] = {64, rows, row_bytes / 128};
  const cuuint64_t strides[2] = {row_bytes, 128};
  const cuuint32_t box[3] = {64, 16, static_cast<cuuint32_t>(row_bytes / 128)};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, slab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (g_debug_tma) std::fprintf(stderr, "[tokenselect] K tensor map encode: %d\n", int(r));
  if (r != CUDA_SUCCESS) return nullptr;
  void* d = nullptr;
  ck(cudaMalloc(&d, sizeof(CUtensorMap)), "cudaMalloc tensor map");
  ck(cudaMemcpyAsync(d, &m, sizeof(CUtensorMap), cudaMemcpyHostToDevice, st), "H2D tensor map");
  ck(cudaStreamSynchronize(st), "sync");
  return d;
}

struct Plan {
  int ctas_per_seq, tpc, s_in_smem, ring_bytes, att_bytes;
  size_t smem;
  const void* fn;
  const void* fn_lean;  // the single-sequence decode-step specialisation (nullptr: none)
  const void* fn_lean_sel;  // its select-only twin (select_for_chunk)
  // the LEAN kernel's layout: S in tensor memory, the rest of smem to the ring
  bool lean_ok;
  int lean_ring_bytes, lean_att_bytes;
  size_t lean_smem;
};

// a kernel's static shared memory (cudaFuncGetAttributes costs microseconds
// of host time; make_plan runs every step)
size_t static_smem(const void* fn) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> known;
  std::lock_guard<std::mutex> lock(mu);
  auto it = known.find(fn);
  if (it != known.end()) return it->second;
  cudaFuncAttributes fa{};
  ck(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
  return known[fn] = fa.sharedSizeBytes;
}

Plan make_plan(int H, int H_kv, int d, int n_seq, int max_T, int att_rows, bool attend = true,
               bool force_spill = false) {
  const DeviceInfo& di = device_info();
  Plan pl{};
  const tsb::ScanGeom g = tsb::scan_geom(H, H_kv, d);
  pl.fn = tsb::decode_kernel_ptr(d, H / H_kv, g.fast != 0, 0);
  pl.fn_lean = pl.fn ? tsb::decode_kernel_ptr(d, H / H_kv, g.fast != 0, 1) : nullptr;
  pl.fn_lean_sel = pl.fn ? tsb::decode_kernel_ptr(d, H / H_kv, g.fast != 0, 2) : nullptr;
  if (!pl.fn) pl.fn = tsb::decode_kernel_ptr(0, 0, false, 0);
  const int base = std::max(max_T, att_rows);
  int c = (base + 63) / 64;
  c = std::max(1, std::min(c, std::max(1, di.num_sms / n_seq)));
  pl.ctas_per_seq = c;
  // 16 candidates: 16-B S rows, and whole 16-token scan stages per CTA (TMA)
  pl.tpc = static_cast<int>(tsb::align_up(static_cast<size_t>(std::max(1, (max_T + c - 1) / c)), 16));
  const int row_bytes = H_kv * d * 2;
  // dynamic shared memory left next to the kernel's static allocation
  size_t stat = static_smem(pl.fn);
  if (pl.fn_lean) stat = std::max(stat, static_smem(pl.fn_lean));
  if (pl.fn_lean_sel) stat = std::max(stat, static_smem(pl.fn_lean_sel));
  const size_t optin = static_cast<size_t>(di.smem_optin) - stat;
  tsb::SmemLayout L = tsb::smem_layout(H, row_bytes, pl.tpc, 1);
  if (L.total <= optin && !g_force_global_s && !force_spill) {
    pl.s_in_smem = 1;
  } else {
    pl.s_in_smem = 0;
    L = tsb::smem_layout(H, row_bytes, pl.tpc, 0);
    if (L.total > optin) fail(TS_INVALID_ARGUMENT, "row too wide for the decode kernel");
  }
  // whatever shared memory is left deepens the K ring
  pl.ring_bytes = static_cast<int>(tsb::kRingBudget + (optin - L.total) / 1024 * 1024);
  L = tsb::smem_layout(H, row_bytes, pl.tpc, pl.s_in_smem, static_cast<size_t>(pl.ring_bytes));
  pl.smem = L.total;
  pl.att_bytes = static_cast<int>(L.frames - L.ring);  // ring + S + keys: dead once the selection is out
  pl.lean_ok = pl.fn_lean && tsb::tmem_fits(H_kv, pl.tpc);
  if (pl.lean_ok) {
    tsb::SmemLayout LL = tsb::smem_layout(H, row_bytes, pl.tpc, tsb::kSTmem);
    pl.lean_ok = LL.total <= optin;
    if (pl.lean_ok) {
      pl.lean_ring_bytes = static_cast<int>(tsb::kRingBudget + (optin - LL.total) / 1024 * 1024);
      LL = tsb::smem_layout(H, row_bytes, pl.tpc, tsb::kSTmem, static_cast<size_t>(pl.lean_ring_bytes));
      pl.lean_smem = LL.total;
      pl.lean_att_bytes = static_cast<int>(LL.frames - LL.ring);
    }
  }
  if (attend && H / H_kv > tsb::kAttMaxG)
    fail(TS_INVALID_ARGUMENT, "more than 8 query heads per KV head is not supported by the decode kernel");
  if (d > 256) fail(TS_INVALID_ARGUMENT, "head_dim > 256 is not supported by the decode kernel");
  if (pl.ctas_per_seq + 1 > tsb::kMaxPrefix) fail(TS_INVALID_ARGUMENT, "too many CTAs per sequence");
  return pl;
}

void launch_decode(DecodeParams& p, const Plan& pl, Workspace& ws, cudaStream_t st) {
  const int n_ctas = p.n_seq * pl.ctas_per_seq;
  // the engine's plain single-sequence step runs the specialisation with the
  // other modes compiled out and S in tensor memory (decode.cu, LEAN)
  const tsb::SeqDesc& s0 = p.seqs[0];
  const bool lean_shape = pl.lean_ok && !g_no_lean && !g_force_global_s && p.n_seq == 1 && p.method == 2 &&
                          !s0.att_list && !s0.no_cur && s0.shard_base == 0 && !s0.cand && s0.sel_rows && !s0.ml_out &&
                          !s0.s_out && (p.page_size & (p.page_size - 1)) == 0;
  const bool lean_step = lean_shape && p.mode == (tsb::kModeSelect | tsb::kModeScore | tsb::kModeCache | tsb::kModeAttend |
                                                  tsb::kModeAppend);
  const bool lean_sel = lean_shape && pl.fn_lean_sel && p.mode == (tsb::kModeSelect | tsb::kModeScore);
  const bool lean = lean_step || lean_sel;
  const void* fn = lean_step ? pl.fn_lean : lean_sel ? pl.fn_lean_sel : pl.fn;
  const size_t smem = lean ? pl.lean_smem : pl.smem;
  const double tq0 = g_host_prof ? now_ns() : 0.0;
  ws.prepare(n_ctas, p.H, p.H_kv, p.d, pl.tpc, lean ? 1 : pl.s_in_smem, p.n_seq, st);
  p.ctas_per_seq = pl.ctas_per_seq;
  p.tpc = pl.tpc;
  p.s_in_smem = lean ? tsb::kSTmem : pl.s_in_smem;
  p.ws_s = ws.s.as<float>();
  p.ws_keys = ws.keys.as<uint32_t>();
  p.ws_m = ws.m.as<float>();
  p.ws_z = ws.z.as<float>();
  p.ws_hist = ws.hist.as<uint32_t>();
  p.ws_cnt = ws.cnt.as<uint32_t>();
  p.ws_nsel = ws.nsel.as<uint32_t>();
  p.ws_sel_tok = ws.sel_tok.as<uint32_t>();
  p.ws_sel_crit = ws.sel_crit.as<float>();
  p.ws_sel_row = ws.sel_row.as<int32_t>();
  p.ws_att = ws.att.as<float>();
  p.ws_acnt = ws.acnt.as<unsigned int>();
  p.bar = ws.bar.as<unsigned int>();
  p.bar_slot = (ws.launches & 1u) ? 32 : 0;  // launches on one workspace are stream-ordered
  p.ring_bytes = lean ? pl.lean_ring_bytes : pl.ring_bytes;
  // whole-stage TMA (general kernel): the kernel checks per stage that its
  // 16 slab rows are consecutive (ascending or descending) and else copies rows
  p.scan_tma = !lean && p.k_tmap ? 1 : 0;
  p.any_select = p.any_radix = 0;
  for (int b = 0; b < p.n_seq; ++b) {
    p.any_select |= p.seqs[b].select;
    p.any_radix |= p.seqs[b].select && p.seqs[b].n_cand > p.k;
  }
  if (g_debug_tma) {
    static std::atomic<int> once{0};
    if (once.fetch_add(1) < 4)
      std::fprintf(stderr, "[tokenselect] launch: lean %d, k_tmap %p, scan_tma %d (page %d, tpc %d, cand_begin %d, cand %p)\n",
                   int(lean), p.k_tmap, p.scan_tma, p.page_size, pl.tpc, p.seqs[0].cand_begin,
                   static_cast<const void*>(p.seqs[0].cand));
  }
  p.att_bytes = lean ? pl.lean_att_bytes : pl.att_bytes;
  p.debug_flags = g_debug_flags;
  if (g_host_prof) g_prof_ld[0] += now_ns() - tq0;
  // the dynamic shared-memory limit is set once per kernel (largest request so far)
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> smem_set;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = smem_set[fn];
  if (smem > have) {
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    have = smem;
  }
  void* args[] = {&p};
  const double t0 = g_host_prof ? now_ns() : 0.0;
  if (g_host_prof) g_prof_ld[1] += t0 - tq0;
  ck(cudaLaunchCooperativeKernel(fn, dim3(n_ctas), dim3(tsb::kDecodeThreads), args, smem, st),
     "decode kernel launch");
  if (g_host_prof) g_prof[3] += now_ns() - t0;
  ws.launches += 1;
  g_launches.fetch_add(1);
}

// Workspace of the single-sequence step kernel (step.cu).
struct StepWorkspace {
  DevBuf mz, hist, cnt, nsel, o, ml, bar;
  unsigned launches = 0;
};

// The step kernel's launch geometry for one sequence with T candidates, or
// ok = false when the shape is outside it (the fused decode kernel then runs).
struct StepPlan {
  bool ok = false;
  int ncta = 0, tpc = 16, spw = 1, stages = 0, G = 0;
  size_t smem = 0;
  const void* fn = nullptr;
};

StepPlan step_plan(const ts_engine_config& c, int T, int W) {
  StepPlan sp;
  const DeviceInfo& di = device_info();
  const int H = static_cast<int>(c.num_heads), Hkv = static_cast<int>(c.num_kv_heads);
  if (g_no_step || c.head_dim != 128 || c.selection_method != TS_HEAD_SOFT_VOTE || H > 64 || Hkv > 16 ||
      tsb::kDecodeConsumers % Hkv || H % Hkv)
    return sp;
  const int G = H / Hkv;
  if (G > 8) return sp;
  const int ncta = di.num_sms;
  if (ncta < 32 || ncta > 272 || (H * 128 + ncta - 1) / ncta > 128) return sp;  // step.cu: 2 * ncta <= threads
  const int nph = tsb::kDecodeConsumers / Hkv;
  const int tpc = static_cast<int>(tsb::align_up(static_cast<size_t>(std::max(1, (T + ncta - 1) / ncta)), 16));
  const int spw = std::max(1, (tpc / 16 + nph - 1) / nph);
  const int cps = G <= 4 ? 2 : 4;
  if (spw * cps > 128) return sp;                                   // TMEM: 128 columns per warp
  if ((static_cast<int>(c.k) + ncta - 1) / ncta > 64 || (W + ncta - 1) / ncta > 64) return sp;
  const size_t row_bytes = static_cast<size_t>(Hkv) * 256;
  const size_t sbytes = 16 * (row_bytes + 16);
  const size_t optin = static_cast<size_t>(di.smem_optin);
  int stages = std::min(16, tsb::kMaxBarPairs / nph);
  while (stages >= 2 && tsb::step_smem_bytes(H, Hkv, tpc, spw, stages) > optin) --stages;
  if (stages < 2) return sp;
  // post-scan aliases of the ring (step.cu): histogram + criticality partials
  // + keys, attention staging + scores + phase sums, and the selected list at its end
  const size_t ring = tsb::align_up(static_cast<size_t>(stages) * sbytes, 1024);
  const size_t tail = ring - static_cast<size_t>(3) * tpc * 4;
  const size_t crit_end = 17 * 1024 + static_cast<size_t>(Hkv) * tpc * 4 + static_cast<size_t>(tpc) * 4;
  const size_t att_end = 2 * tsb::kStepRowsPerBatch * row_bytes + (tsb::kStepRowsPerBatch + 1) * 64 * 4 +
                         static_cast<size_t>(nph) * H * 128 * 4;
  const size_t merge_end = static_cast<size_t>(4 * ncta + ncta * 128 + 8 + 128 * ((ncta + 7) / 8)) * 4;
  if (crit_end > tail || att_end > tail || merge_end > tail) return sp;
  sp.fn = tsb::step_kernel_ptr(G);
  if (!sp.fn) return sp;
  sp.ok = true;
  sp.ncta = ncta;
  sp.tpc = tpc;
  sp.spw = spw;
  sp.stages = stages;
  sp.G = G;
  sp.smem = tsb::step_smem_bytes(H, Hkv, tpc, spw, stages);
  return sp;
}

void launch_step(tsb::StepParams& p, const StepPlan& sp, StepWorkspace& ws, cudaStream_t st) {
  const int ncta = sp.ncta, ncp = (ncta + 3) & ~3;
  ws.mz.ensure(static_cast<size_t>(p.H) * ncp * 8);
  ws.hist.ensure(2 * tsb::kRadixBins * 4);
  ws.cnt.ensure(static_cast<size_t>(ncta) * 4);
  ws.nsel.ensure(static_cast<size_t>(ncta) * 4);
  ws.o.ensure(static_cast<size_t>(ncta) * p.H * 128 * 4);
  ws.ml.ensure(static_cast<size_t>(ncta) * p.H * 8);
  if (!ws.bar.p) {
    ws.bar.ensure(256);
    ck(cudaMemsetAsync(ws.bar.p, 0, 256, st), "memset barrier");
  }
  p.tpc = sp.tpc;
  p.stages_per_warp = sp.spw;
  p.ring_stages = sp.stages;
  p.ws_mz = ws.mz.as<float2>();
  p.ws_hist = ws.hist.as<uint32_t>();
  p.ws_cnt = ws.cnt.as<uint32_t>();
  p.ws_nsel = ws.nsel.as<uint32_t>();
  p.ws_o = ws.o.as<float>();
  p.ws_ml = ws.ml.as<float2>();
  p.bar = ws.bar.as<unsigned int>();
  p.bar_slot = (ws.launches & 1u) ? 32 : 0;
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> smem_set;
  {
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = smem_set[sp.fn];
    if (sp.smem > have) {
      ck(cudaFuncSetAttribute(sp.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sp.smem)),
         "cudaFuncSetAttribute");
      have = sp.smem;
    }
  }
  void* args[] = {&p};
  const double t0 = g_host_prof ? now_ns() : 0.0;
  ck(cudaLaunchCooperativeKernel(sp.fn, dim3(ncta), dim3(tsb::kStepThreads), args, sp.smem, st), "step kernel launch");
  if (g_host_prof) g_prof[3] += now_ns() - t0;
  ws.launches += 1;
  g_launches.fetch_add(1);
}

// selattn::Rng::index semantics (rng.hpp:19-26) on std::mt19937_64, so the
// shuffled free list is the reference's permutation.
struct RefRng {
  std::mt19937_64 e;
  explicit RefRng(uint64_t seed) : e(seed) {}
  double uniform() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  size_t index(size_t n) { return static_cast<size_t>(uniform() * static_cast<double>(n)) % n; }
};

}  // namespace

// =================================================================== pool
struct ts_pool {
  size_t page_size = 1, H_kv = 0, d = 0, row = 0, total_frames = 0;
  uint16_t* k_slab = nullptr;
  uint16_t* v_slab = nullptr;
  void* k_tmap = nullptr;  // device CUtensorMap over the K slab (scan stages in one TMA op), or nullptr
  std::vector<uint32_t> free_list;
  struct Seq {
    std::vector<uint32_t> frames;
    size_t len = 0;
    int32_t* d_pt = nullptr;
    int32_t* h_pt = nullptr;  // pinned mirror of the page table (uploads stay asynchronous)
  };
  std::unordered_map<uint32_t, Seq> seqs;
  uint32_t next_id = 0;
  cudaStream_t stream = nullptr;
  Workspace ws;
  DevBuf st_a, st_b, st_c, st_d, st_e, st_f, st_split;  // staging

  ~ts_pool() {
    for (auto& kv : seqs)
      if (kv.second.d_pt) cudaFree(kv.second.d_pt);
    for (auto& kv : seqs)
      if (kv.second.h_pt) cudaFreeHost(kv.second.h_pt);
    if (k_slab) cudaFree(k_slab);
    if (v_slab) cudaFree(v_slab);
    if (k_tmap) cudaFree(k_tmap);
    if (stream) cudaStreamDestroy(stream);
  }

  Seq& state(uint32_t id) {
    auto it = seqs.find(id);
    if (it == seqs.end()) fail(TS_INVALID_ARGUMENT, "PagedKvPool: unknown or released sequence " + std::to_string(id));
    return it->second;
  }
  const Seq& state(uint32_t id) const { return const_cast<ts_pool*>(this)->state(id); }

  int64_t slab_row(const Seq& s, size_t pos) const {
    return static_cast<int64_t>(s.frames[pos / page_size]) * static_cast<int64_t>(page_size) +
           static_cast<int64_t>(pos % page_size);
  }

  // Allocates frames for t more tokens (kv_pool.cpp:63-76) and uploads the
  // new page-table entries (the slab rows follow from the page table on the
  // device).
  void reserve(Seq& s, size_t t, cudaStream_t st) {
    const size_t frames_now = (s.len + page_size - 1) / page_size;
    const size_t frames_after = (s.len + t + page_size - 1) / page_size;
    const size_t need = frames_after - frames_now;
    if (need > free_list.size())
      fail(TS_CAPACITY, "append_kv: pool exhausted (need " + std::to_string(need) + " frames, " +
                            std::to_string(free_list.size()) + " free)");
    for (size_t i = 0; i < need; ++i) {
      s.frames.push_back(free_list.back());
      s.h_pt[frames_now + i] = static_cast<int32_t>(free_list.back());  // entries are written once per sequence
      free_list.pop_back();
    }
    if (need)
      ck(cudaMemcpyAsync(s.d_pt + frames_now, s.h_pt + frames_now, need * sizeof(int32_t), cudaMemcpyHostToDevice,
                         st),
         "page table upload");
  }

  // sync = false: the caller's later work on `st` is stream-ordered after
  // the append (the engine's prefill); the public pool API stays synchronous.
  // reserved: the caller ran reserve(t) already (the engine's prefill, so
  // that the append launch follows the attention directly: pdl, a
  // programmatic launch after it)
  void append(uint32_t id, const void* k, const void* v, size_t t, bool bf16, size_t* first,
              size_t* last, cudaStream_t st, bool sync = true, bool reserved = false, bool pdl = false) {
    Seq& s = state(id);
    const size_t f = s.len;
    if (first) *first = f;
    if (last) *last = f + t;
    if (t == 0) return;
    if (!reserved) reserve(s, t, st);  // rows come from the page table on the device (no host round trip)
    const size_t n = t * row;
    if (bf16) {
      const uint16_t* kd = dev_in(static_cast<const uint16_t*>(k), n, st_b, st);
      const uint16_t* vd = dev_in(static_cast<const uint16_t*>(v), n, st_c, st);
      ck(tsb::launch_kv_append(k_slab, v_slab, nullptr, nullptr, kd, vd, nullptr, static_cast<int>(t),
                               static_cast<int>(row), st, s.d_pt, static_cast<int64_t>(s.len),
                               static_cast<int>(page_size)),
         "kv_append");
    } else {
      const float* kd = dev_in(static_cast<const float*>(k), n, st_b, st);
      const float* vd = dev_in(static_cast<const float*>(v), n, st_c, st);
      ck(tsb::launch_kv_append(k_slab, v_slab, kd, vd, nullptr, nullptr, nullptr, static_cast<int>(t),
                               static_cast<int>(row), st, s.d_pt, static_cast<int64_t>(s.len),
                               static_cast<int>(page_size), pdl),
         "kv_append");
    }
    g_launches.fetch_add(1);
    if (sync) ck(cudaStreamSynchronize(st), "append sync");
    s.len += t;
  }
};

// ================================================================= engine
// One step of a KV-sequence-sharded decode (config 4), kept between the
// per-exchange launches of this shard.
struct ShardStep {
  const float *q = nullptr, *k = nullptr, *v = nullptr;
  size_t base = 0, n_global = 0, n_local_len = 0;
  int32_t cand_first = 0, T = 0, sel_on = 0;
};

struct ts_engine {
  ts_engine_config cfg{};
  int rank = 0, world = 1;  // sharded decode: this shard's rank among `world`
  ShardStep shard;
  DevBuf s_att, s_natt;     // sharded attend: attended local rows + count
  DevBuf s_blk, s_out;      // ts_shard_decode_step: exchanged blocks, staged output
  std::unique_ptr<ts_pool> pool;
  // multi-layer engine: n_layers x B sequences in one pool, each
  // (layer, sequence) with its own Selection Cache entry; the calls act on
  // the current layer (ts_engine_set_layer)
  std::vector<uint32_t> seq_ids;  // [L][B]
  size_t B = 1, L = 1, layer = 0;
  size_t li(size_t b) const { return layer * B + b; }
  uint32_t sid(size_t b) const { return seq_ids[li(b)]; }
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // per-sequence Selection Cache entries (device)
  DevBuf cached_q, sel, sel_crit, sel_rows;
  // step IO staging (device) + pinned host mirrors
  DevBuf d_q, d_k, d_v, d_out;
  float* h_q = nullptr;
  float* h_k = nullptr;
  float* h_v = nullptr;
  float* h_out = nullptr;
  CacheState* h_cache = nullptr;
  // h_out's device alias (mapped pinned memory): the synchronous host-buffer
  // decode writes its output and cache states there directly, no D2H copy
  // (nullptr: not mappable, or TS_NO_ZERO_COPY)
  char* h_out_dev = nullptr;
  // set for one engine_step: the launch mirrors the cache states into h_out_dev
  bool mirror_cache = false;
  bool mirror_done = false;  // the last engine_step's launches wrote the mirror
  uint32_t* h_sel = nullptr;
  Workspace ws;
  StepWorkspace sws;  // the single-sequence step kernel's
  // frames the last decode step appended, per sequence (-1: none); a step
  // the device rejected (zero query) is rolled back with them
  std::vector<int64_t> last_frames;
  bool last_unchecked = false;  // decode_async: the step's error flag is read at the next sync / stats
  // device phase trace (%globaltimer stamps of CTA 0), when enabled
  DevBuf trace;
  bool trace_on = false;
  // prefill scratch
  DevBuf p_qmean, p_sel, p_crit, p_selrows, p_state, p_att, p_natt, p_bad, p_q, p_k, p_v, p_out, p_split, p_trace;
  // host-buffer prefill: the chunk's K/V copies run on their own stream,
  // behind the query's, while the selection (which needs only the query) runs
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_q = nullptr, ev_kv = nullptr;

  ~ts_engine() {
    if (ev_q) cudaEventDestroy(ev_q);
    if (ev_kv) cudaEventDestroy(ev_kv);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (h_q) cudaFreeHost(h_q);
    if (h_k) cudaFreeHost(h_k);
    if (h_v) cudaFreeHost(h_v);
    if (h_out) cudaFreeHost(h_out);
    if (h_sel) cudaFreeHost(h_sel);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
  size_t W() const { return cfg.num_heads * cfg.head_dim; }
  size_t KW() const { return cfg.num_kv_heads * cfg.head_dim; }
  // [B x H*d output | L x B cache states], 256-B aligned split
  size_t out_bytes() const { return (B * W() * 4 + 255) / 256 * 256; }
  size_t out_block_bytes() const { return out_bytes() + L * B * sizeof(CacheState); }
  CacheState* cache(size_t b) const {
    return reinterpret_cast<CacheState*>(d_out.as<char>() + out_bytes()) + li(b);
  }
  CacheState* hcache(size_t b) const { return h_cache + li(b); }
  float* cq(size_t b) const { return cached_q.as<float>() + li(b) * W(); }
  uint32_t* sl(size_t b) const { return sel.as<uint32_t>() + li(b) * std::max<size_t>(cfg.k, 1); }
  float* sc(size_t b) const { return sel_crit.as<float>() + li(b) * std::max<size_t>(cfg.k, 1); }
  int32_t* sr(size_t b) const { return sel_rows.as<int32_t>() + li(b) * std::max<size_t>(cfg.k, 1); }
};

namespace {

void validate_cfg(const ts_engine_config& c) {
  if (c.num_heads == 0 || c.num_kv_heads == 0 || c.head_dim == 0)
    fail(TS_INVALID_ARGUMENT, "EngineConfig: head counts and head_dim must be >= 1");
  if (c.num_heads % c.num_kv_heads != 0)
    fail(TS_INVALID_ARGUMENT, "EngineConfig: num_heads must be a multiple of num_kv_heads");
  if (c.chunk_size == 0) fail(TS_INVALID_ARGUMENT, "EngineConfig: chunk_size must be >= 1");
  if (c.block_size == 0) fail(TS_INVALID_ARGUMENT, "EngineConfig: block_size must be >= 1");
  if (c.selection_method < 0 || c.selection_method > 2) fail(TS_INVALID_ARGUMENT, "select_with: bad method");
}

void check_method_supported(int m, bool sharded = false) {
  if (m == TS_HEAD_VOTE && sharded)
    fail(TS_INVALID_ARGUMENT, "head_vote selection is not supported by the sharded decode (per-head top-k across "
                              "shards); use head_soft_vote or topk");
}

DecodeParams base_params(const ts_pool* pool, int H, int H_kv, int d, int k, int method, int mode) {
  DecodeParams p{};
  p.k_slab = pool ? pool->k_slab : nullptr;
  p.k_tmap = pool ? pool->k_tmap : nullptr;
  p.v_slab = pool ? pool->v_slab : nullptr;
  p.k_slab_w = pool ? pool->k_slab : nullptr;
  p.v_slab_w = pool ? pool->v_slab : nullptr;
  p.page_size = pool ? static_cast<int>(pool->page_size) : 1;
  p.H = H;
  p.H_kv = H_kv;
  p.d = d;
  p.k = k;
  p.method = method;
  p.mode = mode;
  p.attn_scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  return p;
}

struct GlobalCtx {
  cudaStream_t stream = nullptr;
  Workspace ws;
  DevBuf a, b, c, d, e, f;
  GlobalCtx() { ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream"); }
};
GlobalCtx& gctx() {
  static GlobalCtx* g = new GlobalCtx();
  return *g;
}

// Standalone selection through the fused kernel (score and/or select modes).
// q: device [H*d] (score mode) ; s_in: device [H*T] (select-from-S mode).
size_t run_select(const ts_pool* pool, const ts_pool::Seq* seq, int H, int H_kv, int d,
                  const float* q, const float* s_in, const uint32_t* cand_dev, size_t T, size_t k,
                  int method, float* s_out_dev, uint32_t* sel_host, double* crit_host, Workspace& ws,
                  DevBuf& b_sel, DevBuf& b_crit, DevBuf& b_state, cudaStream_t st, bool do_select) {
  const int mode = (s_in ? tsb::kModeSIn : tsb::kModeScore) | (do_select ? tsb::kModeSelect : 0) |
                   (s_out_dev ? tsb::kModeSOut : 0);
  DecodeParams p = base_params(pool, H, H_kv, d, static_cast<int>(k), method, mode);
  p.n_seq = 1;
  SeqDesc& sd = p.seqs[0];
  sd.page_table = seq ? seq->d_pt : nullptr;
  sd.n_cached = seq ? static_cast<int32_t>(seq->len) : 0;
  sd.cand_begin = 0;
  sd.n_cand = static_cast<int32_t>(T);
  sd.cand = cand_dev;
  sd.select = 1;
  sd.q = q;
  sd.s_in = s_in;
  sd.s_out = s_out_dev;
  sd.append_frame = -1;
  sd.append_page = -1;
  const size_t kk = std::max<size_t>(std::min(k, T), 1);
  sd.sel = static_cast<uint32_t*>(b_sel.ensure(kk * 4));
  sd.sel_crit = static_cast<float*>(b_crit.ensure(kk * 4));
  sd.cache = static_cast<CacheState*>(b_state.ensure(sizeof(CacheState)));
  ck(cudaMemsetAsync(sd.cache, 0, sizeof(CacheState), st), "memset");
  const Plan pl = make_plan(H, H_kv, d, 1, static_cast<int>(T), 1, false);
  if (method == TS_HEAD_VOTE && do_select) {
    // select_head_vote (vote.cu) over S: given, or scored here into the workspace
    const float* S = s_in;
    if (!S) {
      float* so = s_out_dev ? s_out_dev : ws.vote_scores(1, H, static_cast<int>(T));
      p.mode = tsb::kModeScore | tsb::kModeSOut;
      sd.s_out = so;
      launch_decode(p, pl, ws, st);
      S = so;
    }
    ck(tsb::launch_head_vote(S, H, static_cast<int>(T), static_cast<int>(k), cand_dev, 0, nullptr, sd.sel,
                             sd.sel_crit, nullptr, &sd.cache->n_sel, ws.vote(H, static_cast<int>(T)), nullptr, st),
       "head vote");
    g_launches.fetch_add(3);
  } else {
    launch_decode(p, pl, ws, st);
  }
  if (!do_select) {
    ck(cudaStreamSynchronize(st), "sync");
    return 0;
  }
  CacheState cs{};
  ck(cudaMemcpyAsync(&cs, sd.cache, sizeof(CacheState), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  const size_t n = static_cast<size_t>(cs.n_sel);
  std::vector<float> crit(n);
  if (n) {
    ck(cudaMemcpyAsync(sel_host, sd.sel, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(crit.data(), sd.sel_crit, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  }
  for (size_t i = 0; i < n; ++i) crit_host[i] = static_cast<double>(crit[i]);
  return n;
}

// the tcgen05 prefill kernel applies (d = 128, G <= 8, not overridden)
bool prefill_uses_tc(int H, int H_kv, int d) {
  return d == 128 && H / H_kv <= 8 && !g_force_cuda_core_prefill && !g_prefill_mma_sync;
}

// C-row sparse attention: the tcgen05 kernel where it applies (d = 128,
// G <= 8), the CUDA-core kernel otherwise.
cudaError_t launch_prefill(tsb::PrefillAttendParams& pa, DevBuf& split_ws, cudaStream_t st) {
  if (pa.win_n_att && !prefill_uses_tc(pa.H, pa.H_kv, pa.d)) return cudaErrorInvalidValue;  // (implicit windows: tcgen05 only)
  if (pa.d == 128 && pa.H / pa.H_kv <= 8 && !g_force_cuda_core_prefill) {
    // bf16 parts of the chunk's K/V, owned by the caller's pool / engine (stream-ordered reuse)
    const size_t base = static_cast<size_t>(2) * (3 * pa.C + std::max(pa.n_att_max, 0)) * pa.H_kv * pa.d * 2;
    const size_t extra = prefill_uses_tc(pa.H, pa.H_kv, pa.d) ? tsb::prefill_tc_extra_ws_bytes(pa, st) + 256 : 0;
    pa.split_ws = static_cast<uint16_t*>(split_ws.ensure(base + extra));
    // tcgen05 (prefill_tc.cu); the mma.sync kernel (prefill.cu) on request (TS_PREFILL_MMA_SYNC=1)
    if (!g_prefill_mma_sync) return tsb::launch_prefill_tc(pa, st);
    return tsb::launch_prefill_flash(pa, st);
  }
  return tsb::launch_prefill_attend(pa, st);
}

// Copy a (host or device) index list to host.
std::vector<uint32_t> host_copy_u32(const uint32_t* p, size_t n) {
  std::vector<uint32_t> v(n);
  if (n == 0) return v;
  if (is_device_ptr(p)) ck(cudaMemcpy(v.data(), p, n * 4, cudaMemcpyDeviceToHost), "D2H");
  else std::memcpy(v.data(), p, n * 4);
  return v;
}

void copy_out(void* dst, const void* src_dev, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  ck(cudaMemcpyAsync(dst, src_dev, bytes, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
     "copy out");
}

}  // namespace

extern "C" {

const char* ts_last_error(void) { return g_err.c_str(); }
const char* ts_version(void) { return "tokenselect-b200 0.1.0 (sm_100a)"; }
uint64_t ts_launch_count(void) { return g_launches.load(); }

void ts_engine_config_default(ts_engine_config* c) {
  c->k = 2048;
  c->n_local = 512;
  c->n_init = 128;
  c->chunk_size = 512;
  c->theta = 0.9;
  c->num_heads = 8;
  c->num_kv_heads = 8;
  c->head_dim = 64;
  c->block_size = 64;
  c->selection_method = TS_HEAD_SOFT_VOTE;
}

ts_status ts_engine_config_validate(const ts_engine_config* cfg) {
  return guarded([&] { validate_cfg(*cfg); });
}

// ------------------------------------------------------------------- pool
ts_status ts_pool_create(size_t capacity_tokens, size_t page_size, size_t num_kv_heads,
                         size_t head_dim, ts_pool** out) {
  return guarded([&] {
    *out = nullptr;
    if (page_size == 0) fail(TS_INVALID_ARGUMENT, "PagedKvPool: page_size must be >= 1");
    if (num_kv_heads * head_dim == 0) fail(TS_INVALID_ARGUMENT, "PagedKvPool: zero row width");
    device_info();
    auto p = std::make_unique<ts_pool>();
    p->page_size = page_size;
    p->H_kv = num_kv_heads;
    p->d = head_dim;
    p->row = num_kv_heads * head_dim;
    p->total_frames = (capacity_tokens + page_size - 1) / page_size;
    const size_t elems = std::max<size_t>(p->total_frames * page_size * p->row, 8);
    ck(cudaMalloc(&p->k_slab, elems * 2), "cudaMalloc K slab");
    ck(cudaMalloc(&p->v_slab, elems * 2), "cudaMalloc V slab");
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "stream");
    ck(cudaMemsetAsync(p->k_slab, 0, elems * 2, p->stream), "memset");
    ck(cudaMemsetAsync(p->v_slab, 0, elems * 2, p->stream), "memset");
    p->k_tmap = encode_k_tmap(p->k_slab, p->total_frames * page_size, p->row * 2, p->stream);
    p->free_list.resize(p->total_frames);
    // highest frame handed out first (kv_pool.cpp:24-27)
    for (size_t i = 0; i < p->total_frames; ++i) p->free_list[i] = static_cast<uint32_t>(i);
    ck(cudaStreamSynchronize(p->stream), "sync");
    *out = p.release();
  });
}

void ts_pool_destroy(ts_pool* pool) { delete pool; }

ts_status ts_pool_create_sequence(ts_pool* pool, uint32_t* seq_id) {
  return guarded([&] {
    ts_pool::Seq s;
    ck(cudaMalloc(&s.d_pt, std::max<size_t>(pool->total_frames, 1) * sizeof(int32_t)), "cudaMalloc page table");
    ck(cudaMallocHost(&s.h_pt, std::max<size_t>(pool->total_frames, 1) * sizeof(int32_t)), "cudaMallocHost page table");
    const uint32_t id = pool->next_id++;
    pool->seqs.emplace(id, std::move(s));
    *seq_id = id;
  });
}

ts_status ts_pool_append_kv(ts_pool* pool, uint32_t seq, const float* k, const float* v, size_t t,
                            size_t* first, size_t* last) {
  return guarded([&] { pool->append(seq, k, v, t, false, first, last, pool->stream); });
}

ts_status ts_pool_append_kv_bf16(ts_pool* pool, uint32_t seq, const uint16_t* k, const uint16_t* v,
                                 size_t t, size_t* first, size_t* last) {
  return guarded([&] { pool->append(seq, k, v, t, true, first, last, pool->stream); });
}

ts_status ts_pool_gather(const ts_pool* cpool, uint32_t seq, const uint32_t* idx, size_t n,
                         float* k_out, float* v_out) {
  return guarded([&] {
    ts_pool* pool = const_cast<ts_pool*>(cpool);
    const ts_pool::Seq& s = pool->state(seq);
    std::vector<uint32_t> ih = host_copy_u32(idx, n);
    std::vector<int64_t> rows(n);
    for (size_t j = 0; j < n; ++j) {
      if (ih[j] >= s.len)
        fail(TS_OUT_OF_RANGE, "gather: index " + std::to_string(ih[j]) + " out of range (logical_len " +
                                  std::to_string(s.len) + ")");
      rows[j] = pool->slab_row(s, ih[j]);
    }
    if (n == 0) return;
    cudaStream_t st = pool->stream;
    int64_t* d_rows = static_cast<int64_t*>(pool->st_a.ensure(n * 8));
    ck(cudaMemcpyAsync(d_rows, rows.data(), n * 8, cudaMemcpyHostToDevice, st), "H2D");
    const size_t bytes = n * pool->row * 4;
    float* kd = k_out ? (is_device_ptr(k_out) ? k_out : static_cast<float*>(pool->st_b.ensure(bytes))) : nullptr;
    float* vd = v_out ? (is_device_ptr(v_out) ? v_out : static_cast<float*>(pool->st_c.ensure(bytes))) : nullptr;
    ck(tsb::launch_kv_gather(pool->k_slab, pool->v_slab, d_rows, static_cast<int>(n), static_cast<int>(pool->row), kd, vd, st),
       "gather");
    g_launches.fetch_add(1);
    if (k_out && kd != k_out) copy_out(k_out, kd, bytes, st);
    if (v_out && vd != v_out) copy_out(v_out, vd, bytes, st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

ts_status ts_pool_release(ts_pool* pool, uint32_t seq) {
  return guarded([&] {
    auto it = pool->seqs.find(seq);
    if (it == pool->seqs.end())
      fail(TS_INVALID_ARGUMENT, "release: unknown or already released sequence " + std::to_string(seq));
    for (uint32_t f : it->second.frames) pool->free_list.push_back(f);
    if (it->second.d_pt) cudaFree(it->second.d_pt);
    if (it->second.h_pt) cudaFreeHost(it->second.h_pt);
    pool->seqs.erase(it);
  });
}

ts_status ts_pool_logical_len(const ts_pool* pool, uint32_t seq, size_t* len) {
  return guarded([&] { *len = pool->state(seq).len; });
}

ts_status ts_pool_shuffle_free_frames(ts_pool* pool, uint64_t seed) {
  return guarded([&] {
    RefRng rng(seed);
    for (size_t i = pool->free_list.size(); i > 1; --i) std::swap(pool->free_list[i - 1], pool->free_list[rng.index(i)]);
  });
}

ts_status ts_pool_page_table_json(const ts_pool* pool, uint32_t seq, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    const ts_pool::Seq& s = pool->state(seq);
    std::string j = "{\"frames\":[";
    for (size_t i = 0; i < s.frames.size(); ++i) {
      if (i) j += ",";
      j += std::to_string(s.frames[i]);
    }
    j += "],\"logical_len\":" + std::to_string(s.len) + ",\"seq_id\":" + std::to_string(seq) + "}";
    if (needed) *needed = j.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, j.size());
      std::memcpy(buf, j.data(), n);
      buf[n] = 0;
    }
  });
}

size_t ts_pool_total_frames(const ts_pool* p) { return p->total_frames; }
size_t ts_pool_free_frames(const ts_pool* p) { return p->free_list.size(); }
size_t ts_pool_page_size(const ts_pool* p) { return p->page_size; }
size_t ts_pool_num_kv_heads(const ts_pool* p) { return p->H_kv; }
size_t ts_pool_head_dim(const ts_pool* p) { return p->d; }

ts_status ts_pool_device_views(const ts_pool* pool, uint32_t seq, const void** k_slab, const void** v_slab,
                               const int32_t** page_table) {
  return guarded([&] {
    const ts_pool::Seq& s = pool->state(seq);
    if (k_slab) *k_slab = pool->k_slab;
    if (v_slab) *v_slab = pool->v_slab;
    if (page_table) *page_table = s.d_pt;
  });
}

// ----------------------------------------------------------------- select
ts_status ts_score_paged(const ts_pool* cpool, uint32_t seq, const float* q, size_t num_heads, size_t head_dim,
                         const uint32_t* candidates, size_t T, size_t block_size, float* s_out) {
  return guarded([&] {
    ts_pool* pool = const_cast<ts_pool*>(cpool);
    if (head_dim != pool->d)
      fail(TS_INVALID_ARGUMENT, "score_paged: query head_dim " + std::to_string(head_dim) +
                                    " does not match pool head_dim " + std::to_string(pool->d));
    if (num_heads == 0 || num_heads % pool->H_kv != 0)
      fail(TS_INVALID_ARGUMENT, "score_paged: H must be a positive multiple of H_kv");
    if (block_size == 0) fail(TS_INVALID_ARGUMENT, "score_paged: block_size must be >= 1");
    const ts_pool::Seq& s = pool->state(seq);
    std::vector<uint32_t> ch = host_copy_u32(candidates, T);
    for (size_t j = 0; j < T; ++j)
      if (ch[j] >= s.len)
        fail(TS_OUT_OF_RANGE, "key_row: index " + std::to_string(ch[j]) + " out of range (logical_len " +
                                  std::to_string(s.len) + ")");
    if (T == 0) return;
    cudaStream_t st = pool->stream;
    const float* qd = dev_in(q, num_heads * head_dim, pool->st_a, st);
    const uint32_t* cd = dev_in(candidates, T, pool->st_b, st);
    const size_t bytes = num_heads * T * 4;
    float* sd = is_device_ptr(s_out) ? s_out : static_cast<float*>(pool->st_c.ensure(bytes));
    DevBuf b1, b2, b3;
    run_select(pool, &s, static_cast<int>(num_heads), static_cast<int>(pool->H_kv), static_cast<int>(head_dim), qd,
               nullptr, cd, T, 0, TS_HEAD_SOFT_VOTE, sd, nullptr, nullptr, pool->ws, b1, b2, b3, st, false);
    if (sd != s_out) {
      copy_out(s_out, sd, bytes, st);
      ck(cudaStreamSynchronize(st), "sync");
    }
  });
}

ts_status ts_select(const float* per_head, size_t num_heads, size_t T, const uint32_t* candidate_idx, size_t k,
                    int method, uint32_t* sel_out, double* crit_out, size_t* n_out) {
  return guarded([&] {
    *n_out = 0;
    if (method < 0 || method > 2) fail(TS_INVALID_ARGUMENT, "select_with: bad method");
    if (T == 0) return;  // pick(): empty criticality -> empty result
    if (k == 0) fail(TS_INVALID_ARGUMENT, "topk_indices: k must be >= 1");
    check_method_supported(method);
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const float* sd = dev_in(per_head, num_heads * T, g.a, st);
    const uint32_t* cd = candidate_idx ? dev_in(candidate_idx, T, g.b, st) : nullptr;
    *n_out = run_select(nullptr, nullptr, static_cast<int>(num_heads), 1, 1, nullptr, sd, cd, T, k, method, nullptr,
                        sel_out, crit_out, g.ws, g.c, g.d, g.e, st, true);
  });
}

ts_status ts_select_for_chunk(const ts_pool* cpool, uint32_t seq, const float* q_chunk, size_t c, size_t width,
                              const uint32_t* candidates, size_t T, size_t k, int method, size_t block_size,
                              uint32_t* sel_out, double* crit_out, size_t* n_out) {
  return guarded([&] {
    *n_out = 0;
    ts_pool* pool = const_cast<ts_pool*>(cpool);
    if (width == 0 || width % pool->d != 0) fail(TS_INVALID_ARGUMENT, "select_for_chunk: chunk width must be H * d_h");
    if (c == 0) fail(TS_INVALID_ARGUMENT, "chunk_mean: empty chunk");
    const size_t H = width / pool->d;
    if (H % pool->H_kv != 0) fail(TS_INVALID_ARGUMENT, "score_paged: H must be a positive multiple of H_kv");
    if (block_size == 0) fail(TS_INVALID_ARGUMENT, "score_paged: block_size must be >= 1");
    if (method < 0 || method > 2) fail(TS_INVALID_ARGUMENT, "select_with: bad method");
    const ts_pool::Seq& s = pool->state(seq);
    std::vector<uint32_t> ch = host_copy_u32(candidates, T);
    for (size_t j = 0; j < T; ++j)
      if (ch[j] >= s.len)
        fail(TS_OUT_OF_RANGE, "key_row: index " + std::to_string(ch[j]) + " out of range (logical_len " +
                                  std::to_string(s.len) + ")");
    if (T == 0) return;
    if (k == 0) fail(TS_INVALID_ARGUMENT, "topk_indices: k must be >= 1");
    check_method_supported(method);
    cudaStream_t st = pool->stream;
    const float* qd = dev_in(q_chunk, c * width, pool->st_a, st);
    float* qm = static_cast<float*>(pool->st_d.ensure(width * 4));
    ck(tsb::launch_chunk_mean(qd, static_cast<int>(c), static_cast<int>(width), qm, st), "chunk_mean");
    g_launches.fetch_add(1);
    const uint32_t* cd = dev_in(candidates, T, pool->st_b, st);
    DevBuf b1, b2, b3;
    *n_out = run_select(pool, &s, static_cast<int>(H), static_cast<int>(pool->H_kv), static_cast<int>(pool->d), qm,
                        nullptr, cd, T, k, method, nullptr, sel_out, crit_out, pool->ws, b1, b2, b3, st, true);
  });
}

// -------------------------------------------------------------- attention
ts_status ts_sparse_attend(const ts_pool* cpool, uint32_t seq, const float* q, const float* k_cur,
                           const float* v_cur, size_t C, size_t num_heads, const uint32_t* forced_init,
                           size_t n_init, const uint32_t* selected, size_t n_sel, const uint32_t* forced_local,
                           size_t n_local, float* out) {
  return guarded([&] {
    ts_pool* pool = const_cast<ts_pool*>(cpool);
    const ts_pool::Seq& s = pool->state(seq);
    // merged() = merge_dedup (tensor.cpp:159-168)
    std::vector<uint32_t> merged;
    for (auto [p, n] : {std::pair{forced_init, n_init}, std::pair{selected, n_sel}, std::pair{forced_local, n_local}}) {
      std::vector<uint32_t> h = host_copy_u32(p, n);
      merged.insert(merged.end(), h.begin(), h.end());
    }
    std::sort(merged.begin(), merged.end());
    merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
    for (uint32_t t : merged)
      if (t >= s.len)
        fail(TS_OUT_OF_RANGE, "gather: index " + std::to_string(t) + " out of range (logical_len " +
                                  std::to_string(s.len) + ")");
    // sdpa_full shape contract (attention.cpp:56-69) with head_dim = q width / H
    if (num_heads == 0) fail(TS_INVALID_ARGUMENT, "sdpa_full: q must be [C x (H * d_h)]");
    const size_t width = num_heads * pool->d;  // callers pass q as [C x H*d_pool]
    const size_t d = pool->d;
    const size_t H_kv = pool->H_kv;
    if (num_heads % H_kv != 0) fail(TS_INVALID_ARGUMENT, "sdpa_full: H must be a multiple of H_kv");
    if (C == 0) return;
    cudaStream_t st = pool->stream;
    const float* qd = dev_in(q, C * width, pool->st_a, st);
    const float* kd = dev_in(k_cur, C * pool->row, pool->st_b, st);
    const float* vd = dev_in(v_cur, C * pool->row, pool->st_c, st);
    const uint32_t* ad = merged.empty() ? nullptr : dev_in(merged.data(), merged.size(), pool->st_e, st);
    const size_t obytes = C * width * 4;
    float* od = is_device_ptr(out) ? out : static_cast<float*>(pool->st_f.ensure(obytes));
    if (C == 1) {
      DecodeParams p = base_params(pool, static_cast<int>(num_heads), static_cast<int>(H_kv), static_cast<int>(d), 0,
                                   TS_HEAD_SOFT_VOTE, tsb::kModeAttend);
      p.n_seq = 1;
      SeqDesc& sdsc = p.seqs[0];
      sdsc.page_table = s.d_pt;
      sdsc.n_cached = static_cast<int32_t>(s.len);
      sdsc.select = 0;
      sdsc.q = qd;
      sdsc.k_new = kd;
      sdsc.v_new = vd;
      sdsc.out = od;
      sdsc.append_frame = -1;
      sdsc.append_page = -1;
      sdsc.att_list = ad ? ad : reinterpret_cast<const uint32_t*>(qd);  // non-null => explicit list
      sdsc.n_att = static_cast<int32_t>(merged.size());
      const Plan pl = make_plan(static_cast<int>(num_heads), static_cast<int>(H_kv), static_cast<int>(d), 1, 0,
                                static_cast<int>(merged.size() + 1));
      launch_decode(p, pl, pool->ws, st);
    } else {
      tsb::PrefillAttendParams pa{};
      pa.q = qd;
      pa.k_cur = kd;
      pa.v_cur = vd;
      pa.k_slab = pool->k_slab;
      pa.v_slab = pool->v_slab;
      pa.page_table = s.d_pt;
      pa.page_size = static_cast<int>(pool->page_size);
      pa.att = ad;
      pa.n_att = static_cast<int>(merged.size());
      pa.n_att_ptr = nullptr;
      pa.n_att_max = pa.n_att;
      pa.C = static_cast<int>(C);
      pa.H = static_cast<int>(num_heads);
      pa.H_kv = static_cast<int>(H_kv);
      pa.d = static_cast<int>(d);
      pa.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
      pa.out = od;
      ck(launch_prefill(pa, pool->st_split, st), "prefill_attend");
      g_launches.fetch_add(1);
    }
    if (od != out) copy_out(out, od, obytes, st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// ------------------------------------------------------------------ engine
namespace {
void check_async_errors(ts_engine* e);  // (defined with the decode path below)
}  // namespace

ts_status ts_engine_create_layers(const ts_engine_config* cfg, size_t capacity_tokens, size_t n_seqs, size_t n_layers,
                                 ts_engine** out) {
  return guarded([&] {
    *out = nullptr;
    validate_cfg(*cfg);
    check_method_supported(cfg->selection_method);
    if (n_seqs == 0) fail(TS_INVALID_ARGUMENT, "AttentionEngine: n_seqs must be >= 1");
    if (n_layers == 0) fail(TS_INVALID_ARGUMENT, "AttentionEngine: n_layers must be >= 1");
    device_info();
    auto e = std::make_unique<ts_engine>();
    e->cfg = *cfg;
    e->B = n_seqs;
    e->L = n_layers;
    const size_t NS = n_seqs * n_layers;  // (layer, sequence) pairs
    ts_pool* p = nullptr;
    // one shared pool, page_size 1 (attention.cpp:219), capacity per sequence
    ts_status rc = ts_pool_create(capacity_tokens * NS, 1, cfg->num_kv_heads, cfg->head_dim, &p);
    if (rc != TS_OK) fail(rc, g_err);
    e->pool.reset(p);
    for (size_t b = 0; b < NS; ++b) {
      uint32_t id;
      rc = ts_pool_create_sequence(p, &id);
      if (rc != TS_OK) fail(rc, g_err);
      e->seq_ids.push_back(id);
    }
    ck(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking), "stream");
    e->stream = e->own_stream;
    const size_t W = e->W(), KW = e->KW(), kk = std::max<size_t>(cfg->k, 1);
    e->cached_q.ensure(NS * W * 4);
    e->sel.ensure(NS * kk * 4);
    e->sel_crit.ensure(NS * kk * 4);
    e->sel_rows.ensure(NS * kk * 4);
    e->d_q.ensure(n_seqs * (W + 2 * KW) * 4);  // q | k | v staging block
    e->d_k.ensure(n_seqs * KW * 4);
    e->d_v.ensure(n_seqs * KW * 4);
    e->d_out.ensure(e->out_block_bytes());  // output | cache states
    ck(cudaMallocHost(&e->h_q, n_seqs * (W + 2 * KW) * 4), "pinned");
    ck(cudaMallocHost(&e->h_k, n_seqs * KW * 4), "pinned");
    ck(cudaMallocHost(&e->h_v, n_seqs * KW * 4), "pinned");
    ck(cudaMallocHost(&e->h_out, e->out_block_bytes()), "pinned");
    e->h_cache = reinterpret_cast<CacheState*>(reinterpret_cast<char*>(e->h_out) + e->out_bytes());
    if (!std::getenv("TS_NO_ZERO_COPY")) {
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, e->h_out, 0) == cudaSuccess) e->h_out_dev = static_cast<char*>(dp);
      else cudaGetLastError();
    }
    std::vector<CacheState> init(NS);
    for (auto& c : init) {
      c = CacheState{};
      c.theta = cfg->theta;  // attention.cpp:222
      c.last_cos = NAN;
      c.first_flag = 1;
      c.last_hit = -1;
    }
    ck(cudaMemcpy(e->cache(0), init.data(), NS * sizeof(CacheState), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemset(e->cached_q.p, 0, NS * W * 4), "memset");
    // the decode workspace at the capacity's candidate count: the per-step
    // plan tracks the growing context, and a reallocation mid-stream would
    // synchronise the device (the GPU idles while the host frees and mallocs)
    if (cfg->k > 0 && capacity_tokens > cfg->n_init + cfg->n_local && !std::getenv("TS_NO_RESERVE")) {
      const int gn = static_cast<int>(std::min<size_t>(tsb::kMaxSeqPerLaunch, n_seqs));
      const int max_T = static_cast<int>(capacity_tokens - cfg->n_init - cfg->n_local);
      const int max_rows = static_cast<int>(cfg->n_init + std::min(cfg->k, capacity_tokens) + cfg->n_local + 1);
      try {
        const Plan pl = make_plan(static_cast<int>(cfg->num_heads), static_cast<int>(cfg->num_kv_heads),
                                  static_cast<int>(cfg->head_dim), gn, max_T, max_rows);
        e->ws.prepare(gn * pl.ctas_per_seq, static_cast<int>(cfg->num_heads), static_cast<int>(cfg->num_kv_heads),
                      static_cast<int>(cfg->head_dim), pl.tpc, pl.s_in_smem, gn, e->stream);
      } catch (const std::exception&) {
        cudaGetLastError();  // (a shape the decode kernel rejects fails at its first step, as before)
      }
    }
    *out = e.release();
  });
}

ts_status ts_engine_create(const ts_engine_config* cfg, size_t capacity_tokens, size_t n_seqs, ts_engine** out) {
  return ts_engine_create_layers(cfg, capacity_tokens, n_seqs, 1, out);
}

ts_status ts_engine_set_layer(ts_engine* eng, size_t layer) {
  return guarded([&] {
    if (layer >= eng->L) fail(TS_INVALID_ARGUMENT, "engine: layer index out of range");
    if (eng->last_unchecked) {  // a pending decode_async step belongs to the current layer
      ck(cudaStreamSynchronize(eng->stream), "sync");
      check_async_errors(eng);
    }
    eng->layer = layer;
  });
}

size_t ts_engine_num_layers(const ts_engine* eng) { return eng->L; }

void ts_engine_destroy(ts_engine* eng) {
  if (g_host_prof && g_prof_n)
    std::fprintf(stderr, "[tokenselect host prof] per step: params %.0f ns, plan %.0f ns, launch_decode %.0f ns (launch api %.0f ns) (%llu steps)\n",
                 g_prof[0] / g_prof_n, g_prof[1] / g_prof_n, g_prof[2] / g_prof_n, g_prof[3] / g_prof_n,
                 static_cast<unsigned long long>(g_prof_n));
  if (g_host_prof && g_prof_n)
    std::fprintf(stderr, "[tokenselect host prof] launch_decode: prepare+fill %.0f ns, before launch api %.0f ns\n",
                 g_prof_ld[0] / g_prof_n, g_prof_ld[1] / g_prof_n);
  if (g_host_prof && g_e2e_n)
    std::fprintf(stderr, "[tokenselect host prof] decode(host bufs): ptr queries %.0f ns, stage+h2d %.0f ns, step %.0f ns, "
                 "d2h issue %.0f ns, sync wait %.0f ns, unpack %.0f ns (%llu calls; packing %.0f ns, h2d api %.0f ns)\n", g_e2e_prof[0] / g_e2e_n,
                 g_e2e_prof[1] / g_e2e_n, g_e2e_prof[2] / g_e2e_n, g_e2e_prof[3] / g_e2e_n, g_e2e_prof[4] / g_e2e_n,
                 g_e2e_prof[5] / g_e2e_n,
                 static_cast<unsigned long long>(g_e2e_n), g_e2e_memcpy / g_e2e_n, g_e2e_h2dapi / g_e2e_n);
  if (g_host_prof) {  // per-engine figures
    std::fill(std::begin(g_prof), std::end(g_prof), 0.0);
    std::fill(std::begin(g_e2e_prof), std::end(g_e2e_prof), 0.0);
    g_prof_n = g_e2e_n = 0;
    g_prof_ld[0] = g_prof_ld[1] = 0;
    g_e2e_memcpy = g_e2e_h2dapi = 0;
  }
  delete eng;
}

ts_status ts_engine_set_stream(ts_engine* eng, void* stream) {
  return guarded([&] { eng->stream = stream ? static_cast<cudaStream_t>(stream) : eng->own_stream; });
}

ts_pool* ts_engine_pool(ts_engine* eng) { return eng->pool.get(); }
uint32_t ts_engine_sequence(const ts_engine* eng, size_t seq) { return eng->sid(seq); }

ts_status ts_engine_append(ts_engine* eng, size_t seq, const float* k, const float* v, size_t t) {
  return guarded([&] {
    if (seq >= eng->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    eng->pool->append(eng->sid(seq), k, v, t, false, nullptr, nullptr, eng->stream);
  });
}

ts_status ts_engine_append_bf16(ts_engine* eng, size_t seq, const uint16_t* k, const uint16_t* v, size_t t) {
  return guarded([&] {
    if (seq >= eng->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    eng->pool->append(eng->sid(seq), k, v, t, true, nullptr, nullptr, eng->stream);
  });
}

namespace {

// One decode step for all sequences (decode_step, attention.cpp:172-200).
// Inputs are device pointers (already staged). Returns per-sequence append
// failure flags (capacity), applied after the step as the reference does.
std::vector<int> engine_step(ts_engine* e, const float* q, const float* k, const float* v, float* out) {
  ts_pool& pool = *e->pool;
  const ts_engine_config& c = e->cfg;
  const size_t W = e->W(), KW = e->KW();
  std::vector<int> cap_fail(e->B, 0);
  e->last_frames.assign(e->B, -1);
  e->mirror_done = false;
  cudaStream_t st = e->stream;
  if (e->B == 1 && e->rank == 0 && e->world == 1) {
    ts_pool::Seq& s = pool.state(e->sid(0));
    const size_t N = s.len;
    const bool sel_on = c.k > 0 && N > c.n_init + c.n_local;
    const int T = sel_on ? static_cast<int>(N - c.n_init - c.n_local) : 0;
    const StepPlan sp = step_plan(c, T, static_cast<int>(c.n_init + c.n_local + 1));
    if (sp.ok) {
      tsb::StepParams p{};
      p.k_slab = pool.k_slab;
      p.v_slab = pool.v_slab;
      p.k_slab_w = pool.k_slab;
      p.v_slab_w = pool.v_slab;
      p.page_table = s.d_pt;
      p.H = static_cast<int>(c.num_heads);
      p.H_kv = static_cast<int>(c.num_kv_heads);
      p.k = static_cast<int>(c.k);
      p.N = static_cast<int>(N);
      p.select = sel_on ? 1 : 0;
      p.cand_begin = static_cast<int>(c.n_init);
      p.T = T;
      p.init_end = static_cast<int>(std::min(c.n_init, N));
      p.lb = static_cast<int>(std::max(N - std::min(c.n_local, N), std::min(c.n_init, N)));
      p.attn_scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c.head_dim)));
      p.q = q;
      p.k_new = k;
      p.v_new = v;
      p.out = out;
      p.cache = e->cache(0);
      p.cached_q = e->cq(0);
      p.sel = e->sl(0);
      p.sel_crit = e->sc(0);
      p.sel_rows = e->sr(0);
      p.append_frame = -1;
      if (pool.free_list.empty()) {
        cap_fail[0] = 1;
      } else {
        const uint32_t f = pool.free_list.back();
        pool.free_list.pop_back();
        s.frames.push_back(f);
        e->last_frames[0] = f;
        p.append_frame = static_cast<int32_t>(f);
      }
      p.trace = e->trace_on ? e->trace.as<unsigned long long>() : nullptr;
      if (p.trace) ck(cudaMemsetAsync(p.trace, 0, kTraceSlots * 8, st), "memset trace");
      launch_step(p, sp, e->sws, st);
      if (!cap_fail[0]) s.len += 1;
      return cap_fail;
    }
  }
  e->mirror_done = e->mirror_cache;
  for (size_t g0 = 0; g0 < e->B; g0 += tsb::kMaxSeqPerLaunch) {
    const double t0 = g_host_prof ? now_ns() : 0.0;
    const size_t gn = std::min<size_t>(tsb::kMaxSeqPerLaunch, e->B - g0);
    DecodeParams p = base_params(&pool, static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                                 static_cast<int>(c.head_dim), static_cast<int>(c.k), c.selection_method,
                                 tsb::kModeCache | tsb::kModeScore | tsb::kModeSelect | tsb::kModeAttend |
                                     tsb::kModeAppend);
    p.n_seq = static_cast<int>(gn);
    int max_T = 0, max_rows = 0;
    for (size_t i = 0; i < gn; ++i) {
      const size_t b = g0 + i;
      ts_pool::Seq& s = pool.state(e->sid(b));
      const size_t N = s.len;
      SeqDesc& sd = p.seqs[i];
      sd.page_table = s.d_pt;
      sd.n_cached = static_cast<int32_t>(N);
      const bool sel_on = c.k > 0 && N > c.n_init + c.n_local;
      sd.select = sel_on ? 1 : 0;
      sd.cand_begin = static_cast<int32_t>(c.n_init);
      sd.n_cand = sel_on ? static_cast<int32_t>(N - c.n_init - c.n_local) : 0;
      sd.cand = nullptr;
      sd.q = q + b * W;
      sd.k_new = k + b * KW;
      sd.v_new = v + b * KW;
      sd.out = out + b * W;
      sd.init_end = static_cast<int32_t>(std::min(c.n_init, N));
      sd.local_begin = static_cast<int32_t>(N - std::min(c.n_local, N));
      sd.att_list = nullptr;
      sd.cache = e->cache(b);
      sd.cached_q = e->cq(b);
      sd.sel = e->sl(b);
      sd.sel_crit = e->sc(b);
      sd.sel_rows = e->sr(b);
      sd.cache_mirror = e->mirror_cache
                            ? reinterpret_cast<CacheState*>(e->h_out_dev + e->out_bytes()) + e->li(b) : nullptr;
      // frame for logical position N (page_size 1): LIFO pop, after-the-step failure
      if (pool.free_list.empty()) {
        cap_fail[b] = 1;
        sd.append_frame = -1;
        sd.append_page = -1;
      } else {
        const uint32_t f = pool.free_list.back();
        pool.free_list.pop_back();
        s.frames.push_back(f);
        e->last_frames[b] = f;
        sd.append_frame = static_cast<int32_t>(f);
        sd.append_slot = 0;
        sd.append_page = static_cast<int32_t>(N);
      }
      max_T = std::max(max_T, sd.n_cand);
      max_rows = std::max(max_rows, static_cast<int>(std::min(c.n_init, N) + std::min(c.k, N) + c.n_local + 1));
    }
    const double t1 = g_host_prof ? now_ns() : 0.0;
    const Plan pl = make_plan(static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                              static_cast<int>(c.head_dim), static_cast<int>(gn), max_T, max_rows);
    const double t2 = g_host_prof ? now_ns() : 0.0;
    if (g_host_prof) {
      g_prof[0] += t1 - t0;
      g_prof[1] += t2 - t1;
      g_prof_n += 1;
    }
    p.trace = e->trace_on ? e->trace.as<unsigned long long>() : nullptr;
    if (p.trace) ck(cudaMemsetAsync(p.trace, 0, kTraceSlots * 8, st), "memset trace");
    const double t3 = g_host_prof ? now_ns() : 0.0;
    if (c.selection_method == TS_HEAD_VOTE) {
      // select_head_vote (selector.cpp:101-111) needs every head's own top-k:
      // (1) Selection Cache decision + S of the missing sequences into the
      // workspace, (2) per sequence the vote kernels (no-ops on a hit),
      // (3) attention over the cache entry's selection + the append
      const int maxT = std::max(1, max_T);
      float* S = e->ws.vote_scores(static_cast<int>(gn), static_cast<int>(c.num_heads), maxT);
      DecodeParams p1 = p;
      p1.mode = tsb::kModeCache | tsb::kModeScore | tsb::kModeSOut;
      for (size_t i = 0; i < gn; ++i) {
        p1.seqs[i].s_out = S + i * c.num_heads * maxT;
        p1.seqs[i].append_frame = -1;
        p1.seqs[i].append_page = -1;
      }
      launch_decode(p1, pl, e->ws, st);
      for (size_t i = 0; i < gn; ++i) {
        const SeqDesc& sd = p.seqs[i];
        if (!sd.select) continue;
        ck(tsb::launch_head_vote(S + i * c.num_heads * maxT, static_cast<int>(c.num_heads), sd.n_cand,
                                 static_cast<int>(c.k), nullptr, sd.cand_begin, sd.page_table, sd.sel, sd.sel_crit,
                                 sd.sel_rows, &sd.cache->n_sel, e->ws.vote(static_cast<int>(c.num_heads), sd.n_cand),
                                 sd.cache, st),
           "head vote");
        g_launches.fetch_add(3);
      }
      p.mode = tsb::kModeAttend | tsb::kModeAppend | tsb::kModeUseCached;
    }
    launch_decode(p, pl, e->ws, st);
    if (g_host_prof) g_prof[2] += now_ns() - t3;
    for (size_t i = 0; i < gn; ++i)
      if (!cap_fail[g0 + i]) pool.state(e->sid(g0 + i)).len += 1;
  }
  return cap_fail;
}

// Undoes the host side of the last step for sequence b (the device skipped
// its append: zero query, reported through CacheState::error).
void rollback_step(ts_engine* e, size_t b) {
  if (b >= e->last_frames.size() || e->last_frames[b] < 0) return;
  ts_pool& pool = *e->pool;
  ts_pool::Seq& s = pool.state(e->sid(b));
  s.frames.pop_back();
  s.len -= 1;
  pool.free_list.push_back(static_cast<uint32_t>(e->last_frames[b]));
  e->last_frames[b] = -1;
}

// decode_async: reads the last step's per-sequence error flags (the stream is
// synchronised by the caller), rolls back the rejected sequences and throws.
void check_async_errors(ts_engine* e) {
  if (!e->last_unchecked) return;
  e->last_unchecked = false;
  std::vector<CacheState> cs(e->B);
  ck(cudaMemcpy(cs.data(), e->cache(0), e->B * sizeof(CacheState), cudaMemcpyDeviceToHost), "D2H");
  bool bad = false;
  for (size_t b = 0; b < e->B; ++b)
    if (cs[b].error) {
      rollback_step(e, b);
      bad = true;
    }
  if (bad) fail(TS_INVALID_ARGUMENT, "lookup_or_select: zero query vector");
}

}  // namespace

ts_status ts_engine_decode(ts_engine* e, const float* q, const float* k, const float* v, float* out, int* cache_hit,
                           uint32_t* sel_out, size_t* n_sel) {
  return guarded([&] {
    const size_t W = e->W(), KW = e->KW(), B = e->B;
    cudaStream_t st = e->stream;
    double tp[7];
    if (g_host_prof) tp[0] = now_ns();
    const bool q_dev = is_device_ptr(q), k_dev = is_device_ptr(k), v_dev = is_device_ptr(v);
    const bool out_dev = is_device_ptr(out);
    if (g_host_prof) tp[1] = now_ns();
    // zero-query check before any mutation (selection_cache.cpp:18-27)
    if (!q_dev) {
      ts_pool& pool = *e->pool;
      for (size_t b = 0; b < B; ++b) {
        const size_t N = pool.state(e->sid(b)).len;
        if (!(e->cfg.k > 0 && N > e->cfg.n_init + e->cfg.n_local)) continue;
        bool nz = false;
        for (size_t i = 0; i < W && !nz; ++i) nz = q[b * W + i] != 0.0f;
        if (!nz) fail(TS_INVALID_ARGUMENT, "lookup_or_select: zero query vector");
      }
    }
    auto stage = [&](const float* src, bool dev, float* pinned, DevBuf& dbuf, size_t n) -> const float* {
      if (dev) return src;
      std::memcpy(pinned, src, n * 4);
      ck(cudaMemcpyAsync(dbuf.p, pinned, n * 4, cudaMemcpyHostToDevice, st), "H2D");
      return dbuf.as<float>();
    };
    const float *qd, *kd, *vd;
    // a host output: written straight into mapped pinned memory, with the
    // cache states mirrored next to it (no D2H copy on the critical path)
    const bool zc = !out_dev && e->h_out_dev != nullptr;
    float* od = out_dev ? out : zc ? reinterpret_cast<float*>(e->h_out_dev) : e->d_out.as<float>();
    if (!q_dev && !k_dev && !v_dev) {
      // host inputs: one pinned staging block, one H2D copy
      std::memcpy(e->h_q, q, B * W * 4);
      std::memcpy(e->h_q + B * W, k, B * KW * 4);
      std::memcpy(e->h_q + B * W + B * KW, v, B * KW * 4);
      const double tc = g_host_prof ? now_ns() : 0.0;
      if (g_host_prof) g_e2e_memcpy += tc - tp[1];
      // a 4-byte copy first: measured on B200 + driver 580 (tools/e2e_time.py),
      // the 24 KB pinned H2D as the first operation on an idle stream costs
      // ~10.5 us of host time, after a tiny one ~1.5 us (the pair ~3.5 us)
      if (!g_no_h2d_primer) {
        ck(cudaMemcpyAsync(e->d_q.p, e->h_q, 4, cudaMemcpyHostToDevice, st), "H2D");
        if (g_host_prof) g_e2e_memcpy += now_ns() - tc;
      }
      const double tc2 = g_host_prof ? now_ns() : 0.0;
      ck(cudaMemcpyAsync(e->d_q.p, e->h_q, (B * W + 2 * B * KW) * 4, cudaMemcpyHostToDevice, st), "H2D");
      if (g_host_prof) g_e2e_h2dapi += now_ns() - tc2;
      qd = e->d_q.as<float>();
      kd = qd + B * W;
      vd = kd + B * KW;
    } else {
      qd = stage(q, q_dev, e->h_q, e->d_q, B * W);
      kd = stage(k, k_dev, e->h_k, e->d_k, B * KW);
      vd = stage(v, v_dev, e->h_v, e->d_v, B * KW);
    }
    if (g_host_prof) tp[2] = now_ns();
    e->mirror_cache = zc;
    std::vector<int> cap_fail;
    try {
      cap_fail = engine_step(e, qd, kd, vd, od);
    } catch (...) {
      e->mirror_cache = false;
      throw;
    }
    e->mirror_cache = false;
    e->last_unchecked = false;  // checked below
    if (g_host_prof) tp[3] = now_ns();
    // every result rides one stream sync: output, cache states and (when
    // requested) the full selection slots
    const size_t kk = std::max<size_t>(e->cfg.k, 1);
    // d_out and the cache states are one device block (and h_out / h_cache
    // one pinned block): a host output rides the same D2H copy
    if (zc) {
      // (the output is host-visible; so are the cache states unless the
      // launch was the opt-in step kernel, which does not mirror them)
      if (!e->mirror_done)
        ck(cudaMemcpyAsync(e->hcache(0), e->cache(0), B * sizeof(CacheState), cudaMemcpyDeviceToHost, st), "D2H");
    } else if (!out_dev)
      ck(cudaMemcpyAsync(e->h_out, od, e->out_block_bytes(), cudaMemcpyDeviceToHost, st), "D2H");
    else
      ck(cudaMemcpyAsync(e->hcache(0), e->cache(0), B * sizeof(CacheState), cudaMemcpyDeviceToHost, st), "D2H");
    if (sel_out) {
      if (!e->h_sel) ck(cudaMallocHost(&e->h_sel, B * kk * 4), "pinned");
      ck(cudaMemcpyAsync(e->h_sel, e->sl(0), B * kk * 4, cudaMemcpyDeviceToHost, st), "D2H sel");  // this layer's slots
    }
    if (g_host_prof) tp[4] = now_ns();
    ck(cudaStreamSynchronize(st), "decode sync");
    if (g_host_prof) tp[5] = now_ns();
    if (!out_dev) std::memcpy(out, e->h_out, B * W * 4);
    ts_pool& pool = *e->pool;
    for (size_t b = 0; b < B; ++b) {
      const CacheState& cs = *e->hcache(b);
      if (cs.error) {
        for (size_t b2 = 0; b2 < B; ++b2)
          if (e->hcache(b2)->error) rollback_step(e, b2);
        fail(TS_INVALID_ARGUMENT, "lookup_or_select: zero query vector");
      }
      // the step ran a lookup iff selection was on for the sequence at step start
      const size_t N_after = pool.state(e->sid(b)).len;
      const size_t N = N_after - (cap_fail[b] ? 0 : 1);
      const bool sel_on = e->cfg.k > 0 && N > e->cfg.n_init + e->cfg.n_local;
      if (cache_hit) cache_hit[b] = sel_on ? cs.last_hit : 0;
      if (sel_out) {
        const size_t n = sel_on ? static_cast<size_t>(cs.n_sel) : 0;
        std::memcpy(sel_out + b * kk, e->h_sel + b * kk, n * 4);
        if (n_sel) n_sel[b] = n;
      }
    }
    if (g_host_prof) {
      tp[6] = now_ns();
      for (int i = 0; i < 6; ++i) g_e2e_prof[i] += tp[i + 1] - tp[i];
      g_e2e_n += 1;
    }
    for (size_t b = 0; b < B; ++b)
      if (cap_fail[b]) fail(TS_CAPACITY, "append_kv: pool exhausted (need 1 frames, 0 free)");
  });
}

ts_status ts_engine_decode_async(ts_engine* e, const float* q, const float* k, const float* v, float* out) {
  return guarded([&] {
    e->last_unchecked = true;
    std::vector<int> cap_fail = engine_step(e, q, k, v, out);
    for (size_t b = 0; b < e->B; ++b)
      if (cap_fail[b]) fail(TS_CAPACITY, "append_kv: pool exhausted (need 1 frames, 0 free)");
  });
}

ts_status ts_engine_force_miss(ts_engine* e, size_t seq) {
  return guarded([&] {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    const int one = 1;
    ck(cudaMemcpyAsync(&e->cache(seq)->first_flag, &one, sizeof(int), cudaMemcpyHostToDevice, e->stream), "H2D");
    ck(cudaStreamSynchronize(e->stream), "sync");
  });
}

ts_status ts_engine_set_trace(ts_engine* e, int enable) {
  return guarded([&] {
    e->trace_on = enable != 0;
    if (e->trace_on) {
      e->trace.ensure(kTraceSlots * 8);
      ck(cudaMemsetAsync(e->trace.p, 0, kTraceSlots * 8, e->stream), "memset");
      ck(cudaStreamSynchronize(e->stream), "sync");
    }
  });
}

ts_status ts_engine_read_trace(ts_engine* e, uint64_t* stamps, size_t n) {
  return guarded([&] {
    if (!e->trace.p) fail(TS_INVALID_ARGUMENT, "trace not enabled");
    ck(cudaStreamSynchronize(e->stream), "sync");
    ck(cudaMemcpy(stamps, e->trace.p, std::min<size_t>(n, kTraceSlots) * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

ts_status ts_engine_set_theta(ts_engine* e, size_t seq, double theta) {
  return guarded([&] {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    ck(cudaMemcpyAsync(&e->cache(seq)->theta, &theta, sizeof(double), cudaMemcpyHostToDevice, e->stream), "H2D");
    ck(cudaStreamSynchronize(e->stream), "sync");
  });
}

ts_status ts_engine_stats(const ts_engine* e, size_t seq, size_t* lookups, size_t* hits, size_t* len, int* last_hit,
                          double* last_cos) {
  return guarded([&] {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    CacheState cs{};
    ck(cudaMemcpyAsync(&cs, e->cache(seq), sizeof(CacheState), cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    // the last (async) step rejected on the device: rolled back and reported
    if (cs.error && e->last_unchecked) check_async_errors(const_cast<ts_engine*>(e));
    if (lookups) *lookups = cs.lookups;
    if (hits) *hits = cs.hits;
    if (len) *len = e->pool->state(e->sid(seq)).len;
    if (last_hit) *last_hit = cs.last_hit;
    if (last_cos) *last_cos = cs.last_cos;
  });
}

ts_status ts_engine_cached_selection(const ts_engine* e, size_t seq, uint32_t* sel_out, double* crit_out,
                                     size_t* n_out) {
  return guarded([&] {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    CacheState cs{};
    ck(cudaMemcpyAsync(&cs, e->cache(seq), sizeof(CacheState), cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    const size_t n = static_cast<size_t>(cs.n_sel);
    *n_out = n;
    if (!n) return;
    std::vector<float> crit(n);
    ck(cudaMemcpy(sel_out, e->sl(seq), n * 4, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(crit.data(), e->sc(seq), n * 4, cudaMemcpyDeviceToHost), "D2H");
    if (crit_out)
      for (size_t i = 0; i < n; ++i) crit_out[i] = crit[i];
  });
}

ts_status ts_engine_cache_entry(const ts_engine* e, size_t seq, float* cached_q, int* first_flag, double* theta) {
  return guarded([&] {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    CacheState cs{};
    ck(cudaMemcpyAsync(&cs, e->cache(seq), sizeof(CacheState), cudaMemcpyDeviceToHost, e->stream), "D2H");
    if (cached_q) ck(cudaMemcpyAsync(cached_q, e->cq(seq), e->W() * 4, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    if (first_flag) *first_flag = cs.first_flag;
    if (theta) *theta = cs.theta;
  });
}

ts_status ts_engine_sync(ts_engine* e) {
  return guarded([&] {
    ck(cudaStreamSynchronize(e->stream), "sync");
    check_async_errors(e);
  });
}

namespace {

void prefill_impl(ts_engine* e, size_t seq, const float* q, const float* k, const float* v, size_t n, float* out,
                  uint32_t* trace_sel, size_t* trace_counts, size_t max_chunks, bool sync) {
  {
    if (seq >= e->B) fail(TS_INVALID_ARGUMENT, "engine: sequence index out of range");
    if (n == 0) fail(TS_INVALID_ARGUMENT, "prefill: empty input");
    const ts_engine_config& c = e->cfg;
    ts_pool& pool = *e->pool;
    const uint32_t sid = e->sid(seq);
    const size_t W = e->W(), KW = e->KW();
    const int H = static_cast<int>(c.num_heads), Hkv = static_cast<int>(c.num_kv_heads), d = static_cast<int>(c.head_dim);
    cudaStream_t st = e->stream;
    const bool q_dev = is_device_ptr(q), k_dev = is_device_ptr(k), v_dev = is_device_ptr(v), o_dev = is_device_ptr(out);
    const size_t kk = std::max<size_t>(c.k, 1);
    size_t trace_off = 0;
    for (size_t begin = 0, chunk = 0; begin < n; begin += c.chunk_size, ++chunk) {
      const size_t len = std::min(c.chunk_size, n - begin);
      const float* qc = q_dev ? q + begin * W : nullptr;
      const float* kc = k_dev ? k + begin * KW : nullptr;
      const float* vc = v_dev ? v + begin * KW : nullptr;
      if (!q_dev) {
        qc = static_cast<float*>(e->p_q.ensure(len * W * 4));
        ck(cudaMemcpyAsync(const_cast<float*>(qc), q + begin * W, len * W * 4, cudaMemcpyHostToDevice, st), "H2D");
      }
      // host K/V: copied on the engine's copy stream once the query's copy
      // (and everything before it on the stream, e.g. the previous chunk's
      // reads of these buffers) is done, overlapping the selection launches
      const bool kv_side = !k_dev || !v_dev;
      if (kv_side) {
        if (!e->copy_stream) {
          ck(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking), "stream");
          ck(cudaEventCreateWithFlags(&e->ev_q, cudaEventDisableTiming), "event");
          ck(cudaEventCreateWithFlags(&e->ev_kv, cudaEventDisableTiming), "event");
        }
        ck(cudaEventRecord(e->ev_q, st), "event");
        ck(cudaStreamWaitEvent(e->copy_stream, e->ev_q, 0), "event");
      }
      if (!k_dev) {
        kc = static_cast<float*>(e->p_k.ensure(len * KW * 4));
        ck(cudaMemcpyAsync(const_cast<float*>(kc), k + begin * KW, len * KW * 4, cudaMemcpyHostToDevice,
                           e->copy_stream), "H2D");
      }
      if (!v_dev) {
        vc = static_cast<float*>(e->p_v.ensure(len * KW * 4));
        ck(cudaMemcpyAsync(const_cast<float*>(vc), v + begin * KW, len * KW * 4, cudaMemcpyHostToDevice,
                           e->copy_stream), "H2D");
      }
      if (kv_side) ck(cudaEventRecord(e->ev_kv, e->copy_stream), "event");
      ts_pool::Seq& s = pool.state(sid);
      const size_t cached = s.len;
      // the chunk's page-table entries now (capacity checked before any work
      // of the chunk), so that its append can follow the attention directly
      pool.reserve(s, len, st);
      uint32_t* psel = static_cast<uint32_t*>(e->p_sel.ensure(kk * 4));
      CacheState* pstate = static_cast<CacheState*>(e->p_state.ensure(sizeof(CacheState)));
      ck(cudaMemsetAsync(pstate, 0, sizeof(CacheState), st), "memset");
      size_t T = 0;
      if (c.k > 0 && cached > c.n_init + c.n_local) T = cached - c.n_init - c.n_local;
      if (T > 0) {
        // select_for_chunk: chunk mean (K9), then the fused score + soft vote + top-k
        float* qm = static_cast<float*>(e->p_qmean.ensure(W * 4));
        ck(tsb::launch_chunk_mean(qc, static_cast<int>(len), static_cast<int>(W), qm, st), "chunk_mean");
        g_launches.fetch_add(1);
        DecodeParams p = base_params(&pool, H, Hkv, d, static_cast<int>(c.k), c.selection_method,
                                     tsb::kModeScore | tsb::kModeSelect);
        p.n_seq = 1;
        SeqDesc& sd = p.seqs[0];
        sd.page_table = s.d_pt;
        sd.n_cached = static_cast<int32_t>(cached);
        sd.cand_begin = static_cast<int32_t>(c.n_init);
        sd.n_cand = static_cast<int32_t>(T);
        sd.select = 1;
        sd.q = qm;
        sd.append_frame = -1;
        sd.append_page = -1;
        sd.cache = pstate;
        sd.sel = psel;
        sd.sel_crit = static_cast<float*>(e->p_crit.ensure(kk * 4));
        sd.sel_rows = static_cast<int32_t*>(e->p_selrows.ensure(kk * 4));  // (the LEAN select-only kernel publishes them)
        const Plan pl = make_plan(H, Hkv, d, 1, static_cast<int>(T), 1, false);
        if (c.selection_method == TS_HEAD_VOTE) {
          float* S = e->ws.vote_scores(1, H, static_cast<int>(T));
          p.mode = tsb::kModeScore | tsb::kModeSOut;
          sd.s_out = S;
          launch_decode(p, pl, e->ws, st);
          ck(tsb::launch_head_vote(S, H, static_cast<int>(T), static_cast<int>(c.k), nullptr, static_cast<int>(c.n_init),
                                   nullptr, psel, sd.sel_crit, nullptr, &pstate->n_sel,
                                   e->ws.vote(H, static_cast<int>(T)), nullptr, st),
             "head vote");
          g_launches.fetch_add(3);
        } else {
          launch_decode(p, pl, e->ws, st);
        }
      }
      if (kv_side) ck(cudaStreamWaitEvent(st, e->ev_kv, 0), "event");  // (the attention reads the chunk's K/V)
      // windows (make_windows) -> device merged list
      const int init_end = static_cast<int>(std::min(c.n_init, cached));
      const int local_begin = static_cast<int>(cached - std::min(c.n_local, cached));
      // merged windows: init U selected U local (<= n_init + k + n_local rows)
      uint32_t* att = static_cast<uint32_t*>(e->p_att.ensure((c.n_init + kk + c.n_local + 1) * 4));
      int* natt = static_cast<int*>(e->p_natt.ensure(16));
      // the tcgen05 attention forms the windows inside its prep launch; the
      // other kernels read the merged list windows_kernel writes
      const bool implicit = prefill_uses_tc(static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                                            static_cast<int>(c.head_dim));
      if (!implicit) {
        unsigned int* bad = static_cast<unsigned int*>(e->p_bad.ensure(16));
        ck(cudaMemsetAsync(bad, 0, 4, st), "memset");
        ck(tsb::launch_windows(psel, T > 0 ? &pstate->n_sel : nullptr, 0, static_cast<int>(cached), init_end,
                               local_begin, att, natt, bad, st),
           "windows");
        g_launches.fetch_add(1);
      }
      float* oc = o_dev ? out + begin * W : static_cast<float*>(e->p_out.ensure(len * W * 4));
      tsb::PrefillAttendParams pa{};
      pa.q = qc;
      pa.k_cur = kc;
      pa.v_cur = vc;
      pa.k_slab = pool.k_slab;
      pa.v_slab = pool.v_slab;
      pa.page_table = s.d_pt;
      pa.page_size = static_cast<int>(pool.page_size);
      pa.att = implicit ? nullptr : att;
      pa.n_att_ptr = natt;
      if (implicit) {
        pa.win_sel = T > 0 ? psel : nullptr;
        pa.win_n_sel = T > 0 ? &pstate->n_sel : nullptr;
        pa.win_init_end = init_end;
        pa.win_local_begin = local_begin;
        pa.win_cached = static_cast<int>(cached);
        pa.win_n_att = natt;
      }
      // init U selected U local, disjoint cached rows
      pa.n_att_max = static_cast<int>(std::min<size_t>(cached, init_end + std::min<size_t>(kk, T) + (cached - local_begin)));
      pa.C = static_cast<int>(len);
      pa.H = H;
      pa.H_kv = Hkv;
      pa.d = d;
      pa.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
      pa.out = oc;
      static const char* ptrace = std::getenv("TS_PREFILL_TRACE");  // dev: stamps -> this file (prefill_tc.cu)
      if (ptrace) {
        pa.trace = static_cast<unsigned long long*>(e->p_trace.ensure(4096 * 8));
        ck(cudaMemsetAsync(pa.trace, 0, 4096 * 8, st), "memset");
      }
      ck(launch_prefill(pa, e->p_split, st), "prefill_attend");
      g_launches.fetch_add(1);
      if (ptrace) {
        std::vector<unsigned long long> h(4096);
        ck(cudaMemcpyAsync(h.data(), pa.trace, 4096 * 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        if (FILE* f = std::fopen(ptrace, "wb")) {
          std::fwrite(h.data(), 8, h.size(), f);
          std::fclose(f);
        }
      }
      if (!o_dev) ck(cudaMemcpyAsync(out + begin * W, oc, len * W * 4, cudaMemcpyDeviceToHost, st), "D2H");
      if (trace_counts && chunk < max_chunks) {
        CacheState cs{};
        ck(cudaMemcpyAsync(&cs, pstate, sizeof(CacheState), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        const size_t ns = T > 0 ? static_cast<size_t>(cs.n_sel) : 0;
        trace_counts[chunk] = ns;
        if (ns && trace_sel) ck(cudaMemcpy(trace_sel + trace_off, psel, ns * 4, cudaMemcpyDeviceToHost), "D2H");
        trace_off += ns;
      }
      // append the chunk after attending (attention.cpp:167)
      static const bool no_pdl = std::getenv("TS_NO_PDL") != nullptr;
      pool.append(sid, kc, vc, len, false, nullptr, nullptr, st, false, true, !no_pdl && implicit);
    }
    if (sync) ck(cudaStreamSynchronize(st), "sync");
  }
}

}  // namespace

ts_status ts_engine_prefill(ts_engine* e, size_t seq, const float* q, const float* k, const float* v, size_t n,
                            float* out, uint32_t* trace_sel, size_t* trace_counts, size_t max_chunks) {
  return guarded([&] { prefill_impl(e, seq, q, k, v, n, out, trace_sel, trace_counts, max_chunks, true); });
}

ts_status ts_engine_prefill_async(ts_engine* e, size_t seq, const float* q, const float* k, const float* v, size_t n,
                                  float* out) {
  return guarded([&] {
    if (!is_device_ptr(q) || !is_device_ptr(k) || !is_device_ptr(v) || !is_device_ptr(out))
      fail(TS_INVALID_ARGUMENT, "prefill_async: q, k, v and out must be device buffers");
    prefill_impl(e, seq, q, k, v, n, out, nullptr, nullptr, 0, false);
  });
}


// ------------------------------------------------------ tensor utilities
// (the free functions of the reference's pybind module, bindings.cpp:60-116)
ts_status ts_softmax_rows(const float* m, size_t rows, size_t cols, float* out) {
  return guarded([&] {
    if (rows == 0 || cols == 0) return;
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const float* md = dev_in(m, rows * cols, g.a, st);
    float* od = is_device_ptr(out) ? out : static_cast<float*>(g.b.ensure(rows * cols * 4));
    ck(tsb::launch_softmax_rows(md, static_cast<int>(rows), static_cast<int>(cols), od, st), "softmax_rows");
    g_launches.fetch_add(1);
    if (od != out) copy_out(out, od, rows * cols * 4, st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

ts_status ts_topk_indices(const double* scores, size_t n, size_t k, uint32_t* out, size_t* n_out) {
  return guarded([&] {
    *n_out = 0;
    if (n == 0) fail(TS_INVALID_ARGUMENT, "topk_indices: empty scores");
    if (k == 0) fail(TS_INVALID_ARGUMENT, "topk_indices: k must be >= 1");
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const double* sd = dev_in(scores, n, g.c, st);
    const size_t take = std::min(k, n);
    uint32_t* od = static_cast<uint32_t*>(g.d.ensure(take * 4 + 16));
    int* nd = reinterpret_cast<int*>(od + take);
    ck(tsb::launch_topk64(sd, static_cast<int>(n), static_cast<int>(k), od, nd, st), "topk_indices");
    g_launches.fetch_add(1);
    int nn = 0;
    ck(cudaMemcpyAsync(&nn, nd, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    copy_out(out, od, take * 4, st);
    ck(cudaStreamSynchronize(st), "sync");
    *n_out = static_cast<size_t>(nn);
  });
}

ts_status ts_cosine(const double* u, const double* v, size_t n, double* out) {
  return guarded([&] {
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const double* ud = dev_in(u, n, g.c, st);
    const double* vd = dev_in(v, n, g.e, st);
    double* od = static_cast<double*>(g.f.ensure(16));
    ck(tsb::launch_cosine(ud, vd, static_cast<int>(n), od, st), "cosine");
    g_launches.fetch_add(1);
    double r = 0.0;
    ck(cudaMemcpyAsync(&r, od, 8, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    if (std::isnan(r)) fail(TS_INVALID_ARGUMENT, "cosine: zero-norm input");
    *out = r;
  });
}

ts_status ts_chunk_mean(const float* q_chunk, size_t c, size_t width, float* out) {
  return guarded([&] {
    if (c == 0) fail(TS_INVALID_ARGUMENT, "chunk_mean: empty chunk");
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const float* qd = dev_in(q_chunk, c * width, g.a, st);
    float* od = is_device_ptr(out) ? out : static_cast<float*>(g.b.ensure(width * 4));
    ck(tsb::launch_chunk_mean(qd, static_cast<int>(c), static_cast<int>(width), od, st), "chunk_mean");
    g_launches.fetch_add(1);
    if (od != out) copy_out(out, od, width * 4, st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

ts_status ts_sdpa_full(const float* q, size_t C, size_t width, const float* k_all, const float* v_all, size_t N,
                       size_t kv_width, size_t num_heads, float* out) {
  return guarded([&] {
    if (num_heads == 0 || width == 0 || width % num_heads != 0)
      fail(TS_INVALID_ARGUMENT, "sdpa_full: q must be [C x (H * d_h)]");
    const size_t d = width / num_heads;
    if (kv_width == 0 || kv_width % d != 0) fail(TS_INVALID_ARGUMENT, "sdpa_full: K/V must be [(N + C) x (H_kv * d_h)]");
    const size_t H_kv = kv_width / d;
    if (num_heads % H_kv != 0) fail(TS_INVALID_ARGUMENT, "sdpa_full: H must be a multiple of H_kv");
    if (N < C) fail(TS_INVALID_ARGUMENT, "sdpa_full: fewer KV rows than query rows");
    if (C == 0) return;
    GlobalCtx& g = gctx();
    cudaStream_t st = g.stream;
    const float* qd = dev_in(q, C * width, g.a, st);
    const float* kd = dev_in(k_all, N * kv_width, g.c, st);
    const float* vd = dev_in(v_all, N * kv_width, g.e, st);
    float* od = is_device_ptr(out) ? out : static_cast<float*>(g.b.ensure(C * width * 4));
    double* ws = static_cast<double*>(g.f.ensure(C * num_heads * N * 8));
    ck(tsb::launch_sdpa_full(qd, kd, vd, static_cast<int>(C), static_cast<int>(N), static_cast<int>(num_heads),
                             static_cast<int>(H_kv), static_cast<int>(d), od, ws, st),
       "sdpa_full");
    g_launches.fetch_add(1);
    if (od != out) copy_out(out, od, C * width * 4, st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// ------------------------------------------------------------ sharded decode
ts_status ts_shard_engine_create(const ts_engine_config* cfg, size_t capacity_tokens, int rank, int world,
                                 ts_engine** out) {
  return guarded([&] {
    if (world < 1 || world > 64 || rank < 0 || rank >= world)
      fail(TS_INVALID_ARGUMENT, "shard: rank must be in [0, world), world in [1, 64]");
    check_method_supported(cfg->selection_method, true);
    ts_status rc = ts_engine_create(cfg, capacity_tokens, 1, out);
    if (rc != TS_OK) fail(rc, g_err);
    (*out)->rank = rank;
    (*out)->world = world;
  });
}

namespace {

// Parameters shared by the stats and select launches of one shard step.
DecodeParams shard_params(ts_engine* e, int mode) {
  ts_pool& pool = *e->pool;
  const ts_engine_config& c = e->cfg;
  const ShardStep& ss = e->shard;
  DecodeParams p = base_params(&pool, static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                               static_cast<int>(c.head_dim), static_cast<int>(c.k), c.selection_method, mode);
  p.n_seq = 1;
  ts_pool::Seq& s = pool.state(e->sid(0));
  SeqDesc& sd = p.seqs[0];
  sd.page_table = s.d_pt;
  sd.n_cached = static_cast<int32_t>(s.len);
  sd.select = ss.sel_on;
  sd.cand_begin = ss.cand_first;
  sd.n_cand = ss.T;
  sd.q = ss.q;
  sd.k_new = ss.k;
  sd.v_new = ss.v;
  sd.append_frame = -1;
  sd.append_page = -1;
  sd.cache = e->cache(0);
  sd.cached_q = e->cq(0);
  sd.sel = e->sl(0);
  sd.sel_crit = e->sc(0);
  sd.sel_rows = e->sr(0);
  sd.shard_base = static_cast<int32_t>(ss.base);
  sd.shard_world = e->world;
  p.trace = e->trace_on ? e->trace.as<unsigned long long>() : nullptr;
  if (p.trace) ck(cudaMemsetAsync(p.trace, 0, kTraceSlots * 8, e->stream), "memset trace");
  return p;
}

Plan shard_plan_for(ts_engine* e) {
  const ts_engine_config& c = e->cfg;
  return make_plan(static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads), static_cast<int>(c.head_dim), 1,
                   e->shard.T, 1, false, /*force_spill=*/true);
}

}  // namespace

ts_status ts_shard_stats(ts_engine* e, const float* q, const float* k, const float* v, size_t base, size_t n_global,
                         float* stats_out) {
  return guarded([&] {
    const ts_engine_config& c = e->cfg;
    ShardStep& ss = e->shard;
    const size_t n_r = e->pool->state(e->sid(0)).len;
    const bool first = e->rank == 0, last = e->rank == e->world - 1;
    if (first && base != 0) fail(TS_INVALID_ARGUMENT, "shard: rank 0 must start at position 0");
    if (base + n_r > n_global) fail(TS_INVALID_ARGUMENT, "shard: rows beyond the global length");
    if (last && base + n_r != n_global) fail(TS_INVALID_ARGUMENT, "shard: the last shard must end the sequence");
    if (e->world > 1 && first && n_r < std::min(c.n_init, n_global))
      fail(TS_INVALID_ARGUMENT, "shard: rank 0 must hold the whole init window");
    if (e->world > 1 && last && n_r < std::min(c.n_local, n_global))
      fail(TS_INVALID_ARGUMENT, "shard: the last shard must hold the whole local window");
    ss.q = q;
    ss.k = k;
    ss.v = v;
    ss.base = base;
    ss.n_global = n_global;
    ss.n_local_len = n_r;
    ss.sel_on = (c.k > 0 && n_global > c.n_init + c.n_local) ? 1 : 0;
    const size_t lo = first ? std::min(c.n_init, n_r) : 0;
    const size_t hi = last ? n_r - std::min(c.n_local, n_r) : n_r;
    ss.cand_first = static_cast<int32_t>(lo);
    ss.T = ss.sel_on && hi > lo ? static_cast<int32_t>(hi - lo) : 0;
    DecodeParams p = shard_params(e, tsb::kModeCache | tsb::kModeScore | tsb::kModeSelect | tsb::kModeShardStats);
    p.seqs[0].shard_stats = stats_out;
    // the kernel writes NaN (unset) over stats_out when it has no fresh statistics
    launch_decode(p, shard_plan_for(e), e->ws, e->stream);
  });
}

ts_status ts_shard_select(ts_engine* e, const float* all_stats, uint32_t* cands_out) {
  return guarded([&] {
    const ts_engine_config& c = e->cfg;
    ck(cudaMemsetAsync(cands_out + 2 * c.k, 0, 4, e->stream), "memset count");
    if (!e->shard.sel_on) return;
    DecodeParams p = shard_params(e, tsb::kModeSelect | tsb::kModeShardSelect);
    p.seqs[0].shard_all = all_stats;
    p.seqs[0].shard_cands = cands_out;
    launch_decode(p, shard_plan_for(e), e->ws, e->stream);
  });
}

ts_status ts_shard_attend(ts_engine* e, const uint32_t* all_cands, float* out_partial, float* ml_out) {
  return guarded([&] {
    const ts_engine_config& c = e->cfg;
    ts_pool& pool = *e->pool;
    const ShardStep& ss = e->shard;
    ts_pool::Seq& s = pool.state(e->sid(0));
    const size_t n_r = s.len, N = ss.n_global;
    const bool first = e->rank == 0, last = e->rank == e->world - 1;
    const size_t ie = std::min(c.n_init, N);
    const size_t lbs = std::max(N - std::min(c.n_local, N), ie);
    const size_t init_hi = first ? std::min(ie, n_r) : 0;
    const size_t loc_lo = last ? std::max(lbs, ss.base) - ss.base : n_r;
    cudaStream_t st = e->stream;
    uint32_t* att = static_cast<uint32_t*>(e->s_att.ensure((n_r + c.k + 8) * 4));
    int* natt = static_cast<int*>(e->s_natt.ensure(16));
    ck(tsb::launch_shard_merge(all_cands, e->world, static_cast<int>(c.k), static_cast<uint32_t>(ie),
                               static_cast<uint32_t>(lbs), static_cast<uint32_t>(ss.base), static_cast<uint32_t>(n_r),
                               static_cast<uint32_t>(init_hi), static_cast<uint32_t>(loc_lo), att, natt, st),
       "shard merge");
    g_launches.fetch_add(1);
    DecodeParams p = base_params(&pool, static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                                 static_cast<int>(c.head_dim), static_cast<int>(c.k), c.selection_method,
                                 tsb::kModeAttend | (last ? tsb::kModeAppend : 0));
    p.n_seq = 1;
    SeqDesc& sd = p.seqs[0];
    sd.page_table = s.d_pt;
    sd.n_cached = static_cast<int32_t>(n_r);
    sd.select = 0;
    sd.q = ss.q;
    sd.k_new = ss.k;
    sd.v_new = ss.v;
    sd.out = out_partial;
    sd.att_list = att;
    sd.n_att_dev = natt;
    sd.n_att = 0;
    sd.no_cur = last ? 0 : 1;
    sd.ml_out = ml_out;
    sd.cache = e->cache(0);
    sd.append_frame = -1;
    sd.append_page = -1;
    bool appended = false;
    if (last) {
      if (pool.free_list.empty()) fail(TS_CAPACITY, "append_kv: pool exhausted (need 1 frames, 0 free)");
      const uint32_t f = pool.free_list.back();
      pool.free_list.pop_back();
      s.frames.push_back(f);
      e->last_frames.assign(1, f);
      sd.append_frame = static_cast<int32_t>(f);
      sd.append_slot = 0;
      sd.append_page = static_cast<int32_t>(n_r);
      appended = true;
    }
    const DeviceInfo& di = device_info();
    const Plan pl = make_plan(static_cast<int>(c.num_heads), static_cast<int>(c.num_kv_heads),
                              static_cast<int>(c.head_dim), 1, 0, di.num_sms * 64);
    p.trace = e->trace_on ? e->trace.as<unsigned long long>() : nullptr;
    if (p.trace) ck(cudaMemsetAsync(p.trace, 0, kTraceSlots * 8, st), "memset trace");
    launch_decode(p, pl, e->ws, st);
    if (appended) s.len += 1;
  });
}

// ---------------------------------------------- in-library data plane
struct ts_comm {
  tsb::Comm c;
};

ts_status ts_comm_unique_id(uint8_t* id128) {
  return guarded([&] { tsb::nccl_unique_id(id128); });
}

ts_status ts_comm_create(const uint8_t* id128, int world, int rank, ts_comm** out) {
  return guarded([&] {
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) fail(TS_INVALID_ARGUMENT, "comm: rank must be in [0, world)");
    device_info();
    auto c = std::make_unique<ts_comm>();
    if (world > 1) tsb::nccl_comm_init(&c->c, id128, world, rank);
    c->c.world = world;
    c->c.rank = rank;
    *out = c.release();
  });
}

void ts_comm_destroy(ts_comm* c) {
  if (!c) return;
  tsb::nccl_comm_destroy(&c->c);
  delete c;
}

// One sharded decode step: stats -> all-gather -> select ->
// all-gather -> attend -> all-gather -> combine, every launch and every
// ncclAllGather on the engine's stream, no host synchronisation (unless out
// is a host pointer). A one-rank communicator (or comm == NULL at world 1)
// passes each block straight to the next phase.
ts_status ts_shard_decode_step(ts_engine* e, ts_comm* comm, const float* q, const float* k, const float* v,
                               size_t base, size_t n_global, float* out) {
  return guarded([&] {
    const ts_engine_config& c = e->cfg;
    const int world = e->world;
    if ((comm ? comm->c.world : 1) != world || (comm ? comm->c.rank : 0) != e->rank)
      fail(TS_INVALID_ARGUMENT, "shard: the communicator's rank / world differ from the shard engine's");
    if (world > 1 && !comm) fail(TS_INVALID_ARGUMENT, "shard: world > 1 needs a communicator");
    cudaStream_t st = e->stream;
    const size_t W = e->W(), KW = e->KW(), H = c.num_heads, kk = std::max<size_t>(c.k, 1);
    const float* qd = dev_in(q, W, e->d_q, st);
    const float* kd = dev_in(k, KW, e->d_k, st);
    const float* vd = dev_in(v, KW, e->d_v, st);
    const size_t n_stats = H * 2, n_cands = 2 * kk + 1, n_pack = W + H * 2;
    float* blk = static_cast<float*>(e->s_blk.ensure((n_stats + n_cands + n_pack) * (world + 1) * 4));
    float* stats = blk;
    uint32_t* cands = reinterpret_cast<uint32_t*>(stats + n_stats);
    float* pack = reinterpret_cast<float*>(cands + n_cands);
    float* all = pack + n_pack;
    float* all_stats = all;
    uint32_t* all_cands = reinterpret_cast<uint32_t*>(all_stats + world * n_stats);
    float* all_pack = reinterpret_cast<float*>(all_cands + world * n_cands);
    auto gather = [&](const void* send, void* recv, size_t words) -> const void* {
      if (world == 1) return send;
      tsb::nccl_all_gather(comm->c, send, recv, words * 4, st);
      return recv;
    };
    ts_status rc = ts_shard_stats(e, qd, kd, vd, base, n_global, stats);
    if (rc != TS_OK) fail(rc, g_err);
    const float* gs = static_cast<const float*>(gather(stats, all_stats, n_stats));
    rc = ts_shard_select(e, gs, cands);
    if (rc != TS_OK) fail(rc, g_err);
    const uint32_t* gc = static_cast<const uint32_t*>(gather(cands, all_cands, n_cands));
    rc = ts_shard_attend(e, gc, pack, pack + W);
    if (rc != TS_OK) fail(rc, g_err);
    const float* gp = static_cast<const float*>(gather(pack, all_pack, n_pack));
    float* od = is_device_ptr(out) ? out : static_cast<float*>(e->s_out.ensure(W * 4));
    rc = ts_shard_combine_packed(gp, world, H, c.head_dim, od, st);
    if (rc != TS_OK) fail(rc, g_err);
    e->last_unchecked = true;  // a zero query is reported by the next sync / stats
    if (od != out) {
      ck(cudaMemcpyAsync(out, od, W * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      check_async_errors(e);
    }
  });
}

ts_status ts_shard_combine(const float* o_all, const float* ml_all, int world, size_t num_heads, size_t head_dim,
                           float* out, void* stream) {
  return guarded([&] {
    device_info();
    ck(tsb::launch_shard_combine(o_all, ml_all, world, static_cast<int>(num_heads), static_cast<int>(head_dim), out,
                                 static_cast<cudaStream_t>(stream)),
       "shard combine");
    g_launches.fetch_add(1);
  });
}

ts_status ts_shard_combine_packed(const float* packed_all, int world, size_t num_heads, size_t head_dim, float* out,
                                  void* stream) {
  return guarded([&] {
    device_info();
    ck(tsb::launch_shard_combine(packed_all, packed_all + num_heads * head_dim, world, static_cast<int>(num_heads),
                                 static_cast<int>(head_dim), out, static_cast<cudaStream_t>(stream), true),
       "shard combine");
    g_launches.fetch_add(1);
  });
}

}  // extern "C"

// cm_api.cu -- the C ABI declared in include/cm.h (validation, graph upload, launch).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "cm.h"
#include "cm_kernel.cuh"
#define CM_API_TU
#include "cm_inst.cuh"

namespace {

thread_local std::string g_err;

cm_status fail(cm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

cm_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return CM_ECUDA;
}

}  // namespace

namespace cmp {
// S of a checkpoint set (R3), one row r of one set per CTA, 0-based: forward nodes
// 0..L-1, loss L.  i >= L (loss, gradients) or i in K: kept while r <= last(i); other forward
// nodes: r <= lastF(i), or 2L - tau(i) < r <= last(i) (recomputed at the backward stage of the
// top tau(i) of i's run of non-checkpoint nodes).  last / lastF from the successor CSR.
__global__ void policy_sstar_kernel(const int32_t* succ_ptr, const int32_t* succ_idx, int n, int L,
                                    const uint8_t* k_sets, float* out, int64_t ld) {
  __shared__ int tau[CM_NMAX];
  const int r = blockIdx.x, set = blockIdx.y;
  const uint8_t* K = k_sets + (size_t)set * L;
  if (threadIdx.x == 0) {
    int top = -1;
    for (int v = L - 1; v >= 0; --v) {
      if (K[v]) top = -1;
      else if (top < 0) top = v;
      tau[v] = top;
    }
  }
  __syncthreads();
  float* row = out + ((size_t)set * n + r) * ld;
  for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) {
    float v = 0.f;
    if (i < r) {
      int last = (int)i, lastF = (int)i;
      for (int e = succ_ptr[i]; e < succ_ptr[i + 1]; ++e) {
        const int j = succ_idx[e];
        last = max(last, j);
        if (j <= L) lastF = max(lastF, j);
      }
      bool keep;
      if (i >= L || K[i]) keep = r <= last;
      else keep = r <= lastF || (2 * L - tau[i] < r && r <= last);
      v = keep ? 1.f : 0.f;
    }
    row[i] = v;
  }
}
}  // namespace cmp

struct cm_graph {
  int32_t n = 0, E = 0;
  int64_t ovh = 0, cost_bound = 0;
  int device = 0, sm_count = 0, smem_optin = 0;
  int32_t blob_bytes = 0;
  int32_t o_pred_ptr = 0, o_pred_idx = 0, o_later = 0, o_succ_ptr = 0, o_succ_idx = 0;
  void* d_blob = nullptr;
  // v2 (stage-sliced) path
  int32_t blob2_bytes = 0;            // M/mscale, C, pred_ptr, pred_idx, node/dep records
  int32_t o_nrec = 0, o_drec = 0, o_qinfo = 0;
  int64_t mscale = 1;                 // gcd of all M (>= 1); the scan works in units of it
  bool scan32 = false;                // sum M / mscale < 2^30: int32 per-stage state
  int32_t n_slot = 0;                 // nodes with a non-adjacent user (K2 A' slots)
  void* d_blob2 = nullptr;
  void* d_nib = nullptr;              // K1 nibble tables of M (checkpoint mass, Eq. 6)
  void* d_nib32 = nullptr;            // int32 copy when scan32 (every row mass < 2^30)
  int32_t nib_entries = 0;
  void* d_ws = nullptr;               // default workspace: two chunk buffers of Sn columns
  int64_t ws_bytes = 0;
  // K1 (rounding) runs on its own stream so it streams chunk c+1 from HBM while K2 scans
  // chunk c; events order the two buffers (ping-pong) against the caller's stream.
  cudaStream_t st_round = nullptr;
  cudaEvent_t ev_start = nullptr, ev_round[2] = {nullptr, nullptr}, ev_scan[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  // fused path: the graph's workspace is used as two halves, alternating per call, each
  // [control words][ring]; a half's control words are zero after every fused call on it
  // (the kernel clears them on exit), so a CM_EVAL_OVERLAP call skips the memset
  int ws_half = 0;
  int64_t ctl_clean[2] = {0, 0};      // leading control words of each half known to be zero
  // completion signal (cm_stream_wait_call): call i stores i into d_seq when its outputs are written
  uint32_t* d_seq = nullptr;
  uint32_t seq = 0;                   // number of the last call (under mu)
  std::mutex mu;
};

namespace {
int kernel_choice() {                 // CM_KERNEL=v1 selects the row-form kernel (A/B tests)
  const char* e = std::getenv("CM_KERNEL");
  return (e && std::strcmp(e, "v1") == 0) ? 1 : 2;
}
constexpr int64_t kDefaultWsBytes = int64_t(1024) << 20; // two 512 MB chunk buffers / fused ring halves
}  // namespace


namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*StreamValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValue32Fn stream_value32(const char* name) {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<StreamValue32Fn>(ptr);
  return nullptr;
}
StreamValue32Fn wait_value32() {
  static StreamValue32Fn fn = stream_value32("cuStreamWaitValue32");
  return fn;
}
StreamValue32Fn write_value32() {
  static StreamValue32Fn fn = stream_value32("cuStreamWriteValue32");
  return fn;
}
// the multi-kernel paths' completion signal: a stream write after their last launch
cudaError_t signal_call(const cm_graph* g, uint32_t seq, cudaStream_t st) {
  StreamValue32Fn fn = write_value32();
  if (!fn) return cudaErrorNotSupported;
  return fn(st, reinterpret_cast<CUdeviceptr>(g->d_seq), seq, 0) == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

// Per-device function-attribute state (cudaFuncSetAttribute is per device): bit flags / sizes
// indexed by device ordinal, under attr_mu.
constexpr int kMaxDev = 64;
std::mutex attr_mu;
struct DevAttrs {
  size_t scan_smem = 0;               // scan_kernel dynamic shared memory set so far
  bool carve = false;                 // carve-out + K1 shared memory set
  size_t v1_smem = 0;                 // row-form kernel
};
DevAttrs g_attrs[kMaxDev];

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// Per-candidate workspace bytes of one chunk buffer: K1 output block + K2 partials.
int64_t cand_bytes(int n, bool m32) { return 4 * (int64_t)cm2::cand_words(n, m32) + 16 * (int64_t)((n + 31) / 32); }
size_t scan_warp_bytes(int n_slot, bool s32, bool tm, int tcols = 256, int q = cm2::kSnRing) {
  const int spill = std::max(0, n_slot - (tm ? tcols : 0));        // A' slots kept in shared memory
  return (size_t)cm2::scan_e_bytes(s32, q) + (size_t)4 * 32 * spill;   // E (+ staged int32 masses, Sn ring), spill
}
// CM_TRACE=1: record timing events around every K1 (round stream) and K2+K3 (caller stream)
// launch of the next call; cm_debug_trace() returns their offsets (debug / overlap check).
struct Trace {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // per chunk: k1 begin, k1 end, k2 begin, k2 end
  int used = 0;
};
// Debug state is per host thread (cm_debug_* report the calling thread's calls).
thread_local Trace g_trace;
// CM_TRACE=2: per-CTA timestamps of fused launches, kTraceCalls regions of 4 x kTraceCtas words
// used in turn; the whole buffer is cleared when region 0 is reused, so consecutive calls
// keep overlapping (no memset between them) for kTraceCalls - 1 calls
constexpr int kTraceCalls = 16, kTraceCtas = 1024;
thread_local uint64_t* g_cta_trace = nullptr;
thread_local int32_t g_cta_trace_n = 0;
thread_local int64_t g_cta_trace_calls = 0;   // fused calls traced so far by this thread
thread_local int32_t g_launches = 0;   // kernels launched by this thread's last cm_round_and_evaluate
bool trace_enabled() {
  const char* e = std::getenv("CM_TRACE");
  return e && std::strcmp(e, "1") == 0;
}
cudaEvent_t trace_event(int i) {
  while ((int)g_trace.ev.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_trace.ev.push_back(e);
  }
  return g_trace.ev[i];
}

bool tmem_enabled() {
  const char* e = std::getenv("CM_TMEM");
  return !(e && std::strcmp(e, "0") == 0);
}

// tuning switches: CM_EVICT_FIRST=1 (default off), CM_PREFETCH=0 (default on)
int env_flag(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// L2 sector promotion of the K1 tensor-map loads.  A block row is 128 bytes; a 256-byte
// promotion also pulls the next 32 nodes of the row (for the diagonal block w = g, entries of
// the never-read upper triangle), yet it measured fastest once rows are 128-byte aligned
// (ld % 32 == 0): 12.97 vs 12.63 M cand/s (128 B) at n = 353 in the two-kernel pipeline.
// CM_L2PROMO = 0 / 64 / 128 / 256 (tuning), default 256 (measured best with 128-byte aligned rows).
CUtensorMapL2promotion promo_of(int v) {
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}
CUtensorMapL2promotion l2_promotion() { return promo_of(env_flag("CM_L2PROMO", 256)); }

// lay: 0 dense (tensor-map TMA), 1 tri4 (gather4 / per-row bulk copies), 2 blocked (one bulk copy per block)
const void* round_fn(int nt, int lay, bool rnd) {
#define CM_R1(NT, L) (rnd ? reinterpret_cast<const void*>(cm2::round_tma_kernel<NT, L, true>) \
                          : reinterpret_cast<const void*>(cm2::round_tma_kernel<NT, L, false>))
#define CM_R(NT) (lay == 1 ? CM_R1(NT, 1) : lay == 2 ? CM_R1(NT, 2) : CM_R1(NT, 0))
  switch (nt) {
    case 1: return CM_R(1);
    case 2: return CM_R(2);
    case 3: return CM_R(3);
    default: return CM_R(4);
  }
#undef CM_R
#undef CM_R1
}
const void* fused_fn(int nt, int lay, bool rnd, bool s32) {
#define CM_F1(NT, L, ET) (rnd ? reinterpret_cast<const void*>(cm2::fused_kernel<NT, L, true, int32_t>) \
                              : reinterpret_cast<const void*>(cm2::fused_kernel<NT, L, false, ET>))
#define CM_F(NT, ET) (lay == 1 ? CM_F1(NT, 1, ET) : lay == 2 ? CM_F1(NT, 2, ET) : CM_F1(NT, 0, ET))
  if (s32) {
    switch (nt) {
      case 1: return CM_F(1, int32_t);
      case 2: return CM_F(2, int32_t);
      case 3: return CM_F(3, int32_t);
      default: return CM_F(4, int32_t);
    }
  }
  switch (nt) {
    case 1: return CM_F(1, int64_t);
    case 2: return CM_F(2, int64_t);
    case 3: return CM_F(3, int64_t);
    default: return CM_F(4, int64_t);
  }
#undef CM_F
#undef CM_F1
}

__global__ void init_keys_kernel(int64_t* best_key, int64_t* best_batch_key, int n_budget) {
  for (int b = threadIdx.x; b < n_budget; b += blockDim.x) {
    best_key[b] = INT64_MAX;
    if (best_batch_key) best_batch_key[b] = INT64_MAX;
  }
}
// CM_EVAL_INIT_KEYS on the launch paths that do not initialise the keys in-kernel
cudaError_t init_keys(const cm_eval_args* a, cudaStream_t st) {
  if (!(a->flags & CM_EVAL_INIT_KEYS) || a->n_budget <= 0) return cudaSuccess;
  init_keys_kernel<<<1, 256, 0, st>>>(a->best_key, a->best_batch_key, a->n_budget);
  ++g_launches;
  return cudaGetLastError();
}

cm_status launch_v2(cm_graph* g, const cm_eval_args* a, cudaStream_t st, int32_t idx_bits) {
  const int n = g->n;
  const int G = (n + 31) / 32;
  const bool m32 = g->scan32;                                       // int32 masses in the blocks
  const int cs = cm2::cand_words(n, m32);
  void* ws = a->workspace ? a->workspace : g->d_ws;
  const int64_t ws_bytes = a->workspace ? a->workspace_bytes : g->ws_bytes;
  if (a->workspace && (reinterpret_cast<uintptr_t>(a->workspace) & 15))
    return fail(CM_EINVAL, "workspace not 16-byte aligned");
  int64_t cap = ws_bytes / 2 / cand_bytes(n, m32);                       // candidates per chunk buffer
  cap &= ~int64_t(31);
  if (cap < std::max<int64_t>(32, a->n_theta)) return fail(CM_EINVAL, "workspace too small");
  const int64_t chunk_s = std::min<int64_t>(cap / a->n_theta, 1 << 20);   // S* per chunk

  // Scan kernel variant: A' in Tensor Memory (+ shared spill) with 8 warps per SM when that
  // fits, else all in shared memory with as many warps as fit.
  const size_t fixed = (size_t)g->blob2_bytes;
  const bool tm = tmem_enabled() && fixed + 8 * scan_warp_bytes(g->n_slot, g->scan32, true) + 1024 <= (size_t)g->smem_optin;
  const size_t wb = scan_warp_bytes(g->n_slot, g->scan32, tm);
  if (fixed + wb > (size_t)g->smem_optin) return fail(CM_ERANGE, "scan kernel: shared memory exceeded");
  const int wpc = tm ? 8 : (int)std::min<size_t>(8, ((size_t)g->smem_optin - fixed) / wb);
  const size_t smem2 = fixed + wb * wpc;
  const void* scan_fn = g->scan32
      ? (tm ? reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, true>) : reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, false>))
      : (tm ? reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, true>) : reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, false>));

  DevAttrs& da = g_attrs[g->device];
  cudaError_t e;
  {
    std::lock_guard<std::mutex> lock(attr_mu);
    if (smem2 > da.scan_smem) {
      for (const void* fn : {reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, false>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, false>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, true>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, true>)}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem2, 48 * 1024));
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(scan_kernel)");
      }
      da.scan_smem = smem2;
    }
  }
  int occ1 = 0, occ2 = 0;
  const int nib_staged = g->d_nib32 ? g->nib_entries : 0;
  const bool bulk = a->layout == CM_LAYOUT_TRI4;                    // K1 stage form: tri4's 5 KB stages
  const int lay = a->layout;                                        // K1 load path (round_fn / fused_fn)
  auto smem1_for = [&](int nt) { return cm2::k1_smem_bytes(nt, nib_staged, bulk); };
  {
    // scan_kernel wants the maximum shared-memory carve-out (its A' arrays are ~210 KB per SM).
    std::lock_guard<std::mutex> lock(attr_mu);
    if (!da.carve) {
      for (int nt = 1; nt <= 4; ++nt)
        for (int lay = 0; lay < 3; ++lay)
          for (int rd = 0; rd < 2; ++rd) {
            const void* fn = round_fn(nt, lay, rd != 0);
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max(cm2::k1_smem_bytes(1, 128 * 32, true), cm2::k1_smem_bytes(4, 128 * 32, true)));
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(round_tma_kernel)");
            e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return cuda_fail(e, "carveout(round_tma_kernel)");
          }
      for (const void* fn : {reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, false>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, false>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int32_t, true>),
                             reinterpret_cast<const void*>(cm2::scan_kernel<int64_t, true>)}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return cuda_fail(e, "carveout(scan_kernel)");
      }
      da.carve = true;
    }
  }
  const bool use_tma = a->layout == CM_LAYOUT_DENSE;
  CUtensorMap tmap;
  cm2::DiagMaps dmaps;
  std::memset(&tmap, 0, sizeof(tmap));
  std::memset(&dmaps, 0, sizeof(dmaps));
  if (use_tma) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(CM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {(cuuint64_t)a->ld, (cuuint64_t)n, (cuuint64_t)a->n_sstar};
    const cuuint64_t strides[2] = {(cuuint64_t)a->ld * 4, (cuuint64_t)a->sstar_stride * 4};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto mk = [&](CUtensorMap* m, CUtensorMapL2promotion pr) {
      return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a->sstar), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    // off-diagonal blocks: 256-byte promotion (CM_L2PROMO); diagonal blocks: none (the rows end there)
    if (mk(&tmap, l2_promotion()) != CUDA_SUCCESS || mk(&dmaps.diag, CU_TENSOR_MAP_L2_PROMOTION_NONE) != CUDA_SUCCESS)
      return fail(CM_EINVAL, "cuTensorMapEncodeTiled failed (alignment / sizes)");
  }
  // tri4: a 2-D map whose rows are the batch's 16-byte units (stride 16 B: overlapping 128-byte
  // rows), read by tile::gather4; every row it can address lies inside the batch buffer.
  int32_t g4 = 0;
  if (bulk && env_flag("CM_GATHER4", 1)) {
    const int64_t floats = (int64_t)a->n_sstar * a->sstar_stride;
    const int64_t rows = floats >= 32 ? (floats - 32) / 4 + 1 : 0;
    EncodeTiledFn enc = encode_tiled();
    if (enc && rows >= 1 && rows < (int64_t(1) << 31) - 64) {
      const cuuint64_t dims[2] = {32, (cuuint64_t)rows};
      const cuuint64_t strides[1] = {16};
      const cuuint32_t box[2] = {32, 1};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a->sstar), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      g4 = r == CUDA_SUCCESS ? 1 : 0;
    }
  }
  const bool rnd = a->rounding == CM_ROUND_RANDOMIZED;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, round_fn(4, lay, rnd), 256, smem1_for(4));
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, scan_fn, 32 * wpc, smem2);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (occ1 < 1 || occ2 < 1) return fail(CM_ERANGE, "kernel does not fit on an SM");

  cm2::RoundParams rp;
  rp.sstar = a->sstar;
  rp.layout = a->layout;
  rp.ld = a->ld;
  rp.stride = a->sstar_stride;
  rp.n = n;
  rp.G = G;
  rp.n_theta = a->n_theta;
  rp.theta = a->theta;
  rp.bw = cm2::block_words(G);
  rp.cs = cs;
  rp.nib = reinterpret_cast<const int64_t*>(g->d_nib);
  rp.nib32 = reinterpret_cast<const int32_t*>(g->d_nib32);
  rp.nib_entries = g->nib_entries;
  rp.brow = cm2::brow_off(n, m32);
  rp.evict_first = env_flag("CM_EVICT_FIRST", 0);   // measured: -2%
  rp.g4 = g4;
  // an S* whose rows' 128-byte windows stay inside the buffer: (s + 1) stride + 32 <= N stride
  rp.g4_end = a->sstar_stride > 0 ? std::max<int64_t>(0, (int64_t)a->n_sstar - (32 + a->sstar_stride - 1) / a->sstar_stride)
                                  : 0;
  rp.rtab = 0;                                        // the fused blocked randomized path sets it
  rp.key0 = (uint32_t)(a->seed & 0xffffffffu);
  rp.key1 = (uint32_t)(a->seed >> 32);
  rp.s0 = (uint32_t)((uint64_t)(a->index_base / a->n_theta) & 0xffffffffu);

  cm2::ScanParams sp;
  sp.blob = reinterpret_cast<const uint4*>(g->d_blob2);
  sp.blob_bytes = g->blob2_bytes;
  sp.n = n;
  sp.o_pred_ptr = 0;
  sp.o_pred_idx = n + 1;
  sp.o_nrec = g->o_nrec;
  sp.o_drec = g->o_drec;
  sp.n_slot = g->n_slot;
  sp.o_qinfo = g->o_qinfo;
  // fused kernel: bit 0 = L2-prefetch a task's blocks when it starts, bit 1 = the next task's
  // (claimed one ahead) when its unit is already filled; the two-kernel scan: nonzero = on
  sp.prefetch = env_flag("CM_PREFETCH", 1);   // measured: 3 -> +8.5 KB/S* DRAM reads, same speed
  sp.cs = cs;
  sp.G = G;
  sp.brow = cm2::brow_off(n, m32);
  sp.mass_bytes = m32 ? 4 : 8;
  sp.r_mask32 = reinterpret_cast<uint32_t*>(a->r_mask);
  sp.s_mask32 = reinterpret_cast<uint32_t*>(a->s_mask);
  sp.warp_bytes = (int32_t)wb;

  cm2::ReduceParams qp;
  qp.G = G;
  qp.index_base = a->index_base;
  qp.ovh = g->ovh;
  qp.mscale = g->mscale;
  qp.idx_bits = idx_bits;
  qp.n_budget = a->n_budget;
  qp.budget = a->budget;
  qp.peak = a->peak;
  qp.cost = a->cost;
  qp.best_key = a->best_key;
  qp.best_batch_key = a->best_batch_key;
  qp.cost_limit = a->cost_limit;
  qp.best_key_mc = a->best_key_mc;
  qp.best_batch_key_mc = a->best_batch_key_mc;

  // ---- fused persistent path (one launch; see cm2::fused_kernel) ----
  if ((g->scan32 || !rnd) && tm && a->n_theta <= 4 && env_flag("CM_FUSED", 1)) {
    const int nt = a->n_theta;
    const size_t wbf = scan_warp_bytes(g->n_slot, g->scan32, true, cm2::fused_tmem_cols(nt, rnd),
                                       cm2::fused_sn_ring(nt, rnd));
    // randomized rounding, blocked layout: the fused kernel's rounding warps keep per-S* Philox
    // tables ([G][8][nt] x 16 bytes per K1 warp) in shared memory (if they do not fit, the
    // smem check below sends the call to the two-kernel pipeline)
    const int rtab = (rnd && a->layout == CM_LAYOUT_BLK) ? G * 8 * nt * 16 : 0;
    const size_t smemf = cm2::fused_k1_bytes(nt, nib_staged, bulk, rtab) + fixed + wbf * cm2::fused_scan_warps(nt, rnd) + 1024;
    const int64_t slot_bytes = 32 * (int64_t)nt * cand_bytes(n, m32);
    const int64_t units = ((int64_t)a->n_sstar + 31) / 32;
    // scan-task tickets: unit-major (default) or windows of CM_WIN units, group-major inside
    // (tuning; measured no gain).  Windows reorder tickets against unit order, so a window's
    // slot predecessors must lie two windows back (W <= R / 2) or a warp blocked on one
    // window task can hold the ticket that would free its slot: clamped below.
    int64_t win = std::max<int64_t>(0, std::min<int64_t>(env_flag("CM_WIN", 0), 256));
    // ring slots: measured (n = 353): 256 -> 13.7, 512 -> 15.8, 768 -> 15.9 M cand/s, 1536 the same;
    // small graphs gain from a deeper ring at the same bytes (VGG16, 44 KB slots: 768 -> 178.6,
    // 4096 -> 210.5 M cand/s): default ~300 MB of slots, 768 .. 4096
    const int64_t ring_auto = std::max<int64_t>(768, std::min<int64_t>(4096, (int64_t(300) << 20) / std::max<int64_t>(1, slot_bytes)));
    int64_t ring_max = std::min<int64_t>(env_flag("CM_RING", (int)ring_auto), 4096);
    int64_t R = std::min<int64_t>(ring_max, units);
    auto ctl_bytes = [](int64_t r) { return (4 * cm2::fused_ctl_words(r) + 255) & ~int64_t(255); };
    // the graph's own workspace: two halves used alternately (CM_EVAL_OVERLAP needs the
    // previous call's ring intact); a caller workspace: one
    const bool own_ws = a->workspace == nullptr;
    const int64_t set_bytes = own_ws ? (ws_bytes / 2) & ~int64_t(255) : ws_bytes;
    const bool overlap = own_ws && (a->flags & CM_EVAL_OVERLAP);
    while (R > 1 && ctl_bytes(R) + R * slot_bytes > set_bytes) --R;
    if (R < units) win = std::min<int64_t>(win, R / 2);             // no slot reuse: any order is safe
    const int64_t total_tasks = win > 0 ? ((units + win - 1) / win) * win * (int64_t)G * nt
                                        : (units - 1) * (int64_t)G * nt +
                                              (int64_t)G * ((((int64_t)a->n_sstar - 32 * (units - 1)) * nt + 31) / 32);
    if (smemf <= (size_t)g->smem_optin && R >= 1 && ctl_bytes(R) + R * slot_bytes <= set_bytes &&
        total_tasks < (int64_t(1) << 31)) {
      const void* fn = fused_fn(nt, lay, rnd, g->scan32);
      {
        std::lock_guard<std::mutex> lock(attr_mu);
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemf);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fused_kernel)");
      }
      const int threads = 32 * cm2::fused_warps(nt, rnd);
      int occf = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, fn, threads, smemf);
      if (e != cudaSuccess) return cuda_fail(e, "occupancy(fused_kernel)");
      if (occf >= 1) {
        // one CTA per SM (all 512 TMEM columns), or as many as fit when a CTA takes fewer columns
        int per_sm = cm2::kFusedTmem == 512 ? 1 : std::min(occf, 512 / cm2::kFusedTmem);
        if (cm2::kFusedTmem < 512) per_sm = std::max(1, std::min(512 / cm2::kFusedTmem, env_flag("CM_FUSED_PER_SM", per_sm)));
        const int grid = g->sm_count * per_sm;
        if (env_flag("CM_DEBUG", 0)) {
          cudaFuncAttributes fa = {};
          cudaFuncGetAttributes(&fa, fn);
          std::fprintf(stderr, "cm: fused_kernel smem %zu (static %zu) threads %d regs %d occupancy %d grid %d ring %lld\n",
                       smemf, fa.sharedSizeBytes, threads, fa.numRegs, occf, grid, (long long)R);
        }
        cm2::FusedParams fp;
        rp.s_begin = 0;
        rp.s_count = a->n_sstar;
        rp.th0 = 0;
        rp.nt = nt;
        rp.sn = nullptr;
        fp.rp = rp;
        fp.rp.rtab = rtab;
        fp.sp = sp;
        fp.sp.warp_bytes = (int32_t)wbf;
        fp.qp = qp;
        fp.init_keys = (a->flags & CM_EVAL_INIT_KEYS) && a->n_budget > 0;
        fp.slot_words = slot_bytes / 4;
        fp.n_slots = (int32_t)R;
        fp.n_sstar = a->n_sstar;
        fp.n_theta = nt;
        fp.n_units = (int32_t)units;
        fp.tpu = G * nt;
        fp.total_tasks = total_tasks;
        fp.win_units = (int32_t)win;
        fp.trace = nullptr;
        if (env_flag("CM_TRACE", 0) == 2 && grid <= kTraceCtas) {
          const size_t region = 4 * (size_t)kTraceCtas;
          if (!g_cta_trace && cudaMalloc(&g_cta_trace, sizeof(uint64_t) * region * kTraceCalls) != cudaSuccess) {
            g_cta_trace = nullptr;
            cudaGetLastError();
          }
          if (g_cta_trace) {
            const int64_t r = g_cta_trace_calls % kTraceCalls;
            if (r == 0) cudaMemsetAsync(g_cta_trace, 0, sizeof(uint64_t) * region * kTraceCalls, st);
            g_cta_trace_n = 4 * grid;
            fp.trace = g_cta_trace + r * region;
            ++g_cta_trace_calls;
          }
        }
        {  // S* per producer ticket: 8 at n = 89, 2 at n = 213 .. ~420, 1 above
          const int gr = n >= 2 ? (n - 2) / 32 + 1 : 1;
          const int blocks = gr * (gr + 1) / 2;
          int c = 1;
          while (c < 8 && 2 * c * blocks <= 64) c *= 2;
          // measured with overlapped calls: n = 353 (66 blocks) 19.55 vs 19.0-19.35 M cand/s at
          // 2 S* per ticket, n = 401 (91) 14.72 vs 14.66; n = 563 (171) better at 1
          if (c == 1 && 2 * blocks <= 190) c = 2;
          fp.claim = env_flag("CM_CLAIM", c);
          if (fp.claim < 1 || fp.claim > 32 || (fp.claim & (fp.claim - 1))) fp.claim = c;
          // scan tasks per consumer ticket (tuning; 1: measured a whole VGG16 unit per ticket
          // at 121 vs 153 M cand/s -- the unit's three tasks then run one after another)
          fp.task_claim = env_flag("CM_TASK_CLAIM", 1);
          if (fp.task_claim < 1 || fp.tpu % fp.task_claim || win > 0) fp.task_claim = 1;
        }
        std::lock_guard<std::mutex> lock(g->mu);
        fp.seq_word = g->d_seq;
        fp.seq = ++g->seq;
        const int half = own_ws ? g->ws_half : 0;
        unsigned char* set_base = reinterpret_cast<unsigned char*>(ws) + half * set_bytes;
        uint32_t* ctl = reinterpret_cast<uint32_t*>(set_base);
        fp.ctl = ctl;
        fp.ring = reinterpret_cast<uint32_t*>(set_base + ctl_bytes(R));
        // (a call with a smaller ring left ring data where this call's control words lie)
        if (!overlap || g->ctl_clean[half] < cm2::fused_ctl_words(R)) {
          e = cudaMemsetAsync(ctl, 0, 4 * (size_t)cm2::fused_ctl_words(R), st);
          if (e != cudaSuccess) return cuda_fail(e, "memset(fused control words)");
        }
        void* args[] = {&fp, &tmap, &dmaps};
        const bool tr = trace_enabled();
        g_trace.used = 0;
        if (tr) cudaEventRecord(trace_event(0), st);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = smemf;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = overlap ? 1 : 0;
        e = cudaLaunchKernelExC(&cfg, fn, args);
        if (e != cudaSuccess) return cuda_fail(e, "launch fused_kernel");
        if (own_ws) {
          g->ctl_clean[half] = cm2::fused_ctl_words(R);   // cleared by the kernel's last CTA
          g->ws_half ^= 1;
        }
        if (tr) {                                    // one "chunk": K1 and K2 share the launch
          cudaEventRecord(trace_event(1), st);
          cudaEventRecord(trace_event(2), st);
          cudaEventRecord(trace_event(3), st);
          g_trace.used = 4;
        }
        g_launches = 1;
        return CM_OK;
      }
    }
  }

  unsigned char* base = reinterpret_cast<unsigned char*>(ws);
  const int64_t half = cap * cand_bytes(n, m32);
  std::lock_guard<std::mutex> lock(g->mu);
  const uint32_t seq = ++g->seq;
  if (!a->workspace) g->ctl_clean[0] = g->ctl_clean[1] = 0;         // chunk buffers overwrite them
  const bool tr = trace_enabled();
  g_trace.used = 0;
  g_launches = 0;
  e = init_keys(a, st);
  if (e != cudaSuccess) return cuda_fail(e, "init keys");
  e = cudaEventRecord(g->ev_start, st);                       // inputs written on `st` before the call
  if (e == cudaSuccess) e = cudaStreamWaitEvent(g->st_round, g->ev_start, 0);
  int c = 0;
  for (int64_t s0 = 0; s0 < a->n_sstar && e == cudaSuccess; s0 += chunk_s, ++c) {
    const int b = c & 1;
    const int sc = (int)std::min<int64_t>(chunk_s, a->n_sstar - s0);
    const int64_t nc = (int64_t)sc * a->n_theta;
    uint32_t* blk = reinterpret_cast<uint32_t*>(base + b * half);
    int64_t* part = reinterpret_cast<int64_t*>(base + b * half + 4 * cap * (int64_t)cs);
    if (g->used[b]) e = cudaStreamWaitEvent(g->st_round, g->ev_scan[b], 0);   // buffer b drained
    if (e != cudaSuccess) break;
    rp.s_begin = s0;
    rp.s_count = sc;
    rp.sn = blk;
    const int64_t warps1 = sc;                                   // a K1 task is one S*
    // one K1 CTA per SM (<= 32k registers): it co-resides with the scan CTA (TMEM variant:
    // 8 warps, 32k registers), so chunk c+1 streams while c scans.
    if (tr) cudaEventRecord(trace_event(4 * c + 0), g->st_round);
#ifdef CM_EXP_NOK1
    for (int th0 = 0; th0 < 0; th0 += 4) {                    // timing experiment: no rounding
#else
    for (int th0 = 0; th0 < a->n_theta; th0 += 4) {          // <= 4 thresholds per S* pass
#endif
      rp.th0 = th0;
      rp.nt = std::min(4, a->n_theta - th0);
      const int wpb = cm2::k1_warps(rp.nt);
      const int grid1 = (int)std::max<int64_t>(1, std::min<int64_t>((warps1 + wpb - 1) / wpb, (int64_t)g->sm_count));
      const int thr1 = 32 * wpb;
      const size_t sm1 = smem1_for(rp.nt);
      void* k1args[] = {&rp, &tmap, &dmaps};
      e = cudaLaunchKernel(round_fn(rp.nt, lay, rnd), dim3((unsigned)grid1), dim3((unsigned)thr1), k1args, sm1, g->st_round);
      if (e != cudaSuccess) break;
    }
    if (e != cudaSuccess) break;
    if (tr) cudaEventRecord(trace_event(4 * c + 1), g->st_round);
    e = cudaEventRecord(g->ev_round[b], g->st_round);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->ev_round[b], 0);
    if (e != cudaSuccess) break;
    if (tr) cudaEventRecord(trace_event(4 * c + 2), st);
#ifdef CM_EXP_NOK2
    e = cudaEventRecord(g->ev_scan[b], st);
    g->used[b] = true;
    continue;
#endif
    sp.ws = blk;
    sp.n_cand = nc;
    sp.n_batch = (int)((nc + 31) / 32);
    sp.part = part;
    sp.out_base = s0 * a->n_theta;
    const int64_t tasks = (int64_t)G * sp.n_batch;
    // TM: one CTA per SM (each allocates all 512 TMEM columns)
    const int64_t max_ctas = tm ? (int64_t)g->sm_count : (int64_t)occ2 * g->sm_count;
    const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>((tasks + wpc - 1) / wpc, max_ctas));
    if (g->scan32) {
      if (tm) cm2::scan_kernel<int32_t, true><<<grid2, 32 * wpc, smem2, st>>>(sp);
      else cm2::scan_kernel<int32_t, false><<<grid2, 32 * wpc, smem2, st>>>(sp);
    } else {
      if (tm) cm2::scan_kernel<int64_t, true><<<grid2, 32 * wpc, smem2, st>>>(sp);
      else cm2::scan_kernel<int64_t, false><<<grid2, 32 * wpc, smem2, st>>>(sp);
    }
    qp.part = part;
    qp.n_cand = nc;
    qp.out_base = sp.out_base;
    cm2::reduce_kernel<0><<<(int)((nc + 255) / 256), 256, 0, st>>>(qp);
    g_launches += (a->n_theta + 3) / 4 + 2;
    if (tr) {
      cudaEventRecord(trace_event(4 * c + 3), st);
      g_trace.used = 4 * (c + 1);
    }
    e = cudaEventRecord(g->ev_scan[b], st);
    g->used[b] = true;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = signal_call(g, seq, st);
  if (e != cudaSuccess) return cuda_fail(e, "launch v2 kernels");
  return CM_OK;
}

}  // namespace

// host-side NVTX range over one C-ABI call (no-op unless a profiler injects NVTX)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

extern "C" {

const char* cm_status_string(cm_status s) {
  switch (s) {
    case CM_OK: return "CM_OK";
    case CM_EINVAL: return "CM_EINVAL: invalid argument";
    case CM_ETOPO: return "CM_ETOPO: edge (i,j) with i >= j (nodes must be topologically numbered)";
    case CM_EDUP: return "CM_EDUP: duplicate edge";
    case CM_ERANGE: return "CM_ERANGE: size or int64 bound out of range";
    case CM_ECUDA: return "CM_ECUDA: CUDA error";
    case CM_ENOMEM: return "CM_ENOMEM: device allocation failed";
  }
  return "unknown cm_status";
}

const char* cm_last_error(void) { return g_err.c_str(); }

void cm_decode_batch_key(int64_t key, int32_t idx_bits, int64_t* b_max, int64_t* idx) {
  if (key == CM_KEY_NONE || key < 0) {
    if (b_max) *b_max = 0;
    if (idx) *idx = -1;
    return;
  }
  if (b_max) *b_max = ((int64_t(1) << 31) - 1) - (key >> idx_bits);
  if (idx) *idx = idx_bits ? (key & ((int64_t(1) << idx_bits) - 1)) : 0;
}

int32_t cm_key_idx_bits(int64_t total_candidates) {
  if (total_candidates <= 1) return 0;
  uint64_t v = (uint64_t)(total_candidates - 1);
  int32_t b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

void cm_decode_key(int64_t key, int32_t idx_bits, int64_t* cost, int64_t* idx) {
  if (key == CM_KEY_NONE || key < 0) {
    if (cost) *cost = -1;
    if (idx) *idx = -1;
    return;
  }
  if (cost) *cost = key >> idx_bits;
  if (idx) *idx = idx_bits ? (key & ((int64_t(1) << idx_bits) - 1)) : 0;
}

cm_status cm_graph_create(int32_t n, const int32_t* pred_ptr, const int32_t* pred_idx,
                          const int64_t* cost, const int64_t* mem, int64_t mem_overhead,
                          cm_graph** out) {
  if (!out) return fail(CM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!pred_ptr || !cost || !mem) return fail(CM_EINVAL, "NULL pred_ptr/cost/mem");
  if (n < 1) return fail(CM_EINVAL, "n < 1");
  if (n > CM_NMAX) return fail(CM_ERANGE, "n > CM_NMAX");
  if (pred_ptr[0] != 0) return fail(CM_EINVAL, "pred_ptr[0] != 0");
  for (int k = 0; k < n; ++k)
    if (pred_ptr[k + 1] < pred_ptr[k]) return fail(CM_EINVAL, "pred_ptr not non-decreasing");
  const int32_t E = pred_ptr[n];
  if (E > CM_EMAX) return fail(CM_ERANGE, "|E| > CM_EMAX");
  if (E > 0 && !pred_idx) return fail(CM_EINVAL, "NULL pred_idx");
  if (mem_overhead < 0) return fail(CM_EINVAL, "mem_overhead < 0");
  for (int k = 0; k < n; ++k) {
    if (cost[k] < 0 || mem[k] < 0) return fail(CM_EINVAL, "negative cost or mem");
    std::set<int32_t> seen;
    for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
      const int32_t i = pred_idx[e];
      if (i < 0) return fail(CM_EINVAL, "negative predecessor index");
      if (i >= k) return fail(CM_ETOPO, "edge (" + std::to_string(i) + "," + std::to_string(k) + ") has i >= j");
      if (!seen.insert(i).second)
        return fail(CM_EDUP, "duplicate edge (" + std::to_string(i) + "," + std::to_string(k) + ")");
    }
  }
  // int64 bounds: every U_{t,k} <= ovh + sum M; every cost <= sum_i (n-i) C_i.
  const int64_t LIM = int64_t(1) << 62;
  int64_t msum = mem_overhead, cbound = 0;
  for (int i = 0; i < n; ++i) {
    if (mem[i] > LIM - msum) return fail(CM_ERANGE, "ovh + sum M overflows 2^62");
    msum += mem[i];
    if (cost[i] > 0 && (int64_t)(n - i) > (LIM - cbound) / cost[i])
      return fail(CM_ERANGE, "sum (n-i) C_i overflows 2^62");
    cbound += (int64_t)(n - i) * cost[i];
  }

  // successor CSR, each list ascending; later[e] = first position in succ(i) after k for
  // the predecessor edge e = (i -> k).
  std::vector<std::vector<int32_t>> users(n);
  for (int k = 0; k < n; ++k)
    for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) users[pred_idx[e]].push_back(k);
  std::vector<int32_t> succ_ptr(n + 1, 0), succ_idx;
  succ_idx.reserve(E);
  for (int i = 0; i < n; ++i) {
    std::sort(users[i].begin(), users[i].end());
    succ_ptr[i + 1] = succ_ptr[i] + (int32_t)users[i].size();
    for (int32_t j : users[i]) succ_idx.push_back(j);
  }
  std::vector<int32_t> pidx(E), later(E);
  for (int k = 0; k < n; ++k) {
    std::vector<int32_t> ps(pred_idx + pred_ptr[k], pred_idx + pred_ptr[k + 1]);
    std::sort(ps.begin(), ps.end());
    for (size_t q = 0; q < ps.size(); ++q) {
      const int32_t i = ps[q];
      pidx[pred_ptr[k] + q] = i;
      const auto it = std::lower_bound(succ_idx.begin() + succ_ptr[i], succ_idx.begin() + succ_ptr[i + 1], k);
      later[pred_ptr[k] + q] = (int32_t)(it - succ_idx.begin()) + 1;
    }
  }

  // blob: M[n] int64, C[n] int64, then int32 arrays
  cm_graph* g = new cm_graph();
  g->n = n;
  g->E = E;
  g->ovh = mem_overhead;
  g->cost_bound = cbound;
  g->o_pred_ptr = 0;
  g->o_pred_idx = g->o_pred_ptr + (n + 1);
  g->o_later = g->o_pred_idx + E;
  g->o_succ_ptr = g->o_later + E;
  g->o_succ_idx = g->o_succ_ptr + (n + 1);
  const int32_t n_i32 = g->o_succ_idx + E;
  size_t bytes = 16 * (size_t)n + 4 * (size_t)n_i32;
  bytes = (bytes + 15) & ~size_t(15);
  g->blob_bytes = (int32_t)bytes;
  std::vector<unsigned char> blob(bytes, 0);
  std::memcpy(blob.data(), mem, 8 * (size_t)n);
  std::memcpy(blob.data() + 8 * (size_t)n, cost, 8 * (size_t)n);
  int32_t* gi = reinterpret_cast<int32_t*>(blob.data() + 16 * (size_t)n);
  std::memcpy(gi + g->o_pred_ptr, pred_ptr, 4 * (size_t)(n + 1));
  if (E) {
    std::memcpy(gi + g->o_pred_idx, pidx.data(), 4 * (size_t)E);
    std::memcpy(gi + g->o_later, later.data(), 4 * (size_t)E);
    std::memcpy(gi + g->o_succ_idx, succ_idx.data(), 4 * (size_t)E);
  }
  std::memcpy(gi + g->o_succ_ptr, succ_ptr.data(), 4 * (size_t)(n + 1));

  cudaError_t e = cudaGetDevice(&g->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, g->device);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&g->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "cm_graph_create: device query");
  }
  e = cudaMalloc(&g->d_blob, bytes);
  if (e != cudaSuccess) {
    delete g;
    cudaGetLastError();
    return fail(CM_ENOMEM, std::string("cm_graph_create: cudaMalloc: ") + cudaGetErrorString(e));
  }
  e = cudaMemcpy(g->d_blob, blob.data(), bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(g->d_blob);
    delete g;
    return cuda_fail(e, "cm_graph_create: cudaMemcpy");
  }
  // v2 blob: M[n]/mscale, C[n] int64, pred_ptr[n+1], pred_idx[E]
  {
    int64_t gd = 0;
    for (int i = 0; i < n; ++i) {
      int64_t a = mem[i], b = gd;
      while (b) { const int64_t t = a % b; a = b; b = t; }
      gd = a;
    }
    g->mscale = gd > 0 ? gd : 1;
    int64_t tot = 0;
    for (int i = 0; i < n; ++i) tot += mem[i] / g->mscale;
    g->scan32 = tot < (int64_t(1) << 31);             // E <= sum M (cm_v2.cuh events)
    if (!g->scan32) g->mscale = 1;
  }
  // + node records {(int32) M_k, e0, ndf | adj << 16, slot_k or -1} and far-dependency
  // records {slot_i | i << 16, (int32) M_i}.  adj: k-1 is a dependency of k (its A' term
  // rides in a register); slot: k has a user other than k+1, so its A' needs storage.
  std::vector<int32_t> slot(n, -1);
  for (int i = 0; i < n; ++i)
    for (int32_t j : users[i])
      if (j != i + 1) { slot[i] = g->n_slot++; break; }
  size_t base2 = (16 * (size_t)n + 4 * (size_t)(n + 1 + E) + 15) & ~size_t(15);
  // node records start one record in: record -1 is a sentinel {0, 0, 0, -1} (no slot), so the
  // walk reads the record of node k-1 without a k > 0 test
  g->o_nrec = (int32_t)(base2 + 16);
  g->o_drec = (int32_t)(base2 + 16 * (size_t)(n + 1));
  g->o_qinfo = (int32_t)(base2 + 16 * (size_t)(n + 1) + 8 * (size_t)E);
  const int nquad = (n + 3) / 4;
  size_t bytes2 = (base2 + 16 * (size_t)(n + 1) + 8 * (size_t)E + 4 * (size_t)nquad + 15) & ~size_t(15);
  g->blob2_bytes = (int32_t)bytes2;
  std::vector<unsigned char> blob2(bytes2, 0);
  std::memcpy(blob2.data(), blob.data(), 16 * (size_t)n + 4 * (size_t)(n + 1 + E));
  for (int i = 0; i < n; ++i) reinterpret_cast<int64_t*>(blob2.data())[i] = mem[i] / g->mscale;
  {
    int32_t* nr = reinterpret_cast<int32_t*>(blob2.data() + g->o_nrec);
    nr[-1] = -1;                                        // sentinel record -1: {0, 0, 0, -1}
    int32_t* dr = reinterpret_cast<int32_t*>(blob2.data() + g->o_drec);
    int32_t ef = 0;
    for (int k = 0; k < n; ++k) {
      int32_t ndf = 0, adj = 0;
      nr[4 * k + 0] = (int32_t)(mem[k] / g->mscale);      // meaningful when scan32
      nr[4 * k + 1] = ef;
      for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
        const int32_t i = pidx[e];
        if (i == k - 1) { adj = 1; continue; }
        dr[2 * ef + 0] = slot[i] | (i << 16);
        dr[2 * ef + 1] = (int32_t)(mem[i] / g->mscale);
        ++ef;
        ++ndf;
      }
      nr[4 * k + 2] = ndf | (adj << 16);
      nr[4 * k + 3] = slot[k];
    }
    int32_t* qi = reinterpret_cast<int32_t*>(blob2.data() + g->o_qinfo);
    for (int q = 0; q < nquad; ++q) {
      int32_t first = -1, msk = 0;
      for (int j = 0; j < 4 && 4 * q + j < n; ++j)
        if (slot[4 * q + j] >= 0) {
          if (first < 0) first = slot[4 * q + j];
          msk |= 1 << j;
        }
      qi[q] = (first < 0 ? 0 : first) | (msk << 16);
    }
  }
  e = cudaMalloc(&g->d_blob2, bytes2);
  if (e == cudaSuccess) e = cudaMemcpy(g->d_blob2, blob2.data(), bytes2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    g->nib_entries = 128 * ((n + 31) / 32);            // 8 nibbles per 32-node block, every block
    std::vector<int64_t> nib(g->nib_entries, 0);
    for (int q = 0; q < g->nib_entries / 16; ++q)
      for (int v = 0; v < 16; ++v)
        for (int j = 0; j < 4; ++j)
          if ((v >> j) & 1 && 4 * q + j < n) nib[16 * q + v] += mem[4 * q + j] / g->mscale;
    e = cudaMalloc(&g->d_nib, 8 * (size_t)g->nib_entries);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_nib, nib.data(), 8 * (size_t)g->nib_entries, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && g->scan32) {
      std::vector<int32_t> nib32(g->nib_entries);
      for (int i = 0; i < g->nib_entries; ++i) nib32[i] = (int32_t)nib[i];
      e = cudaMalloc(&g->d_nib32, 4 * (size_t)g->nib_entries);
      if (e == cudaSuccess)
        e = cudaMemcpy(g->d_nib32, nib32.data(), 4 * (size_t)g->nib_entries, cudaMemcpyHostToDevice);
    }
  }
  if (e == cudaSuccess) {
    const int64_t per = cand_bytes(n, g->scan32);
    int64_t want = kDefaultWsBytes;
    if (const char* env = std::getenv("CM_WS_MB")) want = std::max<int64_t>(1, std::atoll(env)) << 20;   // tuning
    g->ws_bytes = std::max<int64_t>(per * 1024, (want / (64 * per)) * 64 * per);
    e = cudaMalloc(&g->d_ws, g->ws_bytes);
    // zeroed once: a candidate block's words that no kernel writes (the masses of rows >= n and
    // of row 0, read 16 bytes at a time and discarded) are then defined memory (initcheck-clean)
    if (e == cudaSuccess) e = cudaMemset(g->d_ws, 0, g->ws_bytes);
  }
  if (e == cudaSuccess) e = cudaMalloc(&g->d_seq, 256);
  if (e == cudaSuccess) e = cudaMemset(g->d_seq, 0, 256);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->st_round, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_start, cudaEventDisableTiming);
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaEventCreateWithFlags(&g->ev_round[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_scan[b], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (g->d_blob2) cudaFree(g->d_blob2);
    if (g->d_ws) cudaFree(g->d_ws);
    if (g->d_nib) cudaFree(g->d_nib);
    if (g->d_nib32) cudaFree(g->d_nib32);
    if (g->d_seq) cudaFree(g->d_seq);
    cudaFree(g->d_blob);
    delete g;
    return fail(CM_ENOMEM, std::string("cm_graph_create: ") + cudaGetErrorString(e));
  }
  *out = g;
  return CM_OK;
}

void cm_graph_destroy(cm_graph* g) {
  if (!g) return;
  if (g->st_round) cudaStreamSynchronize(g->st_round);
  for (int b = 0; b < 2; ++b) {
    if (g->ev_round[b]) cudaEventDestroy(g->ev_round[b]);
    if (g->ev_scan[b]) cudaEventDestroy(g->ev_scan[b]);
  }
  if (g->ev_start) cudaEventDestroy(g->ev_start);
  if (g->st_round) cudaStreamDestroy(g->st_round);
  if (g->d_blob) cudaFree(g->d_blob);
  if (g->d_blob2) cudaFree(g->d_blob2);
  if (g->d_ws) cudaFree(g->d_ws);
  if (g->d_nib) cudaFree(g->d_nib);
  if (g->d_nib32) cudaFree(g->d_nib32);
  if (g->d_seq) cudaFree(g->d_seq);
  delete g;
}

// Debug: after a CM_TRACE=1 call has completed, writes per-chunk (k1_begin, k1_end,
// k2_begin, k2_end) in ms relative to the first k1_begin; returns the number of values.
int32_t cm_debug_trace(float* out, int32_t max_values) {
  int32_t m = 0;
  if (g_trace.used == 0) return 0;
  cudaEventSynchronize(g_trace.ev[g_trace.used - 1]);
  for (int i = 0; i < g_trace.used && m < max_values; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_trace.ev[0], g_trace.ev[i]);
    out[m++] = ms;
  }
  return m;
}

int32_t cm_debug_last_launches(void) { return g_launches; }

int32_t cm_debug_cta_trace_at(int32_t back, uint64_t* out, int32_t max_values) {
  if (!g_cta_trace || !out || back < 0 || back >= kTraceCalls || back >= g_cta_trace_calls) return 0;
  const int64_t r = (g_cta_trace_calls - 1 - back) % kTraceCalls;
  const int32_t m = std::min(max_values, g_cta_trace_n);
  if (cudaMemcpy(out, g_cta_trace + r * 4 * (int64_t)kTraceCtas, sizeof(uint64_t) * (size_t)m,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return m;
}

int32_t cm_debug_cta_trace(uint64_t* out, int32_t max_values) { return cm_debug_cta_trace_at(0, out, max_values); }

uint32_t cm_last_call_seq(const cm_graph* g) {
  if (!g) return 0;
  std::lock_guard<std::mutex> lock(const_cast<cm_graph*>(g)->mu);
  return g->seq;
}

cm_status cm_stream_wait_call(const cm_graph* g, uint32_t seq, cm_stream stream) {
  if (!g) return fail(CM_EINVAL, "NULL graph");
  StreamValue32Fn fn = wait_value32();
  if (!fn) return fail(CM_ECUDA, "cuStreamWaitValue32 unavailable");
  const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(g->d_seq), seq,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(CM_ECUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
  return CM_OK;
}

cm_status cm_policy_sstar(const cm_graph* g, int32_t L, int32_t n_sets, const uint8_t* k_sets, float* sstar,
                          int64_t ld, cm_stream stream) {
  if (!g || L < 1 || L > g->n || n_sets < 0 || n_sets > 65535 || ld < g->n || (n_sets > 0 && (!k_sets || !sstar)))
    return fail(CM_EINVAL, "cm_policy_sstar: bad arguments");
  if (n_sets == 0) return CM_OK;
  const int32_t* gi = reinterpret_cast<const int32_t*>(reinterpret_cast<const unsigned char*>(g->d_blob) + 16 * (size_t)g->n);
  cmp::policy_sstar_kernel<<<dim3((unsigned)g->n, (unsigned)n_sets), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      gi + g->o_succ_ptr, gi + g->o_succ_idx, g->n, L, k_sets, sstar, ld);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "launch policy_sstar_kernel");
  return CM_OK;
}

int64_t cm_workspace_bytes(const cm_graph* g, int64_t chunk_candidates) {
  if (!g || chunk_candidates < 1) return -1;
  return 2 * cand_bytes(g->n, g->scan32) * ((chunk_candidates + 31) & ~int64_t(31));   // two buffers
}

int64_t cm_sstar_floats(int32_t n, int32_t layout, int64_t ld) {
  if (n < 1) return -1;
  switch (layout) {
    case CM_LAYOUT_DENSE: return ld >= n ? (int64_t)n * ld : -1;
    case CM_LAYOUT_TRI4: {
      const int64_t q = n >> 2, m = n & 3;
      return 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
    }
    case CM_LAYOUT_BLK: return cm2::blk_size(n);
  }
  return -1;
}

int32_t cm_graph_n(const cm_graph* g) { return g ? g->n : -1; }
int64_t cm_graph_cost_bound(const cm_graph* g) { return g ? g->cost_bound : -1; }

cm_status cm_round_and_evaluate(const cm_graph* g, const cm_eval_args* a, cm_stream stream) {
  const NvtxRange nvtx("cm_round_and_evaluate");
  if (!g || !a) return fail(CM_EINVAL, "NULL graph or args");
  const int n = g->n;
  if (a->n_sstar < 0 || a->n_theta < 1 || a->n_budget < 0) return fail(CM_EINVAL, "bad counts");
  if (a->layout != CM_LAYOUT_DENSE && a->layout != CM_LAYOUT_TRI4 && a->layout != CM_LAYOUT_BLK)
    return fail(CM_EINVAL, "bad layout");
  if (a->rounding != CM_ROUND_THRESHOLD && a->rounding != CM_ROUND_RANDOMIZED) return fail(CM_EINVAL, "bad rounding");
  if (a->rounding == CM_ROUND_RANDOMIZED && a->index_base % a->n_theta != 0)
    return fail(CM_EINVAL, "randomized rounding: index_base must be a multiple of n_theta (samples)");
  if (a->layout == CM_LAYOUT_DENSE && (a->ld < n || (a->ld & 3)))
    return fail(CM_EINVAL, "ld must be >= n and a multiple of 4");
  const int64_t min_stride = cm_sstar_floats(n, a->layout, a->ld);
  if (a->n_sstar > 0) {
    if (a->sstar_stride < min_stride || (a->sstar_stride & 3))
      return fail(CM_EINVAL, "sstar_stride too small or not a multiple of 4");
    // n = 1 has no strict-lower entries: nothing is read, sstar may be NULL (an empty tri4 batch)
    if (min_stride > 0 && (!a->sstar || (reinterpret_cast<uintptr_t>(a->sstar) & 15)))
      return fail(CM_EINVAL, "sstar NULL or not 16-byte aligned");
    if (!a->sstar && n > 1) return fail(CM_EINVAL, "sstar NULL");
    if ((!a->theta && a->rounding == CM_ROUND_THRESHOLD) || !a->peak || !a->cost)
      return fail(CM_EINVAL, "NULL theta/peak/cost");
  }
  if (a->n_budget > 0 && (!a->budget || !a->best_key)) return fail(CM_EINVAL, "NULL budget/best_key");
  if (a->best_key_mc || a->best_batch_key_mc) {
    if (a->flags & CM_EVAL_INIT_KEYS)
      return fail(CM_EINVAL, "multicast keys: CM_EVAL_INIT_KEYS would race other ranks' reductions");
    if ((a->best_key_mc && !a->best_key) || (a->best_batch_key_mc && !a->best_batch_key))
      return fail(CM_EINVAL, "multicast keys need the local (unicast) view too");
    if ((reinterpret_cast<uintptr_t>(a->best_key_mc) | reinterpret_cast<uintptr_t>(a->best_batch_key_mc)) & 7)
      return fail(CM_EINVAL, "multicast keys not 8-byte aligned");
  }
  if (a->best_batch_key && cm_key_idx_bits(a->total_candidates) > 32)
    return fail(CM_ERANGE, "max-batch keys need total_candidates <= 2^32");
  if (a->n_budget > 4096) return fail(CM_ERANGE, "n_budget > 4096");
  const int64_t n_cand = (int64_t)a->n_sstar * a->n_theta;
  if (a->index_base < 0 || a->total_candidates < a->index_base + n_cand)
    return fail(CM_EINVAL, "total_candidates < index_base + n_sstar*n_theta");
  const int32_t idx_bits = cm_key_idx_bits(a->total_candidates);
  if (idx_bits > 62 || (idx_bits > 0 && g->cost_bound >= (int64_t(1) << (63 - idx_bits))))
    return fail(CM_ERANGE, "cost bound does not fit the packed key; use fewer candidates per key space");
  {
    int cur = -1;
    const cudaError_t ed = cudaGetDevice(&cur);
    if (ed != cudaSuccess) return cuda_fail(ed, "cudaGetDevice");
    if (cur != g->device)
      return fail(CM_EINVAL, "the graph lives on device " + std::to_string(g->device) + ", current device is " +
                                 std::to_string(cur));
    if (g->device >= kMaxDev) return fail(CM_ERANGE, "device ordinal >= 64");
  }
  g_launches = 0;
  if (n_cand == 0) {
    cm_graph* gm = const_cast<cm_graph*>(g);
    std::lock_guard<std::mutex> lock(gm->mu);
    const uint32_t seq = ++gm->seq;
    cudaError_t e0 = init_keys(a, reinterpret_cast<cudaStream_t>(stream));
    if (e0 == cudaSuccess) e0 = signal_call(g, seq, reinterpret_cast<cudaStream_t>(stream));
    return e0 == cudaSuccess ? CM_OK : cuda_fail(e0, "init keys");
  }
  if (kernel_choice() == 2 && (size_t)g->blob2_bytes + scan_warp_bytes(g->n_slot, g->scan32, false) <= (size_t)g->smem_optin) {
    cudaError_t e0 = cudaGetLastError();                 // surface earlier asynchronous faults
    if (e0 != cudaSuccess) return cuda_fail(e0, "earlier asynchronous error");
    return launch_v2(const_cast<cm_graph*>(g), a, reinterpret_cast<cudaStream_t>(stream), idx_bits);
  }
  if (a->rounding != CM_ROUND_THRESHOLD || a->best_batch_key || a->layout == CM_LAYOUT_BLK || a->best_key_mc)
    return fail(CM_ERANGE, "randomized rounding / max-batch / the blocked layout / multicast keys need the "
                           "stage-sliced kernels (graph too large for them)");

  const int G = (n + 31) / 32;
  const int tri_words = 16 * G * (G + 1);
  const int threads = 32 * G;
  const size_t fixed = (size_t)g->blob_bytes + 2 * 8 * (size_t)((a->n_budget + 1) & ~1) + 8 * 96 +
                       4 * (size_t)tri_words;
  const size_t per_theta = 4 * (size_t)tri_words;
  if (fixed + per_theta > (size_t)g->smem_optin)
    return fail(CM_ERANGE, "shared memory: graph + one threshold's bit rows exceed the per-CTA limit");
  int theta_chunk = (int)std::min<size_t>((size_t)a->n_theta, ((size_t)g->smem_optin - fixed) / per_theta);
  theta_chunk = std::max(1, std::min(theta_chunk, 8));
  // prefer a chunk that splits n_theta evenly
  const int n_tchunks = (a->n_theta + theta_chunk - 1) / theta_chunk;
  theta_chunk = (a->n_theta + n_tchunks - 1) / n_tchunks;
  const size_t smem = fixed + per_theta * theta_chunk;

  cudaError_t e = cudaGetLastError();                   // surface earlier asynchronous faults
  if (e != cudaSuccess) return cuda_fail(e, "earlier asynchronous error");
  {
    std::lock_guard<std::mutex> lock(attr_mu);
    DevAttrs& da = g_attrs[g->device];
    if (smem > da.v1_smem) {
      e = cudaFuncSetAttribute(cmk::round_evaluate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(smem, 48 * 1024));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      da.v1_smem = smem;
    }
  }
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cmk::round_evaluate_kernel, threads, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (occ < 1) return fail(CM_ERANGE, "kernel does not fit on an SM");
  const int64_t items = (int64_t)a->n_sstar * n_tchunks;
  const int grid = (int)std::min<int64_t>(items, (int64_t)occ * g->sm_count);

  cmk::Params p;
  p.blob = reinterpret_cast<const uint4*>(g->d_blob);
  p.blob_bytes = g->blob_bytes;
  p.n = n;
  p.E = g->E;
  p.o_pred_ptr = g->o_pred_ptr;
  p.o_pred_idx = g->o_pred_idx;
  p.o_later = g->o_later;
  p.o_succ_ptr = g->o_succ_ptr;
  p.o_succ_idx = g->o_succ_idx;
  p.ovh = g->ovh;
  p.sstar = a->sstar;
  p.layout = a->layout;
  p.ld = a->ld;
  p.stride = a->sstar_stride;
  p.n_sstar = a->n_sstar;
  p.n_theta = a->n_theta;
  p.theta_chunk = theta_chunk;
  p.n_tchunks = n_tchunks;
  p.theta = a->theta;
  p.n_budget = a->n_budget;
  p.budget = a->budget;
  p.index_base = a->index_base;
  p.idx_bits = idx_bits;
  p.peak = a->peak;
  p.cost = a->cost;
  p.best_key = a->best_key;
  p.r_mask = a->r_mask;
  p.s_mask = a->s_mask;
  p.tri_words = tri_words;
  e = init_keys(a, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "init keys");
  cmk::round_evaluate_kernel<<<grid, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  ++g_launches;
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    cm_graph* gm = const_cast<cm_graph*>(g);
    std::lock_guard<std::mutex> lock(gm->mu);
    e = signal_call(g, ++gm->seq, reinterpret_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "launch round_evaluate_kernel");
  return CM_OK;
}

}  // extern "C"

// cm_api.cu -- the C ABI declared in include/cm.h (validation, graph upload, launch).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "cm.h"
#include "cm_kernel.cuh"

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

struct cm_graph {
  int32_t n = 0, E = 0;
  int64_t ovh = 0, cost_bound = 0;
  int device = 0, sm_count = 0, smem_optin = 0;
  int32_t blob_bytes = 0;
  int32_t o_pred_ptr = 0, o_pred_idx = 0, o_later = 0, o_succ_ptr = 0, o_succ_idx = 0;
  void* d_blob = nullptr;
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
  *out = g;
  return CM_OK;
}

void cm_graph_destroy(cm_graph* g) {
  if (!g) return;
  if (g->d_blob) cudaFree(g->d_blob);
  delete g;
}

int32_t cm_graph_n(const cm_graph* g) { return g ? g->n : -1; }
int64_t cm_graph_cost_bound(const cm_graph* g) { return g ? g->cost_bound : -1; }

cm_status cm_round_and_evaluate(const cm_graph* g, const cm_eval_args* a, cm_stream stream) {
  if (!g || !a) return fail(CM_EINVAL, "NULL graph or args");
  const int n = g->n;
  if (a->n_sstar < 0 || a->n_theta < 1 || a->n_budget < 0) return fail(CM_EINVAL, "bad counts");
  if (a->layout != CM_LAYOUT_DENSE && a->layout != CM_LAYOUT_TRI4) return fail(CM_EINVAL, "bad layout");
  int64_t min_stride;
  if (a->layout == CM_LAYOUT_DENSE) {
    if (a->ld < n || (a->ld & 3)) return fail(CM_EINVAL, "ld must be >= n and a multiple of 4");
    min_stride = (int64_t)n * a->ld;
  } else {
    const int64_t q = n >> 2, m = n & 3;
    min_stride = 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
  }
  if (a->n_sstar > 0) {
    if (a->sstar_stride < min_stride || (a->sstar_stride & 3))
      return fail(CM_EINVAL, "sstar_stride too small or not a multiple of 4");
    if (!a->sstar || (reinterpret_cast<uintptr_t>(a->sstar) & 15))
      return fail(CM_EINVAL, "sstar NULL or not 16-byte aligned");
    if (!a->theta || !a->peak || !a->cost) return fail(CM_EINVAL, "NULL theta/peak/cost");
  }
  if (a->n_budget > 0 && (!a->budget || !a->best_key)) return fail(CM_EINVAL, "NULL budget/best_key");
  if (a->n_budget > 4096) return fail(CM_ERANGE, "n_budget > 4096");
  const int64_t n_cand = (int64_t)a->n_sstar * a->n_theta;
  if (a->index_base < 0 || a->total_candidates < a->index_base + n_cand)
    return fail(CM_EINVAL, "total_candidates < index_base + n_sstar*n_theta");
  const int32_t idx_bits = cm_key_idx_bits(a->total_candidates);
  if (idx_bits > 62 || (idx_bits > 0 && g->cost_bound >= (int64_t(1) << (63 - idx_bits))))
    return fail(CM_ERANGE, "cost bound does not fit the packed key; use fewer candidates per key space");
  if (n_cand == 0) return CM_OK;

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
  static std::mutex mu;
  static size_t smem_set = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > smem_set) {
      e = cudaFuncSetAttribute(cmk::round_evaluate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(smem, 48 * 1024));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      smem_set = smem;
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
  cmk::round_evaluate_kernel<<<grid, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "launch round_evaluate_kernel");
  return CM_OK;
}

}  // extern "C"

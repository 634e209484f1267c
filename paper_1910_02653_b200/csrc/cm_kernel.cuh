// cm_kernel.cuh -- sm_100a kernels for Checkmate two-phase rounding + memory accounting.
//
// One CTA evaluates one S* (for a chunk of thresholds) at a time, persistent over the
// batch.  Thread r owns stage t = r+1 (T = n stages).  Per candidate:
//
//   round   (a1)  warps stream S* rows from HBM (coalesced 16-byte loads, one pass for all
//                 thresholds of the chunk), compare > theta in fp32 and pack the bits with
//                 warp shuffles into S rows kept in shared memory (Eq. 12b).
//   seed    (a2)  R_t = e_t | (S_{t+1} & ~S_t)      (Alg. 2 lines 2-5)
//   close   (a3)  walk the set bits of R_t from high to low; node k pushes its DEPS(k) not
//                 in S_t into R_t -- the paper's "reverse topological order for each stage,
//                 right to left" scan; work ~ closure visits.
//   events  (a4-a6) walk R_t from low to high: U += M_k, relpeak = max(relpeak, U),
//                 then subtract GC(k) = sum of M_i freed at k, FREE per Eq. 9:
//                 i in DEPS(k) u {k}, not in S_{t+1}, no later user of i computed in stage t.
//   base          U_{t,0} = ovh + sum_{i in S_t} M_i (Eq. 6) as a prefix over stages of
//                 delta_t = M(S_{t+1} \ S_t) - M(S_t \ S_{t+1}), a block-wide int64 scan.
//   peak          max_t (U_{t,0} + relpeak_t) (Eqs. 6-7; the max over k is attained at a
//                 compute step, Q9), cost = sum_t sum_{k in R_t} C_k (objective (1)).
//   keys    (a7)  per budget: min over feasible candidates of (cost << idx_bits | idx), kept
//                 per CTA in shared memory and folded into the global keys with one
//                 atomicMin per budget per CTA at the end.
//
// Shared-memory bit rows use a per-row-block layout: rows 32g..32g+31 hold words 0..g
// (a row r has bits i < r only), word w of row r at  32*g*(g+1)/2 + 32*w + (r & 31).
// Each lane touches only its own row (or row r+1), so every access is bank-conflict free.
#pragma once
#include <stdint.h>

namespace cmk {

constexpr unsigned FULL = 0xffffffffu;

struct Params {
  // graph blob (device global), copied into shared memory by every CTA
  const uint4* blob;
  int32_t blob_bytes;      // multiple of 16
  int32_t n, E;
  int32_t o_pred_ptr, o_pred_idx, o_later, o_succ_ptr, o_succ_idx;  // int32 offsets after M, C
  int64_t ovh;
  // batch
  const float* sstar;
  int32_t layout;
  int64_t ld, stride;
  int32_t n_sstar, n_theta, theta_chunk, n_tchunks;
  const float* theta;
  int32_t n_budget;
  const int64_t* budget;
  int64_t index_base;
  int32_t idx_bits;
  int64_t* peak;
  int64_t* cost;
  int64_t* best_key;
  uint64_t* r_mask;
  uint64_t* s_mask;
  int32_t tri_words;       // 32*G*(G+1)/2, G = ceil(n/32)
};

__device__ __forceinline__ int tri_addr(int r, int w) {
  const int g = r >> 5;
  return 16 * g * (g + 1) + 32 * w + (r & 31);
}

__device__ __forceinline__ int64_t row_offset(const Params& p, int r) {
  if (p.layout == 0) return (int64_t)r * p.ld;
  const int64_t q = r >> 2, m = r & 3;                     // sum_{r'<r} roundup4(r')
  return 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
}

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t o = __shfl_up_sync(FULL, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_max(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = max(v, (int64_t)__shfl_xor_sync(FULL, v, d));
  return v;
}

__device__ __forceinline__ int64_t warp_sum(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
  return v;
}

__global__ void __launch_bounds__(1024) round_evaluate_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int n = p.n;

  // ---- shared-memory carve (host computes the same sizes) ----
  unsigned char* sp = smem;
  const int64_t* M = reinterpret_cast<const int64_t*>(sp);
  const int64_t* C = M + n;
  const int32_t* gi = reinterpret_cast<const int32_t*>(sp + 16 * n);
  const int32_t* pred_ptr = gi + p.o_pred_ptr;
  const int32_t* pred_idx = gi + p.o_pred_idx;
  const int32_t* later = gi + p.o_later;
  const int32_t* succ_ptr = gi + p.o_succ_ptr;
  const int32_t* succ_idx = gi + p.o_succ_idx;
  sp += p.blob_bytes;
  int64_t* best = reinterpret_cast<int64_t*>(sp);             sp += 8 * ((p.n_budget + 1) & ~1);
  int64_t* bud = reinterpret_cast<int64_t*>(sp);              sp += 8 * ((p.n_budget + 1) & ~1);
  int64_t* red = reinterpret_cast<int64_t*>(sp);              sp += 8 * 96;
  uint32_t* Sb = reinterpret_cast<uint32_t*>(sp);             sp += 4 * (size_t)p.tri_words * p.theta_chunk;
  uint32_t* Rr = reinterpret_cast<uint32_t*>(sp);

  // ---- one-time: graph blob + budgets into shared memory ----
  for (int i = tid; i < p.blob_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = p.blob[i];
  for (int b = tid; b < p.n_budget; b += blockDim.x) {
    best[b] = INT64_MAX;
    bud[b] = p.budget[b];
  }
  __syncthreads();

  const int64_t n_items = (int64_t)p.n_sstar * p.n_tchunks;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int s = (int)(item / p.n_tchunks);
    const int th0 = (int)(item % p.n_tchunks) * p.theta_chunk;
    const int nth = min(p.theta_chunk, p.n_theta - th0);
    const float* S0 = p.sstar + (int64_t)s * p.stride;

    // ================= a1: round all rows for all thresholds of the chunk =================
    for (int r = warp; r < n; r += nwarps) {
      const float* row = S0 + row_offset(p, r);
      const int nwords = (r >> 5) + 1;                 // words 0..r>>5 are stored for row r
      for (int c = 0; 4 * c < nwords; ++c) {
        const int e0 = c * 128 + lane * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e0 < r) v = __ldcs(reinterpret_cast<const float4*>(row + e0));
        const int w = 4 * c + (lane >> 3);
        for (int j = 0; j < nth; ++j) {
          const float th = __ldg(p.theta + th0 + j);
          uint32_t nib = (uint32_t)((e0 + 0 < r) & (v.x > th)) |
                         ((uint32_t)((e0 + 1 < r) & (v.y > th)) << 1) |
                         ((uint32_t)((e0 + 2 < r) & (v.z > th)) << 2) |
                         ((uint32_t)((e0 + 3 < r) & (v.w > th)) << 3);
          uint32_t x = nib << ((lane & 7) * 4);
          x |= __shfl_xor_sync(FULL, x, 1);
          x |= __shfl_xor_sync(FULL, x, 2);
          x |= __shfl_xor_sync(FULL, x, 4);
          if ((lane & 7) == 0 && w < nwords) Sb[(size_t)j * p.tri_words + tri_addr(r, w)] = x;
        }
      }
    }
    __syncthreads();

    for (int j = 0; j < nth; ++j) {
      const uint32_t* Sj = Sb + (size_t)j * p.tri_words;
      const int r = tid;
      int64_t delta = 0, relpeak = INT64_MIN, cost_t = 0;
      if (r < n) {
        const int gr = r >> 5;
        const bool has_next = r + 1 < n;               // S_{n+1} = 0 (Q3)
        // ---- a2: seed ----
        for (int w = 0; w <= gr; ++w) {
          const uint32_t sn = has_next ? Sj[tri_addr(r + 1, w)] : 0u;
          Rr[tri_addr(r, w)] = sn & ~Sj[tri_addr(r, w)];
        }
        Rr[tri_addr(r, gr)] |= 1u << (r & 31);
        // ---- a3: closure, right to left ----
        for (int w = gr; w >= 0; --w) {
          uint32_t x = Rr[tri_addr(r, w)];
          while (x) {
            const int b = 31 - __clz(x);
            x &= ~(1u << b);
            const int k = 32 * w + b;
            for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
              const int i = pred_idx[e];
              const int wi = i >> 5;
              const uint32_t bi = 1u << (i & 31);
              if (Sj[tri_addr(r, wi)] & bi) continue;
              const int a = tri_addr(r, wi);
              const uint32_t old = Rr[a];
              if (!(old & bi)) {
                Rr[a] = old | bi;
                if (wi == w) x |= bi;
              }
            }
          }
        }
        // ---- a4-a6: events left to right ----
        int64_t U = 0;
        for (int w = 0; w <= gr; ++w) {
          uint32_t x = Rr[tri_addr(r, w)];
          while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            const int k = 32 * w + b;
            U += M[k];
            relpeak = max(relpeak, U);
            cost_t += C[k];
            int64_t gc = 0;
            for (int e = pred_ptr[k]; e < pred_ptr[k + 1]; ++e) {
              const int i = pred_idx[e];
              if (has_next && (Sj[tri_addr(r + 1, i >> 5)] >> (i & 31) & 1u)) continue;
              bool last_use = true;
              for (int q = later[e]; q < succ_ptr[i + 1]; ++q) {
                const int jj = succ_idx[q];
                if (jj > r) break;
                if (Rr[tri_addr(r, jj >> 5)] >> (jj & 31) & 1u) { last_use = false; break; }
              }
              if (last_use) gc += M[i];
            }
            if (!(has_next && (Sj[tri_addr(r + 1, k >> 5)] >> (k & 31) & 1u))) {
              bool unused = true;
              for (int q = succ_ptr[k]; q < succ_ptr[k + 1]; ++q) {
                const int jj = succ_idx[q];
                if (jj > r) break;
                if (Rr[tri_addr(r, jj >> 5)] >> (jj & 31) & 1u) { unused = false; break; }
              }
              if (unused) gc += M[k];
            }
            U -= gc;
          }
        }
        // ---- base: delta_t = M(S_{t+1} \ S_t) - M(S_t \ S_{t+1}) ----
        for (int w = 0; w <= gr; ++w) {
          const uint32_t sc = Sj[tri_addr(r, w)];
          const uint32_t sn = has_next ? Sj[tri_addr(r + 1, w)] : 0u;
          uint32_t add = sn & ~sc, sub = sc & ~sn;
          while (add) { const int b = __ffs(add) - 1; add &= add - 1; delta += M[32 * w + b]; }
          while (sub) { const int b = __ffs(sub) - 1; sub &= sub - 1; delta -= M[32 * w + b]; }
        }
      }
      // ---- block-wide exclusive scan of delta -> U_{t,0}; max peak; sum cost ----
      int64_t incl = warp_incl_scan(delta, lane);
      if (lane == 31) red[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int64_t v = lane < nwarps ? red[lane] : 0;
        int64_t sc = warp_incl_scan(v, lane);
        red[32 + lane] = sc - v;                       // exclusive warp prefix
      }
      __syncthreads();
      const int64_t base = p.ovh + red[32 + warp] + incl - delta;
      int64_t pk = (r < n) ? base + relpeak : INT64_MIN;
      pk = warp_max(pk);
      int64_t cs = warp_sum(cost_t);
      __syncthreads();                                  // everyone has read red[32+warp]
      if (lane == 0) { red[warp] = pk; red[32 + warp] = cs; }
      __syncthreads();
      if (warp == 0) {
        int64_t a = lane < nwarps ? red[lane] : INT64_MIN;
        int64_t b2 = lane < nwarps ? red[32 + lane] : 0;
        a = warp_max(a);
        b2 = warp_sum(b2);
        if (lane == 0) { red[64] = a; red[65] = b2; }
      }
      __syncthreads();
      const int64_t cand_peak = red[64], cand_cost = red[65];
      const int64_t local = (int64_t)s * p.n_theta + th0 + j;
      if (tid == 0) {
        p.peak[local] = cand_peak;
        p.cost[local] = cand_cost;
      }
      const int64_t key = (cand_cost << p.idx_bits) | (p.index_base + local);
      for (int b = tid; b < p.n_budget; b += blockDim.x)
        if (cand_peak <= bud[b] && key < best[b]) best[b] = key;
      // ---- optional masks ----
      if ((p.r_mask || p.s_mask) && r < n) {
        const int W64 = (n + 63) >> 6, gr = r >> 5;
        const size_t o = ((size_t)local * n + r) * W64;
        for (int w = 0; w < W64; ++w) {
          if (p.r_mask) {
            const uint64_t lo = (2 * w <= gr) ? Rr[tri_addr(r, 2 * w)] : 0u;
            const uint64_t hi = (2 * w + 1 <= gr) ? Rr[tri_addr(r, 2 * w + 1)] : 0u;
            p.r_mask[o + w] = lo | (hi << 32);
          }
          if (p.s_mask) {
            const uint64_t lo = (2 * w <= gr) ? Sj[tri_addr(r, 2 * w)] : 0u;
            const uint64_t hi = (2 * w + 1 <= gr) ? Sj[tri_addr(r, 2 * w + 1)] : 0u;
            p.s_mask[o + w] = lo | (hi << 32);
          }
        }
      }
      __syncthreads();                                  // red[] reuse; Rr reuse by next threshold
    }
  }
  __syncthreads();
  for (int b = tid; b < p.n_budget; b += blockDim.x)
    if (best[b] != INT64_MAX)
      atomicMin(reinterpret_cast<long long*>(p.best_key + b), (long long)best[b]);
}

}  // namespace cmk

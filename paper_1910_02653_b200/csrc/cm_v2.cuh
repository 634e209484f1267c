// cm_v2.cuh -- stage-sliced sm_100a kernels for Checkmate two-phase rounding (Alg. 2,
// PAPER.md:389-415) and the Eq. 6-9 memory accounting.
//
// "Stage-sliced": a 32-bit word holds one node's bit for 32 consecutive stages.  A lane
// owns a group g of 32 stages (rows 32g..32g+31, 0-based row r = stage t-1) of one
// candidate, so every bitwise step of the method runs for 32 stages at once and the control
// flow (a walk over the graph) is identical in all lanes: no per-stage divergence, however
// recomputation is distributed over the stages.
//
// K1 round_pack_kernel (HBM-bound).  Task = (S*, row group g).  For each 32x32 block
//   (w = 0..g) lane l loads row r = 32g+l+1 with 16-byte streaming loads, compares > theta
//   (a1: strict, fp32, NaN -> 0) into a row word, and a 5-step shuffle
//   transpose turns the 32 row words into column words
//       Sn_g[i]  bit b = S_{row 32g+b+1, node i} = S_{t+1}   for stage t = 32g+b+1,
//   i.e. the NEXT stage's checkpoint bits (S_{n+1} = 0).  The current stage's
//   bits follow from them: Sw_g = (Sn_g << 1) | (Sn_{g-1} >> 31).  One S* read serves every
//   threshold.
//
// K2 scan_kernel (ALU / latency-bound).  One warp evaluates cpw candidates, lanes =
//   (candidate, group).  A single pass over nodes k = n-1 .. 0 (reverse topological order,
//   the paper's right-to-left repair scan), push form:
//     R_k   = ((Sn_k | Acc_k) & ~Sw_k) | diag_k      a2 seed S_{t+1} & ~S_t, e_t; a3 closure
//             Acc_k = OR of R_j over the users j > k (all visited before k)
//     FREE  i in DEPS(k): R_k & ~Sn_i & ~Acc_i       Eq. 9: k computed, i not kept, no later user
//           i = k:        R_k & ~Sn_k & ~Acc_k       the i = k term of Eq. 8
//     Acc_i |= R_k
//   Memory: with D = U_{t,k} - U_{t,end} run backwards and MX = max over computes of D,
//   only E = MX - D matters:  frees:  E -= M_i ;  compute of k:  E = max(E, 0) + M_k.
//   Then peak_t = U_{t,0} + E_t (the max over k is reached at a compute,
//   DESIGN.md Q9), with U_{t,0} = ovh + mass_t (Eq. 6) from K1.  The per-stage int64 E sits
//   in shared memory and is touched only at set bits (events).
//
// Layout of one candidate's column array in the workspace: group g holds nodes 0..32g+31 at
// word offset grp_off(g) = 16 g (g+1) (16-byte aligned).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace cm2 {

constexpr unsigned FULL = 0xffffffffu;

__host__ __device__ __forceinline__ int grp_off(int g) { return 16 * g * (g + 1); }
__host__ __device__ __forceinline__ int block_words(int G) { return 16 * G * (G + 1); }
// workspace words per candidate: [Sn columns: block_words][mass: n int64][brow: G x G u32]
// brow row g = the row-form words of S row 32g (bits over nodes), the bit S_t for t = 32g+1
// that a group-g pass cannot derive from its own Sn columns.
__host__ __device__ __forceinline__ int cand_words(int n) {
  const int G = (n + 31) / 32;
  return (block_words(G) + 2 * n + G * G + 3) & ~3;
}
__host__ __device__ __forceinline__ int brow_off(int n) { return block_words((n + 31) / 32) + 2 * n; }

__device__ __forceinline__ int64_t row_offset(int layout, int64_t ld, int r) {
  if (layout == 0) return (int64_t)r * ld;
  const int64_t q = r >> 2, m = r & 3;                     // sum_{r'<r} roundup4(r')
  return 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
}

// 32x32 bit transpose across a warp: in, lane l holds row word l (bit c = A[l][c]);
// out, lane l holds column word l (bit r = A[r][l]).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t M = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                     : j == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(FULL, x, j);
    const bool hi = (lane & j) != 0;
    const uint32_t t = hi ? (y >> j) : (y << j);
    const uint32_t K = hi ? ~M : M;
    x = (x & K) | (t & ~K);
  }
  return x;
}

// The same transpose with the per-lane select folded into a rotate: t = rotl(y, s_j) with
// s_j = j (lane bit j clear) or 32 - j (set); the bits a rotate wraps around land exactly
// where the stage's keep-mask K_j drops them.  3 instructions per stage (SHFL, SHF.L.W, LOP3).
struct Transposer {
  uint32_t K[5];
  uint32_t sh[5];
  __device__ __forceinline__ explicit Transposer(int lane) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int j = 16 >> k;
      const uint32_t M = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                       : j == 2 ? 0x33333333u : 0x55555555u;
      const bool hi = (lane & j) != 0;
      K[k] = hi ? ~M : M;
      sh[k] = hi ? 32u - j : (uint32_t)j;
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t y = __shfl_xor_sync(FULL, x, 16 >> k);
      const uint32_t t = __funnelshift_l(y, y, sh[k]);
      x = (x & K[k]) | (t & ~K[k]);
    }
    return x;
  }
};

// ------------------------------------------------------------------------------------ K1
struct RoundParams {
  const float* sstar;
  int32_t layout;
  int64_t ld, stride;
  int32_t n, G;
  int64_t s_begin;            // first S* of this chunk (batch-relative)
  int32_t s_count;
  int32_t n_theta;            // all thresholds (block index stride)
  int32_t th0, nt;            // this launch handles thresholds th0 .. th0+nt-1, nt <= 4
  const float* theta;
  uint32_t* sn;               // out: candidate block (s - s_begin) * n_theta + j, cs words each:
  int32_t cs;                 //   [Sn columns: bw words][mass: n int64]
  int32_t bw;
  const int64_t* nib;         // nibble tables: nib[p*16 + v] = sum_{j<4, bit j of v} M[4p + j]
  const int32_t* nib32;       // the same in int32 when every row mass fits (else nullptr)
  int32_t nib_entries;        // 128 * G
  int32_t brow;               // word offset of brow in a candidate block
};

// ---- bulk-async copy + mbarrier helpers (sm_90+ PTX; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
// 3-D tensor-map TMA: box {32 nodes, 32 rows, 1 S*} at (x = node, y = row, z = S*).
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}

// K1 for the dense layout.  Per S* the warp walks the blocks (g, w), g = 0..G-1, w = 0..g:
// rows r = 32g+1+l, l = 0..31 (the S_{t+1} rows of group g's stages) x nodes 32w..32w+31.
// One elected lane loads a block with a single 3-D tensor-map TMA (rows >= n zero-filled) in
// the 128-byte swizzle (16-byte chunk c of tile row l lands at chunk c ^ (l & 7)), so lane l
// reads its own row with 8 conflict-free LDS.128.  One ballot per node q of x[q] > theta
// (Alg. 2 line 1) yields node q's column word over the 32 rows -- the form K2
// consumes; the 32 words pass through a 32-word shared slot to lane q, which masks them to
// the strict lower triangle, stores them, and transposes them into row words for the row's
// checkpoint mass mass_r = sum_{i in S_r} M_i (the Eq. 6 sum, from 4-bit
// tables) and for row 32(g+1)'s word (the brow operand of K2).
constexpr int kStages = 2;     // 64 KB per CTA: co-resides with the TMEM scan CTA (144 KB)
constexpr int kK1Warps = 8;
// Shared layout (bytes from a 1024-aligned base): tiles, mbarriers, NT column-word slots per
// warp (one per threshold, so the NT chains interleave), then the staged int32 mass tables.
struct K1Smem {
  float tile[kK1Warps][kStages][32][32];      // 4 KB tiles, 1024-byte aligned (swizzle atom)
  uint64_t bar[kK1Warps][kStages];
};
__host__ __device__ constexpr size_t k1_cols_off() { return sizeof(K1Smem); }
__host__ __device__ constexpr size_t k1_nib_off(int nt) { return sizeof(K1Smem) + (size_t)kK1Warps * nt * 128; }
// dynamic bytes to request: + 1024 slack for aligning the base
__host__ __device__ constexpr size_t k1_smem_bytes(int nt, int nib_entries) {
  return k1_nib_off(nt) + 4 * (size_t)nib_entries + 1024;
}

// NT = thresholds per pass (1..4, a compile-time count so the per-threshold work of one block
// -- ballots, mass lookups, transposes -- forms NT independent instruction chains).
template <int NT>
__global__ void __maxnreg__(128) round_tma_kernel(const RoundParams p, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char k1raw[];
  unsigned char* k1smem = k1raw + ((1024u - (smem_u32(k1raw) & 1023u)) & 1023u);
  K1Smem& sm = *reinterpret_cast<K1Smem*>(k1smem);
  int32_t* nib32 = reinterpret_cast<int32_t*>(k1smem + k1_nib_off(NT));   // p.nib32 staged (if any)
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t(*cols_w)[32] = reinterpret_cast<uint32_t(*)[32]>(k1smem + k1_cols_off()) + NT * wl;
  const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int G = p.G;
  if (p.nib32)
    for (int i = threadIdx.x; i < p.nib_entries; i += blockDim.x) nib32[i] = p.nib32[i];
  if (lane == 0)
    for (int st = 0; st < kStages; ++st) mbar_init(&sm.bar[wl][st], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  float th[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) th[j] = p.theta[p.th0 + j];
  const Transposer transpose(lane);
  const bool scaled32 = p.nib32 != nullptr;
  const uint32_t row_base = smem_u32(&sm.tile[wl][0][lane][0]);     // stage 0, this lane's row
  const uint32_t swz = (uint32_t)(lane & 7) << 4;

  // Producer cursor (ps, pg, pw) runs kStages-1 blocks ahead of the consumer.  No proxy
  // fence before re-filling a stage: its previous contents were consumed (ballots issued on
  // the loaded values, then __syncwarp) before the refill is issued.
  int ps = wid, pg = 0, pw = 0, pstage = 0;
  auto issue = [&]() {
    if (ps >= p.s_count) return;
    if (lane == 0) {
      mbar_expect_tx(&sm.bar[wl][pstage], 32u * 32u * 4u);
      tma_load_3d(&sm.tile[wl][pstage][0][0], &tmap, 32 * pw, 32 * pg + 1, (int)(p.s_begin + ps),
                  &sm.bar[wl][pstage]);
    }
    pstage = pstage + 1 == kStages ? 0 : pstage + 1;
    if (++pw > pg) {
      pw = 0;
      if (++pg == G) { pg = 0; ps += nw; }
    }
  };
  for (int d = 0; d < kStages - 1; ++d) issue();

  int cstage = 0;
  uint32_t phase_bits = 0u;                                         // bit st = parity of stage st
  for (int s = wid; s < p.s_count; s += nw) {
    uint32_t* out = p.sn + ((int64_t)s * p.n_theta + p.th0) * p.cs;
    for (int g = 0; g < G; ++g) {
      const int rq = 32 * g + lane + 1;                             // row owned by this lane
      // rows of the group that exist (r < n): bits [0, hi)
      const int hi = p.n - 1 - 32 * g;
      const uint32_t rows_ok = hi >= 32 ? FULL : (hi <= 0 ? 0u : (1u << hi) - 1u);
      int64_t mass[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) mass[j] = 0;
      for (int w = 0; w <= g; ++w) {
        issue();
        mbar_wait(&sm.bar[wl][cstage], (phase_bits >> cstage) & 1u);
        phase_bits ^= 1u << cstage;
        const uint32_t rb = row_base + (uint32_t)cstage * (32u * 32u * 4u);
        float x[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rb + (((uint32_t)c << 4) ^ swz)));
          x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
        cstage = cstage + 1 == kStages ? 0 : cstage + 1;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q = 0; q < 32; ++q) cols_w[j][q] = __ballot_sync(FULL, x[q] > th[j]);
        __syncwarp();                                               // tile read, ballots stored
        // Column mask of node i = 32w + lane: rows r = 32g+1+b with i < r (strict lower
        // triangle: b >= 32(w-g) + lane) and r < n.  Zero-filled / upper entries never leak.
        const int lo = 32 * (w - g) + lane;
        const uint32_t cmask = rows_ok & (lo <= 0 ? FULL : (lo >= 32 ? 0u : FULL << lo));
        uint32_t word[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) word[j] = cols_w[j][lane] & cmask;   // node i's column
        __syncwarp();
        const int node = 32 * w + lane;
        const int brow_at = p.brow + (g + 1) * G + w;               // row 32(g+1)'s word (lane 31)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          uint32_t* oj = out + (int64_t)j * p.cs;
          oj[grp_off(g) + node] = word[j];
          word[j] = transpose(word[j]);                             // row rq's word over block w
          if (lane == 31 && g + 1 < G) oj[brow_at] = word[j];
        }
        if (scaled32) {                                             // scaled masses fit int32
          const unsigned char* tb = reinterpret_cast<const unsigned char*>(nib32 + 128 * w);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int32_t m32 = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t off = q == 0 ? (word[j] << 2) & 0x3Cu : (word[j] >> (4 * q - 2)) & 0x3Cu;
              m32 += *reinterpret_cast<const int32_t*>(tb + 64 * q + off);
            }
            mass[j] += m32;
          }
        } else {
          const int64_t* tw = p.nib + 128 * w;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int64_t ms = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) ms += __ldg(tw + 16 * q + ((word[j] >> (4 * q)) & 15u));
            mass[j] += ms;
          }
        }
      }
      if (rq < p.n) {
#pragma unroll
        for (int j = 0; j < NT; ++j) reinterpret_cast<int64_t*>(out + (int64_t)j * p.cs + p.bw)[rq] = mass[j];
      }
    }
  }
}

// K1 for the packed tri4 layout (rows of irregular stride).  Per task (S*, g) the warp covers rows r_q = 32g+1+q, q = 0..31 (the S_{t+1} rows of the
// group's stages), 32 nodes (block w) at a time.  Lane = node: row q of the block is one
// coalesced 128-byte load, one compare (a1, strict fp32 '>', NaN -> 0) and one ballot, which
// is already the packed row word.  The 32 row words go through a 32-word shared slot to
// lane q, which transposes them into column words and adds the checkpoint mass of its
// row, mass_r = sum_{i in S_r} M_i (the Eq. 6 sum), from 4-bit tables.
// Out-of-triangle elements are replaced by NaN, which compares false for every theta.
__global__ void __launch_bounds__(256) round_ldg_kernel(const RoundParams p) {
  __shared__ uint32_t rows_w[8][32];                              // per-warp ballot slot
  __shared__ int64_t rows_off[8][32];                             // per-warp row offsets
  const int64_t* nib = p.nib;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int tasks = p.s_count * p.G;
  const float qnan = __int_as_float(0x7fffffff);
  for (int task = wid; task < tasks; task += nw) {
    const int s = task / p.G;
    const int g = task - s * p.G;
    const float* S0 = p.sstar + (p.s_begin + s) * p.stride;
    uint32_t* out = p.sn + ((int64_t)s * p.n_theta + p.th0) * p.cs;
    const int rq = 32 * g + lane + 1;                               // row owned by this lane
    rows_off[wl][lane] = row_offset(p.layout, p.ld, rq);
    __syncwarp();
    const bool full_rows = (32 * g + 32) < p.n;                     // every r_q exists
    int64_t mass[4] = {0, 0, 0, 0};
    for (int w = 0; w <= g; ++w) {
      const int node = 32 * w + lane;
      float x[32];
      if (w < g && full_rows) {                                     // interior block: no masking
#pragma unroll
        for (int q = 0; q < 32; ++q) x[q] = __ldcs(S0 + rows_off[wl][q] + node);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int r = 32 * g + 1 + q;
          x[q] = (r < p.n && node < r) ? __ldcs(S0 + rows_off[wl][q] + node) : qnan;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= p.nt) break;
        const float th = __ldg(p.theta + p.th0 + j);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t b = __ballot_sync(FULL, x[q] > th);
          rows_w[wl][q] = b;                                        // uniform value: one store
        }
        __syncwarp();
        const uint32_t word = rows_w[wl][lane];                     // row r_q's word, block w
        __syncwarp();
        int64_t ms = 0;
        if (word) {
          const int64_t* tw = nib + 128 * w;
#pragma unroll
          for (int q = 0; q < 8; ++q) ms += __ldg(tw + 16 * q + ((word >> (4 * q)) & 15u));
        }
        uint32_t* oj = out + (int64_t)j * p.cs;
        if (lane == 31 && g + 1 < p.G) oj[p.brow + (g + 1) * p.G + w] = word;   // row 32(g+1)
        oj[grp_off(g) + node] = transpose32(word, lane);
        mass[j] += ms;
      }
    }
    if (rq < p.n) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < p.nt) reinterpret_cast<int64_t*>(out + (int64_t)j * p.cs + p.bw)[rq] = mass[j];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------ K2
// Group-major scan: a task is (stage group g, 32 candidates); lane l works on candidate
// c0 + l.  The stages of different groups never interact (stage t needs only S_t, S_{t+1}
// and the graph), so a group pass is a complete, independent evaluation of its 32 stages;
// all lanes walk the same node range k = min(n,32g+32)-1 .. 0 in lockstep.
// Shared memory per warp: Sn[node][lane], Acc[node][lane] (u32) and E[stage][lane] (int64),
// every access lane-contiguous (bank-conflict free).
struct ScanParams {
  const uint4* blob;          // M[n] int64, C[n] int64, pred_ptr[n+1], pred_idx[E] (int32)
  int32_t blob_bytes;
  int32_t n, o_pred_ptr, o_pred_idx;
  int32_t o_nrec, o_drec;     // byte offsets of the node / dependency records in the blob
  const uint32_t* ws;         // chunk workspace from K1 (cs words per candidate)
  int32_t cs, G, brow;
  int64_t n_cand;             // candidates in this chunk
  int32_t n_batch;            // ceil(n_cand / 32)
  int64_t* part;              // out: [n_cand][G] x {peak_g - ovh, cost_g}
  uint32_t* r_mask32;         // optional masks (u64 words seen as pairs of u32)
  uint32_t* s_mask32;
  int64_t out_base;           // local index of the chunk's first candidate
  int32_t warp_bytes;         // shared bytes per warp region
};

// A' storage of one warp.  TM = false: shared memory [node][lane].  TM = true: nodes < tmc
// live in Tensor Memory -- lane = TMEM lane (this warp's 32-lane quarter), node = TMEM
// column, accessed with tcgen05.ld/st.32x32b (one column, all 32 lanes, uniform address)
// -- and nodes >= tmc spill to shared memory.  Stores are made visible to later loads by
// tcgen05.wait::st, issued once per node step (fence_st).
template <bool TM>
struct AView {
  uint32_t* sm;
  uint32_t taddr;
  int tmc;
  int lane;
  // MODE 0: shared only; 1: decide per access (node < tmc -> TMEM); 2: TMEM only.
  template <int MODE>
  __device__ __forceinline__ uint32_t ldm(int k) const {
    if (TM && (MODE == 2 || (MODE == 1 && k < tmc))) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr + (uint32_t)k) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v) :: "memory");
      return v;
    }
    return sm[32 * (k - tmc) + lane];
  }
  template <int MODE>
  __device__ __forceinline__ void stm(int k, uint32_t v) const {
    if (TM && (MODE == 2 || (MODE == 1 && k < tmc)))
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr + (uint32_t)k), "r"(v) : "memory");
    else
      sm[32 * (k - tmc) + lane] = v;
  }
  __device__ __forceinline__ uint32_t ld(int k) const { return ldm<TM ? 1 : 0>(k); }
  __device__ __forceinline__ void st(int k, uint32_t v) const { stm<TM ? 1 : 0>(k, v); }
  __device__ __forceinline__ void st4(int k, uint4 v) const {   // nodes k..k+3, k % 4 == 0
    if (TM && k < tmc)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                   :: "r"(taddr + (uint32_t)k), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else {
      sm[32 * (k + 0 - tmc) + lane] = v.x;
      sm[32 * (k + 1 - tmc) + lane] = v.y;
      sm[32 * (k + 2 - tmc) + lane] = v.z;
      sm[32 * (k + 3 - tmc) + lane] = v.w;
    }
  }
  __device__ __forceinline__ void fence_st() const {
    if (TM) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
};

// One node k of the group-g pass for dependency count ND (0..4; ND = 4 also walks any
// further dependencies).  Specialised so the event loop carries exactly ND free masks.
// drec[e] = {i, (int32) M_i} (M_i read from the int64 array when ET is int64).
template <int ND, typename ET, bool TM, int MODE>
__device__ __forceinline__ void node_step(int k, uint32_t Rk, uint32_t a, ET Mk, int e0, int nd,
                                          const int2* __restrict__ drec,
                                          const int64_t* __restrict__ M, const AView<TM>& A, ET* E,
                                          int lane, uint32_t& a_next) {
  uint32_t f[ND > 0 ? ND : 1];
  ET mi[ND > 0 ? ND : 1];
#pragma unroll
  for (int j = 0; j < ND; ++j) {                                   // FREE_{t,i,k} = R_k & ~A'_i
    const int2 d = drec[e0 + j];
    const int i = d.x;
    const bool nb = (i == k - 1);
    const uint32_t ai = nb ? a_next : A.template ldm<MODE>(i);
    f[j] = Rk & ~ai;
    A.template stm<MODE>(i, ai | Rk);                               // A'_i |= R_k
    if (nb) a_next = ai | Rk;
    mi[j] = sizeof(ET) == 4 ? (ET)d.y : (ET)M[i];
  }
  if (ND == 4) {
    for (int e = e0 + 4; e < e0 + nd; ++e) {                       // in-degree > 4 (rare)
      const int2 d = drec[e];
      const int i = d.x;
      const bool nb = (i == k - 1);
      const uint32_t ai = nb ? a_next : A.template ldm<MODE>(i);
      uint32_t fx = Rk & ~ai;
      A.template stm<MODE>(i, ai | Rk);
      if (nb) a_next = ai | Rk;
      const ET Mi = sizeof(ET) == 4 ? (ET)d.y : (ET)M[i];
      for (; fx; fx &= fx - 1) E[32 * (__ffs(fx) - 1) + lane] -= Mi;
    }
  }
  const uint32_t selff = Rk & ~a;                                   // FREE_{t,k,k}
  // every free at k lies in a stage that computes k: E = max(E - GC(k), 0) + M_k.
  // Up to four stage bits per round: their loads issue together (latency, not issue, bound).
  for (uint32_t x = Rk; x;) {
    int b[4];
    bool v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = x != 0u;
      b[u] = v[u] ? __ffs(x) - 1 : 0;
      x &= x - 1;
    }
    ET ev[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ev[u] = v[u] ? E[32 * b[u] + lane] : (ET)0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((selff >> b[u]) & 1u) ev[u] -= Mk;
#pragma unroll
      for (int j = 0; j < ND; ++j)
        if ((f[j] >> b[u]) & 1u) ev[u] -= mi[j];
      ev[u] = (ev[u] > 0 ? ev[u] : (ET)0) + Mk;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v[u]) E[32 * b[u] + lane] = ev[u];
  }
}

// Walk the quads q = q_hi .. q_lo (nodes 4q+3 .. 4q) of a group pass.  MODE as in AView.
// nrec[k] = {(int32) M_k, e0, nd, -} with C_k from the int64 array.
template <typename ET, bool TM, int MODE>
__device__ __forceinline__ void walk(int q_hi, int q_lo, int nk, int g, bool live, const uint4* sn4,
                                     const uint32_t* brow, const int4* __restrict__ nrec,
                                     const int2* __restrict__ drec, const int64_t* __restrict__ M,
                                     const int64_t* __restrict__ C, const AView<TM>& A, ET* E, int lane,
                                     uint4& cur, uint32_t& a_next, uint32_t& bword, uint32_t& bnext,
                                     int64_t& costL) {
  for (int q = q_hi; q >= q_lo; --q) {
    const uint4 nxt = (q > 0 && live) ? __ldcg(sn4 + q - 1) : make_uint4(0u, 0u, 0u, 0u);
    if ((q & 7) == 7) {                                             // entered a new 32-node block
      bword = bnext;
      const int wb = (q >> 3) - 1;
      bnext = (g > 0 && wb >= 0 && wb < g && live) ? brow[wb] : 0u;
    }
#pragma unroll
    for (int u = 3; u >= 0; --u) {
      const int k = 4 * q + u;
      if (k >= nk) continue;                                        // warp-uniform
      const uint32_t sn = u == 3 ? cur.w : u == 2 ? cur.z : u == 1 ? cur.y : cur.x;
      const uint32_t sw = (sn << 1) | ((bword >> (k & 31)) & 1u);   // S_t from S_{t+1} and row 32g
      A.fence_st();                                                 // earlier stores visible
      const uint32_t a = a_next;                                    // A'_k = Sn_k | Acc_k (complete)
      a_next = k > 0 ? A.template ldm<(MODE == 1) ? 1 : MODE>(k - 1) : 0u;   // prefetch
      const uint32_t diag = ((k >> 5) == g) ? (1u << (k & 31)) : 0u;
      const uint32_t Rk = (a & ~sw) | diag;                         // a2 seed + a3 closure
      A.template stm<MODE>(k, Rk);                                  // slot now holds R column
      if (!__any_sync(FULL, Rk != 0u)) continue;                    // computed in no lane
      const int4 rec = nrec[k];
      const ET Mk = sizeof(ET) == 4 ? (ET)rec.x : (ET)M[k];
      costL += (int64_t)__popc(Rk) * C[k];
      const int e0 = rec.y, nd = rec.z;
      switch (nd) {                                                 // warp-uniform
        case 0: node_step<0, ET, TM, MODE>(k, Rk, a, Mk, e0, nd, drec, M, A, E, lane, a_next); break;
        case 1: node_step<1, ET, TM, MODE>(k, Rk, a, Mk, e0, nd, drec, M, A, E, lane, a_next); break;
        case 2: node_step<2, ET, TM, MODE>(k, Rk, a, Mk, e0, nd, drec, M, A, E, lane, a_next); break;
        case 3: node_step<3, ET, TM, MODE>(k, Rk, a, Mk, e0, nd, drec, M, A, E, lane, a_next); break;
        default: node_step<4, ET, TM, MODE>(k, Rk, a, Mk, e0, nd, drec, M, A, E, lane, a_next); break;
      }
    }
    cur = nxt;
  }
}

// ET = int32_t when every M is a multiple of a scale s with sum M/s < 2^30 (the host checks;
// exact), else int64_t.  M in the blob, the masses and the results are in units of s.
// TM: A' of nodes < 256 in Tensor Memory (8 warps, one CTA per SM, 512 TMEM columns:
// warp w uses lane quarter w % 4 and columns 256 * (w / 4) ..).
template <typename ET, bool TM>
__global__ void __launch_bounds__(256, 2) scan_kernel(const ScanParams p) {   // <= 128 regs: co-resides with K1
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = p.n, G = p.G;
  const int64_t* M = reinterpret_cast<const int64_t*>(smem);
  const int64_t* C = M + n;
  const int32_t* gi = reinterpret_cast<const int32_t*>(smem + 16 * n);
  const int4* nrec = reinterpret_cast<const int4*>(smem + p.o_nrec);
  const int2* drec = reinterpret_cast<const int2*>(smem + p.o_drec);
  (void)gi;
  unsigned char* wr = smem + p.blob_bytes + (size_t)warp * p.warp_bytes;
  ET* E = reinterpret_cast<ET*>(wr);                               // [32 stages][32 lanes]
  uint32_t* Asm = reinterpret_cast<uint32_t*>(E + 32 * 32);         // [node][lane] (spill part)
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < p.blob_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = p.blob[i];
  if (TM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  AView<TM> A;
  A.sm = Asm;
  A.lane = lane;
  A.tmc = TM ? min(p.n, 256) : 0;
  A.taddr = TM ? tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2) : 0u;

  const int tasks = G * p.n_batch;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int task = gw; task < tasks; task += nwarps) {
    const int g = G - 1 - task / p.n_batch;                         // big groups first
    const int64_t c = (int64_t)(task % p.n_batch) * 32 + lane;
    const bool live = c < p.n_cand;
    const int nk = min(n, 32 * (g + 1));                            // nodes 0..nk-1
    const int nq = (nk + 3) >> 2;                                   // uint4 blocks of Sn
    const uint32_t* cw = p.ws + (live ? c : 0) * p.cs;
    const uint4* sn4 = reinterpret_cast<const uint4*>(cw + grp_off(g));
    // A'_i = Sn_i | Acc_i (Acc = OR of R over visited users): the closure reads Sn_k | Acc_k and
    // every FREE test reads Sn_i | Acc_i, so one array serves both.  Start: A' = Sn.
    {  // software-pipelined: the loads of 8 quads are in flight while the previous 8 are stored
      uint4 va[8], vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) va[u] = (live && u < nq) ? __ldcg(sn4 + u) : make_uint4(0u, 0u, 0u, 0u);
      for (int q0 = 0; q0 < nq; q0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          vb[u] = (live && q0 + 8 + u < nq) ? __ldcg(sn4 + q0 + 8 + u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i0 = 4 * (q0 + u);
          if (i0 >= nk) break;                                      // warp-uniform
          if (TM && i0 < A.tmc) A.st4(i0, va[u]);                   // tmc % 4 == 0 or tmc == n
          else {
            if (i0 + 0 < nk) A.st(i0 + 0, va[u].x);
            if (i0 + 1 < nk) A.st(i0 + 1, va[u].y);
            if (i0 + 2 < nk) A.st(i0 + 2, va[u].z);
            if (i0 + 3 < nk) A.st(i0 + 3, va[u].w);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) va[u] = vb[u];
      }
    }
    for (int b = 0; b < 32; ++b) E[32 * b + lane] = (ET)0;
    __syncwarp();
    const uint32_t* brow = cw + p.brow + g * G;                     // S row 32g, row form
    int64_t costL = 0;
    uint4 cur = live ? __ldcg(sn4 + nq - 1) : make_uint4(0u, 0u, 0u, 0u);
    A.fence_st();
    uint32_t a_next = A.ld(nk - 1);
    // row 32g's word for the current 32-node block; the next block's word is prefetched
    uint32_t bword = (g > 0 && ((nq - 1) >> 3) < g && live) ? brow[(nq - 1) >> 3] : 0u;
    uint32_t bnext = (g > 0 && ((nq - 1) >> 3) >= 1 && ((nq - 1) >> 3) - 1 < g && live)
                         ? brow[((nq - 1) >> 3) - 1] : 0u;
    // the first quad's block word is bword; the walk reloads bword/bnext at block entries
    // (q & 7 == 7), so prime bnext with the current block for a block-aligned first quad
    if (((nq - 1) & 7) == 7) bnext = bword;
    if (!TM) {
      walk<ET, TM, 0>(nq - 1, 0, nk, g, live, sn4, brow, nrec, drec, M, C, A, E, lane, cur, a_next, bword,
                      bnext, costL);
    } else {
      const int qb = A.tmc >> 2;                                      // quads with k >= tmc: mixed
      if (nq - 1 >= qb)
        walk<ET, TM, 1>(nq - 1, qb, nk, g, live, sn4, brow, nrec, drec, M, C, A, E, lane, cur, a_next, bword,
                        bnext, costL);
      walk<ET, TM, 2>(min(nq - 1, qb - 1), 0, nk, g, live, sn4, brow, nrec, drec, M, C, A, E, lane, cur, a_next,
                      bword, bnext, costL);
    }
    // ---- group result: max_t (mass_t + E_t) over this group's stages, cost sum ----
    const int64_t* mass = reinterpret_cast<const int64_t*>(cw + block_words(G));
    int64_t mv[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) {                                  // issue all 32 loads first
      const int r = 32 * g + b;
      mv[b] = (r && r < n && live) ? __ldcg(mass + r) : 0;
    }
    int64_t pk = INT64_MIN;
#pragma unroll
    for (int b = 0; b < 32; ++b)
      if (32 * g + b < n) pk = max(pk, mv[b] + (int64_t)E[32 * b + lane]);
    if (live) {
      int64_t* pp = p.part + 2 * (c * G + g);
      pp[0] = pk;
      pp[1] = costL;
    }
    if (p.r_mask32 || p.s_mask32) {                                 // verification output
      A.fence_st();
      __syncwarp();
      const int W32 = 2 * ((n + 63) >> 6);
      uint32_t* scratch = reinterpret_cast<uint32_t*>(E);             // E is dead: [32 nodes][32 lanes]
      for (int w = 0; w <= g; ++w) {
        for (int j = 0; j < 32; ++j) {
          const int node = 32 * w + j;
          scratch[32 * j + lane] = node < nk ? A.ld(node) : 0u;      // R column, own candidate
        }
        __syncwarp();
        for (int cl = 0; cl < 32; ++cl) {
          const int64_t cc = (int64_t)(task % p.n_batch) * 32 + cl;
          if (cc >= p.n_cand) break;                                // warp-uniform
          const uint32_t* ccw = p.ws + cc * p.cs;
          const int row = 32 * g + lane;
          const int node = 32 * w + lane;
          const uint32_t rc = scratch[32 * lane + cl];
          uint32_t sc = node < nk ? ccw[grp_off(g) + node] : 0u;
          const uint32_t bb = (g > 0 && w < g) ? ccw[p.brow + g * G + w] : 0u;
          sc = (sc << 1) | ((bb >> lane) & 1u);
          const uint32_t xr = transpose32(rc, lane);
          const uint32_t xs = transpose32(sc, lane);
          if (row < n) {
            const size_t o = ((size_t)(p.out_base + cc) * n + row) * W32;
            if (p.r_mask32) p.r_mask32[o + w] = xr;
            if (p.s_mask32) p.s_mask32[o + w] = xs;
          }
        }
        __syncwarp();
      }
      const int row = 32 * g + lane;                                // zero the words above the block diagonal
      for (int cl = 0; cl < 32; ++cl) {
        const int64_t cc = (int64_t)(task % p.n_batch) * 32 + cl;
        if (cc >= p.n_cand || row >= n) break;
        const size_t o = ((size_t)(p.out_base + cc) * n + row) * W32;
        for (int w = g + 1; w < W32; ++w) {
          if (p.r_mask32) p.r_mask32[o + w] = 0u;
          if (p.s_mask32) p.s_mask32[o + w] = 0u;
        }
      }
    }
    __syncwarp();
  }
  if (TM) {
    A.fence_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem_base) : "memory");
  }
}

// ------------------------------------------------------------------------------------ K3
// Per candidate: peak = ovh + max_g part_peak, cost = sum_g part_cost; then the a7 keys.
struct ReduceParams {
  const int64_t* part;
  int32_t G;
  int64_t n_cand, out_base, index_base;
  int64_t ovh, mscale;        // peak = ovh + mscale * max_g part
  int32_t idx_bits, n_budget;
  const int64_t* budget;
  int64_t* peak;
  int64_t* cost;
  int64_t* best_key;
};

__global__ void __launch_bounds__(256) reduce_kernel(const ReduceParams p) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p.n_cand) return;
  const int64_t* pp = p.part + 2 * c * p.G;
  int64_t pk = INT64_MIN, cs = 0;
  for (int g = 0; g < p.G; ++g) {
    pk = max(pk, __ldcg(pp + 2 * g));
    cs += __ldcg(pp + 2 * g + 1);
  }
  pk = p.ovh + p.mscale * pk;
  const int64_t local = p.out_base + c;
  p.peak[local] = pk;
  p.cost[local] = cs;
  const int64_t key = (cs << p.idx_bits) | (p.index_base + local);
  for (int b = 0; b < p.n_budget; ++b) {
    if (pk <= __ldg(p.budget + b)) {
      const int64_t cur = *reinterpret_cast<volatile const int64_t*>(p.best_key + b);
      if (key < cur) atomicMin(reinterpret_cast<long long*>(p.best_key + b), (long long)key);
    }
  }
}

}  // namespace cm2

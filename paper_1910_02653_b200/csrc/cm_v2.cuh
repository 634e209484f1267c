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
  int32_t evict_first;        // S* loads with an L2 evict-first policy
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
// S* is read exactly once: the loads carry an L2 evict-first policy so the stream does not
// push the K1 -> K2 workspace out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      :: "r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* ptr) {
  asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(ptr));
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
// Warps per CTA, TMA stages per warp and the register cap depend on NT: with one threshold
// K1 runs 12 warps x 3 stages at <= 80 registers (30k registers, ~150 KB), so it still
// co-resides with the TMEM scan CTA (8 warps x 128 registers, ~50 KB) while hiding more latency.
#ifndef CM_K1_WARPS1
#define CM_K1_WARPS1 8
#endif
#ifndef CM_K1_STAGES1
#define CM_K1_STAGES1 2
#endif
#ifndef CM_K1_REGS1
#define CM_K1_REGS1 128
#endif
__host__ __device__ constexpr int k1_warps(int nt) { return nt == 1 ? CM_K1_WARPS1 : 8; }
__host__ __device__ constexpr int k1_stages(int nt) { return nt == 1 ? CM_K1_STAGES1 : 2; }
// Shared layout (bytes from a 1024-aligned base): tiles [warp][stage][32][32] f32 (4 KB each,
// 1024-byte aligned: the swizzle atom), mbarriers [warp][stage], NT column-word slots per warp
// (one per threshold, so the NT chains interleave), then the staged int32 mass tables.
__host__ __device__ constexpr size_t k1_bar_off(int nt) { return (size_t)k1_warps(nt) * k1_stages(nt) * 4096; }
__host__ __device__ constexpr size_t k1_cols_off(int nt) { return k1_bar_off(nt) + (size_t)k1_warps(nt) * k1_stages(nt) * 8; }
__host__ __device__ constexpr size_t k1_nib_off(int nt) { return k1_cols_off(nt) + (size_t)k1_warps(nt) * nt * 128; }
// dynamic bytes to request: + 1024 slack for aligning the base
__host__ __device__ constexpr size_t k1_smem_bytes(int nt, int nib_entries) {
  return k1_nib_off(nt) + 4 * (size_t)nib_entries + 1024;
}

// NT = thresholds per pass (1..4, a compile-time count so the per-threshold work of one block
// -- ballots, mass lookups, transposes -- forms NT independent instruction chains).
template <int NT>
__global__ void __maxnreg__(NT == 1 ? CM_K1_REGS1 : 128) round_tma_kernel(const RoundParams p, const __grid_constant__ CUtensorMap tmap) {
  constexpr int kSt = k1_stages(NT);
  extern __shared__ __align__(1024) unsigned char k1raw[];
  unsigned char* k1smem = k1raw + ((1024u - (smem_u32(k1raw) & 1023u)) & 1023u);
  int32_t* nib32 = reinterpret_cast<int32_t*>(k1smem + k1_nib_off(NT));   // p.nib32 staged (if any)
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  float(*tiles)[32][32] = reinterpret_cast<float(*)[32][32]>(k1smem) + kSt * wl;   // [stage]
  uint64_t* bars = reinterpret_cast<uint64_t*>(k1smem + k1_bar_off(NT)) + kSt * wl;
  uint32_t(*cols_w)[32] = reinterpret_cast<uint32_t(*)[32]>(k1smem + k1_cols_off(NT)) + NT * wl;
  const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int G = p.G;
  // row groups with a row r = 32g+1+l < n; the Sn columns of later groups are all zero
  // (S_{n+1} = 0) and K2 does not read them
  const int Gr = p.n >= 2 ? (p.n - 2) / 32 + 1 : 0;
  if (Gr == 0) return;
  if (p.nib32)
    for (int i = threadIdx.x; i < p.nib_entries; i += blockDim.x) nib32[i] = p.nib32[i];
  if (lane == 0)
    for (int st = 0; st < kSt; ++st) mbar_init(&bars[st], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  float th[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) th[j] = p.theta[p.th0 + j];
  const Transposer transpose(lane);
  const bool scaled32 = p.nib32 != nullptr;
  const uint32_t row_base = smem_u32(&tiles[0][lane][0]);            // stage 0, this lane's row
  const uint64_t pol = p.evict_first ? l2_evict_first_policy() : 0ull;
  const uint32_t swz = (uint32_t)(lane & 7) << 4;

  // Producer cursor (ps, pg, pw) runs kSt-1 blocks ahead of the consumer.  No proxy
  // fence before re-filling a stage: its previous contents were consumed (ballots issued on
  // the loaded values, then __syncwarp) before the refill is issued.
  int ps = wid, pg = 0, pw = 0, pstage = 0;
  auto issue = [&]() {
    if (ps >= p.s_count) return;
    if (lane == 0) {
      mbar_expect_tx(&bars[pstage], 32u * 32u * 4u);
      if (pol)
        tma_load_3d(&tiles[pstage][0][0], &tmap, 32 * pw, 32 * pg + 1, (int)(p.s_begin + ps), &bars[pstage], pol);
      else
        tma_load_3d(&tiles[pstage][0][0], &tmap, 32 * pw, 32 * pg + 1, (int)(p.s_begin + ps), &bars[pstage]);
    }
    pstage = pstage + 1 == kSt ? 0 : pstage + 1;
    if (++pw > pg) {
      pw = 0;
      if (++pg == Gr) { pg = 0; ps += nw; }
    }
  };
  for (int d = 0; d < kSt - 1; ++d) issue();

  int cstage = 0;
  uint32_t phase_bits = 0u;                                         // bit st = parity of stage st
  for (int s = wid; s < p.s_count; s += nw) {
    uint32_t* out = p.sn + ((int64_t)s * p.n_theta + p.th0) * p.cs;
    for (int g = 0; g < Gr; ++g) {
      const int rq = 32 * g + lane + 1;                             // row owned by this lane
      // rows of the group that exist (r < n): bits [0, hi)
      const int hi = p.n - 1 - 32 * g;
      const uint32_t rows_ok = hi >= 32 ? FULL : (hi <= 0 ? 0u : (1u << hi) - 1u);
      int64_t mass[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) mass[j] = 0;
      for (int w = 0; w <= g; ++w) {
        issue();
        mbar_wait(&bars[cstage], (phase_bits >> cstage) & 1u);
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
        cstage = cstage + 1 == kSt ? 0 : cstage + 1;
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
#ifndef CM_EXP_NOMASS
          word[j] = transpose(word[j]);                             // row rq's word over block w
#endif
          if (lane == 31 && g + 1 < G) oj[brow_at] = word[j];
        }
#ifdef CM_EXP_NOMASS
        if (false) {
#else
        if (scaled32) {                                             // scaled masses fit int32
#endif
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
//
// A'_i = Sn_i | Acc_i is kept only where it has to be: a node whose only user is i+1 (the
// "adjacent" edge i -> i+1) needs no storage -- its Acc is one register carried from step
// i+1 to step i.  Nodes with a non-adjacent user get a slot (host-assigned, nrec.w), slots
// < 256 in Tensor Memory, the rest in shared memory.  Per warp in shared memory: E[stage][lane]
// and the spilled slots [slot][lane].
struct ScanParams {
  const uint4* blob;          // M[n] int64, C[n] int64, pred_ptr, pred_idx, nrec, drec
  int32_t blob_bytes;
  int32_t n, o_pred_ptr, o_pred_idx;
  int32_t o_nrec, o_drec;     // byte offsets of the node / dependency records in the blob
  int32_t n_slot;             // nodes with a non-adjacent user
  int32_t o_qinfo;            // byte offset of the per-quad slot info (first slot | mask << 16)
  int32_t prefetch;           // L2-prefetch the warp's next task
  uint32_t* ws;               // chunk workspace from K1 (cs words per candidate)
  int32_t cs, G, brow;
  int64_t n_cand;             // candidates in this chunk
  int32_t n_batch;            // ceil(n_cand / 32)
  int64_t* part;              // out: [n_cand][G] x {peak_g - ovh, cost_g}
  uint32_t* r_mask32;         // optional masks (u64 words seen as pairs of u32)
  uint32_t* s_mask32;
  int64_t out_base;           // local index of the chunk's first candidate
  int32_t warp_bytes;         // shared bytes per warp region
};

// Slot storage of one warp.  TM = false: shared memory [slot][lane].  TM = true: slots < tmc
// live in Tensor Memory -- lane = TMEM lane (this warp's 32-lane quarter), slot = TMEM
// column, accessed with tcgen05.ld/st.32x32b (one column, all 32 lanes, uniform address)
// -- and slots >= tmc spill to shared memory.  A load after a store of the same column is
// ordered by tcgen05.wait::st (the walk tracks pending stores).
template <bool TM>
struct AView {
  uint32_t* sm;
  uint32_t taddr;
  int tmc;
  int lane;
  // MODE 0: shared only; 1: decide per access (slot < tmc -> TMEM); 2: TMEM only.
  template <int MODE>
  __device__ __forceinline__ bool in_tmem(int s) const { return TM && (MODE == 2 || (MODE == 1 && s < tmc)); }
  template <int MODE>
  __device__ __forceinline__ uint32_t ld_async(int s) const {   // TMEM: value valid after wait_ld()
    uint32_t v;
    if (in_tmem<MODE>(s))
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr + (uint32_t)s) : "memory");
    else
      v = sm[32 * (s - tmc) + lane];
    return v;
  }
  __device__ __forceinline__ void wait_ld(uint32_t& v) const {
    if (TM) asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v) :: "memory");
  }
  template <int MODE>
  __device__ __forceinline__ void st(int s, uint32_t v) const {
    if (in_tmem<MODE>(s))
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr + (uint32_t)s), "r"(v) : "memory");
    else
      sm[32 * (s - tmc) + lane] = v;
  }
  __device__ __forceinline__ void wait_st() const {
    if (TM) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // slots s..s+3, all in TMEM (TM, s + 3 < tmc)
  __device__ __forceinline__ void st4(int s, uint4 v) const {
    if (TM)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                   :: "r"(taddr + (uint32_t)s), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
};

// Events of one computing node k: for every stage bit b of R_k (stage b computes k), in the
// backward walk, first the frees at k (Eq. 9: the masks f_j with masses m_j, and the i = k
// self-free sf with M_k), then the compute: E_b = max(E_b - frees, 0) + M_k.  NM dependency
// masks (compile-time).  A round takes up to W stage bits of x (their loads issue together);
// the width follows the warp's largest per-lane event count (REDUX), so nodes whose lanes
// compute in one or two stages do not pay for four-wide rounds.
template <int W, int NM, typename ET>
__device__ __forceinline__ void event_round(uint32_t& x, uint32_t sf, ET Mk, const uint32_t* f, const ET* m,
                                            ET* E, int lane) {
  int b[W];
  bool v[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    v[u] = x != 0u;
    b[u] = v[u] ? __ffs(x) - 1 : 0;
    x &= x - 1;
  }
  ET ev[W];
#pragma unroll
  for (int u = 0; u < W; ++u) ev[u] = v[u] ? E[32 * b[u] + lane] : (ET)0;
#pragma unroll
  for (int u = 0; u < W; ++u) {
    if ((sf >> b[u]) & 1u) ev[u] -= Mk;
#pragma unroll
    for (int j = 0; j < NM; ++j)
      if ((f[j] >> b[u]) & 1u) ev[u] -= m[j];
    ev[u] = (ev[u] > 0 ? ev[u] : (ET)0) + Mk;
  }
#pragma unroll
  for (int u = 0; u < W; ++u)
    if (v[u]) E[32 * b[u] + lane] = ev[u];
}
template <int NM, typename ET>
__device__ __forceinline__ void events(uint32_t Rk, uint32_t sf, ET Mk, const uint32_t* f, const ET* m,
                                       ET* E, int lane) {
  const unsigned mx = __reduce_max_sync(FULL, (unsigned)__popc(Rk));
  uint32_t x = Rk;
  if (mx <= 1) event_round<1, NM, ET>(x, sf, Mk, f, m, E, lane);
  else if (mx == 2) event_round<2, NM, ET>(x, sf, Mk, f, m, E, lane);
  else
    while (__any_sync(FULL, x != 0u)) event_round<4, NM, ET>(x, sf, Mk, f, m, E, lane);
}

// The far (non-adjacent) dependencies of node k (NDF of them; NDF = 3 also walks any further
// ones, applying their frees first), the adjacent one (mask fa, mass ma; zero when absent),
// then the events.  drec[e] = {slot_i | i << 16, (int32) M_i}.
template <int NDF, typename ET, bool TM, int MODE>
__device__ __forceinline__ void node_step(uint32_t Rk, uint32_t sf, ET Mk, uint32_t fa, ET ma, int e0, int ndf,
                                          const int2* __restrict__ drec, const int64_t* __restrict__ M,
                                          const AView<TM>& A, ET* E, int lane, bool& st_pending) {
  uint32_t f[NDF + 1];
  ET m[NDF + 1];
  f[NDF] = fa;
  m[NDF] = ma;
  if (NDF > 0) {
    int sl[NDF > 0 ? NDF : 1];
    uint32_t ai[NDF > 0 ? NDF : 1];
#pragma unroll
    for (int j = 0; j < NDF; ++j) {
      const int2 d = drec[e0 + j];
      sl[j] = d.x & 0xffff;
      m[j] = sizeof(ET) == 4 ? (ET)d.y : (ET)M[d.x >> 16];
    }
    if (st_pending) A.wait_st();
#pragma unroll
    for (int j = 0; j < NDF; ++j) ai[j] = A.template ld_async<MODE>(sl[j]);
#pragma unroll
    for (int j = 0; j < NDF; ++j) A.wait_ld(ai[j]);
#pragma unroll
    for (int j = 0; j < NDF; ++j) {
      f[j] = Rk & ~ai[j];                                           // FREE_{t,i,k} = R_k & ~A'_i
      A.template st<MODE>(sl[j], ai[j] | Rk);                       // A'_i |= R_k
    }
    st_pending = true;
  }
  if (NDF == 3) {
    for (int e = e0 + 3; e < e0 + ndf; ++e) {                       // more far deps (rare)
      const int2 d = drec[e];
      const int s = d.x & 0xffff;
      A.wait_st();
      uint32_t ai = A.template ld_async<MODE>(s);
      A.wait_ld(ai);
      A.template st<MODE>(s, ai | Rk);
      const ET Mi = sizeof(ET) == 4 ? (ET)d.y : (ET)M[d.x >> 16];
      for (uint32_t fx = Rk & ~ai; fx; fx &= fx - 1) E[32 * (__ffs(fx) - 1) + lane] -= Mi;
    }
  }
  events<NDF + 1, ET>(Rk, sf, Mk, f, m, E, lane);
}

// Walk the quads q = q_hi .. q_lo (nodes 4q+3 .. 4q) of a group pass.
// nrec[k] = {(int32) M_k, e0, ndf | adj << 16, slot_k or -1}.
template <typename ET, bool TM, int MODE, bool RSTORE>
__device__ __forceinline__ void walk(int q_hi, int nk, int g, bool live, bool lsn, const uint4* sn4, uint32_t* rcol,
                                     const uint32_t* brow, const int4* __restrict__ nrec,
                                     const int2* __restrict__ drec, const int64_t* __restrict__ M,
                                     const int64_t* __restrict__ C, const AView<TM>& A, ET* E, int lane,
                                     int64_t& costL) {
  uint4 cur = lsn ? __ldcg(sn4 + q_hi) : make_uint4(0u, 0u, 0u, 0u);
  // row 32g's word for the current 32-node block; the next block's word is prefetched
  uint32_t bword = (g > 0 && (q_hi >> 3) < g && live) ? brow[q_hi >> 3] : 0u;
  uint32_t bnext = (g > 0 && (q_hi >> 3) >= 1 && (q_hi >> 3) - 1 < g && live) ? brow[(q_hi >> 3) - 1] : 0u;
  if ((q_hi & 7) == 7) bnext = bword;      // a block-aligned first quad reloads at entry
  int4 rec1 = nrec[nk - 1];                                         // record of the next node
  uint32_t acc = 0u;                                                // Acc_k from user k+1
  uint32_t bslot = 0u;                                              // A'_k base when k has a slot
  bool st_pending = true;                                           // init stores precede
  if (rec1.w >= 0) {
    A.wait_st();
    bslot = A.template ld_async<MODE>(rec1.w);
    A.wait_ld(bslot);
    st_pending = false;
  }
  for (int q = q_hi; q >= 0; --q) {
    const uint4 nxt = (q > 0 && lsn) ? __ldcg(sn4 + q - 1) : make_uint4(0u, 0u, 0u, 0u);
    if ((q & 7) == 7) {                                             // entered a new 32-node block
      bword = bnext;
      const int wb = (q >> 3) - 1;
      bnext = (g > 0 && wb >= 0 && wb < g && live) ? brow[wb] : 0u;
    }
#pragma unroll
    for (int u = 3; u >= 0; --u) {
      const int k = 4 * q + u;
      if (k >= nk) continue;                                        // warp-uniform
      const int4 rec = rec1;
      rec1 = k > 0 ? nrec[k - 1] : make_int4(0, 0, 0, -1);
      const int64_t Ck = C[k];
      const uint32_t sn = u == 3 ? cur.w : u == 2 ? cur.z : u == 1 ? cur.y : cur.x;
      const uint32_t sn1 = u == 3 ? cur.z : u == 2 ? cur.y : u == 1 ? cur.x : nxt.w;   // Sn_{k-1}
      const uint32_t a = (rec.w >= 0 ? bslot : sn) | acc;           // A'_k, complete
      const uint32_t sw = (sn << 1) | ((bword >> (k & 31)) & 1u);   // S_t from S_{t+1} and row 32g
      const uint32_t diag = ((k >> 5) == g) ? (1u << (k & 31)) : 0u;
      const uint32_t Rk = (a & ~sw) | diag;                         // a2 seed + a3 closure
      if (RSTORE && live) rcol[k] = Rk;                             // verification output
      // base of A'_{k-1}: its slot (final: every far user j > k is done; the adjacent user k
      // contributes through acc) or Sn_{k-1}
      uint32_t b1 = sn1;
      if (rec1.w >= 0) {
        if (st_pending) { A.wait_st(); st_pending = false; }
        b1 = A.template ld_async<MODE>(rec1.w);
      }
      acc = 0u;
      if (__any_sync(FULL, Rk != 0u)) {                             // computed in some lane
        const ET Mk = sizeof(ET) == 4 ? (ET)rec.x : (ET)M[k];
        costL += (int64_t)__popc(Rk) * Ck;
        const bool adj = (rec.z >> 16) != 0;
        if (rec1.w >= 0) A.wait_ld(b1);
        const uint32_t fa = adj ? Rk & ~b1 : 0u;                    // FREE_{t,k-1,k}
        const ET ma = sizeof(ET) == 4 ? (ET)rec1.x : (k > 0 ? (ET)M[k - 1] : (ET)0);
        if (adj) acc = Rk;                                          // Acc_{k-1} |= R_k
        const uint32_t sf = Rk & ~a;                                // FREE_{t,k,k}
        const int ndf = rec.z & 0xffff;
        switch (ndf) {                                              // warp-uniform
          case 0: node_step<0, ET, TM, MODE>(Rk, sf, Mk, fa, ma, rec.y, ndf, drec, M, A, E, lane, st_pending); break;
          case 1: node_step<1, ET, TM, MODE>(Rk, sf, Mk, fa, ma, rec.y, ndf, drec, M, A, E, lane, st_pending); break;
          case 2: node_step<2, ET, TM, MODE>(Rk, sf, Mk, fa, ma, rec.y, ndf, drec, M, A, E, lane, st_pending); break;
          default: node_step<3, ET, TM, MODE>(Rk, sf, Mk, fa, ma, rec.y, ndf, drec, M, A, E, lane, st_pending); break;
        }
      } else if (rec1.w >= 0) {
        A.wait_ld(b1);
      }
      bslot = b1;
    }
    cur = nxt;
  }
}

// Write one 32x32 mask block set (rows 32g..32g+31 of the 32 candidates of the task) from
// column words: col(cl, node) for candidate cl of the batch.  S: S_t words from the Sn columns
// and row 32g (brow); R: the R columns the walk stored over the Sn columns.
template <bool IS_S>
__device__ void emit_mask(const ScanParams& p, uint32_t* out, int g, int nk, int64_t batch0, int lane,
                          uint32_t* scratch) {
  const int n = p.n, G = p.G;
  const int W32 = 2 * ((n + 63) >> 6);
  const int row = 32 * g + lane;
  for (int cl = 0; cl < 32; ++cl) {
    const int64_t cc = batch0 + cl;
    if (cc >= p.n_cand) break;                                      // warp-uniform
    const uint32_t* ccw = p.ws + cc * p.cs;
    for (int w = 0; w <= g; ++w) {
      const int node = 32 * w + lane;
      uint32_t sc = node < nk && (!IS_S || 32 * g + 1 < n) ? ccw[grp_off(g) + node] : 0u;
      if (IS_S) {
        const uint32_t bb = (g > 0 && w < g) ? ccw[p.brow + g * G + w] : 0u;
        sc = (sc << 1) | ((bb >> lane) & 1u);
      }
      const uint32_t x = transpose32(sc, lane);
      if (row < n) out[((size_t)(p.out_base + cc) * n + row) * W32 + w] = x;
    }
    if (row < n)
      for (int w = g + 1; w < W32; ++w) out[((size_t)(p.out_base + cc) * n + row) * W32 + w] = 0u;
  }
  (void)scratch;
}

// ET = int32_t when every M is a multiple of a scale s with sum M/s < 2^30 (the host checks;
// exact), else int64_t.  M in the blob, the masses and the results are in units of s.
// TM: slots < 256 in Tensor Memory (8 warps, one CTA per SM, 512 TMEM columns: warp w uses
// lane quarter w % 4 and columns 256 * (w / 4) ..).
template <typename ET, bool TM>
__global__ void __launch_bounds__(256, 2) scan_kernel(const ScanParams p) {   // <= 128 regs: co-resides with K1
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = p.n, G = p.G;
  const int64_t* M = reinterpret_cast<const int64_t*>(smem);
  const int64_t* C = M + n;
  const int4* nrec = reinterpret_cast<const int4*>(smem + p.o_nrec);
  const int2* drec = reinterpret_cast<const int2*>(smem + p.o_drec);
  const int32_t* qinfo = reinterpret_cast<const int32_t*>(smem + p.o_qinfo);
  unsigned char* wr = smem + p.blob_bytes + (size_t)warp * p.warp_bytes;
  ET* E = reinterpret_cast<ET*>(wr);                               // [32 stages][32 lanes]
  uint32_t* Asm = reinterpret_cast<uint32_t*>(E + 32 * 32);         // [slot][lane] (spill part)
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
  A.tmc = TM ? min(p.n_slot, 256) : 0;
  A.taddr = TM ? tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2) : 0u;
  const bool all_tm = TM && p.n_slot <= 256;

  const int tasks = G * p.n_batch;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int task = gw; task < tasks; task += nwarps) {
    const int g = G - 1 - task / p.n_batch;                         // big groups first
    const int64_t batch0 = (int64_t)(task % p.n_batch) * 32;
    const int64_t c = batch0 + lane;
    const bool live = c < p.n_cand;
    const int nk = min(n, 32 * (g + 1));                            // nodes 0..nk-1
    const int nq = (nk + 3) >> 2;                                   // uint4 blocks of Sn
    uint32_t* cw = p.ws + (live ? c : 0) * p.cs;
    const uint4* sn4 = reinterpret_cast<const uint4*>(cw + grp_off(g));
    const bool lsn = live && 32 * g + 1 < n;                        // K1 wrote Sn for this group
    {  // pull the warp's next task (Sn columns, row-32g words, masses) towards L2 meanwhile
      const int tn = task + nwarps;
      if (p.prefetch && tn < tasks) {
        const int gn = G - 1 - tn / p.n_batch;
        const int64_t cn = (int64_t)(tn % p.n_batch) * 32 + lane;
        if (cn < p.n_cand) {
          const unsigned char* b = reinterpret_cast<const unsigned char*>(p.ws + cn * p.cs);
          const unsigned char* col = b + 4 * (size_t)grp_off(gn);
          if (32 * gn + 1 < n) {                                    // the group has Sn columns
            for (int off = 0; off < 128 * (gn + 1); off += 128) prefetch_l2(col + off);
            prefetch_l2(col + 128 * (gn + 1) - 4);                  // the block is 16-byte aligned
          }
          prefetch_l2(b + 4 * ((size_t)p.brow + (size_t)gn * G));
          const unsigned char* ms = b + 4 * (size_t)block_words(G) + 8 * (size_t)(32 * gn);
          prefetch_l2(ms);
          prefetch_l2(ms + 128);
          prefetch_l2(ms + 255);
        }
      }
    }
    if (p.s_mask32) emit_mask<true>(p, p.s_mask32, g, nk, batch0, lane, nullptr);   // before R overwrites
    // slots: A'_i = Sn_i (Acc_i = 0) for the slotted nodes of the pass.  qinfo[q] = first slot
    // of quad q | (4-bit mask of its slotted nodes) << 16 (slots ascend with the node index).
    {  // software-pipelined: the loads of 8 quads are in flight while the previous 8 are stored
      uint4 va[8], vb[8];
      int qa[8], qb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        va[u] = (lsn && u < nq) ? __ldcg(sn4 + u) : make_uint4(0u, 0u, 0u, 0u);
        qa[u] = u < nq ? qinfo[u] : 0;
      }
      for (int q0 = 0; q0 < nq; q0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          vb[u] = (lsn && q0 + 8 + u < nq) ? __ldcg(sn4 + q0 + 8 + u) : make_uint4(0u, 0u, 0u, 0u);
          qb[u] = q0 + 8 + u < nq ? qinfo[q0 + 8 + u] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i0 = 4 * (q0 + u);
          if (i0 >= nk) break;                                      // warp-uniform
          const uint32_t wv[4] = {va[u].x, va[u].y, va[u].z, va[u].w};
          int s = qa[u] & 0xffff;
          const int msk = (qa[u] >> 16) & (i0 + 4 <= nk ? 15 : (1 << (nk - i0)) - 1);
          if (msk == 15 && all_tm) {                                // four consecutive slots
            A.st4(s, va[u]);
            continue;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if ((msk >> j) & 1) {
              if (!TM) A.template st<0>(s, wv[j]);
              else if (all_tm) A.template st<2>(s, wv[j]);
              else A.template st<1>(s, wv[j]);
              ++s;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          va[u] = vb[u];
          qa[u] = qb[u];
        }
      }
    }
    for (int b = 0; b < 32; ++b) E[32 * b + lane] = (ET)0;
    __syncwarp();
    const uint32_t* brow = cw + p.brow + g * G;                     // S row 32g, row form
    int64_t costL = 0;
    uint32_t* rcol = cw + grp_off(g);
    if (p.r_mask32) {
      if (!TM) walk<ET, TM, 0, true>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
      else if (all_tm) walk<ET, TM, 2, true>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
      else walk<ET, TM, 1, true>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
    } else {
      if (!TM) walk<ET, TM, 0, false>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
      else if (all_tm) walk<ET, TM, 2, false>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
      else walk<ET, TM, 1, false>(nq - 1, nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL);
    }
    A.wait_st();                                                    // next task re-fills the slots
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
    if (p.r_mask32) {
      __syncwarp();
      __threadfence_block();
      emit_mask<false>(p, p.r_mask32, g, nk, batch0, lane, nullptr);
    }
    __syncwarp();
  }
  if (TM) {
    A.wait_st();
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

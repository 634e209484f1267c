// cm_v2.cuh -- stage-sliced sm_100a kernels for Checkmate two-phase rounding (Alg. 2,
// PAPER.md:389-415) and the Eq. 6-9 memory accounting.
//
// "Stage-sliced": a 32-bit word holds one node's bit for 32 consecutive stages (group g =
// rows 32g..32g+31, 0-based row r = stage t-1), so every bitwise step of the method runs for
// 32 stages at once, and a warp takes lane = candidate with the same group in all lanes: the
// control flow (a walk over the graph) is uniform however recomputation is distributed.
//
// K1 body (k1_body; HBM-bound), per S*: for each 32x32 block (g, w <= g) -- rows 32g+1+l,
//   nodes 32w.. -- lane l reads its row from a TMA-staged tile, packs x > theta (a1,
//   strict, fp32, NaN -> 0) into its row word, adds the row's checkpoint mass
//   (the Eq. 6 sum) from 4-bit tables, and a 5-step shuffle transpose gives the column words
//       Sn_g[i]  bit b = S_{row 32g+b+1, node i} = S_{t+1}   for stage t = 32g+b+1,
//   i.e. the NEXT stage's checkpoint bits (S_{n+1} = 0).  The current stage's
//   bits follow from them and row 32g's word (brow).  One S* read serves up to 4 thresholds
//   (or 4 random samples, RAND: Philox4x32-10, one block per 4 nodes and sample, R1).
//
// K2 task (scan_task; latency / ALU-bound), per (group g, 32 candidates): one pass over nodes
//   k = nk-1 .. 0 (reverse topological order, the paper's right-to-left scan):
//     R_k   = ((Sn_k | Acc_k) & ~Sw_k) | diag_k      a2 seed S_{t+1} & ~S_t, e_t; a3 closure
//             Acc_k = OR of R_j over the users j > k (all visited before k)
//     FREE  i in DEPS(k): R_k & ~Sn_i & ~Acc_i       Eq. 9: k computed, i not kept, no later user
//           i = k:        R_k & ~Sn_k & ~Acc_k       the i = k term of Eq. 8
//     Acc_i |= R_k
//   Memory: with D = U_{t,k} - U_{t,end} run backwards and MX = max over computes of D,
//   only E = MX - D matters:  frees:  E -= M_i ;  compute of k:  E = max(E, 0) + M_k.
//   Then peak_t = U_{t,0} + E_t (the max over k is reached at a compute,
//   DESIGN.md Q9), with U_{t,0} = ovh + mass_t (Eq. 6) from K1.
//
// Reduce (reduce_one): per candidate max / sum over groups, the a7 per-budget keys and the
//   optional max-batch keys.
//
// Kernels: fused_kernel (one persistent launch; K1 warps and K2 warps per CTA, hand-off through
// a ring in global memory -- the default path), or round_tma_kernel + scan_kernel +
// reduce_kernel on two streams (the two-kernel pipeline: > 4 thresholds, randomized rounding
// with the int64 state, or no shared-memory / TMEM fit).
//
// Build-time switches: tuning (CM_K1_WARPS1, CM_K1_STAGES1, CM_K1_REGS1, CM_KF2,
// CM_DIAG_BULK, CM_DIAG_SPLIT) and timing experiments that break the results on purpose
// (CM_EXP_L2INPUT: every S* read from 64 L2-resident ones; CM_EXP_NOSCAN: no walks;
// CM_EXP_NOFENCE: no hand-off fences) -- tools/build_variant.py builds them into tune/.
//
// Layout of one candidate block: group g's Sn columns (nodes 0..32g+31) at word offset
// grp_off(g) = 16 g (g+1) (whole 128-byte lines), then the masses, then brow.
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
// m32: the masses are int32 (the int32 scan state: every row mass fits), else int64.
__host__ __device__ __forceinline__ int mass_words(int n, bool m32) { return m32 ? ((n + 31) & ~31) : 2 * n; }
__host__ __device__ __forceinline__ int cand_words(int n, bool m32) {
  const int G = (n + 31) / 32;
  return (block_words(G) + mass_words(n, m32) + G * G + 3) & ~3;
}
__host__ __device__ __forceinline__ int brow_off(int n, bool m32) { return block_words((n + 31) / 32) + mass_words(n, m32); }

__device__ __forceinline__ int64_t row_offset(int layout, int64_t ld, int r) {
  if (layout == 0) return (int64_t)r * ld;
  const int64_t q = r >> 2, m = r & 3;                     // sum_{r'<r} roundup4(r')
  return 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
}

// CM_LAYOUT_BLK, the blocked strict lower triangle (include/cm.h): row group g = rows
// 32g+1 .. 32g+h_g (h_g = min(32, n-1-32g)), blocks w = 0..g of 32 nodes, stored group after
// group, block after block, every block chunk-major (16-byte chunk c = nodes 32w+4c .. +3):
// off-diagonal blocks chunk c of row l at chunk h_g c + l, the diagonal block chunk c of rows
// l = 4c .. h_g-1 at chunk B_c + l - 4c.  So K1 lane l reads chunk c at 16 l + a per-chunk
// constant (an immediate offset for the full groups), and a quarter-warp's reads of one chunk
// are 8 consecutive 16-byte units (no bank conflict).  Every group but the last is full
// (h = 32): 128 g (g-1) + 144 g chunks precede group g.
__host__ __device__ __forceinline__ int blk_rows(int n, int g) { return min(32, n - 1 - 32 * g); }
__host__ __device__ __forceinline__ int blk_diag_chunks(int h) {
  int c = 0;
  for (int k = 0; k < 8; ++k) c += max(0, h - 4 * k);
  return c;
}
__host__ __device__ __forceinline__ int64_t blk_block_off(int g, int w, int h) {   // floats
  return 4 * (128 * (int64_t)g * (g - 1) + 144 * (int64_t)g) + (int64_t)32 * h * w;
}
__host__ __device__ __forceinline__ int64_t blk_size(int n) {                      // floats per S*
  if (n < 2) return 0;
  const int Gr = (n - 2) / 32 + 1, h = blk_rows(n, Gr - 1);
  return blk_block_off(Gr - 1, Gr - 1, h) + 4 * (int64_t)blk_diag_chunks(h);
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
      uint32_t y;                                                   // (inline: no divergence check)
      asm volatile("shfl.sync.bfly.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(y) : "r"(x), "r"(16 >> k));
      const uint32_t t = __funnelshift_l(y, y, sh[k]);
      // x = (x & K) | (t & ~K) as ONE lop3 (left to itself ptxas splits it into three)
      asm("lop3.b32 %0, %0, %1, %2, 0xE4;" : "+r"(x) : "r"(t), "r"(K[k]));
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
  // randomized rounding (R1): S = u < S*, u from Philox4x32-10 with counter
  // (node / 4, row, global S* index, sample) and key (key0, key1), word node % 4; sample j = th0 + j
  uint32_t key0, key1;
  uint32_t s0;                // global index of batch S* 0 (mod 2^32)
  int32_t g4;                 // tri4: tile::gather4 through the 16-byte-unit tensor map (else per-row copies)
  int64_t g4_end;             // batch-relative: S* from here on take per-row copies (window past the end)
  int32_t rtab;               // RAND, fused blocked path: bytes per K1 warp of the per-S* Philox table (0: none)
};

// w |= (x[q] > th) << q for q = Q0 .. Q0+15 (strict fp32 compare, NaN -> 0): a setp and a
// predicated or per element, which ptxas emits as FSETP + @P VIADD (the bits are disjoint).
template <int Q>
__device__ __forceinline__ void pack_gt1(uint32_t& w, float v, float th) {
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
      : "+r"(w) : "f"(v), "f"(th), "n"(1u << Q));
}
template <int Q0, int K = 0>
__device__ __forceinline__ void pack_gt(uint32_t& w, const float* x, float th) {
  if constexpr (K < 16) {
    pack_gt1<Q0 + K>(w, x[Q0 + K], th);
    pack_gt<Q0, K + 1>(w, x, th);
  }
}

// The same 32 compares with packed fp32: d = theta - x by FADD2 (sub.rn.f32x2, no flush to zero)
// for a pair of elements, and x > theta  <=>  sign(d) = 1: the rounded difference keeps the
// exact difference's sign (denormals are kept), x = theta gives +0, NaN gives the canonical
// NaN 0x7fffffff (sign 0), and theta is +0 rather than -0 (the caller adds 0.0f: -0 - (+0) =
// -0 would set the bit for x = +0).  Each sign bit is funnel-shifted into the word (SHF): 1.5
// instructions per element instead of 2.  Bit q of the word = element q; two chains (q >= 16,
// q < 16) for ILP.  tt = theta in both halves.
__device__ __forceinline__ uint32_t pack_sub(const uint64_t (&xp)[16], uint64_t tt) {
  uint32_t hi = 0u, lo = 0u;
#pragma unroll
  for (int k = 15; k >= 8; --k) {
    uint64_t d, e;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(tt), "l"(xp[k]));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(e) : "l"(tt), "l"(xp[k - 8]));
    hi = __funnelshift_l((uint32_t)(d >> 32), hi, 1);                // element 2k+1
    hi = __funnelshift_l((uint32_t)d, hi, 1);                        // element 2k
    lo = __funnelshift_l((uint32_t)(e >> 32), lo, 1);                // element 2k-15
    lo = __funnelshift_l((uint32_t)e, lo, 1);                        // element 2k-16
  }
  return (hi << 16) | lo;
}

// Philox4x32-10 (Salmon et al., SC'11); the uniform is (word >> 8) * 2^-24, exact in fp32.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;             // one IMAD.WIDE.U32 each
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
  }
  return c;
}
__device__ __forceinline__ float uniform24(uint32_t w) { return (float)(w >> 8) * 5.9604644775390625e-8f; }

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
// 1-D bulk copy global -> shared (SASS UBLKCP): `bytes` % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// tile::gather4 (sm_100a): four rows y0..y3 of a 2-D tensor map, box {32, 1}, into dst.
__device__ __forceinline__ void tma_gather4(uint32_t dst, const void* tmap, int y0, int y1, int y2, int y3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"(dst), "l"(tmap), "r"(0), "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(smem_u32(bar)) : "memory");
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
// TMA stages per rounding warp (one threshold).  Measured with overlapped calls, 2 -> 3:
// ResNet-50 19.5 -> 19.86, U-Net 46.2 -> 49.5, MobileNet 14.7 -> 15.4 M cand/s (4: 19.77)
#ifndef CM_K1_STAGES1
#define CM_K1_STAGES1 3
#endif
#ifndef CM_K1_REGS1
#define CM_K1_REGS1 128
#endif
__host__ __device__ constexpr int k1_warps(int nt) { return nt == 1 ? CM_K1_WARPS1 : 8; }
// (2+ thresholds / samples: 3 stages measured 8.60 vs 8.70 M cand/s at 4 samples -- ALU-bound)
#ifndef CM_K1_STAGESN
#define CM_K1_STAGESN 2
#endif
__host__ __device__ constexpr int k1_stages(int nt) { return nt == 1 ? CM_K1_STAGES1 : CM_K1_STAGESN; }
// Shared layout (bytes from a 1024-aligned base): tiles [warp][stage][32][32] f32 (4 KB each,
// 1024-byte aligned: the swizzle atom), mbarriers [warp][stage], NT column-word slots per warp
// (one per threshold, so the NT chains interleave), then the staged int32 mass tables.
// A stage holds one 32 x 32 block.  TMA (dense): 4 KB, 128-byte swizzled rows.  BULK (tri4):
// rows at a 144-byte pitch (one 16-byte chunk of skew per row), so lane l reading 16-byte
// chunk c of its row hits bank group (l + c) % 8: conflict-free without a swizzle.
constexpr int kBulkPitch = 144;
// tri4 (bulk): 5 KB so a stage holds either the swizzled 4 KB gather4 tile (1024-aligned) or
// the 144-byte-pitch per-row form of the fallback.
__host__ __device__ constexpr size_t k1_stage_bytes(bool bulk) { return bulk ? 5120 : 4096; }
__host__ __device__ constexpr size_t k1_bar_off(int nt, bool bulk = false) {
  return ((size_t)k1_warps(nt) * k1_stages(nt) * k1_stage_bytes(bulk) + 1023) & ~(size_t)1023;
}
__host__ __device__ constexpr size_t k1_cols_off(int nt, bool bulk = false) {
  return k1_bar_off(nt, bulk) + (size_t)k1_warps(nt) * k1_stages(nt) * 8;
}
// (512-byte aligned: a block's 8 x 16-entry int32 table is one 512-byte run, so an entry's
// address is table | (nibble << 2) plus an immediate 64 q -- one LOP3 per lookup)
__host__ __device__ constexpr size_t k1_nib_off(int nt, bool bulk = false) {
  return (k1_cols_off(nt, bulk) + (size_t)k1_warps(nt) * nt * 128 + 511) & ~(size_t)511;
}
// the Philox tables [K1 warp][rtab bytes], after the staged mass tables
__host__ __device__ constexpr size_t k1_rtab_off(int nt, int nib_entries, bool bulk) {
  return (k1_nib_off(nt, bulk) + 4 * (size_t)nib_entries + 15) / 16 * 16;
}
// dynamic bytes to request: + 1024 slack for aligning the base
__host__ __device__ constexpr size_t k1_smem_bytes(int nt, int nib_entries, bool bulk = false) {
  return k1_nib_off(nt, bulk) + 4 * (size_t)nib_entries + 1024;
}

// NT = thresholds per pass (1..4, a compile-time count so the per-threshold work of one block
// -- ballots, mass lookups, transposes -- forms NT independent instruction chains).
// BULK = false: dense layout, one 3-D tensor-map TMA per block (rows >= n zero-filled, 128-byte
// swizzle).  BULK = true: packed tri4 layout (row r at the float offset sum_{r'<r} roundup4(r'),
// not an affine map, so no tensor map): lane l issues one 1-D bulk copy of its own row's
// segment, nodes 32w .. min(32w+32, roundup4(r))-1 -- exactly the stored strict-lower entries
// (plus < 4 floats of row padding), so the HBM stream is the algorithmic one.  Rows >= n are
// not copied; whatever a stage holds outside the copied segments is masked away below (cmask).
// Where K1 writes candidate block (S* s, threshold th0 + j): begin(s) gives the block of
// threshold th0 (blocks of one S* are consecutive, cs words each) and end(s) runs after every
// word of S* s is written.  K1Plain: the chunk buffer of the two-kernel pipeline.
// first() / next(s) give the S* a warp processes, in order (K1Plain: a static stride).
struct K1Plain {
  static constexpr bool kTab = false;                             // no per-S* Philox table (rtab)
  uint32_t* sn;
  int32_t n_theta, th0, cs;
  int32_t wid, nw;
  __device__ __forceinline__ int first() const { return wid; }
  __device__ __forceinline__ int next(int s) const { return s + nw; }
  __device__ __forceinline__ uint32_t* begin(int s) const { return sn + ((int64_t)s * n_theta + th0) * cs; }
  __device__ __forceinline__ void end(int) const {}
};

// Per-CTA K1 set-up (staged mass table, mbarriers); the caller synchronises the CTA after it.
template <int NT, int LAY, bool RAND>
__device__ __forceinline__ void k1_setup(const RoundParams& p, unsigned char* k1smem, int nwarps1, int tid,
                                         int nthreads) {
  constexpr bool BULK = LAY == 1;
  constexpr int kSt = k1_stages(NT);
  int32_t* nib32 = reinterpret_cast<int32_t*>(k1smem + k1_nib_off(NT, BULK));
  if (p.nib32)
    for (int i = tid; i < p.nib_entries; i += nthreads) nib32[i] = p.nib32[i];
  uint64_t* bars = reinterpret_cast<uint64_t*>(k1smem + k1_bar_off(NT, BULK));
  if (tid < nwarps1 * kSt) mbar_init(&bars[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Dense diagonal blocks (w = g): the full {32, 32} box through a map without L2 promotion (the
// rows end inside the block).  Measured: reading only the rows' stored prefixes (boxes of 8x8,
// 16x8 and 32x16 nodes x rows, 2 816 instead of 4 096 bytes) cut the L2 -> SM bytes by 14 KB
// per S* but not one DRAM byte -- a missed 32-byte sector brings its whole 128-byte line from
// DRAM -- and cost 4 % more instructions; the blocked layout (CM_LAYOUT_BLK) removes the bytes.
struct DiagMaps {
  CUtensorMap diag;    // box {32 nodes, 32 rows}, SWIZZLE_128B, no promotion
};

// a1 word of one 32 x 32 block (row r = rq of this lane, nodes 32w ..): randomized rounding
// (R1): sample th0 + j of node i-1 = 32w + q in row rq is word q % 4 of the Philox
// block with counter (8w + q / 4, rq, global S* index, th0 + j): one block per four
// consecutive nodes and sample, and S = [w 2^-32 < x] exactly.  With X = x 2^32 (exact: a
// power-of-two scale; x > 2^96 or inf -> +inf, always; NaN stays NaN, never) and f = rz(w)
// (cvt.rz: the largest float <= w), [w < X] = [f < X] -- X is a float, so X <= w iff X <= f --
// and [f < X] = sign(f - X) in fp32: a nonzero difference of floats never rounds to 0, f = X
// gives +0, NaN the canonical NaN (sign 0).  Per element and sample: one I2FP, half a packed
// FADD2 (sub.rn.f32x2) and one funnel shift of the sign into the word; X once per element
// (half a packed FMUL2).  Two pack chains (elements 0..15 and 16..31); CM_RAND_ILP Philox
// blocks in flight.
#ifndef CM_RAND_ILP
#define CM_RAND_ILP 2
#endif
// KB Philox blocks advanced round by round together (independent chains side by side, so the
// IMAD.WIDE -> LOP3 latency of one chain is covered by the others)
template <int KB>
__device__ __forceinline__ void philox_xk(uint4 (&c)[KB], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0[KB], p1[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      p0[b] = (uint64_t)0xD2511F53u * c[b].x;
      p1[b] = (uint64_t)0xCD9E8D57u * c[b].z;
    }
#pragma unroll
    for (int b = 0; b < KB; ++b)
      c[b] = make_uint4((uint32_t)(p1[b] >> 32) ^ c[b].y ^ k0, (uint32_t)p1[b], (uint32_t)(p0[b] >> 32) ^ c[b].w ^ k1,
                        (uint32_t)p0[b]);
  }
}
// CM_RAND_CMP 1: the same exact compare in integers -- C = ceil(x 2^32) once per element
// (cvt.rpi.u32.f32 of the exact x 2^32, saturating: x <= 0 and NaN -> 0, never; x >= 1 ->
// 2^32 - 1, so [x >= 1] is OR-ed in from one packed compare against nextbelow(1)), and
// [w < C] = [w < x 2^32] since C is the least integer >= x 2^32.  Per sample the carry of
// w - C is shifted into the word (sub.cc + addc: one ALU IADD3 and one IMAD.X on the FMA pipe
// instead of I2FP + funnel shift; the F2I runs on the XU pipe once per element).  On sm_100a
// the carry after sub.cc is the no-borrow flag [w >= C] (the other polarity fails the parity
// tests), so the word is complemented.  Bit-exact (profiles r2aw, r2ax) but measured slower at
// 1 and 2 samples (9.68 / 9.99 vs 9.96 / 10.24 M cand/s) and +1 % at 4: off (0: fp32 sign form).
#ifndef CM_RAND_CMP
#define CM_RAND_CMP 0
#endif
// Philox4x32-10 rounds 3..9 (0-based) of KB blocks from the state after round 2 (k0, k1 the base key)
template <int KB>
__device__ __forceinline__ void philox_tail_xk(uint4 (&c)[KB], uint32_t k0, uint32_t k1) {
  k0 += 2u * 0x9E3779B9u;
  k1 += 2u * 0xBB67AE85u;
#pragma unroll
  for (int r = 3; r < 10; ++r) {
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
    uint64_t p0[KB], p1[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      p0[b] = (uint64_t)0xD2511F53u * c[b].x;
      p1[b] = (uint64_t)0xCD9E8D57u * c[b].z;
    }
#pragma unroll
    for (int b = 0; b < KB; ++b)
      c[b] = make_uint4((uint32_t)(p1[b] >> 32) ^ c[b].y ^ k0, (uint32_t)p1[b], (uint32_t)(p0[b] >> 32) ^ c[b].w ^ k1,
                        (uint32_t)p0[b]);
  }
}
// The per-S* Philox table (RoundParams::rtab): rounds 0-2 of a block depend on the lane only
// through its row rq (counter word 1, entering round 0 by XOR); the rest of rounds 0-2 depends
// on (node block w, q4, sample j) and the S* number, so each warp computes it once per S* for
// all (w, q4, j), lane-parallel: entry {w1 ^ k1_1, y2 ^ k0_2, hi(M0 x2) ^ k1_2, lo(M0 x2)} with
// (x1, y1, z1, w1) the round-0 output without the row, y2 = lo(M1 z1), x2 = hi(M1 z1) ^ y1 ^ k0_1.
// A lane then finishes round 1 with P = M0 x1 (x1 = hi(M1 S*) ^ row ^ k0, once per group) and
// round 2 with one IMAD.WIDE: z2 = hi(P) ^ A, x3 = hi(M1 z2) ^ B, y3 = lo(M1 z2), z3 = C ^ lo(P),
// w3 = D -- the same bits as the plain block (oracle R1), ~2 IMAD.WIDE and ~4 ALU ops fewer.
__device__ __forceinline__ void rand_table_build(uint32_t tab, int Gr, int NTs, uint32_t sg, const RoundParams& p) {
  const int lane = threadIdx.x & 31;
  const uint32_t k0 = p.key0, k1 = p.key1;
  const uint64_t q2 = (uint64_t)0xCD9E8D57u * sg;
  const uint32_t y1 = (uint32_t)q2;
  const int ne = Gr * 8 * NTs;
  for (int e = lane; e < ne; e += 32) {
    const int j = e % NTs, wq = e / NTs;                            // wq = 8 w + q4
    const uint64_t p0 = (uint64_t)0xD2511F53u * (uint32_t)wq;
    const uint32_t z1 = (uint32_t)(p0 >> 32) ^ (uint32_t)(p.th0 + j) ^ k1, w1 = (uint32_t)p0;
    const uint64_t q = (uint64_t)0xCD9E8D57u * z1;
    const uint32_t x2 = (uint32_t)(q >> 32) ^ y1 ^ (k0 + 0x9E3779B9u);
    const uint64_t r = (uint64_t)0xD2511F53u * x2;
    const uint32_t A = w1 ^ (k1 + 0xBB67AE85u), B = (uint32_t)q ^ (k0 + 2u * 0x9E3779B9u);
    const uint32_t C = (uint32_t)(r >> 32) ^ (k1 + 2u * 0xBB67AE85u), D = (uint32_t)r;
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(tab + 16u * (uint32_t)e), "r"(A), "r"(B), "r"(C), "r"(D)
                 : "memory");
  }
}
template <int NT, bool TAB = false>
__device__ __forceinline__ void rand_words(uint32_t (&word)[NT], const uint64_t (&xp)[16], int w, int rq, uint32_t sg,
                                           const RoundParams& p, uint32_t tab = 0u) {
  if constexpr (TAB) {                                              // the per-S* Philox table
    const uint64_t q2 = (uint64_t)0xCD9E8D57u * sg;
    const uint32_t x1 = (uint32_t)(q2 >> 32) ^ (uint32_t)rq ^ p.key0;
    const uint64_t P = (uint64_t)0xD2511F53u * x1;
    const uint32_t hP = (uint32_t)(P >> 32), lP = (uint32_t)P;
    uint64_t X[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(X[k]) : "l"(xp[k]), "l"(0x4f8000004f800000ull));
    auto pack4 = [&](uint32_t& acc, const uint4& o, int k0) {
      uint64_t f23, f01, d23, d01;
      asm("{\n\t.reg .f32 a, b;\n\tcvt.rz.f32.u32 a, %1;\n\tcvt.rz.f32.u32 b, %2;\n\tmov.b64 %0, {a, b};\n\t}"
          : "=l"(f23) : "r"(o.z), "r"(o.w));
      asm("{\n\t.reg .f32 a, b;\n\tcvt.rz.f32.u32 a, %1;\n\tcvt.rz.f32.u32 b, %2;\n\tmov.b64 %0, {a, b};\n\t}"
          : "=l"(f01) : "r"(o.x), "r"(o.y));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(f23), "l"(X[k0 + 1]));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(f01), "l"(X[k0]));
      acc = __funnelshift_l((uint32_t)(d23 >> 32), acc, 1);
      acc = __funnelshift_l((uint32_t)d23, acc, 1);
      acc = __funnelshift_l((uint32_t)(d01 >> 32), acc, 1);
      acc = __funnelshift_l((uint32_t)d01, acc, 1);
    };
    auto start = [&](int q4, int j) {                               // the state after round 2
      uint4 e;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                   : "r"(tab + 16u * (uint32_t)((8 * w + q4) * NT + j)));
      const uint32_t z2 = hP ^ e.x;
      const uint64_t p1 = (uint64_t)0xCD9E8D57u * z2;
      return make_uint4((uint32_t)(p1 >> 32) ^ e.y, (uint32_t)p1, e.z ^ lP, e.w);
    };
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      uint32_t hi = 0u, lo = 0u;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        uint4 o[2] = {start(q + 4, j), start(q, j)};
        philox_tail_xk<2>(o, p.key0, p.key1);
        pack4(hi, o[0], 2 * (q + 4));
        pack4(lo, o[1], 2 * q);
      }
      word[j] = (hi << 16) | lo;
    }
    return;
  }
  if constexpr (CM_RAND_CMP == 1) {
    uint32_t C[32];                                                 // ceil(x 2^32), saturated
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint64_t X;
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(X) : "l"(xp[k]), "l"(0x4f8000004f800000ull));
      asm("cvt.rpi.u32.f32 %0, %1;" : "=r"(C[2 * k]) : "f"(__uint_as_float((uint32_t)X)));
      asm("cvt.rpi.u32.f32 %0, %1;" : "=r"(C[2 * k + 1]) : "f"(__uint_as_float((uint32_t)(X >> 32))));
    }
    const uint32_t ge1 = pack_sub(xp, 0x3f7fffff3f7fffffull);      // x > nextbelow(1) = x >= 1
    auto bpack4 = [&](uint32_t& acc, const uint4& o, int e0) {      // elements e0 .. e0 + 3, descending
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int e = 3; e >= 0; --e)
        asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
            : "+r"(acc) : "r"(ow[e]), "r"(C[e0 + e]));
    };
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      uint32_t hi = 0u, lo = 0u;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        uint4 o[2] = {make_uint4((uint32_t)(8 * w + q + 4), (uint32_t)rq, sg, (uint32_t)(p.th0 + j)),
                      make_uint4((uint32_t)(8 * w + q), (uint32_t)rq, sg, (uint32_t)(p.th0 + j))};
        philox_xk<2>(o, p.key0, p.key1);
        bpack4(hi, o[0], 4 * (q + 4));
        bpack4(lo, o[1], 4 * q);
      }
      word[j] = ~((hi << 16) | lo) | ge1;                          // the shifted-in bits are [w >= C]
    }
    return;
  }
  uint64_t X[16];                                                   // x 2^32, elements 2k, 2k+1
#pragma unroll
  for (int k = 0; k < 16; ++k) asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(X[k]) : "l"(xp[k]), "l"(0x4f8000004f800000ull));
  auto pack4 = [&](uint32_t& acc, const uint4& o, int k0) {         // elements 2k0 .. 2k0 + 3, descending
    uint64_t f23, f01, d23, d01;
    asm("{\n\t.reg .f32 a, b;\n\tcvt.rz.f32.u32 a, %1;\n\tcvt.rz.f32.u32 b, %2;\n\tmov.b64 %0, {a, b};\n\t}"
        : "=l"(f23) : "r"(o.z), "r"(o.w));
    asm("{\n\t.reg .f32 a, b;\n\tcvt.rz.f32.u32 a, %1;\n\tcvt.rz.f32.u32 b, %2;\n\tmov.b64 %0, {a, b};\n\t}"
        : "=l"(f01) : "r"(o.x), "r"(o.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(f23), "l"(X[k0 + 1]));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(f01), "l"(X[k0]));
    acc = __funnelshift_l((uint32_t)(d23 >> 32), acc, 1);           // element 2k0 + 3
    acc = __funnelshift_l((uint32_t)d23, acc, 1);                   // element 2k0 + 2
    acc = __funnelshift_l((uint32_t)(d01 >> 32), acc, 1);           // element 2k0 + 1
    acc = __funnelshift_l((uint32_t)d01, acc, 1);                   // element 2k0
  };
  constexpr int KH = CM_RAND_ILP / 2;                               // blocks per chain per step
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    uint32_t hi = 0u, lo = 0u;
#pragma unroll
    for (int q = 4 - KH; q >= 0; q -= KH) {                         // blocks q .. q+KH-1 (lo), +4 (hi)
      uint4 o[2 * KH];
#pragma unroll
      for (int b = 0; b < KH; ++b) {
        o[b] = make_uint4((uint32_t)(8 * w + q + b + 4), (uint32_t)rq, sg, (uint32_t)(p.th0 + j));
        o[KH + b] = make_uint4((uint32_t)(8 * w + q + b), (uint32_t)rq, sg, (uint32_t)(p.th0 + j));
      }
      philox_xk<2 * KH>(o, p.key0, p.key1);
#pragma unroll
      for (int b = KH - 1; b >= 0; --b) {
        pack4(hi, o[b], 2 * (q + b + 4));
        pack4(lo, o[KH + b], 2 * (q + b));
      }
    }
    word[j] = (hi << 16) | lo;
  }
}

#ifndef CM_BLK_EVICT_FIRST
#define CM_BLK_EVICT_FIRST 1
#endif
// K1 software pipelining (block w's finish after block w+1's pack): measured 0.5-2 % slower
// on every config (ResNet-50 21.40 vs 21.44, VGG16 209 vs 214, rand1 9.80 vs 9.96 M cand/s;
// profiles r2au) -- the rounding warps are not latency-bound here: off
#ifndef CM_K1_PIPE
#define CM_K1_PIPE 0
#endif

// K1 for the blocked layout (CM_LAYOUT_BLK): the same per-block steps as k1_body, with the
// bookkeeping hoisted out of the block loop -- a group's row masks, store pointers and table
// base are set once per group (running pointers inside it), and the producer cursor is a
// running source pointer whose block sizes follow from (pg, pw) alone.
// MS: the mass tables -- 0 decided at run time (p.nib32 set or not), 1 int32 (staged), 2 int64.
template <int NT, bool RAND, int MS, class Hooks>
__device__ __forceinline__ void k1_body_blk(const RoundParams& p, unsigned char* k1smem, int wl, int* sq,
                                            const Hooks& hk, int Gr) {
  constexpr int kSt = k1_stages(NT);
  constexpr uint32_t kStageBytes = 4096u;
  const int lane = threadIdx.x & 31;
  const uint32_t tiles = smem_u32(k1smem) + (uint32_t)(kSt * kStageBytes) * (uint32_t)wl;
  const uint32_t bars = smem_u32(k1smem + k1_bar_off(NT, false)) + 8u * (uint32_t)(kSt * wl);
  const uint32_t nibs = smem_u32(k1smem + k1_nib_off(NT, false));
  const uint32_t rtabw = smem_u32(k1smem + k1_rtab_off(NT, p.nib32 ? p.nib_entries : 0, false)) +
                         (uint32_t)p.rtab * (uint32_t)wl;
  const int G = p.G, n = p.n;
  const int64_t cs = p.cs;
  uint64_t tt[NT];                                                  // theta (-0 -> +0) in both halves
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const uint32_t b = __float_as_uint(RAND ? 0.f : p.theta[p.th0 + j] + 0.0f);
    tt[j] = ((uint64_t)b << 32) | b;
  }
  const Transposer transpose(lane);
  const bool scaled32 = MS == 0 ? p.nib32 != nullptr : MS == 1;
  // every group but the last (h_last rows) is full: 4 KB off-diagonal, 2 304-byte diagonal blocks
  const int h_last = blk_rows(n, Gr - 1);
  const uint32_t off_last = 128u * (uint32_t)h_last, diag_last = 16u * (uint32_t)blk_diag_chunks(h_last);
#if CM_BLK_EVICT_FIRST
  const uint64_t pol = l2_evict_first_policy();
#endif


  // ---- producer cursor (S* ps, block (pg, pw), stage pstage), kSt - 1 blocks ahead
  int ps = hk.first(), pg = 0, pw = 0;
  uint32_t pstage = 0;
  unsigned qhead = 0, qtail = 0;                                    // sq ring (warp-uniform)
  if (lane == 0) sq[0] = ps;
  ++qhead;
  const float* psrc = ps < p.s_count ? p.sstar + (p.s_begin + ps) * p.stride : p.sstar;
  auto issue = [&]() {
    if (ps >= p.s_count) return;
    const bool last = pg == Gr - 1;
    const uint32_t bytes = pw < pg ? (last ? off_last : 4096u) : (last ? diag_last : 2304u);
    if (lane == 0) {
      const uint32_t bar = bars + 8u * pstage;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
#if CM_BLK_EVICT_FIRST
      // S* is read exactly once: an L2 evict-first policy keeps the stream from pushing the
      // ring (written by these warps, read back by the scan warps) out of L2 (measured: 4 KB
      // per S* fewer ring read-backs from DRAM, ResNet-50 +1.9 %, U-Net +3.7 %; the ring's
      // write-back, 10.6 KB per S*, stays -- evict-last ring stores or discarding a reduced
      // unit's lines (CM_DISCARD) changed neither the bytes nor the rate)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   :: "r"(tiles + kStageBytes * pstage), "l"(psrc), "r"(bytes), "r"(bar), "l"(pol) : "memory");
#else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(tiles + kStageBytes * pstage), "l"(psrc), "r"(bytes), "r"(bar) : "memory");
#endif
    }
    psrc += bytes >> 2;
    pstage = pstage + 1 == (uint32_t)kSt ? 0u : pstage + 1;
    if (++pw > pg) {
      pw = 0;
      if (++pg == Gr) {
        pg = 0;
        ps = hk.next(ps);
        if (lane == 0) sq[qhead & 7] = ps;
        ++qhead;
        if (ps < p.s_count) psrc = p.sstar + (p.s_begin + ps) * p.stride;
      }
    }
  };
#pragma unroll
  for (int d = 0; d < kSt - 1; ++d) issue();

  // ---- consumer
  uint32_t cstage = 0, cpar = 0;
  auto wait_block = [&]() {                                         // returns the stage's smem address
    issue();
    const uint32_t bar = bars + 8u * cstage;
    asm volatile("{\n\t.reg .pred p;\n\tWAITB_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAITB_%=;\n\t}" :: "r"(bar), "r"(cpar) : "memory");
    const uint32_t st0 = tiles + kStageBytes * cstage;
    if (++cstage == (uint32_t)kSt) {
      cstage = 0;
      cpar ^= 1u;
    }
    return st0;
  };
  for (;;) {
    __syncwarp();
    const int s = sq[qtail & 7];
    ++qtail;
    if (s >= p.s_count) break;
    uint32_t* out = hk.begin(s);
    const uint32_t sg = p.s0 + (uint32_t)(p.s_begin + s);           // RAND: global S* index
    if constexpr (RAND && Hooks::kTab) {                            // this S*'s Philox table
      __syncwarp();                                                 // the previous S*'s reads are done
      rand_table_build(rtabw, Gr, NT, sg, p);
      __syncwarp();
    }
    for (int g = 0; g < Gr; ++g) {
      const int rq = 32 * g + lane + 1;                             // row owned by this lane
      // row masks (a1 reads i < t only, rows < n): FULL off the diagonal, nodes 32g .. rq-1 on it
      const uint32_t rm_off = rq < n ? FULL : 0u;
      const uint32_t rm_diag = rq < n ? (lane == 31 ? FULL : (2u << lane) - 1u) : 0u;
      uint32_t* colp = out + grp_off(g) + lane;                     // node 32w+lane's column word
      uint32_t* browp = out + p.brow + (g + 1) * G;                 // row 32(g+1) = lane 31's row
      const bool wbrow = lane == 31 && g + 1 < G;
      uint32_t tb = nibs;                                           // block w's mass table
      int32_t mass32[NT];
      int64_t mass[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) mass32[j] = 0, mass[j] = 0;
      // one block in two halves: pack (xp holds this lane's row, elements 2k, 2k+1 in xp[k]) ->
      // the row word; finish -> the stage-sliced column word (transpose), row 32(g+1)'s word and
      // the row's checkpoint mass.  CM_K1_PIPE: block w's finish runs after block w+1's pack, so
      // the two dependency chains (FADD2 / funnel shifts, SHFL transpose / mass lookups) of
      // consecutive blocks interleave in one basic block.
      auto pack = [&](const uint64_t (&xp)[16], uint32_t rmask, int w, uint32_t (&word)[NT]) {
        if (RAND) {
          rand_words<NT, RAND && Hooks::kTab>(word, xp, w, rq, sg, p, rtabw);
#pragma unroll
          for (int j = 0; j < NT; ++j) word[j] &= rmask;
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) word[j] = pack_sub(xp, tt[j]) & rmask;
        }
      };
      const int64_t* tw64 = p.nib;                                  // int64 tables of the next block
      auto finish = [&](const uint32_t (&word)[NT]) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          if (wbrow) browp[j * cs] = word[j];
          colp[j * cs] = transpose(word[j]);                        // bit b = row 32g+1+b
        }
        ++browp;
        colp += 32;
#ifndef CM_EXP_NOMASS
        if (scaled32) {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int32_t v[8];
            const uint32_t wd = word[j];
            auto ent = [&](uint32_t sh) {                           // (nibble << 2) | table: one LOP3
              uint32_t a;
              asm("lop3.b32 %0, %1, 0x3C, %2, 0xEA;" : "=r"(a) : "r"(sh), "r"(tb));
              return a;
            };
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[0]) : "r"(ent(wd << 2)));
#define CM_NIB(Q) asm volatile("ld.shared.u32 %0, [%1+" #Q "*64];" : "=r"(v[Q]) : "r"(ent(wd >> (4 * Q - 2))))
            CM_NIB(1); CM_NIB(2); CM_NIB(3); CM_NIB(4); CM_NIB(5); CM_NIB(6); CM_NIB(7);
#undef CM_NIB
            mass32[j] += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
          }
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int64_t ms = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) ms += __ldg(tw64 + 16 * q + ((word[j] >> (4 * q)) & 15u));
            mass[j] += ms;
          }
        }
#endif
        tb += 512u;
        tw64 += 128;
      };
      // one body for every block (the hot loop stays small next to K2's in the instruction
      // cache); only the 8 shared loads depend on the block's form
      const bool bfull = g < Gr - 1 || h_last == 32;
      uint32_t pend[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) pend[j] = 0u;
      for (int w = 0; w <= g; ++w) {
        const uint32_t st0 = wait_block();
        const uint32_t rb = st0 + 16u * (uint32_t)lane;
        uint64_t xp[16];
        if (w < g && bfull) {                                       // chunk-major 32-row block
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(xp[2 * c]), "=l"(xp[2 * c + 1]) : "r"(rb + 512u * c));
        } else if (bfull) {                                         // chunk-major diagonal, h = 32
          constexpr uint32_t kDiag[8] = {0, 448, 832, 1152, 1408, 1600, 1728, 1792};   // 16 (B_c - 4c)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(xp[2 * c]), "=l"(xp[2 * c + 1]) : "r"(rb + kDiag[c]));
        } else if (w < g) {                                         // partial group: chunk stride h_last
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];"
                         : "=l"(xp[2 * c]), "=l"(xp[2 * c + 1]) : "r"(rb + 16u * (uint32_t)h_last * c));
        } else {
          // partial diagonal: chunk c of this lane's row at byte 16 (B_c + lane - 4c) for the rows
          // that have chunk c (lane >= 4c), any in-stage address for the others (bits masked)
          int b = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t a = lane >= 4 * c ? st0 + 16u * (uint32_t)(b + lane - 4 * c) : st0;
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(xp[2 * c]), "=l"(xp[2 * c + 1]) : "r"(a));
            b += max(0, h_last - 4 * c);
          }
        }
        uint32_t word[NT];
        pack(xp, w < g ? rm_off : rm_diag, w, word);
        if (CM_K1_PIPE) {
          if (w > 0) finish(pend);
#pragma unroll
          for (int j = 0; j < NT; ++j) pend[j] = word[j];
        } else {
          finish(word);
        }
      }
      if (CM_K1_PIPE) finish(pend);
      if (rq < n) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          if (scaled32) reinterpret_cast<int32_t*>(out + (int64_t)j * cs + p.bw)[rq] = mass32[j];
          else reinterpret_cast<int64_t*>(out + (int64_t)j * cs + p.bw)[rq] = mass[j];
        }
      }
    }
    hk.end(s);
  }
}

// K1 body of one warp: S* s = hk.first(), hk.next(s), ... while < s_count; wl = the warp's
// index among the CTA's K1 warps (its stage ring).  The TMA cursor runs ahead of the
// consumer and may enter the next S* (or several, for tiny graphs) first: the S* indices it
// takes queue in `sq` (8 per warp) until the consumer reaches them.
// RAND: randomized rounding, sample th0 + j instead of threshold th0 + j (one Philox block
// per four consecutive nodes and sample).
template <int NT, int LAY, bool RAND, class Hooks, int MS = 0>
__device__ __forceinline__ void k1_body(const RoundParams& p, const CUtensorMap* tmap, const DiagMaps* dmaps,
                                        unsigned char* k1smem,
                                        int wl, int* sq, const Hooks& hk) {
  constexpr bool BULK = LAY == 1;                                   // tri4
  constexpr bool BLK = LAY == 2;                                    // blocked triangle: k1_body_blk
  constexpr int kSt = k1_stages(NT);
  constexpr uint32_t kStageBytes = (uint32_t)k1_stage_bytes(BULK);
  int32_t* nib32 = reinterpret_cast<int32_t*>(k1smem + k1_nib_off(NT, BULK));   // p.nib32 staged (if any)
  const int lane = threadIdx.x & 31;
  unsigned char* tiles = k1smem + (size_t)kSt * kStageBytes * wl;                   // [stage] of this warp
  uint64_t* bars = reinterpret_cast<uint64_t*>(k1smem + k1_bar_off(NT, BULK)) + kSt * wl;
  const int G = p.G;
  // row groups with a row r = 32g+1+l < n; the Sn columns of later groups are all zero
  // (S_{n+1} = 0) and K2 does not read them
  const int Gr = p.n >= 2 ? (p.n - 2) / 32 + 1 : 0;
  if (Gr == 0) {
    for (int s = hk.first(); s < p.s_count; s = hk.next(s)) { hk.begin(s); hk.end(s); }
    return;
  }
  if constexpr (BLK) {
    k1_body_blk<NT, RAND, MS>(p, k1smem, wl, sq, hk, Gr);
    return;
  }
  uint64_t tt[NT];                                                  // theta (-0 -> +0) in both halves
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const uint32_t b = __float_as_uint(RAND ? 0.f : p.theta[p.th0 + j] + 0.0f);
    tt[j] = ((uint64_t)b << 32) | b;
  }
  const Transposer transpose(lane);
  const bool scaled32 = p.nib32 != nullptr;
  const uint32_t tiles_u32 = smem_u32(tiles);
  // tri4 read by gather4 lands in the same 128-byte-swizzled form as the dense tensor tiles.
  // The batch's last S* (the last ceil(32 / stride) for tiny graphs) cannot use it -- a row's
  // 128-byte window may run past the buffer -- so those take per-row bulk copies of exactly the
  // stored floats into the 144-byte-pitch form.
  auto pitched_of = [&](int s_rel) { return BULK && (!p.g4 || p.s_begin + s_rel >= p.g4_end); };
  const uint64_t pol = (LAY == 0 && p.evict_first) ? l2_evict_first_policy() : 0ull;

  // Producer cursor (ps, pg, pw) runs kSt-1 blocks ahead of the consumer.  No proxy
  // fence before re-filling a stage: its previous contents were consumed (ballots issued on
  // the loaded values, then __syncwarp) before the refill is issued.
  int ps = hk.first(), pg = 0, pw = 0, pstage = 0;
  unsigned qhead = 0, qtail = 0;                                    // sq ring (warp-uniform)
  if (lane == 0) sq[0] = ps;
  ++qhead;
  auto issue = [&]() {
    if (ps >= p.s_count) return;
    if (BULK && !pitched_of(ps)) {
      // tri4 through a 2-D tensor map whose "rows" are the batch's 16-byte units (an
      // overlapping stride): block row r = 32 pg + 1 + lane starts at unit (offset of S* ps +
      // offset of row r + 32 pw) / 4.  Eight tile::gather4 loads (lanes 0, 4, .., 28) each
      // place four rows, so the stage holds the swizzled 32 x 32 tile of the dense path, and
      // the bytes fetched are the stored triangle itself (plus the next rows' heads where a
      // row ends inside the block, which other blocks read anyway).
      const int r = 32 * pg + 1 + lane;
      const int y = (int)((((p.s_begin + ps) * p.stride) + row_offset(1, 0, r) + 32 * pw) >> 2);
      const int y1 = __shfl_down_sync(FULL, y, 1), y2 = __shfl_down_sync(FULL, y, 2), y3 = __shfl_down_sync(FULL, y, 3);
      if (lane == 0) mbar_expect_tx(&bars[pstage], 32u * 32u * 4u);
      __syncwarp();
      if ((lane & 3) == 0)
        tma_gather4(tiles_u32 + (uint32_t)pstage * kStageBytes + 128u * (uint32_t)lane, tmap, y, y1, y2, y3, &bars[pstage]);
    } else if (BULK) {
      // this lane's row r = 32 pg + 1 + lane, nodes 32 pw .. : the stored part of the block
      const int r = 32 * pg + 1 + lane;
      const int len = r < p.n ? min(32, ((r + 3) & ~3) - 32 * pw) : 0;   // floats, % 4 == 0, > 0 if r < n
      const uint32_t total = __reduce_add_sync(FULL, (uint32_t)len) * 4u;
      if (lane == 0) mbar_expect_tx(&bars[pstage], total);
      __syncwarp();
      if (len > 0) {
        const float* src = p.sstar + (p.s_begin + ps) * p.stride + row_offset(1, 0, r) + 32 * pw;
        bulk_load(tiles_u32 + (uint32_t)pstage * kStageBytes + (uint32_t)lane * kBulkPitch, src, 4u * (uint32_t)len,
                  &bars[pstage]);
      }
    } else if (lane == 0) {
#ifdef CM_EXP_L2INPUT
      const int z = (int)((p.s_begin + ps) & 63);                   // timing experiment
#else
      const int z = (int)(p.s_begin + ps);
#endif
      unsigned char* dst = tiles + (size_t)pstage * kStageBytes;
      mbar_expect_tx(&bars[pstage], 32u * 32u * 4u);
      const CUtensorMap* tm = pw == pg ? &dmaps->diag : tmap;
      if (pol) tma_load_3d(dst, tm, 32 * pw, 32 * pg + 1, z, &bars[pstage], pol);
      else tma_load_3d(dst, tm, 32 * pw, 32 * pg + 1, z, &bars[pstage]);
    }
    pstage = pstage + 1 == kSt ? 0 : pstage + 1;
    if (++pw > pg) {
      pw = 0;
      if (++pg == Gr) {
        pg = 0;
        ps = hk.next(ps);
        if (lane == 0) sq[qhead & 7] = ps;
        ++qhead;
      }
    }
  };
  for (int d = 0; d < kSt - 1; ++d) issue();

  int cstage = 0;
  uint32_t phase_bits = 0u;                                         // bit st = parity of stage st
  for (;;) {
    __syncwarp();
    const int s = sq[qtail & 7];
    ++qtail;
    if (s >= p.s_count) break;
    uint32_t* out = hk.begin(s);
    for (int g = 0; g < Gr; ++g) {
      const int rq = 32 * g + lane + 1;                             // row owned by this lane
      int64_t mass[NT];
      int32_t mass32[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) mass[j] = 0, mass32[j] = 0;
      for (int w = 0; w <= g; ++w) {
        issue();
        mbar_wait(&bars[cstage], (phase_bits >> cstage) & 1u);
        phase_bits ^= 1u << cstage;
        // this lane's row in the stage: the 144-byte-pitch per-row form (tri4 fallback) or the
        // 128-byte-swizzled 32 x 32 tile
        const bool pitched = pitched_of(s);
        const uint32_t st0 = tiles_u32 + (uint32_t)cstage * kStageBytes;
        const uint32_t rb = st0 + (uint32_t)lane * (pitched ? (uint32_t)kBulkPitch : 128u);
        const uint32_t sw = pitched ? 0u : (uint32_t)(lane & 7) << 4;
        uint64_t xp[16];                                            // elements (2k, 2k+1) of the row
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];"
                       : "=l"(xp[2 * c]), "=l"(xp[2 * c + 1]) : "r"(rb + (((uint32_t)c << 4) ^ sw)));
        cstage = cstage + 1 == kSt ? 0 : cstage + 1;
        // Row word of this lane's row r = rq over block w: bit q = S_{r, 32w+q} = [x_q > theta]
        // (a1: strict fp32 '>', NaN -> 0), masked to the strict lower triangle (32w+q < r) and
        // to rows r < n, so zero-filled or stale stage contents never leak.
        const int rem = rq - 32 * w;                                // >= 1: nodes 32w .. rq-1 exist
        const uint32_t rmask = rq >= p.n ? 0u : (rem >= 32 ? FULL : (1u << rem) - 1u);
        uint32_t word[NT];
        if (RAND) {                                                 // a1 randomized: u < S*
          rand_words<NT>(word, xp, w, rq, p.s0 + (uint32_t)(p.s_begin + s), p);
#pragma unroll
          for (int j = 0; j < NT; ++j) word[j] &= rmask;
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) word[j] = pack_sub(xp, tt[j]) & rmask;
        }
        const int node = 32 * w + lane;
        const int brow_at = p.brow + (g + 1) * G + w;               // row 32(g+1) = lane 31's row
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          uint32_t* oj = out + (int64_t)j * p.cs;
          if (lane == 31 && g + 1 < G) oj[brow_at] = word[j];
          oj[grp_off(g) + node] = transpose(word[j]);               // node 32w+lane's column: bit b = row 32g+1+b
        }
#ifndef CM_EXP_NOMASS                                               // timing experiment: no masses
        if (scaled32) {                                             // scaled masses fit int32 (every row's)
          const uint32_t tb = smem_u32(nib32) + 512u * (uint32_t)w;   // 512-byte aligned
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            int32_t v[8];
            const uint32_t wd = word[j];
            // entry address (nibble << 2) | table: one LOP3 ((a & 0x3C) | c, LUT 0xEA) per lookup
            auto ent = [&](uint32_t sh) {
              uint32_t a;
              asm("lop3.b32 %0, %1, 0x3C, %2, 0xEA;" : "=r"(a) : "r"(sh), "r"(tb));
              return a;
            };
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[0]) : "r"(ent(wd << 2)));
#define CM_NIB(Q) asm volatile("ld.shared.u32 %0, [%1+" #Q "*64];" : "=r"(v[Q]) : "r"(ent(wd >> (4 * Q - 2))))
            CM_NIB(1); CM_NIB(2); CM_NIB(3); CM_NIB(4); CM_NIB(5); CM_NIB(6); CM_NIB(7);
#undef CM_NIB
            mass32[j] += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
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
#endif
      }
      if (rq < p.n) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          if (scaled32) reinterpret_cast<int32_t*>(out + (int64_t)j * p.cs + p.bw)[rq] = mass32[j];
          else reinterpret_cast<int64_t*>(out + (int64_t)j * p.cs + p.bw)[rq] = mass[j];
        }
      }
    }
    hk.end(s);
  }
}

template <int NT, int LAY, bool RAND>
__global__ void __maxnreg__(NT == 1 ? CM_K1_REGS1 : 128) round_tma_kernel(const RoundParams p, const __grid_constant__ CUtensorMap tmap,
                                                                    const __grid_constant__ DiagMaps dmaps) {
  extern __shared__ __align__(1024) unsigned char k1raw[];
  unsigned char* k1smem = k1raw + ((1024u - (smem_u32(k1raw) & 1023u)) & 1023u);
  k1_setup<NT, LAY, RAND>(p, k1smem, (int)(blockDim.x >> 5), (int)threadIdx.x, (int)blockDim.x);
  __syncthreads();
  __shared__ int sq[32][8];
  const K1Plain hk{p.sn, p.n_theta, p.th0, p.cs, (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5),
                   (int)((gridDim.x * blockDim.x) >> 5)};
  k1_body<NT, LAY, RAND>(p, &tmap, &dmaps, k1smem, (int)(threadIdx.x >> 5), sq[threadIdx.x >> 5], hk);
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
// int32 state: the task's 32 checkpoint masses staged into shared memory by cp.async at the
// task start (CM_STAGE_MASS=1, 4 KB per scan warp) or read from the ring at the end (default:
// measured within 1 %, and the 32 KB per CTA pay for the Sn rings).
#ifndef CM_STAGE_MASS
#define CM_STAGE_MASS 0
#endif
constexpr bool kStageMassCfg = CM_STAGE_MASS != 0;
// The walk's Sn words come through a per-warp shared-memory ring of CM_SN_RING quads (16 bytes
// per lane each, cp.async.cg, CM_SN_RING - 1 quads = 4 (CM_SN_RING - 1) nodes ahead); 0: the
// quads ride in registers two quads ahead.
#ifndef CM_SN_RING
#define CM_SN_RING 8
#endif
// The int64 state keeps the registers (its 8 KB E per warp leaves no room for rings at n ~ 560).
constexpr int kSnRing = CM_SN_RING;
static_assert(kSnRing == 0 || (kSnRing >= 2 && (kSnRing & (kSnRing - 1)) == 0), "ring of a power of two quads");
__host__ __device__ constexpr int sn_ring_quads(bool s32, int q = kSnRing) { return s32 ? q : 0; }
__host__ __device__ constexpr int scan_e_bytes(bool s32, int q = kSnRing) {
  return (s32 ? 4 * 32 * 32 * (kStageMassCfg ? 2 : 1) : 8 * 32 * 32) + 512 * sn_ring_quads(s32, q);
}

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
  int32_t mass_bytes;         // 4 (int32 state) or 8 per mass entry in a candidate block
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
// ordered by tcgen05.wait::st (the walk tracks pending stores).  The TMEM asm carries no
// "memory" clobber: TMEM is not memory, volatile asm keeps the ld / st / wait order, and
// register operands order the uses -- so shared-memory work (E) may move across them.
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
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr + (uint32_t)s));
    else
      v = sm[32 * (s - tmc) + lane];
    return v;
  }
  __device__ __forceinline__ void wait_ld(uint32_t& v) const {
    if (TM) asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v));
  }
  __device__ __forceinline__ void wait_ld3(uint32_t& v0, uint32_t& v1, uint32_t& v2) const {
    if (TM) asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v0), "+r"(v1), "+r"(v2));
  }
  template <int MODE>
  __device__ __forceinline__ void st(int s, uint32_t v) const {
    if (in_tmem<MODE>(s))
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(taddr + (uint32_t)s), "r"(v));
    else
      sm[32 * (s - tmc) + lane] = v;
  }
  __device__ __forceinline__ void wait_st() const {
    if (TM) asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  // slots s..s+3, all in TMEM (TM, s + 3 < tmc)
  __device__ __forceinline__ void st4(int s, uint4 v) const {
    if (TM)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                   :: "r"(taddr + (uint32_t)s), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  }
};

// Events of one computing node k: for every stage bit b of x (stage b computes k), in the
// backward walk, first the frees at k (Eq. 9: the masks f_j with masses m_j, and the i = k
// self-free sf with M_k), then the compute: E_b = max(E_b - frees, 0) + M_k (E is a memory
// rise, at most sum M, and every intermediate lies in [-sum M, sum M]: the int32 state needs
// only sum M / gcd < 2^31).  NM dependency masks (compile-time).  A round takes up to W
// stage bits of x, highest first (FLO yields the index; stages are independent, so the order
// is free), and their loads issue together; the width follows the warp's largest per-lane
// event count (REDUX), so nodes whose lanes compute in one or two stages do not pay for
// four-wide rounds.  x excludes the diagonal stage t = k: that compute is the first event of
// stage t in the walk (R_{t,k} = 0 for k > t), so it always leaves E_t = M_t and the scan
// initialises E with it instead.
// E[stage][lane] is addressed in the shared window: eaddr = &E[0][lane], stage b at eaddr +
// 32 b sizeof(ET).  A slot takes bit b = bfind(x) (0xffffffff when x = 0) and sel = 1 << b (0
// then: a shift by 32 or more clears the word), so an empty slot needs no select; its load and
// store are predicated off by sel = 0.
template <typename ET>
__device__ __forceinline__ void lds_if(ET& v, uint32_t addr, uint32_t sel) {
  if constexpr (sizeof(ET) == 4)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u32 %0, [%1];\n\t}"
                 : "+r"(v) : "r"(addr), "r"(sel) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u64 %0, [%1];\n\t}"
                 : "+l"(v) : "r"(addr), "r"(sel) : "memory");
}
template <typename ET>
__device__ __forceinline__ void sts_if(uint32_t addr, uint32_t sel, ET v) {
  if constexpr (sizeof(ET) == 4)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p st.shared.u32 [%0], %2;\n\t}"
                 :: "r"(addr), "r"(sel), "r"(v) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p st.shared.u64 [%0], %2;\n\t}"
                 :: "r"(addr), "r"(sel), "l"(v) : "memory");
}
template <int W, int NM, typename ET>
__device__ __forceinline__ void event_round(uint32_t& x, uint32_t sf, ET Mk, const uint32_t* f, const ET* m,
                                            uint32_t eaddr) {
  uint32_t sel[W], addr[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    uint32_t b;
    asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(x));                   // highest set bit, ~0 if none
    asm("shl.b32 %0, %1, %2;" : "=r"(sel[u]) : "r"(1u), "r"(b));   // 0 if none
    addr[u] = eaddr + b * (uint32_t)(32 * sizeof(ET));
    x ^= sel[u];
  }
  ET ev[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    ev[u] = (ET)0;
    lds_if(ev[u], addr[u], sel[u]);
  }
#pragma unroll
  for (int u = 0; u < W; ++u) {
    ET fr = (sf & sel[u]) ? Mk : (ET)0;
#pragma unroll
    for (int j = 0; j < NM; ++j)
      if (f[j] & sel[u]) fr += m[j];
    ev[u] = max(ev[u] - fr, (ET)0) + Mk;                             // every term within [-sum M, sum M]
  }
#pragma unroll
  for (int u = 0; u < W; ++u) sts_if(addr[u], sel[u], ev[u]);
}
template <int NM, typename ET>
__device__ __forceinline__ void events(uint32_t x, uint32_t sf, ET Mk, const uint32_t* f, const ET* m,
                                       ET* E, int lane) {
  const unsigned mx = __reduce_max_sync(FULL, (unsigned)__popc(x));
  if (mx == 0) return;
  const uint32_t eaddr = smem_u32(E) + (uint32_t)(sizeof(ET) * lane);
  if (mx == 1) event_round<1, NM, ET>(x, sf, Mk, f, m, eaddr);
  else if (mx == 2) event_round<2, NM, ET>(x, sf, Mk, f, m, eaddr);
  else
    while (__any_sync(FULL, x != 0u)) event_round<4, NM, ET>(x, sf, Mk, f, m, eaddr);
}

// The far (non-adjacent) dependencies of node k (ndf of them, warp-uniform; three in
// registers, any further ones applied first in a rare loop), the adjacent one (mask fa, mass
// ma; zero when absent), then the events.  drec[e] = {slot_i | i << 16, (int32) M_i}.
// One body for every ndf: the walk's hot loop must stay small (instruction-cache resident
// next to the rounding code on the same SM).
template <typename ET, bool TM, int MODE>
__device__ __forceinline__ void node_step(uint32_t Rk, uint32_t diag, uint32_t sf, ET Mk, uint32_t fa, ET ma, int e0,
                                          int ndf, const int2* __restrict__ drec, const int64_t* __restrict__ M,
                                          const AView<TM>& A, ET* E, int lane, bool& st_pending) {
  if (ndf == 0) {
    events<1, ET>(Rk & ~diag, sf, Mk, &fa, &ma, E, lane);
    return;
  }
  if (ndf == 1) {                                                   // the common far case
    const int2 d = drec[e0];
    const int s0 = d.x & 0xffff;
    uint32_t f[2] = {0u, fa};
    ET m[2] = {sizeof(ET) == 4 ? (ET)d.y : (ET)M[d.x >> 16], ma};
    if (st_pending) A.wait_st();
    uint32_t a0 = A.template ld_async<MODE>(s0);
    A.wait_ld(a0);
    f[0] = Rk & ~a0;                                                // FREE_{t,i,k} = R_k & ~A'_i
    A.template st<MODE>(s0, a0 | Rk);                               // A'_i |= R_k
    st_pending = true;
    events<2, ET>(Rk & ~diag, sf, Mk, f, m, E, lane);
    return;
  }
  uint32_t f[4] = {0u, 0u, 0u, fa};
  ET m[4] = {(ET)0, (ET)0, (ET)0, ma};
  int sl[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < 3; ++j)
    if (j < ndf) {
      const int2 d = drec[e0 + j];
      sl[j] = d.x & 0xffff;
      m[j] = sizeof(ET) == 4 ? (ET)d.y : (ET)M[d.x >> 16];
    }
  if (st_pending) A.wait_st();
  uint32_t ai[3] = {0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < 3; ++j)
    if (j < ndf) ai[j] = A.template ld_async<MODE>(sl[j]);
  A.wait_ld3(ai[0], ai[1], ai[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j)
    if (j < ndf) {
      f[j] = Rk & ~ai[j];                                           // FREE_{t,i,k} = R_k & ~A'_i
      A.template st<MODE>(sl[j], ai[j] | Rk);                       // A'_i |= R_k
    }
  st_pending = true;
  for (int e = e0 + 3; e < e0 + ndf; ++e) {                         // more far deps (rare)
    const int2 d = drec[e];
    const int s = d.x & 0xffff;
    A.wait_st();
    uint32_t ai1 = A.template ld_async<MODE>(s);
    A.wait_ld(ai1);
    A.template st<MODE>(s, ai1 | Rk);
    const ET Mi = sizeof(ET) == 4 ? (ET)d.y : (ET)M[d.x >> 16];
    for (uint32_t fx = Rk & ~ai1 & ~diag; fx; fx &= fx - 1) E[32 * (__ffs(fx) - 1) + lane] -= Mi;
  }
  events<4, ET>(Rk & ~diag, sf, Mk, f, m, E, lane);
}

// Sn ring of Q quads: quad q of the group's Sn column (nodes 4q .. 4q+3, 16 bytes per lane)
// lives in slot q mod Q; one cp.async group per quad, issued Q - 1 quads ahead,
// zero-filled for quads below 0 or candidates / groups without Sn.
template <int Q>
__device__ __forceinline__ void sn_fetch(uint32_t snr, const uint4* sn4, int q, bool lsn) {
  const bool v = lsn && q >= 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n\tcp.async.commit_group;"
               :: "r"(snr + ((uint32_t)(q & (Q - 1)) << 9)), "l"(sn4 + (v ? q : 0)), "r"(v ? 16 : 0)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// Walk the nodes k = nk-1 .. 0 of a group pass, one node per iteration.
// nrec[k] = {(int32) M_k, e0, ndf | adj << 16, slot_k or -1}.
template <typename ET, bool TM, int MODE, bool RSTORE, int Q = kSnRing>
__device__ __forceinline__ void walk(int nk, int g, bool live, bool lsn, const uint4* sn4, uint32_t* rcol,
                                     const uint32_t* brow, const int4* __restrict__ nrec,
                                     const int2* __restrict__ drec, const int64_t* __restrict__ M,
                                     const int64_t* __restrict__ C, const AView<TM>& A, ET* E, int lane,
                                     int64_t& costL, uint32_t snr) {
  const int k0 = nk - 1;
  constexpr int kQ = sn_ring_quads(sizeof(ET) == 4, Q);
  static_assert(kQ == 0 || (kQ >= 2 && (kQ & (kQ - 1)) == 0), "ring of a power of two quads");
  constexpr bool kRing = kQ > 0;
  // registers (no ring): Sn words of the quad holding k and of the two quads below, loaded two
  // quads ahead.  Ring: quads k0/4 .. k0/4 - kQ + 1 in flight, sp = the address of Sn_{k-1}.
  uint4 quad = make_uint4(0u, 0u, 0u, 0u), nquad = quad, n2quad = quad;
  uint32_t sp = 0u;
  uint32_t sn1;
  if constexpr (kRing) {
#pragma unroll
    for (int i = 0; i < kQ; ++i) sn_fetch<kQ>(snr, sn4, (k0 >> 2) - i, lsn);
    cp_async_wait<kQ - 1>();
    sp = snr + ((uint32_t)((k0 >> 2) & (kQ - 1)) << 9) + 4u * (uint32_t)(k0 & 3);
    sn1 = lds_u32(sp);                                              // Sn_k0
  } else {
    quad = lsn ? __ldcg(sn4 + (k0 >> 2)) : make_uint4(0u, 0u, 0u, 0u);
    nquad = (lsn && (k0 >> 2) > 0) ? __ldcg(sn4 + (k0 >> 2) - 1) : make_uint4(0u, 0u, 0u, 0u);
    n2quad = (lsn && (k0 >> 2) > 1) ? __ldcg(sn4 + (k0 >> 2) - 2) : make_uint4(0u, 0u, 0u, 0u);
    sn1 = (k0 & 3) == 3 ? quad.w : (k0 & 3) == 2 ? quad.z : (k0 & 3) == 1 ? quad.y : quad.x;
  }
  // row 32g's word for k's 32-node block (blocks w < g only; nodes >= 32g are never in S_32g)
  // and, prefetched, for the block below
  const uint32_t bword = (g > 0 && (k0 >> 5) < g && live) ? __ldcg(brow + (k0 >> 5)) : 0u;
  uint32_t bnext = (g > 0 && (k0 >> 5) >= 1 && live) ? __ldcg(brow + (k0 >> 5) - 1) : 0u;
  uint32_t bcur = bword << (31 - (k0 & 31));                        // bit 31 = node k's bit of row 32g
  uint32_t dg = 1u << (k0 - 32 * g);                                // e_t for k in 32g .. k0 (k0 >= 32g)
  int4 rec1 = nrec[k0];                                             // record of the next node
  // Sn_k: the previous step's Sn_{k-1}, so each step extracts one word
  uint32_t acc = 0u;                                                // Acc_k from user k+1
  uint32_t bslot = 0u;                                              // A'_k base when k has a slot
  bool st_pending = true;                                           // init stores precede
  if (rec1.w >= 0) {
    A.wait_st();
    bslot = A.template ld_async<MODE>(rec1.w);
    A.wait_ld(bslot);
    st_pending = false;
  }
#pragma unroll 1
  for (int k = k0; k >= 0; --k) {
    const int u = k & 3;
    const int4 rec = rec1;
    rec1 = nrec[k - 1];                                             // k = 0: the sentinel record
    const int64_t Ck = C[k];
    const uint32_t sn = sn1;
    if constexpr (kRing) {                                          // Sn_{k-1} from the ring
      if (u == 0) {
        // quad k/4 - 1 must have landed; slot k/4 is consumed: refill it kQ quads below
        cp_async_wait<kQ - 2>();
        sp = snr + ((uint32_t)(((k >> 2) - 1) & (kQ - 1)) << 9) + 12u;
        sn1 = lds_u32(sp);
        sn_fetch<kQ>(snr, sn4, (k >> 2) - kQ, lsn);
      } else {
        sp -= 4u;
        sn1 = lds_u32(sp);
      }
    } else {  // Sn_{k-1}: component u-1 of the quad, or the next quad's last word (branch-free selects)
      const uint32_t c01 = (u & 2) ? quad.y : quad.x;              // u = 2 -> y, u = 1 -> x
      const uint32_t c = u == 3 ? quad.z : c01;
      sn1 = u == 0 ? nquad.w : c;
    }
    const uint32_t a = (rec.w >= 0 ? bslot : sn) | acc;             // A'_k, complete
    const uint32_t sw = __funnelshift_l(bcur, sn, 1);               // S_t from S_{t+1} and row 32g
    const uint32_t diag = dg;                                       // stage t = k of this group
    dg >>= 1;
    bcur <<= 1;
    const uint32_t Rk = (a & ~sw) | diag;                           // a2 seed + a3 closure
    if (RSTORE && live) rcol[k] = Rk;                               // verification output
    // base of A'_{k-1}: its slot (final: every far user j > k is done; the adjacent user k
    // contributes through acc) or Sn_{k-1}
    uint32_t b1 = sn1;
    if (rec1.w >= 0) {
      if (st_pending) { A.wait_st(); st_pending = false; }
      b1 = A.template ld_async<MODE>(rec1.w);
    }
    acc = 0u;
    if (__any_sync(FULL, Rk != 0u)) {                               // computed in some lane
      const ET Mk = sizeof(ET) == 4 ? (ET)rec.x : (ET)M[k];
      costL += (int64_t)__popc(Rk) * Ck;
      const bool adj = (rec.z >> 16) != 0;
      if (rec1.w >= 0) A.wait_ld(b1);
      const uint32_t fa = adj ? Rk & ~b1 : 0u;                      // FREE_{t,k-1,k}
      const ET ma = sizeof(ET) == 4 ? (ET)rec1.x : (k > 0 ? (ET)M[k - 1] : (ET)0);
      if (adj) acc = Rk;                                            // Acc_{k-1} |= R_k
      const uint32_t sf = Rk & ~a;                                  // FREE_{t,k,k}
      node_step<ET, TM, MODE>(Rk, diag, sf, Mk, fa, ma, rec.y, rec.z & 0xffff, drec, M, A, E, lane, st_pending);
    } else if (rec1.w >= 0) {
      A.wait_ld(b1);
    }
    bslot = b1;
    if (!kRing && u == 0) {                                         // next node is in the quad below
      quad = nquad;                                                 // loads run two quads ahead
      nquad = n2quad;
      n2quad = (lsn && (k >> 2) >= 3) ? __ldcg(sn4 + (k >> 2) - 3) : make_uint4(0u, 0u, 0u, 0u);
    }
    if ((k & 31) == 0) {                                            // next node is in the block below
      bcur = bnext;
      bnext = (g > 0 && (k >> 5) >= 2 && live) ? __ldcg(brow + (k >> 5) - 2) : 0u;
    }
  }
  if constexpr (kRing) cp_async_wait<0>();                          // the next task reuses the slots
}

// Write one 32x32 mask block set (rows 32g..32g+31 of the 32 candidates of the task) from
// column words: col(cl, node) for candidate cl of the batch.  S: S_t words from the Sn columns
// and row 32g (brow); R: the R columns the walk stored over the Sn columns.
template <bool IS_S>
__device__ void emit_mask(const ScanParams& p, const uint32_t* ws, int64_t n_cand, int64_t out_base, uint32_t* out,
                          int g, int nk, int64_t batch0, int lane) {
  const int n = p.n, G = p.G;
  const int W32 = 2 * ((n + 63) >> 6);
  const int row = 32 * g + lane;
  for (int cl = 0; cl < 32; ++cl) {
    const int64_t cc = batch0 + cl;
    if (cc >= n_cand) break;                                        // warp-uniform
    const uint32_t* ccw = ws + cc * p.cs;
    for (int w = 0; w <= g; ++w) {
      const int node = 32 * w + lane;
      uint32_t sc = node < nk && (!IS_S || 32 * g + 1 < n) ? __ldcg(ccw + grp_off(g) + node) : 0u;
      if (IS_S) {
        const uint32_t bb = (g > 0 && w < g) ? __ldcg(ccw + p.brow + g * G + w) : 0u;
        sc = (sc << 1) | ((bb >> lane) & 1u);
      }
      const uint32_t x = transpose32(sc, lane);
      if (row < n) out[((size_t)(out_base + cc) * n + row) * W32 + w] = x;
    }
    if (row < n)
      for (int w = g + 1; w < W32; ++w) out[((size_t)(out_base + cc) * n + row) * W32 + w] = 0u;
  }
}

// Scratch of one K2 warp: shared-memory views (graph blob, E, spilled A' slots) and TMEM.
template <typename ET, bool TM>
struct ScanCtx {
  const int64_t* M;
  const int64_t* C;
  const int4* nrec;
  const int2* drec;
  const int32_t* qinfo;
  ET* E;                      // [32 stages][32 lanes]
  ET* massbuf;                // [chunk][32 lanes][16 bytes]: the task's checkpoint masses (rows 32g ..)
  uint32_t snr;               // shared address of this lane's 16 bytes in quad slot 0 of the Sn ring
  AView<TM> A;
  bool all_tm;
};

// tcols: TMEM columns per warp (512 / warps per lane quarter); slots beyond spill to shared memory.
template <typename ET, bool TM, int Q = kSnRing>
__device__ __forceinline__ ScanCtx<ET, TM> scan_ctx(const ScanParams& p, unsigned char* smem, int wk, uint32_t tmem_base,
                                                    int tcols) {
  ScanCtx<ET, TM> x;
  const int lane = threadIdx.x & 31;
  x.M = reinterpret_cast<const int64_t*>(smem);
  x.C = x.M + p.n;
  x.nrec = reinterpret_cast<const int4*>(smem + p.o_nrec);
  x.drec = reinterpret_cast<const int2*>(smem + p.o_drec);
  x.qinfo = reinterpret_cast<const int32_t*>(smem + p.o_qinfo);
  unsigned char* wr = smem + p.blob_bytes + (size_t)wk * p.warp_bytes;
  x.E = reinterpret_cast<ET*>(wr);
  x.massbuf = reinterpret_cast<ET*>(wr + 32 * 32 * sizeof(ET));           // int32 state only
  x.snr = smem_u32(wr + scan_e_bytes(sizeof(ET) == 4, Q) - 512 * sn_ring_quads(sizeof(ET) == 4, Q)) + 16u * (uint32_t)lane;
  x.A.sm = reinterpret_cast<uint32_t*>(wr + scan_e_bytes(sizeof(ET) == 4, Q));   // [slot][lane] (spill part)
  x.A.lane = lane;
  x.A.tmc = TM ? min(p.n_slot, tcols) : 0;
  // TMEM: a warp reaches lane quarter (CTA warp index % 4); K2 warp wk takes columns 256 (wk / 4) ..
  x.A.taddr = TM ? tmem_base + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16) + (uint32_t)(tcols * (wk >> 2)) : 0u;
  x.all_tm = TM && p.n_slot <= tcols;
  return x;
}

// L2-prefetch the candidate blocks a later task (group gn, candidates cn = first + lane) reads.
__device__ __forceinline__ void scan_prefetch(const ScanParams& p, const uint32_t* ws, int64_t n_cand, int gn,
                                              int64_t cn) {
  const int n = p.n, G = p.G;
  if (cn >= n_cand) return;
  const unsigned char* b = reinterpret_cast<const unsigned char*>(ws + cn * p.cs);
  const unsigned char* col = b + 4 * (size_t)grp_off(gn);
  if (32 * gn + 1 < n) {                                            // the group has Sn columns
    for (int off = 0; off < 128 * (gn + 1); off += 128) prefetch_l2(col + off);
    prefetch_l2(col + 128 * (gn + 1) - 4);                          // the block is 16-byte aligned
  }
  prefetch_l2(b + 4 * ((size_t)p.brow + (size_t)gn * G));
  const unsigned char* ms = b + 4 * (size_t)block_words(G) + (size_t)p.mass_bytes * (32 * gn);
  prefetch_l2(ms);
  if (p.mass_bytes == 8) prefetch_l2(ms + 128);
}

// One K2 task: stage group g of the 32 candidates batch0 .. batch0+31 of a buffer `ws` holding
// n_cand candidate blocks; writes part[c][g] = {max_t (mass_t + E_t) over the group's stages,
// the group's cost} and (optionally) the group's rows of the R / S masks (global candidate
// index out_base + c).  Everything the task reads from `ws` bypasses L1 (.cg): the fused kernel
// rewrites a ring slot in the same launch.
template <typename ET, bool TM, int Q = kSnRing>
__device__ __forceinline__ void scan_task(const ScanParams& p, const ScanCtx<ET, TM>& x, int g, int64_t batch0,
                                          uint32_t* ws, int64_t n_cand, int64_t* part, int64_t out_base) {
  const int lane = threadIdx.x & 31;
  const int n = p.n, G = p.G;
  const int64_t* M = x.M;
  const int64_t* C = x.C;
  const int4* nrec = x.nrec;
  const int2* drec = x.drec;
  const int32_t* qinfo = x.qinfo;
  ET* E = x.E;
  const AView<TM>& A = x.A;
  const bool all_tm = x.all_tm;
  const int64_t c = batch0 + lane;
  const bool live = c < n_cand;
  const int nk = min(n, 32 * (g + 1));                            // nodes 0..nk-1
  const int nq = (nk + 3) >> 2;                                   // uint4 blocks of Sn
  uint32_t* cw = ws + (live ? c : 0) * p.cs;
  const uint4* sn4 = reinterpret_cast<const uint4*>(cw + grp_off(g));
  const bool lsn = live && 32 * g + 1 < n;                        // K1 wrote Sn for this group
  // the group's 32 checkpoint masses (Eq. 6 sums, rows 32g ..; ET-wide: 128 or 256 bytes)
  // -> shared memory [chunk j][lane][16 bytes], asynchronously
  constexpr int kMassChunks = 2 * (int)sizeof(ET);
  constexpr bool kStageMass = kStageMassCfg && sizeof(ET) == 4;     // else read at the end (.cg)
  if (kStageMass && live) {
    const char* msrc = reinterpret_cast<const char*>(cw + block_words(G)) + 32 * sizeof(ET) * (size_t)g;
    const uint32_t mdst = smem_u32(x.massbuf) + 16u * (uint32_t)lane;
#pragma unroll
    for (int j = 0; j < kMassChunks; ++j)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(mdst + 512u * (uint32_t)j), "l"(msrc + 16 * j)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (p.s_mask32) emit_mask<true>(p, ws, n_cand, out_base, p.s_mask32, g, nk, batch0, lane);   // before R overwrites
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
  // E_t after stage t's first event, the compute of its own node t (see events())
  for (int b = 0; b < 32; ++b) E[32 * b + lane] = 32 * g + b < n ? (ET)M[32 * g + b] : (ET)0;
  __syncwarp();
  const uint32_t* brow = cw + p.brow + g * G;                     // S row 32g, row form
  int64_t costL = 0;
  uint32_t* rcol = cw + grp_off(g);
  if (p.r_mask32) {
    if (!TM) walk<ET, TM, 0, true, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
    else if (all_tm) walk<ET, TM, 2, true, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
    else walk<ET, TM, 1, true, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
  } else {
    if (!TM) walk<ET, TM, 0, false, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
    else if (all_tm) walk<ET, TM, 2, false, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
    else walk<ET, TM, 1, false, Q>(nk, g, live, lsn, sn4, rcol, brow, nrec, drec, M, C, A, E, lane, costL, x.snr);
  }
  A.wait_st();                                                    // next task re-fills the slots
  // ---- group result: max_t (mass_t + E_t) over this group's stages, cost sum ----
  // the group's checkpoint masses were copied to shared memory at the task start
  int64_t pk = INT64_MIN;
  if (kStageMass) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    constexpr int kPer = 16 / (int)sizeof(ET);                      // masses per 16-byte chunk
#pragma unroll 4
    for (int j = 0; j < kMassChunks; ++j) {
      ET mv[kPer];
      *reinterpret_cast<uint4*>(mv) = reinterpret_cast<const uint4*>(x.massbuf)[32 * j + lane];
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        const int b = kPer * j + e, r = 32 * g + b;
        if (r < n) pk = max(pk, (r ? (int64_t)mv[e] : 0) + (int64_t)E[32 * b + lane]);
      }
    }
  } else if (sizeof(ET) == 4) {
    // the group's 32 int32 masses (rows 32g .., 128 bytes, L2-prefetched with the task)
    const uint4* m4 = reinterpret_cast<const uint4*>(cw + block_words(G)) + 8 * g;
    uint4 mv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) mv[j] = live ? __ldcg(m4 + j) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t w4[4] = {mv[j].x, mv[j].y, mv[j].z, mv[j].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int b = 4 * j + e, r = 32 * g + b;
        if (r < n) pk = max(pk, (r ? (int64_t)(int32_t)w4[e] : 0) + (int64_t)E[32 * b + lane]);
      }
    }
  } else {
    const int64_t* mass = reinterpret_cast<const int64_t*>(cw + block_words(G));
#pragma unroll
    for (int b0 = 0; b0 < 32; b0 += 8) {                            // 8 loads in flight at a time
      int64_t mv[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int r = 32 * g + b0 + b;
        mv[b] = (r && r < n && live) ? __ldcg(mass + r) : 0;
      }
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (32 * g + b0 + b < n) pk = max(pk, mv[b] + (int64_t)E[32 * (b0 + b) + lane]);
    }
  }
  if (live) {
    int64_t* pp = part + 2 * (c * G + g);
    pp[0] = pk;
    pp[1] = costL;
  }
  if (p.r_mask32) {
    __syncwarp();
    __threadfence_block();
    emit_mask<false>(p, ws, n_cand, out_base, p.r_mask32, g, nk, batch0, lane);
  }
  __syncwarp();
}

// ET = int32_t when every M is a multiple of a scale s with sum M/s < 2^30 (the host checks;
// exact), else int64_t.  M in the blob, the masses and the results are in units of s.
// TM: slots < 256 in Tensor Memory (8 warps, one CTA per SM, 512 TMEM columns: warp w uses
// lane quarter w % 4 and columns 256 * (w / 4) ..).
template <typename ET, bool TM>
__global__ void __launch_bounds__(256, 2) scan_kernel(const ScanParams p) {   // <= 128 regs: co-resides with K1
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
#ifdef CM_EXP_SCAN_PAD
  __shared__ uint32_t pad[8];                                       // diagnostic: moves tmem_base
  if (threadIdx.x < 8) pad[threadIdx.x] = 0u;
#endif
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
  const ScanCtx<ET, TM> x = scan_ctx<ET, TM>(p, smem, warp, TM ? tmem_base : 0u, 256);
  const int G = p.G;
  const int lane = threadIdx.x & 31;
  const int tasks = G * p.n_batch;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int task = gw; task < tasks; task += nwarps) {
    const int g = G - 1 - task / p.n_batch;                         // big groups first
    const int64_t batch0 = (int64_t)(task % p.n_batch) * 32;
    const int tn = task + nwarps;                                   // pull the next task towards L2
    if (p.prefetch && tn < tasks)
      scan_prefetch(p, p.ws, p.n_cand, G - 1 - tn / p.n_batch, (int64_t)(tn % p.n_batch) * 32 + lane);
    scan_task<ET, TM>(p, x, g, batch0, p.ws, p.n_cand, p.part, p.out_base);
  }
  if (TM) {
    x.A.wait_st();
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
  // max-batch epilogue (Eq. 13): candidates with cost <= cost_limit compete
  // per budget for the largest B_max = floor((b - ovh) / (peak - ovh)) >= 1 (capped at 2^31-1);
  // key ((2^31-1 - B_max) << idx_bits) | idx, atomicMin into best_batch_key (nullptr: off)
  int64_t cost_limit;
  int64_t* best_batch_key;
  // a8 in the reduce step: NVLink multicast views of best_key / best_batch_key
  // (nullptr: atomics on the local buffers).  multimem.red.min reaches every GPU's replica.
  int64_t* best_key_mc;
  int64_t* best_batch_key_mc;
};

// MIN of key into *p: a multicast address (every participating GPU's replica, reduced in the
// NVSwitch) or the local buffer.  Keys are >= 0, so the signed MIN is the key order.
__device__ __forceinline__ void key_min(int64_t* local, int64_t* mc, int b, int64_t key) {
  if (mc)
    asm volatile("multimem.red.relaxed.sys.global.min.s64 [%0], %1;" :: "l"(mc + b), "l"(key) : "memory");
  else
    atomicMin(reinterpret_cast<long long*>(local + b), (long long)key);
}

// peak / cost / a7 keys of candidate c (part rows c, output index out_base + c).
__device__ __forceinline__ void reduce_one(const ReduceParams& p, const int64_t* part, int64_t c, int64_t out_base) {
  const int64_t* pp = part + 2 * c * p.G;
  int64_t pk = INT64_MIN, cs = 0;
  for (int g = 0; g < p.G; ++g) {
    pk = max(pk, __ldcg(pp + 2 * g));
    cs += __ldcg(pp + 2 * g + 1);
  }
  pk = p.ovh + p.mscale * pk;
  const int64_t local = out_base + c;
  p.peak[local] = pk;
  p.cost[local] = cs;
  const int64_t key = (cs << p.idx_bits) | (p.index_base + local);
  for (int b = 0; b < p.n_budget; ++b) {
    if (pk <= __ldg(p.budget + b)) {
      const int64_t cur = *reinterpret_cast<volatile const int64_t*>(p.best_key + b);
      if (key < cur) key_min(p.best_key, p.best_key_mc, b, key);
    }
  }
  if (p.best_batch_key && cs <= p.cost_limit) {
    constexpr int64_t kCap = (int64_t(1) << 31) - 1;
    for (int b = 0; b < p.n_budget; ++b) {
      const int64_t bu = __ldg(p.budget + b);
      const int64_t bm = bu < p.ovh ? 0 : (pk <= p.ovh ? kCap : min(kCap, (bu - p.ovh) / (pk - p.ovh)));
      if (bm >= 1) {
        const int64_t k2 = ((kCap - bm) << p.idx_bits) | (p.index_base + local);
        const int64_t cur = *reinterpret_cast<volatile const int64_t*>(p.best_batch_key + b);
        if (k2 < cur) key_min(p.best_batch_key, p.best_batch_key_mc, b, k2);
      }
    }
  }
}

template <int = 0>
__global__ void __launch_bounds__(256) reduce_kernel(const ReduceParams p) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p.n_cand) return;
  reduce_one(p, p.part, c, p.out_base);
}

// ------------------------------------------------------------------------------------ fused
// One persistent launch per call (n_theta <= 4, int32 scan state, A' in TMEM): every CTA runs
// KF1 = k1_warps(NT) rounding warps (the K1 body) and KF2 = 8 scan warps (the K2 task body)
// side by side, handing the stage-sliced S columns over through a ring of R slots in global
// memory that stays L2-resident (a slot = one unit of 32 S*: 32 n_theta candidate blocks plus
// their per-group partials, ~0.43 MB at n = 353).  Unit u lives in slot u % R.
//   K1 warp, S* s of unit u = s / 32:  wait freed[slot] >= u / R  (the slot's previous unit is
//     scanned and reduced), write the blocks, then fence + filled[slot] += 1.
//   K2 warp: take task tickets in order (one atomic per task: dynamic balance over tasks of very
//     different length); task (u, g, batch) waits filled[slot] >= 32 (u / R) + |u|, runs the scan
//     task, fences, done[slot] += 1; the warp that completes unit u reduces its candidates
//     (peak, cost, per-budget keys: the K3 step) right there, then freed[slot] += 1.
// Deadlock-free: the smallest unwritten S* belongs to a unit whose slot predecessor is complete
// (all its S* are smaller), and tickets are issued in unit order, so that predecessor's tasks
// are held by warps that can run them.  One launch removes the two-kernel pipeline's fill and
// drain, its per-chunk prologues and tails, and the DRAM round trip of the chunk buffers.
struct FusedParams {
  RoundParams rp;             // rp.s_begin = 0, rp.s_count = n_sstar, rp.th0 = 0, rp.nt = n_theta
  ScanParams sp;              // per-task buffer fields unused
  ReduceParams qp;            // part / n_cand / out_base unused
  uint32_t* ring;             // n_slots slots of slot_words words
  int64_t slot_words;         // 32 n_theta cs words of candidate blocks, then the partials
  int32_t n_slots;
  uint32_t* ctl;              // [0] task ticket, [1 + slot] filled, [1 + R + slot] done,
                              // [1 + 2R + slot] freed, [1 + 3R] S* ticket, [2 + 3R] CTAs
                              // exited, [3 + 3R] key-init state; fused_ctl_words(R) words, zero
                              // at launch and zeroed again by the last CTA to exit
  int32_t n_sstar, n_theta;
  int32_t n_units;
  int32_t tpu;                // tasks of a full unit: G * n_theta
  int64_t total_tasks;
  int32_t claim;              // S* per producer ticket (power of two <= 32)
  int32_t task_claim;         // scan tasks per consumer ticket (divides tpu)
  int32_t win_units;          // ticket windows (units), 0: unit-major order
  uint64_t* trace;            // debug (CM_TRACE=2): per CTA {start, K1 end, ~first unit-0 task, K2 end} ns
  int32_t init_keys;          // CM_EVAL_INIT_KEYS: the first CTA sets the keys to INT64_MAX
  uint32_t* seq_word;         // completion signal (cm_stream_wait_call): the last CTA out stores
  uint32_t seq;               //   seq here once every output of the call is written
};
__host__ __device__ constexpr int64_t fused_ctl_words(int64_t R) { return 4 + 3 * R; }

// Kernel exit: every warp of the CTA (both roles) has stopped touching the control words;
// the last CTA out zeroes them, so the next call on this workspace half can skip the memset
// (and start while this one drains: CM_EVAL_OVERLAP).
__device__ __forceinline__ void fused_exit(const FusedParams& fp) {
  __shared__ uint32_t last;
  // Let the next call (CM_EVAL_OVERLAP) be scheduled -- its CTAs then take SMs as this call's
  // CTAs exit -- but only once the call before this one has completed: the next call reuses
  // that call's workspace half, and a CTA that cannot get TMEM yet may already be resident
  // when shared memory allows two CTAs per SM, so residency alone does not order them.
  // Thread 0 (rounding warp 0) gets here when its production ends, well before the tail.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
  // (non-.aligned barrier: the rounding and the scan warps reach it from different code)
  asm volatile("barrier.sync 2, %0;" :: "r"((int)blockDim.x) : "memory");
  const int64_t words = fused_ctl_words(fp.n_slots);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(fp.ctl + 2 + 3 * (int64_t)fp.n_slots, 1u) == gridDim.x - 1;
  }
  asm volatile("barrier.sync 2, %0;" :: "r"((int)blockDim.x) : "memory");
  if (last && threadIdx.x == 0 && fp.seq_word) {
    // every CTA fenced its outputs before its exit count, and this CTA saw all the counts:
    // publish the call's number to a stream wait on another stream (system-scope release)
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(fp.seq_word), "r"(fp.seq) : "memory");
  }
  if (last) {
    __threadfence();
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) fp.ctl[i] = 0u;
    __threadfence();
  }
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// lane 0 waits until *p >= target (then the warp proceeds); exponential back-off sleep.  The
// counters only grow: poll with relaxed loads (an acquire load invalidates L1 -- CCTL.IVALL --
// every time) and acquire once when the target is reached.
// CAP: the back-off ceiling in ns -- a producer waiting for a ring slot waits on the scan (a
// long wait when the scan binds: its polls would only take issue slots from the scan warps).
#ifndef CM_SLOT_WAIT_NS
#define CM_SLOT_WAIT_NS 8192
#endif
template <uint32_t CAP = 1024>
__device__ __forceinline__ void warp_wait_geq(const uint32_t* p, uint32_t target) {
  if ((threadIdx.x & 31) == 0) {
    uint32_t ns = 32;
    while (ld_relaxed(p) < target) {
      __nanosleep(ns);
      ns = ns < CAP ? 2 * ns : ns;
    }
    (void)ld_acquire(p);
  }
  __syncwarp();
}

struct K1Ring {
  static constexpr bool kTab = true;                              // randomized: the per-S* Philox table
  uint32_t* ring;
  int64_t slot_words;
  int32_t n_slots, n_theta, cs;
  uint32_t* ctl;
  int32_t claim;              // S* per ticket (a power of two <= 32: a claim never straddles a unit)
  int32_t s_count;
  // S* tickets (in order across all K1 warps; a CTA that starts late simply takes later ones).
  // Small graphs take several consecutive S* per ticket, so the fence and the count are paid
  // once per claim rather than once per S*.
  __device__ __forceinline__ int first() const {
    uint32_t t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ctl + 1 + 3 * n_slots, 1u);
    return (int)__shfl_sync(FULL, t, 0) * claim;
  }
  __device__ __forceinline__ int next(int s) const { return ((s + 1) & (claim - 1)) ? s + 1 : first(); }
  __device__ __forceinline__ uint32_t* begin(int s) const {
    const int u = s >> 5, slot = u % n_slots, k = u / n_slots;
    if (k > 0 && (s & (claim - 1)) == 0) warp_wait_geq<CM_SLOT_WAIT_NS>(ctl + 1 + 2 * n_slots + slot, (uint32_t)k);
    return ring + (int64_t)slot * slot_words + (int64_t)(s & 31) * n_theta * cs;
  }
  __device__ __forceinline__ void end(int s) const {
    if ((s & (claim - 1)) != claim - 1 && s != s_count - 1) return;   // not the claim's last S*
#ifndef CM_EXP_NOFENCE
    __threadfence();                                                // this lane's blocks, then the count
#endif
    __syncwarp();
    if ((threadIdx.x & 31) == 0) atomicAdd(ctl + 1 + (s >> 5) % n_slots, (uint32_t)((s & (claim - 1)) + 1));
  }
};

#ifndef CM_KF2
#define CM_KF2 8
#endif
// scan warps per fused CTA.  Measured: 10 (96 registers, spills) 17.3 vs 18.5 M cand/s for 8;
// setmaxnreg to rebalance registers needs whole warpgroups (10 scan warps hang), and 12 do
// not fit in shared memory at n = 353.
// With 2-4 thresholds (deterministic) a S* carries N_theta candidates for the scan, so those
// instances run 12 scan warps (registers rebalanced by setmaxnreg, Sn rings of 4 quads to fit
// shared memory): N_theta = 4 at ResNet-50 16.2 -> 17.7 M cand/s.  (At one threshold 12 scan
// warps measured +7 % for R-heavy S* families but -5 % for G1 and -12 % for VGG16; randomized
// rounding's K1 needs more than the 72 registers the rebalance leaves it.)
#ifndef CM_KF2N
#define CM_KF2N 12
#endif
#ifndef CM_SN_RING_N
#define CM_SN_RING_N 4
#endif
// randomized rounding with 2-4 samples: scan warps (tuning; its K1 keeps CM_FUSED_K1_REGS_RAND)
#ifndef CM_KF2N_RAND
#define CM_KF2N_RAND CM_KF2
#endif
__host__ __device__ constexpr int fused_scan_warps(int nt, bool rand) {
  return nt >= 2 ? (rand ? CM_KF2N_RAND : CM_KF2N) : CM_KF2;
}
__host__ __device__ constexpr int fused_sn_ring(int nt, bool rand) {
  return fused_scan_warps(nt, rand) > 8 ? CM_SN_RING_N : kSnRing;
}
#ifndef CM_FUSED_TMEM
#define CM_FUSED_TMEM 512
#endif
constexpr int kFusedTmem = CM_FUSED_TMEM;                           // TMEM columns per CTA (512: one CTA per SM)
__host__ __device__ constexpr int fused_tmem_cols(int nt, bool rand) {   // per scan warp
  return kFusedTmem / ((fused_scan_warps(nt, rand) + 3) / 4);
}
__host__ __device__ constexpr int fused_warps(int nt, bool rand) { return k1_warps(nt) + fused_scan_warps(nt, rand); }
// dynamic shared memory: [K1 region, 1024-aligned][K2: graph blob, per-warp E / spill]
__host__ __device__ constexpr size_t fused_k1_bytes(int nt, int nib_entries, bool bulk, int rtab = 0) {
  return (k1_nib_off(nt, bulk) + 4 * (size_t)nib_entries + 15) / 16 * 16 + (size_t)k1_warps(nt) * rtab + 1023 &
         ~(size_t)1023;
}

// Register rebalance (setmaxnreg, whole warpgroups): more than 16 warps per CTA leave fewer than
// 128 registers per thread at launch; the rounding warps then drop to CM_FUSED_K1_REGS (the K1
// body needs ~72) and the scan warps grow by what they released -- an increase is served from
// the CTA's own pool of released registers only (USETMAXREG.TRY_ALLOC.CTAPOOL spins until it
// can be), so sum of increases <= sum of decreases, or the scan warps wait forever.
#ifndef CM_FUSED_K1_REGS
#define CM_FUSED_K1_REGS 72
#endif
#ifndef CM_FUSED_K1_REGS_RAND
#define CM_FUSED_K1_REGS_RAND 88
#endif
__host__ __device__ constexpr int fused_k1_regs(bool rand) { return rand ? CM_FUSED_K1_REGS_RAND : CM_FUSED_K1_REGS; }
__host__ __device__ constexpr int fused_launch_regs(int nt, bool rand) {
  return (65536 / (32 * fused_warps(nt, rand))) / 8 * 8;
}
__host__ __device__ constexpr int fused_k2_regs(int nt, bool rand) {
  return (fused_launch_regs(nt, rand) + k1_warps(nt) * (fused_launch_regs(nt, rand) - fused_k1_regs(rand)) /
          fused_scan_warps(nt, rand)) / 8 * 8;
}

// ET: the scan state (int32 when sum M / gcd < 2^31, else int64).
template <int NT, int LAY, bool RAND, typename ET>
#ifndef CM_FUSED_MINB
#define CM_FUSED_MINB 1
#endif
__global__ void __launch_bounds__(32 * fused_warps(NT, RAND), CM_FUSED_MINB) fused_kernel(const FusedParams fp,
                                                                         const __grid_constant__ CUtensorMap tmap,
                                                                         const __grid_constant__ DiagMaps dmaps) {
  constexpr int KF1 = k1_warps(NT);
  constexpr int KF2 = fused_scan_warps(NT, RAND);
  constexpr int kQ = fused_sn_ring(NT, RAND);
  // warp roles: the rounding warps take the low (default) or, with CM_K1_HIGH, the high warp
  // indices -- the SMSP arbiter favours higher warp ids
#ifdef CM_K1_HIGH
  constexpr bool kK1High = true;
#else
  constexpr bool kK1High = false;
#endif
  constexpr int kFirstScanWarp = kK1High ? 0 : KF1;
  extern __shared__ __align__(1024) unsigned char fraw[];
  unsigned char* base = fraw + ((1024u - (smem_u32(fraw) & 1023u)) & 1023u);
  unsigned char* k1smem = base;
  unsigned char* k2smem = base + fused_k1_bytes(NT, fp.rp.nib32 ? fp.rp.nib_entries : 0, LAY == 1, fp.rp.rtab);
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ScanParams& sp = fp.sp;
  if (fp.init_keys && threadIdx.x == 0 &&
      atomicCAS(fp.ctl + 3 + 3 * (int64_t)fp.n_slots, 0u, 1u) == 0u) {       // first CTA in
    for (int b = 0; b < fp.qp.n_budget; ++b) {
      fp.qp.best_key[b] = INT64_MAX;
      if (fp.qp.best_batch_key) fp.qp.best_batch_key[b] = INT64_MAX;
    }
    __threadfence();
    atomicExch(fp.ctl + 3 + 3 * (int64_t)fp.n_slots, 2u);
  }
  k1_setup<NT, LAY, RAND>(fp.rp, k1smem, KF1, (int)threadIdx.x, (int)blockDim.x);
  for (int i = threadIdx.x; i < sp.blob_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(k2smem)[i] = sp.blob[i];
  if (warp == kFirstScanWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(kFusedTmem) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (fp.trace && threadIdx.x == 0) fp.trace[4 * blockIdx.x] = globaltimer();

  constexpr bool kRebal = fused_warps(NT, RAND) > 16;
  static_assert(!kRebal || (KF1 % 4 == 0 && KF2 % 4 == 0 && !kK1High), "warpgroup roles");
  static_assert(!kRebal || (fused_k1_regs(RAND) <= fused_launch_regs(NT, RAND) && fused_k2_regs(NT, RAND) <= 256),
                "register pool");
  if (kK1High ? warp >= KF2 : warp < KF1) {                         // ---- rounding (K1) warps
    if constexpr (kRebal) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(fused_k1_regs(RAND)));
    __shared__ int sq[KF1][8];
    const int w1 = kK1High ? warp - KF2 : warp;
    const K1Ring hk{fp.ring, fp.slot_words, fp.n_slots, fp.n_theta, fp.rp.cs, fp.ctl, fp.claim, fp.n_sstar};
    // the int32 scan state <=> the int32 mass tables (both: every row mass fits, cm_api.cu)
    k1_body<NT, LAY, RAND, K1Ring, sizeof(ET) == 4 ? 1 : 2>(fp.rp, &tmap, &dmaps, k1smem, w1, sq[w1], hk);
    if (fp.trace && lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(fp.trace + 4 * blockIdx.x + 1), globaltimer());
    fused_exit(fp);
    return;
  }
  // ---- scan (K2) warps
  if constexpr (kRebal) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(fused_k2_regs(NT, RAND)));
  const int wk = warp - kFirstScanWarp;
  const ScanCtx<ET, true> x = scan_ctx<ET, true, kQ>(sp, k2smem, wk, tmem_base, fused_tmem_cols(NT, RAND));
  const int G = sp.G;
  const int R = fp.n_slots;
  const int64_t unit_cands = 32 * (int64_t)fp.n_theta;
  // tickets are claimed one task ahead, so the next task's blocks can be pulled into L2 while
  // the current one scans (when its unit is already filled)
  auto claim = [&]() {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(fp.ctl, 1u);
    return __shfl_sync(FULL, t, 0);
  };
  struct Task {
    int u, g, batch, slot, k, ns;
    int64_t ncand;
    bool valid;
  };
  // Ticket order.  win_units == 0: unit by unit, big groups first inside a unit.  Otherwise
  // windows of win_units units, each ordered (group descending, unit, batch), so the longest
  // tasks of the batch's last units are claimed early and the launch does not end on one
  // long walk (tickets of a short last window / unit that name no task are skipped).
  auto decode = [&](uint32_t t) {
    Task d;
    int sub;
    if (fp.win_units == 0) {
      d.u = (int)(t / (uint32_t)fp.tpu);
      sub = (int)(t - (uint32_t)d.u * (uint32_t)fp.tpu);
    } else {
      const uint32_t per_win = (uint32_t)fp.win_units * (uint32_t)fp.tpu;
      const uint32_t w = t / per_win, r = t - w * per_win;
      const uint32_t per_g = (uint32_t)fp.win_units * (uint32_t)fp.n_theta;   // full-unit batches
      const uint32_t gi = r / per_g, rr = r - gi * per_g;
      d.u = (int)(w * (uint32_t)fp.win_units + rr / (uint32_t)fp.n_theta);
      sub = (int)(gi * (uint32_t)fp.n_theta + rr % (uint32_t)fp.n_theta);
    }
    d.valid = d.u < fp.n_units;
    d.ns = d.valid ? min(32, fp.n_sstar - 32 * d.u) : 0;            // S* of this unit
    d.ncand = (int64_t)d.ns * fp.n_theta;
    const int nb = fp.win_units == 0 ? (int)((d.ncand + 31) / 32) : fp.n_theta;   // batches per group slot
    d.g = G - 1 - sub / nb;                                         // big groups first
    d.batch = sub % nb;
    d.valid = d.valid && (int64_t)d.batch * 32 < d.ncand;
    d.slot = d.u % R;
    d.k = d.u / R;
    return d;
  };
  // A ticket covers tc consecutive tasks (tc divides tpu, so a claim stays inside one unit):
  // small graphs take a whole unit per ticket and pay the fence and the count once per unit.
  const uint32_t tc = (uint32_t)fp.task_claim;
  bool keys_ready = false;
  uint32_t t = claim();
  while ((int64_t)t * tc < fp.total_tasks) {
    const uint32_t t_next = claim();
    const uint32_t t0 = t * tc;
    const Task d0 = decode(t0);
    if (!d0.valid) {                                                // a ticket that names no task
      t = t_next;
      continue;
    }
    const int u = d0.u, slot = d0.slot, k = d0.k, ns = d0.ns;
    const int64_t ncand = d0.ncand;
    const int nb = (int)((ncand + 31) / 32);
    const uint32_t tasks_u = (uint32_t)(G * nb);
    uint32_t* ws = fp.ring + (int64_t)slot * fp.slot_words;
    int64_t* part = reinterpret_cast<int64_t*>(ws + unit_cands * sp.cs);
    warp_wait_geq(fp.ctl + 1 + slot, (uint32_t)(32 * k + ns));
    if (fp.trace && lane == 0 && u == 0)                            // first unit ready (any warp)
      atomicMax(reinterpret_cast<unsigned long long*>(fp.trace + 4 * blockIdx.x + 2), ~globaltimer());   // min
    uint32_t cnt = 0;
    for (uint32_t j = 0; j < tc; ++j) {
      const uint32_t tt = t0 + j;
      if ((int64_t)tt >= fp.total_tasks) break;                     // the last unit may be short
      const Task d = decode(tt);
      if (sp.prefetch & 1) scan_prefetch(sp, ws, ncand, d.g, (int64_t)d.batch * 32 + lane);
      if ((sp.prefetch & 2) && tc == 1 && (int64_t)t_next < fp.total_tasks) {
        const Task e = decode(t_next);
        bool ready = false;
        if (lane == 0) ready = ld_acquire(fp.ctl + 1 + e.slot) >= (uint32_t)(32 * e.k + e.ns);
        if (__shfl_sync(FULL, ready, 0))
          scan_prefetch(sp, fp.ring + (int64_t)e.slot * fp.slot_words, e.ncand, e.g, (int64_t)e.batch * 32 + lane);
      }
#ifndef CM_EXP_NOSCAN
      scan_task<ET, true, kQ>(sp, x, d.g, (int64_t)d.batch * 32, ws, ncand, part, (int64_t)u * unit_cands);
#endif
      ++cnt;
    }
#ifndef CM_EXP_NOFENCE
    __threadfence();                                                // reads done, partials visible
#endif
    __syncwarp();
    uint32_t old = 0;
    if (lane == 0) old = atomicAdd(fp.ctl + 1 + R + slot, cnt);
    old = __shfl_sync(FULL, old, 0);
    if (old + cnt == (uint32_t)fp.tpu * (uint32_t)k + tasks_u) {     // last task of unit u: reduce it
      if (fp.init_keys && !keys_ready) {                            // the keys are initialised
        warp_wait_geq(fp.ctl + 3 + 3 * R, 2u);
        keys_ready = true;
      }
      __threadfence();
      for (int64_t c = lane; c < ncand; c += 32) reduce_one(fp.qp, part, c, (int64_t)u * unit_cands);
#ifdef CM_DISCARD
      // the slot's data is dead: drop its L2 lines without writing them back to DRAM
      __syncwarp();
      for (int64_t l = lane; l < fp.slot_words / 32; l += 32)
        asm volatile("discard.global.L2 [%0], 128;" :: "l"(ws + 32 * l) : "memory");
#endif
      __threadfence();                                              // partials read: release the slot
      __syncwarp();
      if (lane == 0) atomicAdd(fp.ctl + 1 + 2 * R + slot, 1u);
    }
    t = t_next;
  }
  x.A.wait_st();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (fp.trace && lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(fp.trace + 4 * blockIdx.x + 3), globaltimer());
  asm volatile("bar.sync 1, %0;" :: "r"(32 * KF2) : "memory");      // the scan warps only
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == kFirstScanWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "n"(kFusedTmem) : "memory");
  fused_exit(fp);
}

}  // namespace cm2

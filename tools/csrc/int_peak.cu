// int_peak.cu -- K-mu: the integer-pipe roofline denominator.
//
// Measurement tool, not product code: every thread of a full-chip grid (SMs x 4 CTAs x 256
// threads) runs long unrolled chains of one instruction class on 8 independent registers
// (enough ILP to cover the 4-cycle pipe latency at one warp instruction per 2 cycles per
// SMSP), and the kernel reads its own SM clock: %clock64 and %globaltimer deltas of each
// CTA give the loaded clock.  Classes (the SASS each asm emits, checked with cuobjdump):
//   0 LOP3   lop3.b32               (alu pipe)
//   1 IADD3  add.u32 of three terms (alu pipe)
//   2 IMAD   mad.lo.u32             (fma pipe)
//   3 LOP3 + IMAD interleaved       (alu + fma pipes together: the integer issue ceiling)
//   4 POPC   popc.b32
//   5 FLO    bfind.u32 (FLO)
//   6 SHFL   shfl.sync.bfly.b32
//   7 FSETP + predicated OR (the K1 compare-and-pack pair, counted as 2 ops)
// Pipe probes (tools/int_peak.py --pipes; which pipe an instruction of the randomized-rounding
// K1 body issues to: a mix with LOP3 that runs at twice LOP3's rate shares no pipe with it):
//   8 IMAD.WIDE.U32  mul.wide.u32 (chained through hi)       9 I2FP.F32.U32  cvt.rn.f32.u32
//  10 SHF.L.W        shf.l.wrap.b32                          11 FFMA2        fma.rn.f32x2 (2 ops)
//  12 IMAD.HI.U32    mul.hi.u32 by a register                13 LOP3 + I2FP
//  14 LOP3 + IMAD.WIDE                                       15 LOP3 + IMAD.HI
//  16 IADD3 + IADD3.X carry pack (sub.cc + addc, 2 ops)      17 LOP3 + FFMA2 (1 + 2 ops)
//  18 LOP3 + SHF                                             19 LOP3 + carry pack (1 + 2 ops)
// ops = threads x iterations x ops per iteration (lane ops).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int CLS>
__device__ __forceinline__ void step(uint32_t (&r)[8], uint64_t (&a)[8], uint32_t k) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (CLS == 0) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(k), "r"(r[(j + 1) & 7]));
    } else if (CLS == 1) {
      asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(r[j]) : "r"(k), "r"(r[(j + 3) & 7]));
    } else if (CLS == 2) {
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(k | 1u), "r"(r[(j + 1) & 7]));
    } else if (CLS == 3) {
      if (j & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(k | 1u), "r"(r[(j + 1) & 7]));
      else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(k), "r"(r[(j + 1) & 7]));
    } else if (CLS == 4) {
      uint32_t t;
      asm volatile("popc.b32 %0, %1;" : "=r"(t) : "r"(r[j] ^ k));
      r[j] += t;   // IADD: not counted (the POPC rate is the number reported)
    } else if (CLS == 5) {
      uint32_t t;
      asm volatile("bfind.u32 %0, %1;" : "=r"(t) : "r"(r[j] | k));
      r[j] ^= t;
    } else if (CLS == 6) {
      asm volatile("shfl.sync.bfly.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(r[j]) : "r"((j & 3) + 1));
    } else if (CLS == 7) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.gt.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
                   : "+r"(r[j]) : "f"(__uint_as_float(r[(j + 1) & 7])), "f"(0.5f), "r"(1u << j));
    } else {
      constexpr int kMix = CLS >= 13 && CLS != 16;                  // odd j: LOP3
      if (kMix && (j & 1)) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(k), "r"(r[(j + 1) & 7]));
      } else if (CLS == 8 || CLS == 14) {
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(a[j]) : "r"((uint32_t)(a[j] >> 32)), "r"(k | 1u));
      } else if (CLS == 9 || CLS == 13) {
        float f;
        asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(r[j]));
        r[j] = __float_as_uint(f);
      } else if (CLS == 10 || CLS == 18) {
        asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(r[j]) : "r"(r[(j + 1) & 7]));
      } else if (CLS == 11 || CLS == 17) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(0x3f8000013f800001ull), "l"(0x3400000034000000ull));
      } else if (CLS == 12 || CLS == 15) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[j]) : "r"(k | 0x80000001u));
      } else {                                                      // 16, 19: carry pack
        asm volatile("{\n\tsub.cc.u32 %0, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
                     : "+r"(r[j]) : "r"(k), "r"(r[(j + 1) & 7]));
      }
    }
  }
}

template <int CLS>
__global__ void __launch_bounds__(256) int_peak_kernel(int iters, uint32_t seed, uint32_t* sink, uint64_t* clk) {
  uint32_t r[8];
  uint64_t a[8];                          // 64-bit chains (IMAD.WIDE, FFMA2 probes)
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = seed * (threadIdx.x + 1) + j, a[j] = 0x3f8000003f800000ull + r[j];
  uint64_t c0, t0;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) step<CLS>(r, a, seed + u);
  }
  uint64_t c1, t1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) x ^= r[j] ^ (uint32_t)a[j] ^ (uint32_t)(a[j] >> 32);
  if (x == 0x12345678u) sink[0] = x;      // keeps the chains live
  if (threadIdx.x == 0) {
    clk[2 * blockIdx.x] = c1 - c0;
    clk[2 * blockIdx.x + 1] = t1 - t0;
  }
}

}  // namespace

extern "C" {

// ops per thread per loop iteration of class cls (lane ops counted per the header)
int cmip_ops_per_iter(int cls) {
  switch (cls) {
    case 1: return 16 * 8 * 2;
    case 7: return 16 * 8 * 2;
    case 11: return 16 * 8 * 2;
    case 16: return 16 * 8 * 2;
    case 17: return 16 * 4 * 3;
    case 19: return 16 * 4 * 3;
    default: return 16 * 8;
  }
}

// Launch class `cls` on `blocks` x 256 threads for `iters` iterations on `stream`; clk
// (device, 2 x blocks u64) receives per CTA {SM cycles, ns}.  Returns a cudaError_t.
int cmip_launch(int cls, int blocks, int iters, uint32_t seed, uint32_t* sink, uint64_t* clk, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (cls) {
    case 0: int_peak_kernel<0><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 1: int_peak_kernel<1><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 2: int_peak_kernel<2><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 3: int_peak_kernel<3><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 4: int_peak_kernel<4><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 5: int_peak_kernel<5><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 6: int_peak_kernel<6><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    case 7: int_peak_kernel<7><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
#define CMIP(C) case C: int_peak_kernel<C><<<blocks, 256, 0, st>>>(iters, seed, sink, clk); break;
    CMIP(8) CMIP(9) CMIP(10) CMIP(11) CMIP(12) CMIP(13) CMIP(14) CMIP(15) CMIP(16) CMIP(17) CMIP(18) CMIP(19)
#undef CMIP
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

}  // extern "C"

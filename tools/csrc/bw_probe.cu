// bw_probe.cu -- measurement tool (not the product): the HBM read ceiling for the fused
// kernel's access pattern.  A persistent grid (one CTA per SM) of `warps` warps; each warp
// streams `bytes`-sized contiguous chunks of a large buffer into `stages` shared-memory
// stages with one 1-D bulk copy (cp.async.bulk, UBLKCP) per chunk, chunk index grid-strided
// over warps, and consumes each stage by one 16-byte shared load per lane (a checksum so the
// loads are not dead).  The rate at 4 KB chunks and the kernel's own warps/stages is the
// denominator the fused kernel's S* stream can reach at best on this part.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void bw_kernel(const unsigned char* src, int64_t n_chunks, int bytes, int stages,
                          unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned char* tiles = sm + (size_t)warp * stages * bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nw * stages * bytes) + warp * stages;
  if (lane < stages)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bars[lane])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, tw = (int64_t)gridDim.x * nw;
  int64_t next = gw;
  int pst = 0;
  auto issue = [&]() {
    if (next < n_chunks && lane == 0) {
      const uint32_t bar = smem_u32(&bars[pst]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(tiles + (size_t)pst * bytes)), "l"(src + next * bytes), "r"(bytes), "r"(bar)
                   : "memory");
    }
    next += tw;
    pst = pst + 1 == stages ? 0 : pst + 1;
  };
  for (int d = 0; d < stages - 1; ++d) issue();
  uint32_t phase = 0;
  int cst = 0;
  unsigned long long acc = 0;
  for (int64_t c = gw; c < n_chunks; c += tw) {
    issue();
    const uint32_t bar = smem_u32(&bars[cst]);
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(bar), "r"((phase >> cst) & 1u) : "memory");
    phase ^= 1u << cst;
    const uint4 v = reinterpret_cast<const uint4*>(tiles + (size_t)cst * bytes)[lane];
    acc += v.x ^ v.w;
    __syncwarp();
    cst = cst + 1 == stages ? 0 : cst + 1;
  }
  if (acc == 0x123456789ull) *sink = acc;
}

}  // namespace

extern "C" int cmbw_launch(const void* src, int64_t total_bytes, int bytes, int warps, int stages, int sms,
                           void* sink, void* stream) {
  const size_t smem = (size_t)warps * stages * bytes + (size_t)warps * stages * 8;
  if (cudaFuncSetAttribute(bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 1;
  bw_kernel<<<sms, 32 * warps, smem, (cudaStream_t)stream>>>(
      static_cast<const unsigned char*>(src), total_bytes / bytes, bytes, stages,
      static_cast<unsigned long long*>(sink));
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

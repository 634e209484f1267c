// gen_sstar.cu -- device version of workloads/sstar.py (input generation only; none of
// the method's arithmetic).  Bit-identical to the numpy generator: integer splitmix64
// hashing, exact 24-bit uniforms, one IEEE-rounded fp32 multiply and one fp32 subtract.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t fmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  return fmix(fmix(fmix(seed ^ (stream << 48)) ^ a) ^ b);
}

__device__ __forceinline__ int64_t row_offset(int layout, int64_t ld, int r) {
  if (layout == 0) return (int64_t)r * ld;
  const int64_t q = r >> 2, m = r & 3;
  return 8 * q * (q - 1) + 12 * q + (m > 0 ? 4 * q : 0) + (m > 1 ? (m - 1) * (4 * q + 4) : 0);
}

// CM_LAYOUT_BLK (include/cm.h): float position of entry (r, i), i < r, within an S*
__device__ __forceinline__ int64_t blk_pos(int n, int r, int i) {
  const int g = (r - 1) >> 5, l = (r - 1) & 31, w = i >> 5, q = i & 31, c = q >> 2, e = q & 3;
  const int h = min(32, n - 1 - 32 * g);
  const int64_t base = 4 * (128 * (int64_t)g * (g - 1) + 144 * (int64_t)g) + (int64_t)32 * h * w;
  if (w < g) return base + 4 * (h * c + l) + e;
  int b = 0;
  for (int k = 0; k < c; ++k) b += max(0, h - 4 * k);
  return base + 4 * (b + l - 4 * c) + e;
}

constexpr int PHI24 = 16777, PSI24 = 16777;
__constant__ int RHO24[3] = {1677722, 5033165, 10066330};
constexpr float INV24 = 1.0f / 16777216.0f;

__global__ void gen_kernel(int n, int L, const int32_t* __restrict__ last, const int32_t* __restrict__ lastF,
                           int family, uint64_t seed, int64_t s_begin, int layout, int64_t ld,
                           int64_t stride, float upper, float sigma_scale, float* __restrict__ out) {
  __shared__ int32_t K[1024];
  __shared__ int32_t tau[1024];
  __shared__ int fam_s;
  const int64_t s = s_begin + blockIdx.x;
  float* dst = out + (int64_t)blockIdx.x * stride;
  if (threadIdx.x == 0) {
    int fam = family;
    if (fam == 3) fam = (fmix(mix64(seed, 7, s, 0)) & 1) ? 2 : 1;
    fam_s = fam;
  }
  __syncthreads();
  const int fam = fam_s;
  if (fam == 1) {
    const int rho24 = RHO24[fmix(mix64(seed, 2, s, 0)) % 3];
    for (int v = threadIdx.x; v < L; v += blockDim.x)
      K[v] = (int)(mix64(seed, 3, s, (uint64_t)v) >> 40) < rho24;
    __syncthreads();
    if (threadIdx.x == 0) {
      int top = -1;
      for (int v = L - 1; v >= 0; --v) {
        if (K[v]) { top = -1; tau[v] = -1; }
        else { if (top < 0) top = v; tau[v] = top; }
      }
    }
    __syncthreads();
  }
  if (layout == 2) {                                  // blocked: fill, then place the entries
    for (int64_t j = threadIdx.x; j < stride; j += blockDim.x) dst[j] = upper;
    __syncthreads();
  }
  for (int r = 0; r < n; ++r) {
    float* row = dst + (layout == 2 ? 0 : row_offset(layout, ld, r));
    const int rowlen = layout == 0 ? (int)ld : layout == 1 ? ((r + 3) & ~3) : r;
    for (int i = threadIdx.x; i < rowlen; i += blockDim.x) {
      if (i >= r) { row[i] = upper; continue; }
      const uint64_t key = ((uint64_t)r << 32) | (uint64_t)i;
      float v;
      if (fam == 2) {
        v = (float)(mix64(seed, 1, s, key) >> 40) * INV24;
      } else {
        bool a;
        if (i >= L) a = r <= last[i];
        else if (K[i]) a = r <= last[i];
        else a = (r <= lastF[i]) || ((2 * L - tau[i] < r) && (r <= last[i]));
        const uint64_t x = mix64(seed, 4, s, key);
        int d = (int)(x & 0xFFFF) + (int)((x >> 16) & 0xFFFF) + (int)((x >> 32) & 0xFFFF) + (int)(x >> 48);
        d = abs(d - 2 * 65535);
        const float g = __fmul_rn((float)d, sigma_scale);
        v = a ? __fsub_rn(1.0f, g) : g;
        const int q = (int)(mix64(seed, 5, s, key) >> 40);
        if (q < PHI24) v = (float)(mix64(seed, 6, s, key) >> 40) * INV24;
        else if (q < PHI24 + PSI24) v = 0.5f;
      }
      if (layout == 2) dst[blk_pos(n, r, i)] = v;
      else row[i] = v;
    }
  }
}

}  // namespace

extern "C" int cmgen_sstar(int n, int L, const int32_t* d_last, const int32_t* d_lastF, int family,
                           uint64_t seed, int64_t s_begin, int32_t count, int layout, int64_t ld,
                           int64_t stride, float upper, float sigma_scale, float* d_out, void* stream) {
  if (count <= 0) return 0;
  if (L > 1024 || n > 1024) return (int)cudaErrorInvalidValue;
  gen_kernel<<<count, 256, 0, (cudaStream_t)stream>>>(n, L, d_last, d_lastF, family, seed, s_begin, layout,
                                                       ld, stride, upper, sigma_scale, d_out);
  return (int)cudaGetLastError();
}

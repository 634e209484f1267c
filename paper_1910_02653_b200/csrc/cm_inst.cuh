// cm_inst.cuh -- the kernel instances.  Each is compiled in its own translation unit
// (k_*.cu, built in parallel); the API translation unit only refers to them.
#pragma once
#include "cm_v2.cuh"

#define CM_ROUND(NT, BULK, RAND) template __global__ void cm2::round_tma_kernel<NT, BULK, RAND>(const cm2::RoundParams, const __grid_constant__ CUtensorMap, const __grid_constant__ cm2::DiagMaps);
#define CM_SCAN(ET, TM) template __global__ void cm2::scan_kernel<ET, TM>(const cm2::ScanParams);
#define CM_FUSED(NT, BULK, RAND, ET) template __global__ void cm2::fused_kernel<NT, BULK, RAND, ET>(const cm2::FusedParams, const __grid_constant__ CUtensorMap, const __grid_constant__ cm2::DiagMaps);
#define CM_REDUCE template __global__ void cm2::reduce_kernel<0>(const cm2::ReduceParams);

#ifdef CM_API_TU
extern CM_ROUND(1, false, false) extern CM_ROUND(1, true, false) extern CM_ROUND(2, false, false) extern CM_ROUND(2, true, false) extern CM_ROUND(3, false, false) extern CM_ROUND(3, true, false) extern CM_ROUND(4, false, false) extern CM_ROUND(4, true, false)
extern CM_ROUND(1, false, true) extern CM_ROUND(1, true, true) extern CM_ROUND(2, false, true) extern CM_ROUND(2, true, true) extern CM_ROUND(3, false, true) extern CM_ROUND(3, true, true) extern CM_ROUND(4, false, true) extern CM_ROUND(4, true, true)
extern CM_SCAN(int32_t, false) extern CM_SCAN(int32_t, true) extern CM_SCAN(int64_t, false) extern CM_SCAN(int64_t, true)
extern CM_FUSED(1, false, false, int32_t) extern CM_FUSED(1, true, false, int32_t) extern CM_FUSED(2, false, false, int32_t) extern CM_FUSED(2, true, false, int32_t) extern CM_FUSED(3, false, false, int32_t) extern CM_FUSED(3, true, false, int32_t) extern CM_FUSED(4, false, false, int32_t) extern CM_FUSED(4, true, false, int32_t)
extern CM_FUSED(1, false, true, int32_t) extern CM_FUSED(1, true, true, int32_t) extern CM_FUSED(2, false, true, int32_t) extern CM_FUSED(2, true, true, int32_t) extern CM_FUSED(3, false, true, int32_t) extern CM_FUSED(3, true, true, int32_t) extern CM_FUSED(4, false, true, int32_t) extern CM_FUSED(4, true, true, int32_t)
extern CM_FUSED(1, false, false, int64_t) extern CM_FUSED(1, true, false, int64_t) extern CM_FUSED(2, false, false, int64_t) extern CM_FUSED(2, true, false, int64_t)
extern CM_FUSED(3, false, false, int64_t) extern CM_FUSED(3, true, false, int64_t) extern CM_FUSED(4, false, false, int64_t) extern CM_FUSED(4, true, false, int64_t)
extern CM_REDUCE
#endif

// cm_inst.cuh -- the kernel instances.  Each is compiled in its own translation unit
// (k_*.cu, built in parallel); the API translation unit only refers to them.  Layouts: 0 dense,
// 1 tri4, 2 blocked (CM_LAYOUT_*).
#pragma once
#include "cm_v2.cuh"

#define CM_ROUND(NT, LAY, RAND) template __global__ void cm2::round_tma_kernel<NT, LAY, RAND>(const cm2::RoundParams, const __grid_constant__ CUtensorMap, const __grid_constant__ cm2::DiagMaps);
#define CM_SCAN(ET, TM) template __global__ void cm2::scan_kernel<ET, TM>(const cm2::ScanParams);
#define CM_FUSED(NT, LAY, RAND, ET) template __global__ void cm2::fused_kernel<NT, LAY, RAND, ET>(const cm2::FusedParams, const __grid_constant__ CUtensorMap, const __grid_constant__ cm2::DiagMaps);
#define CM_REDUCE template __global__ void cm2::reduce_kernel<0>(const cm2::ReduceParams);

#ifdef CM_API_TU
extern CM_ROUND(1, 0, false) extern CM_ROUND(1, 1, false) extern CM_ROUND(1, 2, false) extern CM_ROUND(2, 0, false) extern CM_ROUND(2, 1, false) extern CM_ROUND(2, 2, false) extern CM_ROUND(3, 0, false) extern CM_ROUND(3, 1, false) extern CM_ROUND(3, 2, false) extern CM_ROUND(4, 0, false) extern CM_ROUND(4, 1, false) extern CM_ROUND(4, 2, false) extern CM_ROUND(1, 0, true) extern CM_ROUND(1, 1, true) extern CM_ROUND(1, 2, true) extern CM_ROUND(2, 0, true) extern CM_ROUND(2, 1, true) extern CM_ROUND(2, 2, true) extern CM_ROUND(3, 0, true) extern CM_ROUND(3, 1, true) extern CM_ROUND(3, 2, true) extern CM_ROUND(4, 0, true) extern CM_ROUND(4, 1, true) extern CM_ROUND(4, 2, true)
extern CM_SCAN(int32_t, false) extern CM_SCAN(int32_t, true) extern CM_SCAN(int64_t, false) extern CM_SCAN(int64_t, true)
extern CM_FUSED(1, 0, false, int32_t) extern CM_FUSED(1, 1, false, int32_t) extern CM_FUSED(1, 2, false, int32_t) extern CM_FUSED(2, 0, false, int32_t) extern CM_FUSED(2, 1, false, int32_t) extern CM_FUSED(2, 2, false, int32_t) extern CM_FUSED(3, 0, false, int32_t) extern CM_FUSED(3, 1, false, int32_t) extern CM_FUSED(3, 2, false, int32_t) extern CM_FUSED(4, 0, false, int32_t) extern CM_FUSED(4, 1, false, int32_t) extern CM_FUSED(4, 2, false, int32_t) extern CM_FUSED(1, 0, true, int32_t) extern CM_FUSED(1, 1, true, int32_t) extern CM_FUSED(1, 2, true, int32_t) extern CM_FUSED(2, 0, true, int32_t) extern CM_FUSED(2, 1, true, int32_t) extern CM_FUSED(2, 2, true, int32_t) extern CM_FUSED(3, 0, true, int32_t) extern CM_FUSED(3, 1, true, int32_t) extern CM_FUSED(3, 2, true, int32_t) extern CM_FUSED(4, 0, true, int32_t) extern CM_FUSED(4, 1, true, int32_t) extern CM_FUSED(4, 2, true, int32_t) extern CM_FUSED(1, 0, false, int64_t) extern CM_FUSED(1, 1, false, int64_t) extern CM_FUSED(1, 2, false, int64_t) extern CM_FUSED(2, 0, false, int64_t) extern CM_FUSED(2, 1, false, int64_t) extern CM_FUSED(2, 2, false, int64_t) extern CM_FUSED(3, 0, false, int64_t) extern CM_FUSED(3, 1, false, int64_t) extern CM_FUSED(3, 2, false, int64_t) extern CM_FUSED(4, 0, false, int64_t) extern CM_FUSED(4, 1, false, int64_t) extern CM_FUSED(4, 2, false, int64_t)
extern CM_REDUCE
#endif

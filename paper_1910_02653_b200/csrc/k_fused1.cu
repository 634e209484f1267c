// Instances: fused persistent kernels, 1 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(1, 0, false, int32_t) CM_FUSED(1, 1, false, int32_t) CM_FUSED(1, 2, false, int32_t)

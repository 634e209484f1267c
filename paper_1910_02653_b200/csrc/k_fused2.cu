// Instances: fused persistent kernels, 2 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(2, 0, false, int32_t) CM_FUSED(2, 1, false, int32_t) CM_FUSED(2, 2, false, int32_t)

// Instances: fused persistent kernels, 3 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, 0, false, int32_t) CM_FUSED(3, 1, false, int32_t) CM_FUSED(3, 2, false, int32_t)

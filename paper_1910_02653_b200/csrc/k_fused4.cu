// Instances: fused persistent kernels, 4 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(4, 0, false, int32_t) CM_FUSED(4, 1, false, int32_t) CM_FUSED(4, 2, false, int32_t)

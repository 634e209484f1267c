// Instances: fused persistent kernels, 1 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(1, false, false, int32_t) CM_FUSED(1, true, false, int32_t)

// Instances: fused persistent kernels, 3 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, false, false, int32_t) CM_FUSED(3, true, false, int32_t)

// Instances: fused persistent kernels, randomized rounding, 1 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(1, 0, true, int32_t) CM_FUSED(1, 1, true, int32_t) CM_FUSED(1, 2, true, int32_t)

// Instances: fused persistent kernels, randomized rounding, 2 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(2, 0, true, int32_t) CM_FUSED(2, 1, true, int32_t) CM_FUSED(2, 2, true, int32_t)

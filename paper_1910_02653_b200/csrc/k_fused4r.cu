// Instances: fused persistent kernels, randomized rounding, 4 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(4, 0, true, int32_t) CM_FUSED(4, 1, true, int32_t) CM_FUSED(4, 2, true, int32_t)

// Instances: fused persistent kernels, randomized rounding, 3 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, 0, true, int32_t) CM_FUSED(3, 1, true, int32_t) CM_FUSED(3, 2, true, int32_t)

// Instances: fused persistent kernels, randomized rounding, 4 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(4, false, true, int32_t) CM_FUSED(4, true, true, int32_t)

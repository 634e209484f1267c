// Instances: fused persistent kernels, randomized rounding, 3 sample(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, false, true, int32_t) CM_FUSED(3, true, true, int32_t)

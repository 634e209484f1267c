// Instances: fused persistent kernels, int64 scan state, 1 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(1, 0, false, int64_t) CM_FUSED(1, 1, false, int64_t) CM_FUSED(1, 2, false, int64_t)

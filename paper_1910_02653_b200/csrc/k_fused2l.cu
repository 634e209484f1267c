// Instances: fused persistent kernels, int64 scan state, 2 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(2, 0, false, int64_t) CM_FUSED(2, 1, false, int64_t) CM_FUSED(2, 2, false, int64_t)

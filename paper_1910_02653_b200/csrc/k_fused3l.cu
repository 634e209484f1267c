// Instances: fused persistent kernels, int64 scan state, 3 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, 0, false, int64_t) CM_FUSED(3, 1, false, int64_t) CM_FUSED(3, 2, false, int64_t)

// Instances: fused persistent kernels, int64 scan state, 2 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(2, false, false, int64_t) CM_FUSED(2, true, false, int64_t)

// Instances: fused persistent kernels, int64 scan state, 3 threshold(s) per pass (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_FUSED(3, false, false, int64_t) CM_FUSED(3, true, false, int64_t)

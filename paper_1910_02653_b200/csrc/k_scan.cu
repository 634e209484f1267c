// Instances: K2 scan kernels (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_SCAN(int32_t, false) CM_SCAN(int32_t, true) CM_SCAN(int64_t, false) CM_SCAN(int64_t, true)

// Instances: K1 randomized-rounding kernels (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_ROUND(1, false, true) CM_ROUND(2, false, true) CM_ROUND(3, false, true) CM_ROUND(4, false, true)
CM_ROUND(1, true, true) CM_ROUND(2, true, true) CM_ROUND(3, true, true) CM_ROUND(4, true, true)

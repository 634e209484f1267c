// Instances: K1 randomized-rounding kernels (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_ROUND(1, 0, true) CM_ROUND(2, 0, true) CM_ROUND(3, 0, true) CM_ROUND(4, 0, true)
CM_ROUND(1, 1, true) CM_ROUND(2, 1, true) CM_ROUND(3, 1, true) CM_ROUND(4, 1, true)
CM_ROUND(1, 2, true) CM_ROUND(2, 2, true) CM_ROUND(3, 2, true) CM_ROUND(4, 2, true)

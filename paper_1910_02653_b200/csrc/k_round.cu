// Instances: K1 rounding kernels and the K3 reduce kernel (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_ROUND(1, 0, false) CM_ROUND(2, 0, false) CM_ROUND(3, 0, false) CM_ROUND(4, 0, false)
CM_ROUND(1, 1, false) CM_ROUND(2, 1, false) CM_ROUND(3, 1, false) CM_ROUND(4, 1, false)
CM_ROUND(1, 2, false) CM_ROUND(2, 2, false) CM_ROUND(3, 2, false) CM_ROUND(4, 2, false)
CM_REDUCE

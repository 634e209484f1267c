// Instances: K1 rounding kernels and the K3 reduce kernel (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_ROUND(1, false) CM_ROUND(2, false) CM_ROUND(3, false) CM_ROUND(4, false)
CM_ROUND(1, true) CM_ROUND(2, true) CM_ROUND(3, true) CM_ROUND(4, true)
CM_REDUCE

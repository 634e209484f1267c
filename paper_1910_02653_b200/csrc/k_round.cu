// Instances: K1 rounding kernels and the K3 reduce kernel (see cm_inst.cuh).
#include "cm_inst.cuh"
CM_ROUND(1, false, false) CM_ROUND(2, false, false) CM_ROUND(3, false, false) CM_ROUND(4, false, false)
CM_ROUND(1, true, false) CM_ROUND(2, true, false) CM_ROUND(3, true, false) CM_ROUND(4, true, false)
CM_REDUCE

// bps_tc_i6.cu — explicit instantiations 7/8 of the tcgen05 kernel (bps_tc_kernel.cuh),
// split across units so that nvcc compiles them in parallel.
#include "bps_tc_kernel.cuh"

BPS_TC_DEFINE(true, true, 2, 64, 1, false, false, 1)
BPS_TC_DEFINE(false, true, 1, 256, 1, false, true, 1)
BPS_TC_DEFINE(false, false, 2, 128, 1, false, false, 1)
BPS_TC_DEFINE(false, false, 1, 256, 1, false, false, 2)
BPS_TC_DEFINE(true, false, 1, 128, 1, true, false, 2)

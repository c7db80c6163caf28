// bps_tc_i5.cu — explicit instantiations 6/8 of the tcgen05 kernel (bps_tc_kernel.cuh),
// split across units so that nvcc compiles them in parallel.
#include "bps_tc_kernel.cuh"

BPS_TC_DEFINE(true, false, 2, 64, 2, false, false, 1)
BPS_TC_DEFINE(false, false, 1, 64, 2, false, false, 1)
BPS_TC_DEFINE(false, true, 1, 128, 2, false, false, 1)
BPS_TC_DEFINE(false, true, 4, 64, 2, false, false, 1)
BPS_TC_DEFINE(false, false, 1, 32, 1, false, false, 1)

// bps_tc_i1.cu — explicit instantiations 2/8 of the tcgen05 kernel (bps_tc_kernel.cuh),
// split across units so that nvcc compiles them in parallel.
#include "bps_tc_kernel.cuh"

BPS_TC_DEFINE(true, false, 1, 128, 2, true, false, 1)
BPS_TC_DEFINE(false, false, 1, 256, 2, false, false, 1)
BPS_TC_DEFINE(false, true, 1, 128, 2, false, true, 1)
BPS_TC_DEFINE(false, true, 2, 128, 2, false, false, 1)
BPS_TC_DEFINE(false, false, 1, 128, 1, false, false, 4)

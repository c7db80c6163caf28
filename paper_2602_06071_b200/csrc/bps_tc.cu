// bps_tc.cu — tcgen05 tensor-core kernel (placeholder until the kernel lands).
#include "bps_internal.h"
namespace bps {
int tc_supported(const SketchParams&, int64_t, bps_dtype, bool, const Placement&) {
  return fail(BPS_ERR_UNSUPPORTED, "tcgen05 variant not built yet");
}
int launch_tc(const SketchParams&, const void*, int64_t, int64_t, bps_dtype, float*, int64_t, bool, const Placement&,
              cudaStream_t) {
  return fail(BPS_ERR_UNSUPPORTED, "tcgen05 variant not built yet");
}
}  // namespace bps

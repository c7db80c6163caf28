// bps_tc.h — host-side interface between the tcgen05 planner/dispatcher (bps_tc.cu) and the
// kernel instantiation units (bps_tc_i*.cu, which include bps_tc_kernel.cuh).  Not installed.
#pragma once
#include <cstddef>
#include <cstdint>

#include "bps_internal.h"

namespace bps {
namespace tcx {

constexpr int kBK = 64;  // K rows (input rows u) per pipeline stage

// CTAs per SM of a kernel configuration: the narrow bf16 row-major tiles (one band tile, no cluster)
// run several independent pipelines per SM — their per-stage cost is handshake latency
// (profiles/r02_narrow_n.md): 2 for the 32- and 64-column tiles (3 for the 32-column tile with 4
// band warps and 2 band buffers measured slower: 1146 vs 1388 GB/s); everything else one CTA per SM.
#ifndef BPS_NARROW_MINB32
#define BPS_NARROW_MINB32 2
#endif
#ifndef BPS_NARROW_MINB
#define BPS_NARROW_MINB 2
#endif
constexpr int narrow_minb(bool f32, bool trans, int nmt, int bn, int cs, int ss) {
  return (!f32 && !trans && nmt == 1 && cs == 1 && ss == 1) ? (bn == 32 ? BPS_NARROW_MINB32 : (bn == 64 ? BPS_NARROW_MINB : 1))
                                                             : 1;
}

// Everything the host decided before choosing a template instantiation.
struct HostPlan {
  int G;            // K-chunks per accumulation group: a function of the sketch only (canonical sums)
  int canon;        // 1: ranges partition the input stream; straddling outputs are finished by
                    //    bps_tc_combine from the group partials in the workspace; 0: "halo" ranges (each
                    //    CTA streams the κ-window of its own outputs, no workspace)
  void* ws;         // canon: workspace (group-partial tiles; scratch)
  size_t ws_bytes;
  int sms;          // multiprocessor count of the current device
};

// One tcgen05 kernel configuration (template arguments of bps_tc_kernel).
#define BPS_TC_INSTANTIATIONS(X)                                                                  \
  X(true, false, 1, 128, 1, true, false, 1)   /* fp32 row-major, T form (data in TMEM)           */ \
  X(true, false, 1, 128, 2, true, false, 1)                                                          \
  X(true, true, 1, 128, 1, false, false, 1)   /* fp32 transposed, one band tile                   */ \
  X(true, true, 1, 128, 2, false, false, 1)                                                          \
  X(true, false, 2, 64, 1, false, false, 1)   /* fp32, κ·B_r in (128, 256]                        */ \
  X(true, false, 2, 64, 2, false, false, 1)                                                          \
  X(true, true, 2, 64, 1, false, false, 1)                                                           \
  X(true, true, 2, 64, 2, false, false, 1)                                                           \
  X(false, false, 1, 256, 1, false, false, 1) /* bf16 row-major                                    */ \
  X(false, false, 1, 256, 2, false, false, 1)                                                        \
  X(false, false, 1, 128, 1, false, false, 1)                                                        \
  X(false, false, 1, 128, 2, false, false, 1)                                                        \
  X(false, false, 1, 64, 1, false, false, 1)  /* narrow n                                          */ \
  X(false, false, 1, 32, 1, false, false, 1)  /* n <= 32: one SW64 atom                            */ \
  X(false, false, 1, 64, 2, false, false, 1)                                                         \
  X(false, true, 1, 256, 1, false, true, 1)   /* bf16 transposed: K-pair boxes + re-layout         */ \
  X(false, true, 1, 256, 2, false, true, 1)                                                          \
  X(false, true, 1, 128, 1, false, true, 1)                                                          \
  X(false, true, 1, 128, 2, false, true, 1)                                                          \
  X(false, true, 1, 256, 1, false, false, 1)  /* bf16 transposed, plain SW128 boxes (B_c % 128)    */ \
  X(false, true, 1, 256, 2, false, false, 1)                                                         \
  X(false, true, 1, 128, 1, false, false, 1)                                                         \
  X(false, true, 1, 128, 2, false, false, 1)                                                         \
  X(false, false, 2, 128, 1, false, false, 1) /* bf16, κ·B_r in (128, 256]                        */ \
  X(false, false, 2, 128, 2, false, false, 1)                                                        \
  X(false, true, 2, 128, 1, false, false, 1)                                                         \
  X(false, true, 2, 128, 2, false, false, 1)                                                         \
  X(false, false, 4, 64, 1, false, false, 1)  /* bf16, κ·B_r in (256, 512]                        */ \
  X(false, false, 4, 64, 2, false, false, 1)                                                         \
  X(false, true, 4, 64, 1, false, false, 1)                                                          \
  X(false, true, 4, 64, 2, false, false, 1) \
  X(false, false, 1, 256, 1, false, false, 2) /* slot split: κ·B_r in (128, 512], row-major     */ \
  X(false, false, 1, 256, 1, false, false, 4)                                                     \
  X(false, false, 1, 128, 1, false, false, 2)                                                     \
  X(false, false, 1, 128, 1, false, false, 4)                                                     \
  X(true, false, 1, 128, 1, false, false, 2)                                                      \
  X(true, false, 1, 128, 1, false, false, 4)                                                      \
  X(true, false, 1, 128, 1, true, false, 2)   /* fp32 slot split in the T form (data in TMEM)    */ \
  X(true, false, 1, 128, 1, true, false, 4)

template <bool F32, bool TRANS, int NMT, int BN_, int CS, bool TF, bool RL, int SS>
int launch_impl(const SketchParams& p, const void* A, int64_t lda, int64_t n, float* Y, int64_t ldy,
                const Placement& pl, const HostPlan& hp, cudaStream_t st);

#define BPS_TC_DECLARE(F, T, NM, B, C, TF_, RL_, SS_)                                                    \
  extern template int launch_impl<F, T, NM, B, C, TF_, RL_, SS_>(const SketchParams&, const void*, int64_t, int64_t, \
                                                            float*, int64_t, const Placement&, const HostPlan&, \
                                                            cudaStream_t);
BPS_TC_INSTANTIATIONS(BPS_TC_DECLARE)
#undef BPS_TC_DECLARE

// canonical workspace: the partial tiles (B_r × BN fp32 each), tiles_per_cta per CTA; pure scratch
// tiles each CTA may write: straddler j (0..κ-1) contributes at most (j+1)·nk/G groups
inline int64_t tiles_per_cta(const SketchParams& p, int G) {
  const int64_t npg = (int64_t)(p.B_c / kBK) / G;
  return (int64_t)p.kappa * (p.kappa + 1) / 2 * npg;
}

}  // namespace tcx
}  // namespace bps

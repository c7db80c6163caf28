// bps_tc.cu — planner and dispatcher of the tcgen05 kernel (the "tc" variant).
// The kernel itself is bps_tc_kernel.cuh, instantiated in bps_tc_i*.cu (compiled in parallel).
//
// The planner picks, from the shape alone: the band M-tiles (κ·B_r ≤ 128/256/512), the column
// tile BN, the 2-CTA band-sharing cluster, the MMA form (T form for fp32 row-major, K-pair
// re-layout for bf16 transposed) and the accumulation group G.  G depends on the sketch only
// (never on n, the device or the decomposition), which is what makes the result canonical:
// Y is the same bit pattern for every column split, every orbit-range split and every SM count
// (R19; SURVEY §8(b) determinism contract).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "bps_tc.h"

namespace bps {
namespace tcx {

// cuTensorMapEncodeTiled through the runtime's driver entry point; resolved once (thread-safe
// function-local static initialisation)
void* encode_tiled_entry() {
  static void* fn = []() -> void* {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return f;
    return nullptr;
  }();
  return fn;
}

namespace {

struct Coverage {
  bool ok = false;
  int nmt = 1;
  int ss = 1;  // slot split (row-major, κ·B_r in (128, 512]): SS CTAs of a cluster share the data
  std::string why;
};

// Slot split applies to the row-major layout when the κ band slots divide into SS = 2 or 4
// groups of ≤ 128 band rows (one M-tile per CTA); disable with BPS_TC_NOSS=1 (A/B knob).
int slot_split(const SketchParams& p, bool transposed) {
  const uint64_t rows = (uint64_t)p.kappa * p.B_r;
  if (transposed || rows <= 128 || rows > 512 || getenv("BPS_TC_NOSS")) return 1;
  const int ss = rows <= 256 ? 2 : 4;
  return (p.kappa % ss == 0 && (uint64_t)(p.kappa / ss) * p.B_r <= 128) ? ss : 1;
}

Coverage coverage(const SketchParams& p, bps_dtype dt, bool transposed) {
  Coverage c;
  if (dt != BPS_F32 && dt != BPS_BF16) {
    c.why = "dtype";
    return c;
  }
  if (p.B_c % kBK != 0) {
    c.why = "tc variant needs B_c % 64 == 0";
    return c;
  }
  const uint64_t rows = (uint64_t)p.kappa * p.B_r;
  c.ss = slot_split(p, transposed);
  if (rows > 512 || (rows > 256 && dt != BPS_BF16 && c.ss == 1)) {
    c.why = "tc variant needs kappa*B_r <= 256 (fp32) or <= 512 (bf16, or fp32 row-major with kappa % 4 == 0)";
    return c;
  }
  if ((uint64_t)p.kappa * p.s > 128) {
    c.why = "tc variant needs kappa*s <= 128";
    return c;
  }
  // more than 2 band tiles: rows ≥ 256 need the row-partitioned fast/dense generators (16-bit
  // stale-entry offsets), i.e. C = B_r/s a power of two and κs a multiple of 4
  if (rows > 256 && c.ss == 1 && p.mode == 0 && ((p.C & (p.C - 1)) != 0 || ((uint64_t)p.kappa * p.s) % 4 != 0)) {
    c.why = "tc variant with kappa*B_r > 256 needs B_r/s a power of two and kappa*s % 4 == 0";
    return c;
  }
  c.nmt = c.ss > 1 ? 1 : (rows <= 128 ? 1 : (rows <= 256 ? 2 : 4));
  c.ok = true;
  return c;
}

// K-chunks per accumulation group: the largest divisor of nk = B_c/64 not above the cap — 128
// (precision: the tensor core's fp32 accumulate is not RN), or nk/2 (≤ 64) for
// blocks of ≤ 128 chunks so that stream ranges can be balanced below one block.  A function of
// the sketch only: the canonical fold of every output is fixed before any launch decision.
int group_for(const SketchParams& p) {
  const int nk = (int)(p.B_c / kBK);
  int cap = nk <= 128 ? std::max(1, std::min(64, nk / 2)) : 128;
  if (const char* e = getenv("BPS_TC_GROUP")) {  // experiment knob (changes the canonical fold)
    const int g = atoi(e);
    if (g >= 1 && nk % g == 0) return g;
  }
  for (int g = cap; g >= 1; --g)
    if (nk % g == 0) return g;
  return 1;
}

int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms <= 0) {
    cudaGetLastError();
    return 148;  // B200
  }
  return sms;
}

struct Choice {
  bool f32, trans, tf, rl;
  int nmt, bn, cs, ss;
};

Choice choose(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl, int nmt, int ss,
              int sms, bool canon, int G) {
  Choice c{};
  c.f32 = dt == BPS_F32;
  c.trans = transposed;
  c.nmt = nmt;
  c.ss = ss;
  if (ss > 1) {  // slot split: one band tile per CTA, no band sharing across column tiles
    c.rl = false;
    c.cs = 1;
    if (c.f32) {
      c.bn = 128;
      // fp32: NT form (hi/lo split in shared memory).  BPS_TC_FORM=tf: the T form (each CTA converts
      // the multicast stage into its TMEM A operand, the ring slot released by every CTA's converters)
      // — parity-green, measured 1.4-2.2x slower on the κ = 8 / 16 fp32 sweep points
      const char* fe = getenv("BPS_TC_FORM");
      c.tf = !transposed && fe && std::string(fe) == "tf";
    } else {
      const int64_t ct256 = (n + 255) / 256, ct128 = (n + 127) / 128, cl = std::max(1, sms / ss);
      const int64_t used256 = ct256 >= cl ? ct256 : ct256 * (cl / ct256);
      const int64_t used128 = ct128 >= cl ? ct128 : ct128 * (cl / ct128);
      c.bn = (used256 * 10 >= used128 * 9 || used256 >= cl) ? 256 : 128;
      if (const char* e = getenv("BPS_TC_BN")) c.bn = atoi(e) == 128 ? 128 : 256;  // tuning knob
    }
    return c;
  }
  const int64_t n_out = pl.range_mode ? pl.n_out : (int64_t)p.M;
  (void)n_out;
  if (c.f32) {
    c.bn = nmt == 1 ? 128 : 64;
  } else if (nmt == 1) {
    // bf16, one band tile: 256 columns per CTA (band reused over twice the columns) unless that
    // leaves SMs idle, then 128; narrow row-major inputs take the 64-column tile with a deep ring
    const int64_t ct256 = (n + 255) / 256, ct128 = (n + 127) / 128;
    const int64_t used256 = ct256 >= sms ? ct256 : ct256 * (sms / ct256);
    const int64_t used128 = ct128 >= sms ? ct128 : ct128 * (sms / ct128);
    c.bn = (used256 * 10 >= used128 * 9 || used256 >= sms) ? 256 : 128;
    if (n <= 64 && !transposed) c.bn = 64;
    // n ≤ 32: a 32-column SW64 tile (no zero-filled half box, half the B-operand reads); BPS_TC_BN=64 off
    if (n <= 32 && !transposed) c.bn = 32;
    if (const char* e = getenv("BPS_TC_BN"))  // tuning knob
      c.bn = atoi(e) == 128 ? 128 : (atoi(e) == 64 && !transposed ? 64 : (atoi(e) == 32 && !transposed && n <= 32 ? 32 : 256));
  } else {
    c.bn = nmt == 2 ? 128 : 64;
  }
  c.tf = c.f32 && !transposed && nmt == 1;
  // bf16 transposed, one band tile: 256-byte K-chunk pairs + in-smem re-layout; ranges must be whole
  // pairs (canon: G even)
  c.rl = !c.f32 && transposed && nmt == 1 && (p.B_c % (2 * kBK)) == 0 && (!canon || G % 2 == 0) &&
         !(getenv("BPS_TC_RL") && atoi(getenv("BPS_TC_RL")) == 0);
  const char* cse = getenv("BPS_TC_CLUSTER");  // tuning knob: 1 (off) or 2 CTAs sharing the band
  int cs = cse ? atoi(cse) : (nmt == 4 ? 1 : 2);  // nmt 4: 64 KB band stages, no cluster (measured 2.1x)
  if (cs != 1 && cs != 2) cs = 2;
  const int64_t nct = (n + c.bn - 1) / c.bn;
  while (cs > 1 && nct % cs) cs /= 2;
  c.cs = cs;
  return c;
}

}  // namespace

int supported_impl(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  (void)transposed;
  Coverage cv = coverage(p, dt, transposed);
  if (!cv.ok) return fail(BPS_ERR_UNSUPPORTED, cv.why);
  const int64_t in_rows = (pl.range_mode ? pl.n_out + (int64_t)p.kappa - 1 : (int64_t)p.M) * (int64_t)p.B_c;
  if (in_rows > 0x7FFFFFFF || n > 0x7FFFFFFF)
    return fail(BPS_ERR_UNSUPPORTED, "tc variant: TMA coordinates exceed int32 (d or n >= 2^31)");
  return BPS_OK;
}

size_t workspace_impl(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  Coverage cv = coverage(p, dt, transposed);
  if (!cv.ok || n <= 0) return 0;
  const int sms = device_sms();
  const int G = group_for(p);
  const Choice c = choose(p, n, dt, transposed, pl, cv.nmt, cv.ss, sms, true, G);
  const int64_t nct = (n + c.bn - 1) / c.bn;
  // grid = nct·R ≤ max(nct, co-resident slots); the 32-column narrow tile runs 2 CTAs per SM (Cfg::MINB)
  const int minb = narrow_minb(c.f32, c.trans, c.nmt, c.bn, c.cs, c.ss);
  const int64_t ctas = std::max<int64_t>(nct, (int64_t)sms * minb);
  // partial tiles + one 8-byte publication flag per CTA (slot-split clusters: ss CTAs per tile)
  return (size_t)ctas * (size_t)tiles_per_cta(p, G) * p.B_r * c.bn * 4 + (size_t)ctas * c.ss * 8;
}

int launch_tc_impl(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y, int64_t ldy,
              bool transposed, const Placement& pl, void* ws, size_t ws_bytes, cudaStream_t st) {
  Coverage cv = coverage(p, dt, transposed);
  if (!cv.ok) return fail(BPS_ERR_UNSUPPORTED, cv.why);
  HostPlan hp{};
  hp.sms = device_sms();
  hp.G = group_for(p);
  const size_t need = workspace_impl(p, n, dt, transposed, pl);
  // canon needs the workspace; an output's group partials must fit the combine kernel's tile list
  hp.canon = ws && need && ws_bytes >= need && ((uintptr_t)ws % 256) == 0 &&
             (int64_t)p.kappa * ((p.B_c / kBK) / hp.G) <= 1024;
  hp.ws = hp.canon ? ws : nullptr;
  hp.ws_bytes = hp.canon ? ws_bytes : 0;
  const Choice c = choose(p, n, dt, transposed, pl, cv.nmt, cv.ss, hp.sms, hp.canon, hp.G);
#define BPS_TC_MATCH(F, T, NM, B, C, TF_, RL_, SS_)                                                       \
  if (c.f32 == F && c.trans == T && c.nmt == NM && c.bn == B && c.cs == C && c.tf == TF_ && c.rl == RL_ && \
      c.ss == SS_)                                                                                        \
    return launch_impl<F, T, NM, B, C, TF_, RL_, SS_>(p, A, lda, n, Y, ldy, pl, hp, st);
  BPS_TC_INSTANTIATIONS(BPS_TC_MATCH)
#undef BPS_TC_MATCH
  return fail(BPS_ERR_UNSUPPORTED, "no tc instantiation for this plan");
}

}  // namespace tcx

int tc_supported(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  return tcx::supported_impl(p, n, dt, transposed, pl);
}
size_t tc_workspace_bytes(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  return tcx::workspace_impl(p, n, dt, transposed, pl);
}
int launch_tc(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y, int64_t ldy,
              bool transposed, const Placement& pl, void* ws, size_t ws_bytes, cudaStream_t st) {
  return tcx::launch_tc_impl(p, A, lda, n, dt, Y, ldy, transposed, pl, ws, ws_bytes, st);
}

}  // namespace bps

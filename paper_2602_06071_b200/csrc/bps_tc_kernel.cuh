// bps_tc_kernel.cuh — the tcgen05 tensor-core kernel for Y = S·A (the "tc" variant) and its
// host launch template.  Included only by the instantiation units bps_tc_i*.cu (parallel
// compilation); the planner/dispatcher is bps_tc.cu.  DESIGN.md §6.2.
//
// Idea: the block sparsity of S is a union of κ permutations that are powers of one
// affine map f.  Ordering input and output blocks along the orbit
// g_i = f^i(0) turns the wiring into a sliding window: output i reads input positions
// i+1..i+κ.  A CTA streams a contiguous range of input positions once (no κ-fold
// re-read), and for each input block p it builds the dense ±1
// "band" B_p = [Φ_{g_{p-1},g_p}; …; Φ_{g_{p-κ},g_p}] (κ·B_r × B_c, bf16 exact, rows
// rotated so output i always lands in slot i mod κ) from the counter hash (R2) and
// feeds it to tcgen05.mma; the data tile (TMA, SW128) is the other operand.
//
// Canonical accumulation (R19): the tensor core's fp32 accumulate is not
// round-to-nearest, so D (TMEM) is fresh for every group of G K-chunks (G a function of
// the sketch only, groups aligned inside input blocks) and the epilogue folds each group
// partial P into a TMEM running sum with IEEE RN adds, in stream order:
//     y_i = scale · ((…((0 + P_1) + P_2) + …) + P_NG),   NG = κ·B_c/(64·G) groups of output i.
// The result therefore does not depend on how the input stream is split between CTAs, on the
// column tile, or on the number of columns: every decomposition computes exactly this fold.
//   * canon (workspace): the stream is split into R group-aligned ranges (one CTA per SM).  The
//     CTA whose range holds an output's first group ("owner") folds its own groups; a CTA holding
//     later groups ("contributor") writes those group partials P to the workspace.  An output that
//     completes inside its owner's range is stored there; one that straddles a range boundary
//     leaves its prefix (unscaled running sum) in Y, and the small bps_tc_combine kernel then adds
//     the partials in stream order and stores it.  No CTA waits for another, no atomics, no
//     pre-zeroing, and the workspace is pure scratch.
//   * halo (no workspace): CTA r owns a contiguous set of outputs and streams their κ-windows
//     itself (κ−1 blocks of halo per range).
//   fp32 input: the converter warps split a = hi + lo (two bf16) and the MMA runs on both
//   (Φ is ±1, exact in bf16) — tf32 would miss the 1e-5 tolerance.
// Non-finite or huge inputs (R12): the dense band multiplies every input by zeros too (0·Inf =
// NaN), so an owner that stores a non-finite value recomputes that output column exactly by
// the sparse definition (Alg. 1): only the κ·s rows an input reaches see it.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <random>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "bps_ptx.cuh"
#include "bps_tc.h"

namespace bps {
namespace tcx {
namespace {

#ifndef BPS_WARP_ARRIVE
#define BPS_WARP_ARRIVE 1
#endif
#ifndef BPS_HOIST_FLAT
#define BPS_HOIST_FLAT 1  // HOIST band generator with flat stale-entry offsets (A/B: -DBPS_HOIST_FLAT=0)
#endif
constexpr int kBandTile = 128 * kBK * 2;  // one M-tile (128 band rows) of a band stage, bytes
constexpr int kMaxRanges = 511;           // canon: stream ranges per column tile (TcArgs::rb)
constexpr int kMaxPeers = 8;              // output broadcast destinations (TcArgs::peer)

// Warp roles (the issue arbiter favours high warp ids, so the latency-critical single-thread
// roles take the last two warps): 0-3 epilogue (TMEM lane quarters 0-3) | 4-11 band
// generator | 12-19 fp32 hi/lo converter (fp32 only) | NWARPS-2 TMA producer |
// NWARPS-1 MMA issuer (+TMEM alloc).
template <bool F32, bool TRANS, int NMT, int BN_, int CS, bool TF, bool RL = false, int SS = 1>
struct Cfg {
  // SS ("slot split", bf16/fp32 row-major NT form, κ·B_r in (128, 512]): the SS CTAs of a cluster
  // take the same range and column tile and split the κ band slots — κ/SS slots (≤ 128 band rows,
  // one M-tile) each; the data stage is loaded once from HBM and multicast to all of them (each
  // CTA issues 1/SS of the rows).  Band sharing across column tiles (CS) is off then.
  static_assert(SS == 1 || (CS == 1 && NMT == 1 && !TRANS && !RL), "SS: row-major, one band tile");
  // TF with SS (fp32): every CTA converts the multicast stage into its own TMEM A operand; a ring
  // slot is free once the converters of ALL the cluster's CTAs have read it (one arrival per warp)
  static_assert(!(TF && SS > 1) || BPS_WARP_ARRIVE, "TF slot split counts warp arrivals");
  static constexpr int CL = CS * SS;  // cluster size
  // PAIR (bf16, SS = 2): the two CTAs run ONE cta_group::2 MMA of M = 256 — each holds its 128 band
  // rows (A) and HALF of the data columns (B); D = its rows × all columns in its own TMEM.  The data
  // tile is loaded once (each CTA its half) instead of multicast whole to both, halving the
  // shared-memory write and read of the data per SM.  Only the leader (rank 0) issues MMAs.
  // Built and parity-green (-DBPS_TC_PAIR=1, scripts/pair_smoke.py), but measured 2.0-2.1x SLOWER
  // than the multicast slot split on the κ = 8 sweep (1.8 vs 3.7 TB/s), also with no MMA and no band
  // generation — not the 2-CTA TMA form, the cluster-scope waits or the proxy fences (each swapped
  // out, profiles/r02_narrow_n.md); off by default.
#ifndef BPS_TC_PAIR
#define BPS_TC_PAIR 0
#endif
  static constexpr bool PAIR = BPS_TC_PAIR && SS == 2 && !F32;
  static constexpr int BNL = PAIR ? BN_ / 2 : BN_;  // data columns held in this CTA's shared memory
  // RL ("re-layout", bf16 transposed layout only): TMA loads TWO K-chunks per box without
  // swizzle (256-byte runs per vector: with vectors megabytes apart, 128-byte runs stream at
  // ~4.6 TB/s and 256-byte runs at ~7.2 TB/s, scripts/tma_probe.cu), into two consecutive ring
  // slots; 4 re-layout warps permute the 16-byte pieces in place into the two SW128 K-major
  // tiles the MMA reads.
  static_assert(!RL || (!F32 && TRANS && NMT == 1), "RL: bf16 transposed, one band tile");
  // TF ("transposed form", fp32 row-major only): the data tile is the MMA A operand, written
  // to TMEM by the converter warps (lane = data column, bf16 pairs along K), and the band is
  // the K-major smem B operand; D = data columns × band rows.  The converters then never
  // write shared memory and the MMA reads only the band from it.
  static_assert(!TF || (F32 && !TRANS && NMT == 1 && BN_ == 128), "TF: fp32 row-major, one band tile");
  static constexpr int BN = BN_;  // data columns per CTA; TMEM = D (NMT·BN) + S (NMT·BN)
  static constexpr int ESZ = F32 ? 4 : 2;
  static constexpr int RAW_STAGE = kBK * BNL * ESZ;
  static constexpr int CONV_HALF = kBK * BN * 2;  // fp32: hi and lo bf16 tiles overwrite the raw stage in place
  static constexpr int BAND_STAGE = NMT * kBandTile;
  // CS > 1: the CTAs of a cluster (same input range, CS column tiles) share the band — band
  // stage t is generated by cluster rank t % CS and bulk-copied to the other CTAs.
#ifndef BPS_NBAND_CLUSTER
#define BPS_NBAND_CLUSTER 4
#endif
  static constexpr int NBAND_CL = NMT == 1 ? BPS_NBAND_CLUSTER : (NMT == 2 ? 4 : 2);  // NMT = 4: 64 KB stages
#ifndef BPS_NBAND_NARROW
#define BPS_NBAND_NARROW 2  // narrow tiles at two CTAs per SM: 2 buffers measured fastest (smalln 1645 vs 1378 with 3)
#endif
  static constexpr int MINB = narrow_minb(F32, TRANS, NMT, BN_, CS, SS);  // CTAs per SM (bps_tc.h)
  static constexpr int NBAND = CS > 1 ? (NBAND_CL < CS ? CS : NBAND_CL)
                                      : ((NMT == 1 && !F32) ? (MINB >= 3 ? 2 : (BN_ <= 64 ? BPS_NBAND_NARROW : 3)) : 2);
  static constexpr int LOCALB = NBAND / CS;  // band buffers this CTA generates into
  static constexpr int BUDGET = MINB >= 3 ? 68 * 1024 : (MINB == 2 ? 100 * 1024 : 210 * 1024);
  static constexpr int NRAW_FIT = (BUDGET - NBAND * BAND_STAGE) / RAW_STAGE;
  // ring depth: 8 stages, 16 for the narrow tile (BN = 64, small n: 8 KB stages, so that enough
  // bytes are in flight)
#ifndef BPS_NARROW_NRAW32
#define BPS_NARROW_NRAW32 12
#endif
  static constexpr int NRAW_MAX = BN_ <= 32 && !F32 ? (MINB >= 3 ? 8 : (MINB == 2 ? BPS_NARROW_NRAW32 : 24))
                                                   : (BN_ <= 64 && !F32 ? (MINB == 2 ? 8 : 16) : 8);
  static constexpr int NRAW = (NRAW_FIT > NRAW_MAX ? NRAW_MAX : NRAW_FIT) & (RL ? ~1 : ~0);  // RL: slot pairs
  static constexpr int OFF_RAW = 0;
  static constexpr int OFF_BAND = OFF_RAW + NRAW * RAW_STAGE;
  static constexpr int OFF_CKEY = OFF_BAND + NBAND * BAND_STAGE;  // [2][256] u64 per-block combo keys
  static constexpr int OFF_CROW = OFF_CKEY + 2 * 256 * 8;  // [128] u32 band-row base σ·B_r + j·C of chunk c
  // epilogue scratch: [0,32) non-finite column bitmap, [32,36) broadcast word, [64,96) fp64
  // partials, [128, 1152) outputs this CTA reached last as a contributor (count + ≤ 255 entries),
  // [1152, 2176) outputs the CTA-wide tail folds (count + entries), [2176, 3200) arrival results of
  // the owned outputs open at the range end
  static constexpr int OFF_FIX = OFF_CROW + 128 * 4;
  static constexpr int OFF_BAR = OFF_FIX + 3200;
  // TF: hi and lo products of a group accumulate into ONE D tile, and D is double-buffered
  // (cols [0,128) and [OFF_D1, OFF_D1+128)) so the MMA runs the next group while the epilogue
  // folds this one; the other forms keep one D (TMEM is full at BN = 256)
  static constexpr int NACC = TF ? 2 : 1;
  static constexpr int NCONVA = TF ? 2 : 0;  // TF: TMEM A stages (hi 32 + lo 32 columns each)
  // raw full/empty, conv full (fp32: per raw stage), band full/empty, acc full, acc free, A full/empty
  // + 1: the epilogue's tail mbarrier (contributor tiles bulk-copied into the idle ring)
  static constexpr int NBARS = 3 * NRAW + 2 * NBAND + 2 * NACC + 2 * NCONVA + 1;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBARS * 8;
  static constexpr int SMEM = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
#ifndef BPS_NBW
#define BPS_NBW 8
#endif
  static constexpr int NBW = MINB >= 3 ? 4 : BPS_NBW;  // band generator warps (4 .. 4+NBW-1)
  static_assert(NBW % 4 == 0 && NBW >= 4 && NBW <= 16, "band warps");
  static constexpr int W_CONV0 = 4 + NBW;  // fp32 converter warps W_CONV0 .. W_CONV0+7
  static constexpr int NCONVW = F32 ? 8 : (RL ? BN_ / 32 : 0);  // converter (fp32 split / RL re-layout) warps
  static constexpr int NWARPS = 4 + NBW + NCONVW + 2;
  static constexpr int NCONVT = NCONVW > 0 ? NCONVW * 32 : 1;  // converter threads
  static constexpr int W_TMA = NWARPS - 2, W_MMA = NWARPS - 1;
  static constexpr int NTHREADS = NWARPS * 32;
  static constexpr int NBANDT = NBW * 32;  // band generator threads
  static constexpr int NCG = NBANDT / 64;  // combo groups per column u
  // fp32: the hi and lo tiles are adjacent along N in smem, so ONE MMA with N = 2·BN reads
  // the band once for both (D columns [0,BN) = band·hi, [BN,2BN) = band·lo).
  static constexpr int DN = TF ? 128 : (F32 ? 2 * BN : BN);  // D columns per M-tile
  static constexpr int SN = TF ? 128 : BN;                    // S columns per M-tile
  static constexpr int OFF_TA = NMT * (DN + SN);              // TF: TMEM A stages start here
  static constexpr int OFF_D1 = OFF_TA + NCONVA * 64;       // TF: second D buffer
  static constexpr int TMEM_NEED = OFF_D1 + (TF ? DN : 0);
  static constexpr uint32_t TMEM_COLS = (TMEM_NEED <= 256) ? 256 : 512;
  static constexpr uint32_t IDESC = ptx::idesc_bf16(PAIR ? 256 : 128, DN, TF ? false : !TRANS);
  static_assert(NRAW >= 2, "smem: raw ring");
  static_assert(TMEM_NEED <= 512 && DN <= 256, "TMEM / MMA N");
  // BN = 32 (bf16 row-major, n ≤ 32): the data tile is one 64-byte-swizzled MN atom (32 columns ×
  // 64 rows, TMA SWIZZLE_64B) — no zero-filled half as with a 64-column box
  static_assert((BN % 64 == 0 || (BN == 32 && !F32 && !TRANS && !TF && SS == 1)) && BN <= 256, "BN");
  static constexpr bool SW64 = BN == 32;
  static_assert(SMEM <= 227 * 1024, "smem");
};

struct TcArgs {
  SketchParams p;
  int64_t n;         // columns of A (row-major) or vectors (transposed)
  float* Y;
  int64_t ldy;
  const void* A;     // input (for the exact recompute of non-finite outputs)
  int64_t lda;
  int range_mode;
  int64_t pos_begin, pos_end;  // owned outputs (range mode)
  int64_t stream_begin;        // first input position of the launch window
  int64_t stream_len;          // number of input positions in the window
  int R;                       // ranges per column tile
  // canon: first stage of range r, r = 0..R (host-computed G·⌊NGt·r/R⌋: no 64-bit divisions on the device)
  int rb[kMaxRanges + 1];
  int nct;                     // column tiles (multiple of the cluster size); CTA = (range, tile)
  int canon;                   // 1: stream ranges + owner/contributor workspace; 0: halo ranges
  int64_t n_out;               // halo: outputs of the launch window; output o is position i_first + o
  int64_t i_first;
  float* W;                    // canon: partial tiles (B_r × BN fp32 each)
  int64_t tpc;                 // canon: tiles per CTA
  int G;                       // K-chunks per accumulation group (divides B_c/64; sketch-only)
  int kgroup;                  // transposed layout: K-chunks whose TMA loads are issued together (≤ NRAW)
  int kstep;                   // stages per band/MMA handshake (1 or 2; 2: narrow bf16 tile, see bps_tc_kernel)
  int band_mn;                 // 1: MN-major band tile written as 16-byte one-hot pieces (C = 8, B_r % 8 == 0)
  int tbox;                    // transposed layout, kgroup > 1: vectors per TMA box (divides BN)
  int nohoist;                 // A/B knob: 1 disables the band generator's register-resident keys
  uint32_t mma_hint;           // MMA issuer's mbarrier suspend-time hint (ns)
  uint32_t sleep_ns;           // TMA producer / band warps: back-off between polls of a not-yet-free
                               // ring slot (0: poll with try_wait only)
  int ab;                      // A/B knob (env BPS_TC_AB): 2 skip contributor tile writes (results
                               // wrong), 4 evict_normal for partials, 8 combine with 128 threads,
                               // 16 combine without programmatic dependent launch, 32 skip the main kernel,
                               // 64 combine element parts not capped at one wave, 128 swap the PDL
                               // trigger position, 256 per-CTA flags (combine does not wait for the grid)
  int dbg;  // experiment switches (env BPS_TC_DEBUG; 0 in production): 1 no band, 2 no convert, 4 no MMA,
            // 8 cycle trace, 16 no band proxy fence, 32 band without hashing,
            // 64 (with 4) ring slots released by thread arrives instead of tcgen05.commit
  unsigned long long* trace;   // dbg & 8: per-CTA cycle counters (16 per CTA), else nullptr
  // output broadcast (row-major orbit ranges; bps_apply_orbit_range_bcast): every FINAL
  // element of Y row r is also stored to row prow0 + r of the npeer destination buffers (peer or
  // local device pointers) and, when mc is set, through the NVLS multicast address mc (multimem.st,
  // one store reaching every GPU bound to it) — the all-gather of block sharding, fused into the
  // epilogue.  Parked prefixes (canon) stay in Y only.
  // canon handoff to bps_tc_combine without waiting for the whole grid: CTA b publishes
  // flags[b] = epoch (release) once its partial tiles and parked prefixes are stored; the combine
  // pass acquires the flags of exactly the CTAs an output needs.  epoch is unique per launch, so the
  // workspace needs no initialisation.  flags == nullptr: griddepcontrol.wait (whole grid)
  unsigned long long* flags;
  unsigned long long epoch;
  int ss;                      // slot-split CTAs per (range, column tile)
  float* peer[kMaxPeers];
  int npeer;
  float* mc;
  int64_t ldp, prow0;
};

// broadcast of one final element / four consecutive ones (row-major)
__device__ __forceinline__ void bcast1(const TcArgs& a, int64_t row, int64_t col, float v) {
  const int64_t off = (a.prow0 + row) * a.ldp + col;
  for (int j = 0; j < a.npeer; ++j) a.peer[j][off] = v;
  if (a.mc) asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(a.mc + off), "f"(v) : "memory");
}
__device__ __forceinline__ void bcast4(const TcArgs& a, int64_t row, int64_t col, float4 v) {
  const int64_t off = (a.prow0 + row) * a.ldp + col;
  if (off & 3) {  // ldp not a multiple of 4: scalar stores
    bcast1(a, row, col, v.x), bcast1(a, row, col + 1, v.y), bcast1(a, row, col + 2, v.z), bcast1(a, row, col + 3, v.w);
    return;
  }
  for (int j = 0; j < a.npeer; ++j) *reinterpret_cast<float4*>(a.peer[j] + off) = v;
  if (a.mc)
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a.mc + off), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Geometry of the canonical stream decomposition (canon mode), shared by bps_tc_kernel (tile
// addresses) and bps_tc_combine (which folds the tiles of a straddling output in stream order).
// Range r covers stream stages [G·⌊NGt·r/R⌋, G·⌊NGt·(r+1)/R⌋); output i's window is stages
// [F_i, F_i + κ·nk), F_i = (i + 1 − stream_begin)·nk; a straddling output's later groups are
// "contributor segments" of the following ranges (wrapping once past position M in full mode).
struct CanonGeom {
  // fields copied by value: holding a reference to the kernel's parameter struct would force it
  // into local memory (its address escapes) and every args access through L1
  float* W;
  const int* rb;  // TcArgs::rb (kernel parameter space)
  int64_t tpc, NGt;
  int nct, nk, bn, G, R, slen, sb, kap, npg, Ts, KN, Br;
  __device__ __forceinline__ CanonGeom(const TcArgs& a, int nk_, int bn_) : nk(nk_), bn(bn_) {
    W = a.W, tpc = a.tpc, nct = a.nct, rb = a.rb;
    G = a.G, R = a.R, slen = (int)a.stream_len, sb = (int)a.stream_begin, kap = (int)a.p.kappa;
    npg = nk / G, Ts = slen * nk, KN = kap * nk, Br = (int)a.p.B_r, NGt = (int64_t)a.stream_len * nk / G;
  }
  __device__ int range_begin(int r) const { return rb[r]; }
  __device__ int range_of(int x) const {  // range holding stream stage x ∈ [0, Ts): binary search
    int lo = 0, hi = R;  // rb[lo] ≤ x < rb[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rb[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
  }
  __device__ int first_stage(int i) const { return (i + 1 - sb) * nk; }
  // partial tile of (range r, column tile ct, straddler j, group lg of the range): TF tiles are
  // row-major [B_r][BN] (lanes = columns), the others column-major [BN][B_r] (lanes = rows)
  __device__ float* tile(int r, int ct, int j, int lg) const {
    return W + (((int64_t)r * nct + ct) * tpc + (int64_t)j * (j + 1) / 2 * npg + lg) * (int64_t)Br * bn;
  }
  // the contributor segments of output i (owner coordinates: F_i ≥ 0) in stream order:
  // fn(range, straddler index j in that range, number of groups)
  template <typename Fn>
  __device__ void walk(int i, Fn&& fn) const {
    const int F = first_stage(i), E = F + KN;
    int x = range_begin(range_of(F) + 1), lap = 0, r = range_of(F) + 1;
    while (x < E) {
      if (r == R) r = 0, ++lap;  // full mode: the window wraps past position M
      const int b0 = range_begin(r), b1 = range_begin(r + 1);
      const int j = (i - lap * slen) - (sb + b0 / nk - kap);
      const int end = (E - lap * Ts) < b1 ? (E - lap * Ts) : b1;
      fn(r, j, (end - b0) / G);
      x = b1 + lap * Ts;
      ++r;
    }
  }
};

// cycle accounting for the BPS_TC_DEBUG=8 trace (compiled in, inactive unless trace != nullptr)
#ifdef BPS_TC_INSTRUMENT
struct Tr {
  unsigned long long* t;
  __device__ __forceinline__ Tr(unsigned long long* p) : t(p) {}
  __device__ __forceinline__ unsigned long long now() const { return t ? clock64() : 0ull; }
  __device__ __forceinline__ void add(int slot, unsigned long long t0) const {
    if (t) t[slot] += clock64() - t0;
  }
};
#define BPS_DBG(x) (args.dbg & (x))
#else
struct Tr {  // production build: instrumentation compiled out
  __device__ __forceinline__ Tr(unsigned long long*) {}
  __device__ __forceinline__ unsigned long long now() const { return 0ull; }
  __device__ __forceinline__ void add(int, unsigned long long) const {}
};
#define BPS_DBG(x) 0
#endif

__device__ __forceinline__ uint32_t mod_pos(int64_t i, uint32_t M) {
  int64_t r = i % (int64_t)M;
  return (uint32_t)(r < 0 ? r + M : r);
}


__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// stores that the combine kernel reads back soon: keep them in L2 (the streamed input is EVICT_FIRST)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep4(float* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_cg_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_cg_f(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// named-barrier OR reduction over `n` threads (bar.red.or)
// Arrival of a whole warp on an mbarrier counted in warps (BPS_WARP_ARRIVE): the lanes' prior
// shared-memory / TMEM accesses are ordered before lane 0's release-arrive by __syncwarp, so the
// barrier sees one arrival per warp instead of 32 (per-thread arrivals on one barrier serialise
// in the barrier unit; 256 of them per stage bounded the narrow-tile pipeline).
constexpr int kArrivePerWarp = BPS_WARP_ARRIVE ? 1 : 32;
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
#if BPS_WARP_ARRIVE
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bar);
#else
  ptx::mbar_arrive(bar);
#endif
}

__device__ __forceinline__ void wait_slot(uint64_t* bar, uint32_t parity, uint32_t ns) {
  if (ns)
    ptx::mbar_wait_sleep(bar, parity, ns);
  else
    ptx::mbar_wait(bar, parity);
}

__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

constexpr uint32_t kEpiBar = 5;
constexpr int kTrSlots = 32;  // BPS_TC_DEBUG=8 trace: cycle counters per CTA  // named barrier of the 4 epilogue warps (ids 1-4 are used by other roles)

// Exact value of Y[row r of output i, column t] by the sparse definition (Alg. 1, P:1688-1709:
// y = scale·Σ_{ℓ,u,j: row(g,ℓ,u,j) = r} σ·A[h_ℓ·B_c + u, t]), computed by the 128 epilogue threads
// (candidates u split by thread, fp64 sums, fixed-order reduction: deterministic).  Used only for
// outputs whose tensor-core value is non-finite (R12).
template <bool F32, bool TRANS>
__device__ float exact_elem(const TcArgs& a, int64_t i, uint32_t r, int64_t t, int et, double* red) {
  const SketchParams& p = a.p;
  const uint32_t g = affine_pow(p, (uint64_t)mod_pos(i, p.M), 0u);
  double acc = 0.0;
  for (uint32_t ell = 1; ell <= p.kappa; ++ell) {
    const int64_t hrow = a.range_mode ? (i + (int64_t)ell - a.pos_begin - 1) * (int64_t)p.B_c
                                      : (int64_t)affine_pow(p, (uint64_t)mod_pos(i + (int64_t)ell, p.M), 0u) * p.B_c;
    for (uint32_t u = (uint32_t)et; u < p.B_c; u += 128) {
      uint32_t hit = 0, neg = 0;
      if (p.mode) {
        const uint64_t z = pattern_hash(p, g, ell, u, 0);
        for (uint32_t j = 0; j < p.s; ++j) {
          const Draw d = affine_draw(p, z, j);
          if (d.row == r) hit = 1, neg = d.neg;
        }
      } else {
        const uint32_t j = r / p.C;
        const Draw d = draw_from_hash(p, pattern_hash(p, g, ell, u, j), j);
        hit = d.row == r;
        neg = d.neg;
      }
      if (!hit) continue;
      const int64_t idx = TRANS ? t * a.lda + hrow + u : (hrow + u) * a.lda + t;
      const float v = F32 ? reinterpret_cast<const float*>(a.A)[idx]
                          : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.A)[idx]);
      acc += neg ? -(double)v : (double)v;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((et & 31) == 0) red[et >> 5] = acc;
  ptx::named_bar_sync(kEpiBar, 128);
  const double tot = ((red[0] + red[1]) + red[2]) + red[3];
  ptx::named_bar_sync(kEpiBar, 128);
  return (float)(tot * (double)p.scale);
}

template <bool F32, bool TRANS, int NMT, int BN_, int CS, bool TF, bool RL, int SS>
__global__ void __launch_bounds__(Cfg<F32, TRANS, NMT, BN_, CS, TF, RL, SS>::NTHREADS,
                                  Cfg<F32, TRANS, NMT, BN_, CS, TF, RL, SS>::MINB)
    bps_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TcArgs args) {
  using K = Cfg<F32, TRANS, NMT, BN_, CS, TF, RL, SS>;
  constexpr int BN = K::BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + K::NRAW;
  uint64_t* conv_full = raw_empty + K::NRAW;  // fp32: stage converted in place, ready for the MMA
  uint64_t* band_full = conv_full + K::NRAW;
  uint64_t* band_empty = band_full + K::NBAND;
  uint64_t* acc_full = band_empty + K::NBAND;
  uint64_t* acc_free = acc_full + K::NACC;
  uint64_t* ta_full = acc_free + K::NACC;  // TF: TMEM A stage written by the converters
  uint64_t* ta_empty = ta_full + K::NCONVA;  // TF: TMEM A stage consumed by the MMA
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + K::OFF_TMEMPTR);
  uint64_t* ckey = reinterpret_cast<uint64_t*>(smem + K::OFF_CKEY);
  uint32_t* crow = reinterpret_cast<uint32_t*>(smem + K::OFF_CROW);

  const SketchParams& p = args.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Tr tr_cta((args.trace && threadIdx.x == 0) ? args.trace + blockIdx.x * kTrSlots : nullptr);
  const unsigned long long t_cta0 = tr_cta.now();
  const uint32_t kappa = p.kappa;
  const int nk = (int)(p.B_c / kBK);
  const int G = args.G;

  // ---- this CTA's column tile and input-stream range
  // canon: ranges partition the stream stages [0, stream_len·nk) at group granularity;
  // halo:  CTA rr owns outputs i ∈ [ilo, ihi) and streams positions ilo+1 .. ihi+κ-1 itself.
  // a cluster = CS consecutive column tiles (band sharing) or SS slot subsets of one tile (SS > 1)
  const int css = SS > 1 ? (int)(blockIdx.x % SS) : 0;  // slot subset of this CTA
  const int cid = SS > 1 ? (int)(blockIdx.x / SS) : (int)blockIdx.x;
  const int ct = cid % args.nct, rr = cid / args.nct;
  const uint32_t kap_l = kappa / SS, sig0 = (uint32_t)css * kap_l;  // this CTA's band slots [sig0, sig0 + kap_l)
  const int64_t col0 = (int64_t)ct * BN;
  // stage s ∈ [S0, S1) of the window = K-chunk s % nk of input position sb + s / nk
  int64_t sb, S0, S1, ilo = 0, ihi = 0;
  const int64_t NGt = args.stream_len * nk / G;  // canon: groups in the stream
  if (args.canon) {
    sb = args.stream_begin;
    S0 = args.rb[rr];
    S1 = args.rb[rr + 1];
  } else {
    const int64_t o0 = args.n_out * rr / args.R, o1 = args.n_out * (rr + 1) / args.R;
    ilo = args.i_first + o0;
    ihi = args.i_first + o1;
    sb = ilo + 1;
    S0 = 0;
    S1 = o1 > o0 ? (o1 - o0 + (int64_t)kappa - 1) * nk : 0;
  }

  // stage indices and positions fit in 32 bits (d < 2^31 ⇒ < 2^25 stages): the role loops use these
  const int S0i = (int)S0, S1i = (int)S1, sbi = (int)sb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < K::NRAW; ++i) {
      // PAIR leader: its own TMA bytes + the peer's forwarded "my half landed" arrival
      ptx::mbar_init(&raw_full[i], (K::PAIR && css == 0) ? 2 : 1);
      // TF: converter warps; SS: every CTA's MMA (multicast data); PAIR: the leader's pair commit
      ptx::mbar_init(&raw_empty[i], TF ? SS * K::NCONVW * kArrivePerWarp : (K::PAIR ? 1 : SS));
      ptx::mbar_init(&conv_full[i], K::NCONVW > 0 ? K::NCONVW * kArrivePerWarp : 1);
    }
    for (int i = 0; i < K::NBAND; ++i) {
      // PAIR: the leader's band warps and (one arrival per warp) the peer's
      ptx::mbar_init(&band_full[i], CS > 1 ? 1 : K::NBW * kArrivePerWarp + (K::PAIR ? K::NBW : 0));
      ptx::mbar_init(&band_empty[i], CS);
    }
    for (int i = 0; i < K::NACC; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_free[i], K::PAIR ? 256 : 128);  // PAIR: both CTAs' epilogues (leader's barrier)
    }
    for (int i = 0; i < K::NCONVA; ++i) {
      ptx::mbar_init(&ta_full[i], K::NCONVW > 0 ? K::NCONVW * kArrivePerWarp : 1);
      ptx::mbar_init(&ta_empty[i], 1);
    }
    ptx::mbar_init(ta_empty + K::NCONVA, 1);  // epilogue tail
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tmap);
  }
  if (threadIdx.x < 40) reinterpret_cast<uint32_t*>(smem + K::OFF_FIX)[threadIdx.x] = 0u;
  if (warp == K::W_MMA) {
    if (K::PAIR)
      ptx::tmem_alloc_pair(tmem_ptr, K::TMEM_COLS);
    else
      ptx::tmem_alloc(tmem_ptr, K::TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (K::CL > 1)
    ptx::cluster_sync();  // peers' barriers are initialised before any remote copy/arrive
  else
    __syncthreads();
  ptx::tc_fence_after();
  // programmatic dependent launch: with the flag handoff the combine pass is triggered as soon as
  // every CTA of this grid has started — its CTAs take SMs freed by finished ranges and fold each
  // straddling output as soon as the CTAs holding its pieces have published them, inside this
  // kernel's tail.  Without flags the trigger sits at the CTA end (BPS_TC_AB & 128 swaps both:
  // early with griddepcontrol.wait measured 1-2 % slower on LS)
  const bool early_trigger = args.flags ? !(args.ab & 128) : (args.ab & 128) != 0;
  if (early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem = *tmem_ptr;               // D: per-group tensor-core accumulator
  const uint32_t tmem_S = tmem + NMT * K::DN;    // S: fp32 running sums (RN adds on CUDA cores)
  const uint32_t tmem_A = tmem + K::OFF_TA;      // TF: A operand stages (data hi | lo)

  if (S1 > S0) {
    if (warp == K::W_TMA) {
      // ===================== TMA producer =====================
      if (lane == 0) {
        const Tr tr(args.trace ? args.trace + blockIdx.x * kTrSlots : nullptr);
        const unsigned long long tstart = tr.now();
        const uint64_t pol = ptx::policy_evict_first();
        int q = sbi + S0i / nk;
        int kc = S0i % nk;
        uint32_t gq = affine_pow(p, (uint64_t)mod_pos(q, p.M), 0u);
        int s = 0;
        uint32_t ph = 0;
        int grp = 0;  // stages of the current K-group still to issue (transposed layout)
        for (int st = S0i; st < S1i; ++st) {
          {
            const int64_t row0 = args.range_mode ? (q - (args.pos_begin + 1)) * (int64_t)p.B_c : (int64_t)gq * p.B_c;
            const unsigned long long t0 = tr.now();
            if (RL) {
              // one unswizzled box = K-chunks kc, kc+1 of BN vectors (256 B per vector) into ring
              // slots s, s+1 (contiguous: NRAW is even and pairs start at even slots)
              if ((kc & 1) == 0) {
                wait_slot(&raw_empty[s], ph ^ 1, args.sleep_ns);
                wait_slot(&raw_empty[s + 1], ph ^ 1, args.sleep_ns);
                tr.add(0, t0);
                ptx::mbar_arrive_expect_tx(&raw_full[s], 2 * K::RAW_STAGE);
                ptx::tma_load_2d(smem + K::OFF_RAW + s * K::RAW_STAGE, &tmap, &raw_full[s], (int32_t)(row0 + kc * kBK),
                                 (int32_t)col0, pol);
              }
            } else if (!TRANS && !F32 && BN == 64 && args.kgroup > 1) {
              // narrow row-major tile (small n): ONE box of 64·kgroup rows fills kgroup consecutive
              // ring slots (the SW128 MN-major tile of a slot is 64 rows × 128 B, so the slots of a
              // group are one contiguous 64·kgroup-row tile); the bytes complete on the group's
              // first slot, which the MMA waits on for every slot of the group
              if (kc % args.kgroup == 0) {
                int s2 = s;
                uint32_t ph2 = ph;
                for (int i = 0; i < args.kgroup; ++i) {
                  wait_slot(&raw_empty[s2], ph2 ^ 1, args.sleep_ns);
                  if (++s2 == K::NRAW) s2 = 0, ph2 ^= 1;
                }
                tr.add(0, t0);
                ptx::mbar_arrive_expect_tx(&raw_full[s], args.kgroup * K::RAW_STAGE);
                ptx::tma_load_2d(smem + K::OFF_RAW + s * K::RAW_STAGE, &tmap, &raw_full[s], (int32_t)col0,
                                 (int32_t)(row0 + kc * kBK), pol);
              }
            } else if (TRANS && args.kgroup > 1) {
              // transposed layout: a stage reads kBK·ESZ bytes of each of BN vectors (128 B for
              // bf16), each vector in another DRAM page.  Issue the K-chunks of an aligned group
              // together, once ALL their ring slots are free, in sub-boxes of tbox vectors
              // alternating over the chunks, so the kgroup pieces of a vector (one contiguous
              // run) reach DRAM a few requests apart and share one row activation.
              if (grp == 0) {
                int m = args.kgroup - kc % args.kgroup;
                if (m > nk - kc) m = nk - kc;
                if (m > S1i - st) m = S1i - st;
                int s2 = s;
                uint32_t ph2 = ph;
                for (int i = 0; i < m; ++i) {
                  wait_slot(&raw_empty[s2], ph2 ^ 1, args.sleep_ns);
                  ptx::mbar_arrive_expect_tx(&raw_full[s2], K::RAW_STAGE);
                  if (++s2 == K::NRAW) s2 = 0, ph2 ^= 1;
                }
                const int vb = args.tbox;
                for (int v0 = 0; v0 < BN; v0 += vb) {
                  int si = s;
                  for (int i = 0; i < m; ++i) {
                    uint8_t* dst = smem + K::OFF_RAW + si * K::RAW_STAGE + v0 * (kBK * K::ESZ);
                    ptx::tma_load_2d(dst, &tmap, &raw_full[si], (int32_t)(row0 + (kc + i) * kBK), (int32_t)(col0 + v0), pol);
                    if (++si == K::NRAW) si = 0;
                  }
                }
                grp = m;
              }
              --grp;
              tr.add(0, t0);
            } else {
              wait_slot(&raw_empty[s], ph ^ 1, args.sleep_ns);
              tr.add(0, t0);
              if (!K::PAIR) ptx::mbar_arrive_expect_tx(&raw_full[s], K::RAW_STAGE);
              uint8_t* dst = smem + K::OFF_RAW + s * K::RAW_STAGE;
              const int32_t r = (int32_t)(row0 + kc * kBK);
              if (K::PAIR) {
                // CTA pair: this CTA loads its half of the columns into its own ring slot; the peer's
                // MMA warp forwards the landing of its half to the leader's barrier
                ptx::mbar_arrive_expect_tx(&raw_full[s], K::RAW_STAGE);
#pragma unroll
                for (int b = 0; b < K::BNL / 64; ++b)
                  ptx::tma_load_2d(dst + b * (kBK * 128), &tmap, &raw_full[s], (int32_t)(col0 + css * K::BNL + 64 * b), r, pol);
              } else if (SS > 1) {
                // slot split: this CTA loads rows [css·PR, (css+1)·PR) of the stage and multicasts them
                // to the SS CTAs of the cluster (same smem offset, completing tx on each one's raw_full)
                constexpr int PR = kBK / SS;
                const uint16_t mask = (uint16_t)((1u << SS) - 1u);
                const int32_t rp = r + css * PR;
                if (F32) {
                  ptx::tma_load_2d_mc(dst + css * PR * BN * 4, &tmap, &raw_full[s], (int32_t)col0, rp, mask, pol);
                } else {
#pragma unroll
                  for (int b = 0; b < BN / 64; ++b)
                    ptx::tma_load_2d_mc(dst + b * (kBK * 128) + css * PR * 128, &tmap, &raw_full[s], (int32_t)(col0 + 64 * b), rp,
                                        mask, pol);
                }
              } else if (!TRANS) {
                if (F32) {
                  ptx::tma_load_2d(dst, &tmap, &raw_full[s], (int32_t)col0, r, pol);
                } else {
#pragma unroll
                  for (int b = 0; b < (BN + 63) / 64; ++b)
                    ptx::tma_load_2d(dst + b * (kBK * 128), &tmap, &raw_full[s], (int32_t)(col0 + 64 * b), r, pol);
                }
              } else {
                ptx::tma_load_2d(dst, &tmap, &raw_full[s], r, (int32_t)col0, pol);
              }
            }
            if (++s == K::NRAW) s = 0, ph ^= 1;
          }
          if (++kc == nk) kc = 0, ++q, gq = affine_step(p, gq);
        }
        tr.add(1, tstart);
      }
    } else if (K::PAIR && warp == K::W_MMA && css != 0) {
      // ============ PAIR peer: forward "my half of stage s landed" to the leader's barrier ============
      if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int st = S0i; st < S1i; ++st) {
          ptx::mbar_wait(&raw_full[s], ph);
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&raw_full[s]), 0));
          if (++s == K::NRAW) s = 0, ph ^= 1;
        }
      }
    } else if (warp == K::W_MMA) {  // PAIR: the leader issues for both CTAs
      // ===================== MMA issuer =====================
      // The whole warp runs the loop (descriptors stay warp-uniform, in uniform registers);
      // one elected lane issues the tcgen05.mma / commit instructions.
      {
        const Tr tr((args.trace && lane == 0) ? args.trace + blockIdx.x * kTrSlots : nullptr);
        const unsigned long long tstart = tr.now();
        int ds = 0, bs = 0;
        uint32_t dph = 0, bph = 0;
        uint64_t* dfull = (F32 || RL) ? conv_full : raw_full;
        uint64_t* dempty = raw_empty;
        constexpr int NDS = K::NRAW;
        const uint32_t data_base = ptx::smem_u32(smem + K::OFF_RAW);
        constexpr int DSTAGE = K::RAW_STAGE;
        const uint32_t band_base = ptx::smem_u32(smem + K::OFF_BAND);
        // Descriptors are built once: per stage only the low word (start address >> 4, 14 bits; smem
        // addresses < 228 KB never carry out of it) moves by the ring slot and the K-step.  Rebuilding
        // them per MMA was a ~45-instruction dependent uniform-datapath chain per stage that bounded
        // the narrow-tile pipeline (~650 cycles of issue per 64-row stage, ncu source view).
        // band: K-major (+32 B per K-step), or MN-major (band_mn: 64-row atoms 8 KB apart, +16 rows of
        // 128 B per K-step) with the matching major bit in the instruction descriptor
        const uint64_t a0 = args.band_mn ? ptx::smem_desc_sw128(band_base, kBK * 128, 1024) : ptx::smem_desc_sw128(band_base, 0, 1024);
        const uint32_t band_ks = args.band_mn ? 128u : 2u;
        const uint32_t idesc = K::IDESC | (args.band_mn ? (TF ? (1u << 16) : (1u << 15)) : 0u);
        // data: K-major SW128 (transposed), MN-major SW128 (64-column atoms, 8 KB apart), or MN-major
        // SW64 (BN = 32: one 32-column atom, 8-row groups 512 B apart; layout type 4)
        const uint64_t b0 = TRANS ? ptx::smem_desc_sw128(data_base, 0, 1024)
                                  : (K::SW64 ? ((ptx::smem_desc_sw128(data_base, kBK * 64, 512) & ~(7ull << 61)) | (4ull << 61))
                                             : ptx::smem_desc_sw128(data_base, kBK * 128, 1024));
        const uint32_t a0lo = (uint32_t)a0, b0lo = (uint32_t)b0;
        const uint64_t a0hi = a0 & 0xFFFFFFFF00000000ull, b0hi = b0 & 0xFFFFFFFF00000000ull;
        int gcount = 0, dbuf = 0;  // groups started; D buffer of the current group
        const int ksm = args.kstep - 1;
        int kc = S0i % nk;
        int gi = kc % G;  // position inside the accumulation group (groups restart at block starts)
        for (int st = S0i; st < S1i; ++st) {
          {
            const bool gstart = st == S0i || gi == 0;
            const bool gend = st == S1i - 1 || kc == nk - 1 || gi == G - 1;
            if (gstart) {
              dbuf = gcount % K::NACC;
              if (gcount >= K::NACC) {  // this D buffer must have been folded into S
                const unsigned long long t0 = tr.now();
                if (K::PAIR && (args.ab & 512))
                  ptx::mbar_wait_cluster(&acc_free[dbuf], (uint32_t)(gcount / K::NACC - 1) & 1u);
                else
                  ptx::mbar_wait(&acc_free[dbuf], (uint32_t)(gcount / K::NACC - 1) & 1u);
                tr.add(2, t0);
                ptx::tc_fence_after();
              }
            }
            unsigned long long t0 = tr.now();
            // kstep = 2 (narrow tile): one handshake per pair of stages — the TMA box of the pair
            // completes on its first slot and the band warps arrive once, on the pair's first buffer
            const int sp = (st - S0i) & ksm;  // position of this stage in its step
            if (sp == 0) {
              // data stage and band stage of this step, polled together
              uint64_t* db = TF ? &ta_full[(st - S0i) & 1] : &dfull[(!TRANS && args.kgroup > 1) ? (ds & ~(args.kgroup - 1)) : ds];
              const uint32_t dp = TF ? ((uint32_t)((st - S0i) >> 1) & 1u) : dph;
              // (PAIR: the peer's band warps and data forwarder arrive here too, with cluster-scope
              // release; a cluster-scope acquire poll measured ~2.5x slower than this wait)
              if (K::PAIR && (args.ab & 512)) {
                while (!ptx::mbar_try_wait2_cluster(db, dp, &band_full[bs], bph)) {
                }
              } else {
                ptx::mbar_wait2(db, dp, &band_full[bs], bph);
              }
            }
            tr.add(3, t0);
            ptx::tc_fence_after();
            const uint32_t alo = a0lo + (uint32_t)bs * (uint32_t)(K::BAND_STAGE >> 4);
            const uint32_t blo = b0lo + (uint32_t)ds * (uint32_t)(DSTAGE >> 4);
            if (ptx::elect_one()) {
            if (TF) {
              const uint32_t ta = tmem_A + (uint32_t)((st - S0i) & 1) * 64;
#pragma unroll
              for (int ks = 0; ks < kBK / 16; ++ks) {
                const uint64_t bdesc = a0hi | (alo + ks * band_ks);  // band (B operand of the T form)
                if (!BPS_DBG(4)) {
                  const uint32_t dt = tmem + (dbuf ? K::OFF_D1 : 0);
                  ptx::mma_bf16_ts(dt, ta + ks * 8, bdesc, idesc, (gstart && ks == 0) ? 0u : 1u);  // hi
                  ptx::mma_bf16_ts(dt, ta + 32 + ks * 8, bdesc, idesc, 1u);                          // lo
                }
              }
            } else
#pragma unroll
            for (int ks = 0; ks < kBK / 16; ++ks) {
#pragma unroll
              for (int m = 0; m < NMT; ++m) {
                const uint64_t adesc = a0hi | (alo + (uint32_t)(m * (kBandTile >> 4)) + (uint32_t)ks * band_ks);
                // data: K-major (+32 B per K-step) or MN-major (+16 rows of 128 B per K-step)
                const uint64_t bdesc = b0hi | (blo + (uint32_t)(TRANS ? ks * 2 : (K::SW64 ? ks * 64 : ks * 128)));
                const uint32_t acc = (gstart && ks == 0) ? 0u : 1u;  // fresh per group
                if (BPS_DBG(4)) {
                } else if (K::PAIR) {
                  ptx::mma_bf16_ss_pair(tmem + m * K::DN, adesc, bdesc, idesc, acc);
                } else {
                  ptx::mma_bf16_ss(tmem + m * K::DN, adesc, bdesc, idesc, acc);
                }
              }
            }
            if (BPS_DBG(64)) {  // experiment (with dbg 4, no MMA issued): release by a thread arrive
              ptx::mbar_arrive(TF ? &ta_empty[(st - S0i) & 1] : &dempty[ds]);
              ptx::mbar_arrive(&band_empty[bs]);
            } else if (TF)
              ptx::mma_commit(&ta_empty[(st - S0i) & 1]);
            else if (K::PAIR)
              ptx::mma_commit_pair(&dempty[ds], (uint16_t)3u);  // both CTAs' halves were read
            else if (SS > 1)
              ptx::mma_commit_multicast(&dempty[ds], (uint16_t)((1u << SS) - 1u));  // every CTA's copy was filled
            else
              ptx::mma_commit(&dempty[ds]);
            if (BPS_DBG(64) || sp != ksm)
              ;  // kstep = 2: the pair's buffers are released together, on its first buffer
            else if (K::PAIR)
              ptx::mma_commit_pair(&band_empty[bs], (uint16_t)3u);  // both CTAs' band stages
            else if (CS > 1)
              ptx::mma_commit_multicast(&band_empty[bs], (uint16_t)((1u << CS) - 1));
            else
              ptx::mma_commit(&band_empty[bs - ksm]);
            if (gend) {
              if (K::PAIR)
                ptx::mma_commit_pair(&acc_full[dbuf], (uint16_t)3u);  // D is ready in both TMEMs
              else
                ptx::mma_commit(&acc_full[dbuf]);
            }
            }  // elect_one
            __syncwarp();
            if (gend) ++gcount;
            if (++ds == NDS) ds = 0, dph ^= 1;
            if (++bs == K::NBAND) bs = 0, bph ^= 1;
          }
          if (++kc == nk) kc = 0, gi = 0;
          else gi = (gi + 1 == G) ? 0 : gi + 1;
        }
        tr.add(5, tstart);
      }
    } else if (warp < 4) {
      // ============ epilogue: fold group partials (fp32 RN), emit / hand over outputs ============
      // Positions and stage indices fit in 32 bits (d < 2^31 ⇒ < 2^25 stages), so the bookkeeping
      // here is 32-bit (register pressure: the fp32 kernels run 704 threads at ≤ 80 registers).
      // ---- output bookkeeping of the epilogue
      const int et = threadIdx.x;  // epilogue threads are 0..127
      uint32_t* fixmap = reinterpret_cast<uint32_t*>(smem + K::OFF_FIX);  // columns to recompute (BN bits)
      double* fixred = reinterpret_cast<double*>(smem + K::OFF_FIX + 64);
      const int Br = (int)p.B_r, krows = (int)(kap_l * p.B_r), kap = (int)kappa, s0 = (int)sig0, kapl = (int)kap_l;
      // slot of output i and whether this CTA holds it (always, unless slot split)
      auto slot_of = [&](int i) { return (int)((uint32_t)(i + kap * 0x10000) % (uint32_t)kap); };
      auto mine = [&](int i) { return SS == 1 || (slot_of(i) >= s0 && slot_of(i) < s0 + kapl); };
      const int sb_ = (int)sb, S0_ = (int)S0, S1_ = (int)S1, ilo_ = (int)ilo, ihi_ = (int)ihi;
      const int pb_ = (int)args.pos_begin, pe_ = (int)args.pos_end;
      auto first_stage = [&](int i) { return (i + 1 - sb_) * nk; };
      // 0: not this CTA's business, 1: owner (folds, finishes and stores), 2: contributor (hands partials over)
      auto role = [&](int i) -> int {
        if (!args.canon) return (i >= ilo_ && i < ihi_) ? 1 : 0;
        if (args.range_mode && (i < pb_ || i >= pe_)) return 0;
        return first_stage(i) >= S0_ ? 1 : 2;
      };
      auto row0_of = [&](int i) -> int64_t {
        return args.range_mode ? (int64_t)(i - pb_) * Br : (int64_t)affine_pow(p, (uint64_t)i, 0u) * Br;
      };
      const int q0c = sb_ + S0_ / nk;  // contributor: straddler j of output i is i - (q0c - κ) ∈ [0, κ)
      const CanonGeom geo(args, nk, BN);
      auto tile_ptr = [&](int r_, int j, int lg) { return geo.tile(r_, ct, j, lg); };
      auto mark_bad = [&](int c) { atomicOr(&fixmap[c >> 5], 1u << (c & 31)); };
      // values the band MMA cannot be trusted with: non-finite (0·Inf in the dense band, hi = Inf
      // for |a| beyond the bf16 range) or a nonzero |y| < 2^-100 — only columns of tiny inputs
      // produce those, and below 2^-117 the bf16 lo part of the fp32 split loses precision
      auto needs_exact = [](float v) {
        const uint32_t b = __float_as_uint(v), e = (b >> 23) & 0xFFu;
        return e == 0xFFu || (e < 27u && (b & 0x7FFFFFFFu) != 0u);
      };
      auto fix_output = [&](int i) {
        const int64_t yr0 = row0_of(i);
        for (int w = 0; w < BN / 32; ++w) {
          uint32_t bits = fixmap[w];
          while (bits) {
            const int c = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t col = col0 + c;
            for (int r = 0; r < Br; ++r) {
              const float v = exact_elem<F32, TRANS>(args, i, (uint32_t)r, col, et, fixred);
              if (et == 0) {
                if (!TRANS) {
                  args.Y[(yr0 + r) * args.ldy + col] = v;
                  if (args.npeer || args.mc) bcast1(args, yr0 + r, col, v);
                } else {
                  args.Y[col * args.ldy + yr0 + r] = v;
                }
              }
            }
          }
        }
        ptx::named_bar_sync(kEpiBar, 128);
        if (et < 8) fixmap[et] = 0u;
        ptx::named_bar_sync(kEpiBar, 128);
      };
      const int qtr = warp & 3;
      const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
      uint64_t keep = policy_evict_last();  // partial tiles and parked prefixes: read by the combine
      if (args.ab & 4) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
      {  // S = 0
        uint32_t z[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) z[t] = 0u;
        for (int c = 0; c < NMT * K::SN; c += 16) ptx::tmem_st16(tmem_S + lane_off + c, z);
        ptx::tmem_wait_st();
      }
      // NT forms: final values (scaled) of 16 consecutive columns cl0.. (local) of Y row yrow
      auto store16 = [&](int64_t yrow, int cl0, const float (&v)[16]) -> bool {
        const int64_t cb = col0 + cl0;
        bool bad = false;
        if (!TRANS) {
          float* y = args.Y + yrow * args.ldy + cb;
          const bool bc = args.npeer || args.mc;
#pragma unroll
          for (int t = 0; t < 16; t += 4) {
            if (cb + t + 3 < args.n) {
              const float4 q4 = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
              *reinterpret_cast<float4*>(y + t) = q4;
              if (bc) bcast4(args, yrow, cb + t, q4);
            } else {
              for (int e = 0; e < 4; ++e)
                if (cb + t + e < args.n) {
                  y[t + e] = v[t + e];
                  if (bc) bcast1(args, yrow, cb + t + e, v[t + e]);
                }
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (cb + t < args.n) args.Y[(cb + t) * args.ldy + yrow] = v[t];
        }
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (cb + t < args.n && needs_exact(v[t])) bad = true, mark_bad(cl0 + t);
        return bad;
      };
      // TF form: one column cl, 16 consecutive rows yrow0.. (row-major Y)
      auto store_col16 = [&](int64_t yrow0, int cl, const float (&v)[16], int t0, int t1) -> bool {
        const int64_t cb = col0 + cl;
        if (cb >= args.n) return false;
        bool bad = false;
        float* y = args.Y + yrow0 * args.ldy + cb;
        const bool bc = args.npeer || args.mc;
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t >= t0 && t < t1) {
            y[(int64_t)t * args.ldy] = v[t];
            if (bc) bcast1(args, yrow0 + t, cb, v[t]);
            bad |= needs_exact(v[t]);
          }
        if (bad) mark_bad(cl);
        return bad;
      };
      // all 128 threads: recompute the marked columns of output i exactly (R12), then clear the map

      int eg = 0;  // groups folded (D buffer eg % NACC)
      const Tr tr((args.trace && threadIdx.x == 0) ? args.trace + blockIdx.x * kTrSlots : nullptr);
      const unsigned long long tstart = tr.now();
      int kc = (int)(S0 % nk);
      int gi = kc % G;
      int q = sb_ + S0_ / nk;
      for (int st = S0_; st < S1_;
           ++st, q += (kc + 1 == nk), gi = (kc + 1 == nk || gi + 1 == G) ? 0 : gi + 1, kc = (kc + 1 == nk) ? 0 : kc + 1) {
        const bool gend = st == S1_ - 1 || kc == nk - 1 || gi == G - 1;
        if (!gend) continue;
        const bool blk_end = kc == nk - 1;
        const int lg = (st - G + 1 - S0_) / G;  // group index inside this range (groups are G-aligned)
        const int qm = (int)((uint32_t)(q - 1) % (uint32_t)kap);  // (q-1) mod κ: slot of output q-1
        // output in slot sig while input block q streams: i ≡ sig (mod κ), q-κ ≤ i ≤ q-1
        auto slot_out = [&](int sig) { return q - 1 - (qm >= sig ? qm - sig : qm + kap - sig); };
        const int db = eg % K::NACC;
        {
          const unsigned long long t0 = tr.now();
          ptx::mbar_wait_sleep(&acc_full[db], (uint32_t)(eg / K::NACC) & 1u, 32);
          tr.add(9, t0);
        }
        ++eg;
        ptx::tc_fence_after();
        bool mybad = false;
        if (TF) {
          // lanes = data columns; TMEM columns = band rows ρ (slot ρ / B_r, row ρ mod B_r)
          const int cl = qtr * 32 + lane;
#pragma unroll 1
          for (int c0 = 0; c0 < krows; c0 += 16) {  // warp-uniform
            uint32_t d[16], sv[16];  // d: hi + lo products of the group (one D tile)
            ptx::tmem_ld16(tmem + (db ? K::OFF_D1 : 0) + lane_off + c0, d);
            ptx::tmem_ld16(tmem_S + lane_off + c0, sv);
            ptx::tmem_wait_ld();
            // the chunk's rows belong to one slot unless B_r is not a multiple of 16: walk its slot runs
            int t0 = 0;
            while (t0 < 16 && c0 + t0 < krows) {
              const int sig = (c0 + t0) / Br, r0 = c0 + t0 - sig * Br;
              const int t1 = min(16, min(t0 + Br - r0, krows - c0));
              const int i = slot_out(s0 + sig);
              const int rl = role(i);
              if (rl == 1) {
                const bool fin = blk_end && i == q - kap;
                float v[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  const float tot = __uint_as_float(sv[t]) + __uint_as_float(d[t]);
                  v[t] = tot * p.scale;
                  if (t >= t0 && t < t1) sv[t] = fin ? 0u : __float_as_uint(tot);
                }
                if (fin) mybad |= store_col16(row0_of(i) + r0 - t0, cl, v, t0, t1);
              } else {
                if (rl == 2 && !(args.ab & 2)) {
                  float* w = tile_ptr(rr, i - (q0c - kap), lg) + (int64_t)(r0 - t0) * BN + cl;
#pragma unroll
                  for (int t = 0; t < 16; ++t)
                    if (t >= t0 && t < t1) st_keep(w + (int64_t)t * BN, __uint_as_float(d[t]), keep);
                }
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  if (t >= t0 && t < t1) sv[t] = 0u;
              }
              t0 = t1;
            }
            ptx::tmem_st16(tmem_S + lane_off + c0, sv);
          }
        } else {
#pragma unroll 1
          for (int m = 0; m < NMT; ++m) {
            const int rho = m * 128 + qtr * 32 + lane;
            const bool valid = rho < krows;
            const int sig = valid ? rho / Br : 0, r = rho - sig * Br;  // local slot
            const int i = slot_out(s0 + sig);
            const int rl = valid ? role(i) : 0;
            const bool fin = rl == 1 && blk_end && i == q - kap;
            float* wcol = rl == 2 ? tile_ptr(rr, i - (q0c - kap), lg) + r : nullptr;  // column-major tile
            const int64_t yrow = fin ? row0_of(i) + r : 0;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 16) {
              uint32_t d[16], sv[16];
              float P[16];
              ptx::tmem_ld16(tmem + lane_off + m * K::DN + c0, d);
              ptx::tmem_ld16(tmem_S + lane_off + m * BN + c0, sv);
              if (F32) {  // hi and lo partial products
                uint32_t dl[16];
                ptx::tmem_ld16(tmem + lane_off + m * K::DN + BN + c0, dl);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 16; ++t) P[t] = __uint_as_float(d[t]) + __uint_as_float(dl[t]);
              } else {
                ptx::tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 16; ++t) P[t] = __uint_as_float(d[t]);
              }
              if (rl == 1) {
                float v[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  const float tot = __uint_as_float(sv[t]) + P[t];
                  v[t] = tot * p.scale;
                  sv[t] = fin ? 0u : __float_as_uint(tot);
                }
                if (fin) mybad |= store16(yrow, c0, v);
              } else {
                if (rl == 2 && !(args.ab & 2)) {
#pragma unroll
                  for (int t = 0; t < 16; ++t) st_keep(wcol + (int64_t)(c0 + t) * Br, P[t], keep);
                }
#pragma unroll
                for (int t = 0; t < 16; ++t) sv[t] = 0u;
              }
              ptx::tmem_st16(tmem_S + lane_off + m * BN + c0, sv);
            }
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        if (K::PAIR && css != 0)
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&acc_free[db]), 0));  // the leader's MMA waits
        else
          ptx::mbar_arrive(&acc_free[db]);
        // ---- group-end bookkeeping (uniform over the 128 epilogue threads)
        if (blk_end && mine(q - kap) && role(q - kap) == 1 && bar_red_or(kEpiBar, 128, mybad)) fix_output(q - kap);
      }
      tr.add(10, tstart);
      // canon, range end: every owned output still open parks its prefix (unscaled running sum) in
      // its Y rows; bps_tc_combine adds the contributors' group partials after the kernel
      if (args.canon) {
        const int q_last = sb_ + (S1_ - 1) / nk;
        const bool full_end = (S1_ - 1) % nk == nk - 1;
        for (int i = q_last - kap + (full_end ? 1 : 0); i <= q_last - 1; ++i) {
          if (role(i) != 1 || !mine(i)) continue;  // uniform
          const int lo = (slot_of(i) - s0) * Br;  // local band rows of its slot
          const int64_t yr0 = row0_of(i);
          if (TF) {
            const int64_t col = col0 + qtr * 32 + lane;
            for (int c0 = lo & ~15; c0 < lo + Br; c0 += 16) {
              uint32_t sv[16];
              ptx::tmem_ld16(tmem_S + lane_off + c0, sv);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int t2 = 0; t2 < 16; ++t2) {
                const int r = c0 + t2 - lo;
                if (r >= 0 && r < Br && col < args.n) st_keep(args.Y + (yr0 + r) * args.ldy + col, __uint_as_float(sv[t2]), keep);
              }
            }
          } else {
#pragma unroll 1
            for (int m = 0; m < NMT; ++m) {
              const int base = m * 128 + qtr * 32;
              if (base + 32 <= lo || base >= lo + Br) continue;  // warp-uniform
              const int r = base + lane - lo;
              const bool in_slot = r >= 0 && r < Br;
#pragma unroll 1
              for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t sv[16];
                ptx::tmem_ld16(tmem_S + lane_off + m * BN + c0, sv);
                ptx::tmem_wait_ld();
                if (!in_slot) continue;
                if (!TRANS && col0 + c0 + 15 < args.n) {
                  float* y = args.Y + (yr0 + r) * args.ldy + col0 + c0;
#pragma unroll
                  for (int t2 = 0; t2 < 16; t2 += 4)
                    st_keep4(y + t2, make_float4(__uint_as_float(sv[t2]), __uint_as_float(sv[t2 + 1]), __uint_as_float(sv[t2 + 2]),
                                                 __uint_as_float(sv[t2 + 3])), keep);
                } else {
#pragma unroll
                  for (int t2 = 0; t2 < 16; ++t2) {
                    const int64_t cb = col0 + c0 + t2;
                    if (cb < args.n) {
                      float* y = TRANS ? args.Y + cb * args.ldy + yr0 + r : args.Y + (yr0 + r) * args.ldy + cb;
                      st_keep(y, __uint_as_float(sv[t2]), keep);
                    }
                  }
                }
              }
            }
          }
        }
        if (args.flags) {
          // every tile and prefix of this CTA is stored: publish them (gpu-scope release)
          __threadfence();
          ptx::named_bar_sync(kEpiBar, 128);
          if (et == 0)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(args.flags + blockIdx.x), "l"(args.epoch) : "memory");
        }
      }
    } else if (warp >= 4 && warp < 4 + K::NBW) {
      // the intra-block mode is a launch constant: specialise the whole generator on it
      auto band_gen = [&](auto affine_tag, auto fast_tag) {
        constexpr bool AFF = decltype(affine_tag)::value;
        // FAST (row-partitioned only): C = B_r/s a power of two and κs a multiple of 4·NCG, so every
        // thread owns a whole number of 4-chunk batches (no tail predication, immediate table
        // offsets), the row offset is a shift, and the stale entries are kept as 16-bit entry
        // offsets (clearing = one extract + one store).  C = 1 (s = B_r) writes every band row of
        // every column each stage, so nothing needs clearing at all.
        // MN8 (C = 8, B_r % 8 == 0, TcArgs::band_mn): MN-major band tile — a chunk's 8 rows at input
        // row u are one 16-byte piece, written whole (one-hot) each stage: no clearing, no prev state
        constexpr bool MN8 = decltype(fast_tag)::value == 7;
        constexpr bool FAST = decltype(fast_tag)::value >= 1 && !MN8;
        constexpr bool FULL = decltype(fast_tag)::value >= 2 && !MN8;  // κs a multiple of 4·NCG: no batch tail
        // HOIST (κs = 4·NCG: exactly one batch of 4 chunks per thread): the thread's 4 keys and
        // row bases live in registers, reloaded once per input block instead of every stage
        constexpr bool HOIST = decltype(fast_tag)::value == 6;
        uint64_t hk[4] = {0, 0, 0, 0};
        uint32_t hc[4] = {0, 0, 0, 0};
        // DENSE (C = B_r/s ∈ {1, 2, 4}): whole 16-byte pieces, CP = C rows per chunk
        constexpr bool DENSE = decltype(fast_tag)::value >= 3 && decltype(fast_tag)::value <= 5;
        constexpr int CP = DENSE ? (1 << (decltype(fast_tag)::value - 3)) : 1;
        constexpr int NPW = FAST ? 8 : 4;  // prev words per buffer
        // ===================== band generator =====================
        // Thread (u, cg) writes column u of every band stage for the row chunks c = cg + NCG·t,
        // c = σ·s + j (slot σ, chunk j).  A chunk's rows [σB_r + jC, +C) are owned by one thread
        // per column, so each thread can clear the single entry it wrote into this buffer
        // NBAND stages ago and write the new one without any barrier (no zero-fill pass).
        const int bt = threadIdx.x - 128;
        const uint32_t u = (uint32_t)bt & (kBK - 1);
        const uint32_t cg = (uint32_t)bt >> 6;  // 0..NCG-1
        const uint32_t ncombo = kap_l * p.s;  // this CTA's (slot, chunk) combos
        const uint32_t T = ncombo > cg ? (ncombo - cg + K::NCG - 1) / K::NCG : 0;  // chunks of this thread (≤ 32)
        const bool zf = ncombo > 16u * K::NCG;  // stale rows no longer fit the prev registers (4 words)
        const uint32_t band_u32 = ptx::smem_u32(smem + K::OFF_BAND);
        const uint32_t ucol = u >> 3, ulo = (u & 7) * 2;
        auto entry = [&](uint32_t sbase, uint32_t rho) {
          // row ρ of the stage at ρ·128 (M-tiles of 128 rows are contiguous: kBandTile = 128·128),
          // SW128: 16-byte chunk index XOR (ρ mod 8)
          static_assert(kBandTile == 128 * 128, "band tile layout");
          return sbase + rho * 128 + (((rho ^ ucol) & 7) << 4) + ulo;
        };
        {  // band buffers start zeroed; chunk row bases (fixed for the whole launch)
          uint4* bz = reinterpret_cast<uint4*>(smem + K::OFF_BAND);
          for (int i = bt; i < K::NBAND * K::BAND_STAGE / 16; i += K::NBANDT) bz[i] = make_uint4(0, 0, 0, 0);
          for (uint32_t c = bt; c < ncombo; c += K::NBANDT) crow[c] = band_crow(p, c / p.s, c % p.s);
        }
        // rows written LOCALB local stages ago: 4 rows per word (κ·B_r ≤ 256), or (FAST) 2 entry
        // offsets per word
        uint32_t prev[K::LOCALB][NPW];
        const uint32_t crank = CS > 1 ? ptx::cluster_ctarank() : 0u;
        int64_t local_no = 0;
  #pragma unroll
        for (int b = 0; b < K::LOCALB; ++b)
  #pragma unroll
          for (int w = 0; w < NPW; ++w) prev[b][w] = 0;
        const uint32_t cshift = 32u - (31u - (uint32_t)__clz(p.C));  // FAST: off = z_hi >> (32 - log2 C)
        if constexpr (HOIST && BPS_HOIST_FLAT) {
          // HOIST: stale entries as full byte offsets, one per chunk (words 0-3); initially the first
          // entry of the thread's own chunk (harmless to clear: zero, or rewritten right after)
  #pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t c = cg + K::NCG * w;
            const uint32_t r = c < ncombo ? band_crow(p, c / p.s, c % p.s) : 0u;
  #pragma unroll
            for (int b = 0; b < K::LOCALB; ++b) prev[b][w] = r * 128u + (((r ^ ucol) & 7u) << 4);
          }
        } else if constexpr (FAST) {
          // before the first write of a buffer, "clear" the first entry of the thread's own chunk
          // (zero in a fresh buffer, and rewritten or left zero by the write that follows)
  #pragma unroll
          for (int w = 0; w < NPW; ++w) {
            uint32_t v = 0;
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t c = cg + K::NCG * (2 * w + h);
              const uint32_t r = c < ncombo ? band_crow(p, c / p.s, c % p.s) : 0u;
              v |= (r * 128u + (((r ^ ucol) & 7u) << 4)) << (16 * h);
            }
  #pragma unroll
            for (int b = 0; b < K::LOCALB; ++b) prev[b][w] = v;
          }
        }
        int bs = 0;
        uint32_t bph = 0;
        int stage_no = 0;
        const int ksm = args.kstep - 1;
        const Tr tr((args.trace && bt == 0) ? args.trace + blockIdx.x * kTrSlots : nullptr);
        const unsigned long long tstart = tr.now();
        int kc = S0i % nk;
        int q = sbi + S0i / nk;
        for (int st = S0i; st < S1i; ++st, q += (kc + 1 == nk), kc = (kc + 1 == nk) ? 0 : kc + 1, ++stage_no) {
          const int par = (int)(q & 1);  // tables double-buffered by block parity
          uint64_t* ck = ckey + par * 256;
          {
            const bool local = CS == 1 || (uint32_t)bs % CS == crank;
            const int sp = stage_no & ksm;  // kstep = 2: wait at the first stage of a pair only
            unsigned long long t0 = tr.now();
            if ((local || bt == 0) && sp == 0) wait_slot(&band_empty[bs], bph ^ 1, args.sleep_ns);
            tr.add(6, t0);
            t0 = tr.now();
            if (kc == 0 || st == S0i) {
              // per input block q: hash key of chunk (σ, j): the output i ≡ σ (mod κ) fed by q is
              // i = q - ℓ with ℓ = ((q - σ - 1) mod κ) + 1
              for (uint32_t c = bt; c < ncombo; c += K::NBANDT) {
                const uint32_t sig = sig0 + c / p.s, j = c % p.s;  // global slot
                const uint32_t ell = mod_pos(q - (int64_t)sig - 1, kappa) + 1;
                const uint32_t g = affine_pow(p, (uint64_t)mod_pos(q - (int64_t)ell, p.M), 0u);
                const uint64_t key = (((uint64_t)g << 40) | ((uint64_t)(ell - 1) << 32) | (uint64_t)band_jfield(p, j)) ^ p.K;
                if constexpr (AFF) {
                  ck[c] = key;
                } else {  // row-partitioned: store the folded key (L1 | P1 << 32), see mix64_folded
                  uint32_t L1, P1;
                  mix64_fold_key(key, L1, P1);
                  ck[c] = ((uint64_t)P1 << 32) | L1;
                }
              }
              ptx::named_bar_sync(1, K::NBANDT);
              if constexpr (HOIST) {
  #pragma unroll
                for (int i = 0; i < 4; ++i) hk[i] = ck[cg + K::NCG * i], hc[i] = crow[cg + K::NCG * i] * 128u;
              }
              tr.add(7, t0);
            }
            const uint64_t uk = (uint64_t)((uint32_t)kc * kBK + u) << 8;
            const uint32_t sbase = band_u32 + bs * K::BAND_STAGE;
            if (!local) {  // band stage generated by cluster peer `bs`: expect its bulk copy
              if (bt == 0) ptx::mbar_arrive_expect_tx(&band_full[bs], K::BAND_STAGE);
              if (++bs == K::NBAND) bs = 0, bph ^= 1;
              continue;
            }
            bool clear = local_no >= K::LOCALB;
            ++local_no;
            const bool zero_fill = AFF ? kap_l > 4u * K::NCG : ((DENSE || MN8) ? false : (zf && p.C > 1u));
            if (zero_fill && clear) {
              // more stale entries per thread than the 4 prev words hold: zero-fill the stage
              // cooperatively, then write (one barrier per stage)
              uint4* bz = reinterpret_cast<uint4*>(smem + K::OFF_BAND + bs * K::BAND_STAGE);
              for (int i = bt; i < K::BAND_STAGE / 16; i += K::NBANDT) bz[i] = make_uint4(0, 0, 0, 0);
              ptx::named_bar_sync(4, K::NBANDT);
            }
            if (zero_fill) clear = false;
            uint32_t nw[NPW];
  #pragma unroll
            for (int w = 0; w < NPW; ++w) nw[w] = 0;
            if (BPS_DBG(1)) {
              // experiment: no band generation (every generator variant)
            } else if constexpr (MN8) {
              // MN-major SW128 band tile: 64-row atoms 8 KB apart, input row u at u·128, the 16-byte
              // piece of rows [ρ0, ρ0+8) at ((ρ0/8 ⊕ u) mod 8)·16.  One hash → the chunk's row offset
              // (R3 with C = 8: z_hi >> 29) and sign → one one-hot piece, one conflict-free store
              const uint32_t x = (uint32_t)uk;  // counter low word: (kc·64 + u) << 8
              const uint32_t urow = sbase + u * 128u;
              for (uint32_t t = 0; t < T; t += 4) {
                uint32_t hi[4], lo[4], cr[4];
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint32_t c = (t + i < T) ? cg + K::NCG * (t + (uint32_t)i) : cg;
                  const uint64_t k = ck[c];
                  cr[i] = crow[c];
                  mix64_folded((uint32_t)k, (uint32_t)(k >> 32), x, hi[i], lo[i]);
                }
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  if (t + (uint32_t)i < T) {
                    const uint32_t off = hi[i] >> 29;
                    const uint32_t val = (0x3F80u | ((lo[i] & 1u) << 15)) << ((off & 1u) << 4);  // ±1.0 bf16
                    const uint32_t ws = off >> 1;
                    const uint32_t rho = cr[i];
                    const uint32_t addr = urow + ((rho >> 6) << 13) + ((((rho >> 3) ^ u) & 7u) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(ws == 0u ? val : 0u),
                                 "r"(ws == 1u ? val : 0u), "r"(ws == 2u ? val : 0u), "r"(ws == 3u ? val : 0u)
                                 : "memory");
                  }
                }
              }
            } else if constexpr (DENSE) {
              // C = B_r/s ∈ {1, 2, 4}: chunk c owns the CP band rows crow[c] .. +CP-1 and has exactly
              // one ±1 per column among them, so every row of the chunk is rewritten each stage as
              // whole 16-byte SW128 pieces (8 columns): per item (chunk, 8-column group) 8
              // independent hashes (ILP 8), CP vector stores, no per-entry addressing and nothing
              // to clear (rows ≥ κB_r stay zero from the initial fill).
              const uint32_t xk = (uint32_t)kc * (uint32_t)kBK;
              for (uint32_t q = (uint32_t)bt; q < ncombo * 8u; q += K::NBANDT) {
                const uint32_t c = q >> 3, ch = q & 7u;
                const uint64_t k = ck[c];
                const uint32_t r0 = crow[c];
                const uint32_t x0 = (xk + ch * 8u) << 8;
                uint32_t v[8], ro[8];
  #pragma unroll
                for (int e = 0; e < 8; ++e) {
                  uint32_t h, l;
                  mix64_folded((uint32_t)k, (uint32_t)(k >> 32), x0 + ((uint32_t)e << 8), h, l);
                  v[e] = (0x3F80u | (l << 15)) & 0xFFFFu;  // ±1.0, sign = z & 1
                  ro[e] = CP == 1 ? 0u : (h >> (32 - (CP == 2 ? 1 : 2)));  // R3: (z_hi · C) >> 32
                }
  #pragma unroll
                for (int rr = 0; rr < CP; ++rr) {
                  uint32_t w[4];
  #pragma unroll
                  for (int j = 0; j < 4; ++j)
                    w[j] = (ro[2 * j] == (uint32_t)rr ? v[2 * j] : 0u) | ((ro[2 * j + 1] == (uint32_t)rr ? v[2 * j + 1] : 0u) << 16);
                  const uint32_t rho = r0 + (uint32_t)rr;
                  const uint32_t addr = sbase + rho * 128u + (((ch ^ rho) & 7u) << 4);
                  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                               "r"(w[3])
                               : "memory");
                }
              }
            } else if constexpr (HOIST && BPS_HOIST_FLAT) {
              // 4 chunks, keys and row-base byte offsets hc[i] = crow·128 in registers.  C ≥ 8 is a power
              // of two, so chunk row bases are multiples of 8 and the SW128 16-byte index of row
              // crow + r is (r ⊕ u/8) mod 8: one shift, one LOP3, one IMAD and one add per entry; the
              // stale entry is a full byte offset (no unpacking)
              const uint32_t x = (uint32_t)uk;  // counter low word: (kc·64 + u) << 8
              const uint32_t ebase = sbase + ulo;
              uint32_t hi[4], lo[4];
  #pragma unroll
              for (int i = 0; i < 4; ++i) mix64_folded((uint32_t)hk[i], (uint32_t)(hk[i] >> 32), x, hi[i], lo[i]);
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const uint32_t r = ptx::shr_clamp(hi[i], cshift);  // R3 for C = 2^m
                const uint32_t off = hc[i] + r * 128u + (((r ^ ucol) & 7u) << 4);
                ptx::st_shared_u16(ebase + prev[0][i], 0);
                nw[i] = off;
                ptx::st_shared_u16(ebase + off, (uint16_t)(0x3F80u | (lo[i] << 15)));  // ±1.0, sign = z & 1
              }
            } else if constexpr (FAST) {
              const uint32_t x = (uint32_t)uk;  // counter low word: (kc·64 + u) << 8
              const uint32_t ebase = sbase + ulo;
              const bool do_clear = !zero_fill && p.C > 1u;
              const bool full = FULL;
              const uint64_t* ckt = ck + cg;
              const uint32_t* crt = crow + cg;
  #pragma unroll
              for (int w = 0; w < 8; ++w) {
                if ((uint32_t)w * 4 >= T) break;
                uint32_t hi[4], lo[4], cr[4];
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint64_t k = HOIST ? hk[i] : ckt[K::NCG * (4 * w + i)];
                  cr[i] = HOIST ? hc[i] / 128u : crt[K::NCG * (4 * w + i)];
                  mix64_folded((uint32_t)k, (uint32_t)(k >> 32), x, hi[i], lo[i]);
                }
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const bool on = full || (uint32_t)(4 * w + i) < T;  // κs/NCG not a multiple of 4: tail
                  const uint32_t rho = cr[i] + ptx::shr_clamp(hi[i], cshift);  // R3 for C = 2^m
                  const uint32_t off = rho * 128u + (((rho ^ ucol) & 7u) << 4);
                  if (w < 4 && on) {
                    if (do_clear) ptx::st_shared_u16(ebase + ((prev[0][2 * w + (i >> 1)] >> (16 * (i & 1))) & 0xFFFFu), 0);
                    nw[2 * w + (i >> 1)] |= off << (16 * (i & 1));
                  }
                  if (on) ptx::st_shared_u16(ebase + off, (uint16_t)(0x3F80u | (lo[i] << 15)));  // ±1.0, sign = z & 1
                }
              }
            } else if constexpr (AFF) {
              // AffineUnique (R18), slot-major: thread (u, cg) owns the whole column u of slots
              // σ ≡ cg (mod NCG): ONE hash per (σ, u) gives α, β and the s signs; the s rows
              // (α·j + β) mod B_r are walked incrementally.  Clearing re-walks last use's (α, β)
              // (kept as α | β<<16 in prev) — same thread, so no barrier.
  #pragma unroll
              for (int t = 0; t < 16; ++t) {
                const uint32_t sig = cg + K::NCG * t;
                if (sig >= kap_l) break;
                const uint32_t base = sig * p.B_r;
                if (t < 4 && clear) {
                  const uint32_t w = prev[0][t & 3], a0 = w & 0xFFFFu;
                  uint32_t r = w >> 16;
                  for (uint32_t j = 0; j < p.s; ++j, r = (r + a0) & p.Brmask)
                    ptx::st_shared_u16(entry(sbase, base + r), 0);
                }
                const uint64_t z = mix64(ck[sig * p.s] ^ uk);
                const uint32_t alpha = (uint32_t)(((((z >> 32) & 0xFFFFu) * p.B_r) >> 16) | 1u);
                const uint32_t beta = (uint32_t)(((z >> 48) * p.B_r) >> 16);
                uint32_t r = beta, zs = (uint32_t)z;
                for (uint32_t j = 0; j < p.s; ++j, r = (r + alpha) & p.Brmask, zs >>= 1)
                  ptx::st_shared_u16(entry(sbase, base + r), (zs & 1u) ? (uint16_t)0xBF80 : (uint16_t)0x3F80);
                if (t < 4) nw[t & 3] = alpha | (beta << 16);
              }
            } else if (!BPS_DBG(1)) {
              // row-partitioned (R1-R3): one hash per (chunk, u).  The 4 chunks of a batch are
              // independent (disjoint row ranges), so the tail of the batch is predicated rather
              // than branched and the compiler interleaves the four hash/store chains.
              const uint32_t x = (uint32_t)uk;  // counter low word: (kc·64 + u) << 8
  #pragma unroll
              for (int w = 0; w < 8; ++w) {
                if ((uint32_t)w * 4 >= T) break;
                uint32_t hi[4], lo[4], cr[4];
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  uint32_t c = cg + K::NCG * (4 * w + i);
                  c = c < ncombo ? c : cg;
                  const uint64_t k = ck[c];
                  cr[i] = crow[c];
                  if (BPS_DBG(32)) {
                    hi[i] = (uint32_t)k ^ x;
                    lo[i] = (uint32_t)(k >> 32);
                  } else {
                    mix64_folded((uint32_t)k, (uint32_t)(k >> 32), x, hi[i], lo[i]);
                  }
                }
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const bool on = (uint32_t)(4 * w + i) < T;
                  if (w < 4 && clear && on) ptx::st_shared_u16(entry(sbase, (prev[0][w & 3] >> (8 * i)) & 0xFFu), 0);
                  const uint32_t rho = cr[i] + __umulhi(hi[i], p.C);  // R3
                  const uint32_t val = 0x3F80u | ((lo[i] & 1u) << 15);  // ±1.0 bf16, sign = z & 1
                  if (on) ptx::st_shared_u16(entry(sbase, rho), (uint16_t)val);
                  if (w < 4 && on) nw[w & 3] |= rho << (8 * i);
                }
              }
            }
  #pragma unroll
            for (int b = 0; b + 1 < K::LOCALB; ++b)
  #pragma unroll
              for (int w = 0; w < NPW; ++w) prev[b][w] = prev[b + 1][w];
  #pragma unroll
            for (int w = 0; w < NPW; ++w) prev[K::LOCALB - 1][w] = nw[w];
            if (sp != ksm) {  // kstep = 2: first stage of a pair — fence and arrive after the second
              if (++bs == K::NBAND) bs = 0, bph ^= 1;
              continue;
            }
            // (PAIR: this CTA's band rows are read by its own SM's tensor core, as part of the leader's
            // pair MMA — the CTA-scope proxy fence plus the cluster-release arrive order them)
            if (!BPS_DBG(16)) ptx::fence_proxy_async_smem();
            if (CS > 1) {
              ptx::named_bar_sync(3, K::NBANDT);  // whole stage written (and fenced) by all band threads
              if (bt == 0) {
                const uint32_t src = band_u32 + bs * K::BAND_STAGE;
                const uint32_t bar = ptx::smem_u32(&band_full[bs]);
                for (uint32_t r = 1; r < (uint32_t)CS; ++r) {
                  const uint32_t peer = (crank + r) % CS;
                  ptx::bulk_copy_to_peer(ptx::mapa(src, peer), src, K::BAND_STAGE, ptx::mapa(bar, peer));
                }
                ptx::mbar_arrive(&band_full[bs]);
              }
            } else {
              if (K::PAIR && css != 0) {  // the leader's MMA reads this CTA's band rows
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&band_full[bs]), 0));
              } else {
                warp_arrive(&band_full[bs - ksm]);
              }
            }
            if (++bs == K::NBAND) bs = 0, bph ^= 1;
          }
        }
        tr.add(8, tstart);
      };
      const uint32_t ncomb = kap_l * p.s;
      if (p.mode)
        band_gen(std::true_type{}, std::integral_constant<int, 0>{});
      else if (p.C == 1u)
        band_gen(std::false_type{}, std::integral_constant<int, 3>{});
      else if (p.C == 2u)
        band_gen(std::false_type{}, std::integral_constant<int, 4>{});
      else if (p.C == 4u)
        band_gen(std::false_type{}, std::integral_constant<int, 5>{});
      else if (args.band_mn)
        band_gen(std::false_type{}, std::integral_constant<int, 7>{});
      else if ((p.C & (p.C - 1u)) == 0u && ncomb == 4u * K::NCG && !args.nohoist)
        band_gen(std::false_type{}, std::integral_constant<int, 6>{});
      else if ((p.C & (p.C - 1u)) == 0u && ncomb % (4u * K::NCG) == 0u)
        band_gen(std::false_type{}, std::integral_constant<int, 2>{});
      else if ((p.C & (p.C - 1u)) == 0u && ncomb % K::NCG == 0u)
        band_gen(std::false_type{}, std::integral_constant<int, 1>{});
      else
        band_gen(std::false_type{}, std::integral_constant<int, 0>{});
    } else if (TF && warp >= K::W_CONV0 && warp < K::W_CONV0 + 8) {
      // ============ TF converter: fp32 column -> TMEM A operand (hi | lo bf16 pairs) ============
      // warp w: TMEM lane quarter w % 4 (data columns 32q..32q+31), K rows 32h..32h+31 (h = (w-12)/4).
      // A stage layout: lane = data column, 32-bit column j holds K rows (2j, 2j+1) (low half = even
      // row); hi at +0..31, lo at +32..63.  The raw stage is released as soon as it is in registers.
      const int cv = threadIdx.x - K::W_CONV0 * 32;
      const int qtr = warp & 3, h = (warp - K::W_CONV0) >> 2;
      const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
      const int col = qtr * 32 + lane;
      int rs = 0;
      uint32_t rph = 0;
      const int total = S1i - S0i;
      for (int it = 0; it < total; ++it) {
        ptx::mbar_wait(&raw_full[rs], rph);
        const float* raw = reinterpret_cast<const float*>(smem + K::OFF_RAW + rs * K::RAW_STAGE) + (h * 32) * BN + col;
        float a[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) a[r] = raw[r * BN];
        warp_arrive(&raw_empty[rs]);  // values are in registers
        if (SS > 1) {  // the multicast refill writes every CTA's copy: release the slot in all of them
          if (lane == 0)
            for (uint32_t pr = 1; pr < (uint32_t)SS; ++pr)
              ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&raw_empty[rs]), ((uint32_t)css + pr) % SS));
        }
        if (++rs == K::NRAW) rs = 0, rph ^= 1;
        const uint32_t ab = (uint32_t)(it & 1);
        ptx::mbar_wait(&ta_empty[ab], (uint32_t)((it >> 1) & 1) ^ 1u);
        ptx::tc_fence_after();
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi[j]) : "f"(a[2 * j + 1]), "f"(a[2 * j]));
          const float r0 = a[2 * j] - __uint_as_float(hi[j] << 16);
          const float r1 = a[2 * j + 1] - __uint_as_float(hi[j] & 0xFFFF0000u);
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo[j]) : "f"(r1), "f"(r0));
        }
        const uint32_t ta = tmem_A + ab * 64 + (uint32_t)h * 16;
        ptx::tmem_st16(ta + lane_off, hi);
        ptx::tmem_st16(ta + lane_off + 32, lo);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        warp_arrive(&ta_full[ab]);
        (void)cv;
      }
    } else if (RL && warp >= K::W_CONV0 && warp < K::W_CONV0 + K::NCONVW) {
      // ===================== RL: unswizzled K-chunk pair -> two SW128 K-major tiles =====================
      // 16-byte piece q of the pair (vector v = q/16, piece c = q%16 of its 256 bytes) moves to
      // tile c/8 (= ring slot rs + c/8), row v, SW128 position (c%8) ^ (v%8).  Reads: a warp
      // reads 512 contiguous bytes; writes: 4 whole 128-byte rows.  In place, so everything
      // is read (registers) before anything is written (named barrier).
      const int cv = threadIdx.x - K::W_CONV0 * 32;
      constexpr int NT = K::NCONVT;
      constexpr int NIT = 2 * K::RAW_STAGE / 16 / NT;
      static_assert(NIT * NT * 16 == 2 * K::RAW_STAGE, "re-layout tiling");
      int rs = 0;
      uint32_t rph = 0;
      for (int st = S0i; st < S1i; st += 2) {
        ptx::mbar_wait(&raw_full[rs], rph);
        uint8_t* base = smem + K::OFF_RAW + rs * K::RAW_STAGE;
        const uint4* src = reinterpret_cast<const uint4*>(base);
        uint4 a[NIT];
#pragma unroll
        for (int i = 0; i < NIT; ++i) a[i] = src[i * NT + cv];
        ptx::named_bar_sync(2, NT);
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const uint32_t q = (uint32_t)(i * NT + cv), v = q >> 4, c = q & 15u;
          *reinterpret_cast<uint4*>(base + (c >> 3) * K::RAW_STAGE + v * 128u + (((c & 7u) ^ (v & 7u)) << 4)) = a[i];
        }
        ptx::fence_proxy_async_smem();
        warp_arrive(&conv_full[rs]);
        warp_arrive(&conv_full[rs + 1]);
        rs += 2;
        if (rs == K::NRAW) rs = 0, rph ^= 1;
      }
    } else if (F32 && !TF && warp >= K::W_CONV0 && warp < K::W_CONV0 + 8) {
      // ===================== fp32 -> (hi, lo) bf16 split =====================
      // a = hi + lo, hi = bf16_rn(a), lo = bf16_rn(a - hi): |a - hi - lo| ≤ 2^-17 |a|.
      // Thread cv owns 4 consecutive MN (or K) elements of rows cv/(BN/4) + RPI·i; the
      // swizzled destination offset is affine in i, so it is precomputed (two parities).
      const int cv = threadIdx.x - K::W_CONV0 * 32;
      constexpr int NT = K::NCONVT;
      constexpr int NIT = kBK * BN / 4 / NT;  // float4 per thread per stage
      static_assert(NIT * NT * 4 == kBK * BN, "converter tiling");
      // destination byte offset of iteration i = off_base[i & 1] + (i >> 1)·dstep (+ i·istep)
      uint32_t off_even, off_odd, istep;
      if (!TRANS) {
        constexpr int F4R = BN / 4;     // float4 per data row
        constexpr int RPI = NT / F4R;   // rows advanced per iteration (8 for BN=128, 16 for BN=64)
        const int rowk0 = cv / F4R, c = (cv % F4R) * 4;
        const int blk = c >> 6, cc = c & 63;
        auto offr = [&](int rk) {
          return (uint32_t)(blk * (kBK * 128) + (rk >> 3) * 1024 + (rk & 7) * 128 + (((cc >> 3) ^ (rk & 7)) << 4) +
                            (cc & 7) * 2);
        };
        off_even = offr(rowk0);
        off_odd = off_even;
        istep = (uint32_t)(RPI / 8) * 1024u;  // RPI is a multiple of 8: (row & 7) is invariant
      } else {
        constexpr int RPI = NT / (kBK / 4);  // vectors advanced per iteration (16)
        const int v0 = cv / (kBK / 4), c = (cv % (kBK / 4)) * 4;
        off_even = (uint32_t)((v0 >> 3) * 1024 + (v0 & 7) * 128 + (((c >> 3) ^ (v0 & 7)) << 4) + (c & 7) * 2);
        off_odd = off_even;
        istep = (uint32_t)(RPI / 8) * 1024u;
      }
      (void)off_odd;
      int rs = 0;
      uint32_t rph = 0;
      const int total = S1i - S0i;
      const Tr tr((args.trace && cv == 0) ? args.trace + blockIdx.x * kTrSlots : nullptr);
      const unsigned long long tstart = tr.now();
      for (int it = 0; it < total; ++it) {
        const unsigned long long t0 = tr.now();
        ptx::mbar_wait(&raw_full[rs], rph);
        tr.add(11, t0);
        uint8_t* stage = smem + K::OFF_RAW + rs * K::RAW_STAGE;
        const float4* rawp = reinterpret_cast<const float4*>(stage) + cv;
        float4 a[NIT];
#pragma unroll
        for (int i = 0; i < NIT; ++i) a[i] = rawp[i * NT];
        ptx::named_bar_sync(2, NT);  // every converter has read its part: the stage can be overwritten
        uint8_t* hbase = stage + off_even;
#pragma unroll
        for (int i = 0; i < (BPS_DBG(2) ? 0 : NIT); ++i) {
          uint32_t h01, h23, l01, l23;
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h01) : "f"(a[i].y), "f"(a[i].x));
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h23) : "f"(a[i].w), "f"(a[i].z));
          const float r0 = a[i].x - __uint_as_float(h01 << 16), r1 = a[i].y - __uint_as_float(h01 & 0xFFFF0000u);
          const float r2 = a[i].z - __uint_as_float(h23 << 16), r3 = a[i].w - __uint_as_float(h23 & 0xFFFF0000u);
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l01) : "f"(r1), "f"(r0));
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l23) : "f"(r3), "f"(r2));
          *reinterpret_cast<uint2*>(hbase + i * istep) = make_uint2(h01, h23);
          *reinterpret_cast<uint2*>(hbase + K::CONV_HALF + i * istep) = make_uint2(l01, l23);
        }
        ptx::fence_proxy_async_smem();
        warp_arrive(&conv_full[rs]);
        if (++rs == K::NRAW) rs = 0, rph ^= 1;
      }
      tr.add(12, tstart);
    }
  }
  if (args.flags && S1 <= S0 && threadIdx.x == 0)  // an empty range has nothing to publish
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(args.flags + blockIdx.x), "l"(args.epoch) : "memory");
  const unsigned long long t_end0 = tr_cta.now();
  ptx::tc_fence_before();
  if (K::CL > 1)
    ptx::cluster_sync();  // no CTA leaves while peers may still copy into it or arrive on its barriers
  else
    __syncthreads();
  tr_cta.add(14, t_end0);
  tr_cta.add(15, t_cta0);
  if (warp == K::W_MMA) {
    ptx::tc_fence_after();
    if (K::PAIR)
      ptx::tmem_dealloc_pair(tmem, K::TMEM_COLS);
    else
      ptx::tmem_dealloc(tmem, K::TMEM_COLS);
  }
  // this CTA's stores are issued: let the combine kernel (programmatic dependent launch) start its
  // prologue; it reads our data only after griddepcontrol.wait (full completion of this grid)
  if (!early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// Straddling outputs of a canon launch: y = scale·((prefix + P_1) + P_2 + …), the prefix parked in Y
// by the owner, the group partials P in stream order from the workspace.  One CTA (256 threads) per
// (output, column tile); outputs that completed inside their owner's range exit at once.  Each
// thread keeps 4 elements and issues the loads of 8 tiles for them at once (32 in flight).
constexpr int kCombineMaxTiles = 1024;  // tile pointers a combine CTA stages (host-checked)

template <bool F32, bool TRANS, int BN, bool TF>
__global__ void __launch_bounds__(256) bps_tc_combine(const __grid_constant__ TcArgs args) {
  constexpr int EPT = 4, TB = 8;  // elements per thread per pass, tiles per load batch
  __shared__ uint32_t fixmap[8];
  __shared__ double red[4];
  __shared__ const float* tiles[kCombineMaxTiles];
  __shared__ int srb[kMaxRanges + 1];
  __shared__ int ntiles;
  const SketchParams& p = args.p;
  const int nk = (int)(p.B_c / kBK);
  CanonGeom geo(args, nk, BN);
  // blockIdx.x = (output o, column tile ct, element part): each CTA takes 1/nsplit of the tile's
  // elements, at most EPT per thread, so that all of them are in flight in one pass
  const unsigned nsplit = gridDim.y;
  const int ct = (int)(blockIdx.x % (unsigned)args.nct), o = (int)(blockIdx.x / (unsigned)args.nct);
  const int part = (int)blockIdx.y;
  const int i = (int)args.i_first + o;  // owner coordinates (first stage o·nk ≥ 0)
  const int F = geo.first_stage(i);
  // the range starts, staged in shared memory: the walk's binary searches on the kernel parameter
  // space (dynamically indexed constant loads, one dependent miss per step) serialised every CTA
  for (int r = (int)threadIdx.x; r <= geo.R; r += (int)blockDim.x) srb[r] = args.rb[r];
  if (threadIdx.x < 8) fixmap[threadIdx.x] = 0u;
  __syncthreads();
  geo.rb = srb;
  if (F + geo.KN <= geo.range_begin(geo.range_of(F) + 1)) {  // finished by its owner
    // with flags, one CTA still orders this grid's completion after the stream kernel's
    if (args.flags && blockIdx.x == 0 && blockIdx.y == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  // flags: the CTA holding output i's slot in range r is (r·nct + ct)·ss + slot / (κ/ss)
  const int css_i = args.ss > 1 ? (int)((uint32_t)(i % (int)p.kappa + (int)p.kappa) % p.kappa) / ((int)p.kappa / args.ss) : 0;
  auto acquire = [&](int r_) {  // spin until CTA (r_, ct) published this launch's epoch
    const unsigned long long* f = args.flags + ((int64_t)r_ * args.nct + ct) * args.ss + css_i;
    unsigned long long v, t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v == args.epoch) break;
      __nanosleep(256);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60000000000ull) __trap();  // 60 s: a lost flag is a bug, fail loudly instead of hanging
    }
  };
  if (threadIdx.x == 0) {
    int nt = 0;
    if (args.flags) acquire(geo.range_of(F));  // the owner's parked prefix
    geo.walk(i, [&](int r_, int j, int ngr) {
      if (args.flags && ngr > 0) acquire(r_);
      for (int g = 0; g < ngr; ++g) tiles[nt++] = geo.tile(r_, ct, j, g);
    });
    ntiles = nt;
  }
  // without flags: programmatic dependent launch — everything above ran while bps_tc_kernel was
  // finishing; its prefixes and partial tiles are visible after this wait
  if (!args.flags) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  const int nt = ntiles, NT = (int)blockDim.x, Br = geo.Br;
  const int el0 = (int)((int64_t)Br * BN * part / nsplit), nel = (int)((int64_t)Br * BN * (part + 1) / nsplit);
  const int64_t col0 = (int64_t)ct * BN;
  const int64_t yr0 = args.range_mode ? (int64_t)(i - args.pos_begin) * Br : (int64_t)affine_pow(p, (uint64_t)i, 0u) * Br;
  float* const Yb = TRANS ? args.Y + col0 * args.ldy + yr0 : args.Y + yr0 * args.ldy + col0;
  bool bad = false;
  for (int e0 = el0 + (int)threadIdx.x; e0 < nel; e0 += EPT * NT) {
    int off[EPT];      // element offset inside a tile (TF: row-major [B_r][BN]; else [BN][B_r])
    int64_t yo[EPT];   // element offset from Yb, or -1
    float acc[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = e0 + k * NT;
      const int r = TF ? e / BN : e % Br, c = TF ? e % BN : e / Br;
      const bool ok = e < nel && col0 + c < args.n;
      off[k] = TF ? r * BN + c : c * Br + r;
      yo[k] = ok ? (TRANS ? (int64_t)c * args.ldy + r : (int64_t)r * args.ldy + c) : -1;
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) acc[k] = yo[k] >= 0 ? __ldcg(Yb + yo[k]) : 0.f;
    // canonical order: acc = ((prefix + P_1) + P_2) + …; the loads of TB tiles are issued together
    for (int t0 = 0; t0 < nt; t0 += TB) {
      float v[TB * EPT];
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        const float* tp = tiles[min(t0 + b, nt - 1)];
#pragma unroll
        for (int k = 0; k < EPT; ++k) v[b * EPT + k] = (t0 + b < nt) ? __ldcg(tp + off[k]) : 0.f;
      }
#pragma unroll
      for (int b = 0; b < TB; ++b)
#pragma unroll
        for (int k = 0; k < EPT; ++k)
          if (t0 + b < nt) acc[k] += v[b * EPT + k];
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (yo[k] >= 0) {
        const float v = acc[k] * p.scale;
        Yb[yo[k]] = v;
        if (!TRANS && (args.npeer || args.mc)) {
          const int e = e0 + k * NT;
          bcast1(args, yr0 + (TF ? e / BN : e % Br), col0 + (TF ? e % BN : e / Br), v);
        }
        const uint32_t bits = __float_as_uint(v), ex = (bits >> 23) & 0xFFu;
        if (ex == 0xFFu || (ex < 27u && (bits & 0x7FFFFFFFu) != 0u)) {  // see needs_exact
          bad = true;
          const int c = TF ? off[k] % BN : off[k] / Br;
          atomicOr(&fixmap[c >> 5], 1u << (c & 31));
        }
      }
  }
  // with flags this grid may overtake the stream kernel's teardown: complete only after it, so that
  // work queued after this apply observes both grids finished
  if (args.flags) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!__syncthreads_or(bad) || threadIdx.x >= 128) return;  // warps 0-3 recompute (exact_elem: 128 threads)
  for (int w = 0; w < BN / 32; ++w) {
    uint32_t bits = fixmap[w];
    while (bits) {
      const int c = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t col = col0 + c;
      for (int r = 0; r < Br; ++r) {
        const float v = exact_elem<F32, TRANS>(args, i, (uint32_t)r, col, (int)threadIdx.x, red);
        if (threadIdx.x == 0) {
          if (!TRANS) {
            args.Y[(yr0 + r) * args.ldy + col] = v;
            if (args.npeer || args.mc) bcast1(args, yr0 + r, col, v);
          } else {
            args.Y[col * args.ldy + yr0 + r] = v;
          }
        }
      }
    }
  }
}

}  // namespace

// A value no earlier launch in this process wrote into any workspace flag, and that stale or
// uninitialised workspace contents match only with probability 2^-64 (random 32-bit salt per process).
inline unsigned long long next_epoch() {
  static const unsigned long long salt = []() {
    std::random_device rd;
    return ((unsigned long long)rd() << 32) ^
           ((unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count() << 16);
  }();
  static std::atomic<unsigned long long> counter{1};
  return (salt & 0xFFFFFFFF00000000ull) | (counter.fetch_add(1) & 0xFFFFFFFFull);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
void* encode_tiled_entry();  // bps_tc.cu (thread-safe lazy driver entry point)

template <bool F32, bool TRANS, int NMT, int BN_, int CS, bool TF, bool RL, int SS>
int launch_impl(const SketchParams& p, const void* A, int64_t lda, int64_t n, float* Y, int64_t ldy,
                const Placement& pl, const HostPlan& hp, cudaStream_t st) {
  using K = Cfg<F32, TRANS, NMT, BN_, CS, TF, RL, SS>;
  constexpr int BN = K::BN;
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(encode_tiled_entry());
  if (!enc) return fail(BPS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  TcArgs a{};
  a.p = p;
  a.n = n;
  a.Y = Y;
  a.ldy = ldy;
  a.A = A;
  a.lda = lda;
  a.range_mode = pl.range_mode;
  a.pos_begin = pl.pos_begin;
  a.pos_end = pl.pos_begin + pl.n_out;
  a.i_first = pl.range_mode ? pl.pos_begin : 0;
  a.n_out = pl.n_out;
  int64_t in_rows;
  if (pl.range_mode) {
    a.stream_begin = pl.pos_begin + 1;
    a.stream_len = pl.n_out + p.kappa - 1;
    in_rows = a.stream_len * (int64_t)p.B_c;
  } else {
    a.stream_begin = 1;
    a.stream_len = p.M;
    in_rows = (int64_t)p.M * p.B_c;
  }
  const int nk = (int)(p.B_c / kBK);
  a.G = hp.G;
  a.dbg = 0;
  a.trace = nullptr;
  a.kgroup = 1;
  if (const char* e = getenv("BPS_TC_KGROUP")) a.kgroup = atoi(e);  // tuning knob (transposed layout)
  if (a.kgroup < 1) a.kgroup = 1;
  if (a.kgroup > K::NRAW) a.kgroup = K::NRAW;  // a group must fit the ring (else the producer waits on itself)
  if (!TRANS) {
    // row-major: grouping only for the narrow bf16 tile (BPS_TC_KGROUP=2/4: 128/256-row boxes;
    // measured no gain on smalln, off by default); a box group never straddles an accumulation group
    if (F32 || BN != 64 || hp.G % a.kgroup || K::NRAW % a.kgroup || a.kgroup > 4 || (a.kgroup & (a.kgroup - 1)))
      a.kgroup = 1;
  }
  // narrow bf16 tile: stage pairs share one data barrier (a 128-row TMA box) and one band
  // handshake, halving the per-stage synchronisation that bounds it (profiles/r02_narrow_n.md);
  // pairs never straddle an accumulation group, block or range (G, nk even; ranges start at groups)
  a.kstep = 1;
  if (!F32 && !TRANS && BN == 64 && CS == 1 && SS == 1 && NMT == 1 && K::NBAND % 2 == 0 && K::NRAW % 2 == 0 &&
      hp.G % 2 == 0 && nk % 2 == 0 && getenv("BPS_TC_KSTEP2")) {  // opt-in: measured slower (n = 64: 2895 vs 3229 GB/s)
    a.kstep = 2;
    a.kgroup = 2;
  }
  a.nohoist = getenv("BPS_TC_NOHOIST") ? 1 : 0;
  // BPS_TC_BANDMN=1 (experiment): MN-major one-hot band pieces for C = 8 row-partitioned sketches —
  // parity-green, measured slower (smalln 1194 vs 1379, LS 5474 vs 5910, grad 5897 vs 6115 GB/s)
  a.band_mn = (p.mode == 0 && p.C == 8u && p.B_r % 8 == 0 && getenv("BPS_TC_BANDMN")) ? 1 : 0;
  a.ab = getenv("BPS_TC_AB") ? atoi(getenv("BPS_TC_AB")) : 0;
  a.mma_hint = getenv("BPS_TC_MMA_HINT") ? (uint32_t)atoi(getenv("BPS_TC_MMA_HINT")) : 0u;  // A/B knob
  a.sleep_ns = getenv("BPS_TC_SLEEP") ? (uint32_t)atoi(getenv("BPS_TC_SLEEP")) : 20u;  // A/B knob
  a.tbox = BN;
  if (const char* e = getenv("BPS_TC_TBOX")) a.tbox = atoi(e);  // tuning knob (transposed layout)
  if (a.tbox < 8 || BN % a.tbox || a.tbox % 8 || a.kgroup == 1) a.tbox = BN;
#ifdef BPS_TC_INSTRUMENT
  {
    const char* e = getenv("BPS_TC_DEBUG");
    a.dbg = e ? atoi(e) : 0;
  }
#endif
  const int64_t n_ct = (n + BN - 1) / BN;
  int dev = 0;
  cudaGetDevice(&dev);
  int slots = hp.sms * K::MINB;
  auto kern = bps_tc_kernel<F32, TRANS, NMT, BN_, CS, TF, RL, SS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
  if (e == cudaSuccess && K::MINB > 1)  // room for MINB CTAs per SM
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  if (K::CL > 1) {  // clusters must fit inside a GPC: not every SM can host one
    static std::atomic<int> cached_slots[64];
    int s = cached_slots[dev & 63].load(std::memory_order_relaxed);
    if (!s) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(K::CL * 64);
      cfg.blockDim = dim3(K::NTHREADS);
      cfg.dynamicSmemBytes = K::SMEM;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = K::CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters <= 0) clusters = hp.sms / K::CL;
      s = clusters * K::CL;
      cached_slots[dev & 63].store(s, std::memory_order_relaxed);
    }
    slots = s;
  }
  a.canon = hp.canon;
  slots /= SS;  // an SS cluster works on one (range, column tile)
  int64_t R = n_ct >= slots ? 1 : slots / n_ct;
  if (a.canon) {
    const int64_t NGt = a.stream_len * nk / hp.G;
    if (R > NGt) R = NGt;
  } else {
    // halo ranges: each re-reads κ-1 blocks; keep that under ~25 % of its own blocks
    if (R > pl.n_out) R = pl.n_out;
    if (p.kappa > 1) {
      const int64_t cap = std::max<int64_t>(1, pl.n_out / (4 * ((int64_t)p.kappa - 1)));
      if (R > cap) R = cap;
    }
  }
  if (const char* e = getenv("BPS_TC_R")) {  // experiment knob: ranges per column tile
    const int64_t r = atoll(e);
    if (r >= 1 && r <= R) R = r;
  }
  if (a.canon && R > kMaxRanges) R = kMaxRanges;
  a.R = (int)R;
  a.nct = (int)n_ct;
  if (pl.bc) {  // fused output broadcast (row-major orbit ranges; the host rejects the transposed layout)
    for (int j = 0; j < pl.bc->npeer; ++j) a.peer[j] = pl.bc->peer[j];
    a.npeer = pl.bc->npeer;
    a.mc = pl.bc->mc;
    a.ldp = pl.bc->ld;
    a.prow0 = pl.bc->row0;
  }
  if (a.canon) {
    const int64_t NGt = a.stream_len * nk / hp.G;
    for (int64_t r = 0; r <= R; ++r) a.rb[r] = (int)(hp.G * (NGt * r / R));
  }
  const int64_t grid = n_ct * R * SS;
  if (grid > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "grid too large");

  if (a.canon) {
    a.tpc = tiles_per_cta(p, hp.G);
    const size_t tiles_bytes = (size_t)(grid / SS) * a.tpc * p.B_r * BN * 4;  // tiles indexed by (range, column tile)
    const size_t need = tiles_bytes + (size_t)grid * 8;                      // + one flag per CTA
    if (!hp.ws || hp.ws_bytes < need) return fail(BPS_ERR_INVALID_ARG, "workspace too small for the tc plan");
    a.W = reinterpret_cast<float*>(hp.ws);
    a.ss = SS;
    if (a.ab & 256) {  // BPS_TC_AB & 256: per-CTA publication flags instead of the whole-grid wait
      // (measured equal on LS/grad/smalln: the combine's cost is its own latency after the last
      // range, not the wait for the grid — profiles/r02_narrow_n.md; kept as an experiment)
      a.flags = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(hp.ws) + tiles_bytes);
      a.epoch = next_epoch();
    }
  }

  // TMA descriptor for the data operand
  CUtensorMap tm;
  const CUtensorMapDataType tdt = F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2], strides[1];
  cuuint32_t box[2], estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = (F32 || RL) ? CU_TENSOR_MAP_SWIZZLE_NONE
                                             : (K::SW64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
  strides[0] = (cuuint64_t)lda * K::ESZ;
  if (!TRANS) {
    dims[0] = (cuuint64_t)n;
    dims[1] = (cuuint64_t)in_rows;
    box[0] = F32 ? BN : (BN < 64 ? BN : 64);
    box[1] = (SS > 1 && !K::PAIR) ? kBK / SS : kBK * a.kgroup;  // SS: each CTA of the cluster loads 1/SS of the rows
  } else {
    dims[0] = (cuuint64_t)in_rows;  // coordinates (d)
    dims[1] = (cuuint64_t)n;        // vectors
    box[0] = RL ? 2 * kBK : kBK;
    box[1] = RL ? BN : a.tbox;
  }
  CUresult cr = enc(&tm, tdt, 2, const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(BPS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));

  auto launch = [&]() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(K::NTHREADS);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = K::CL;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, tm, a);
  };
#ifdef BPS_TC_INSTRUMENT
  if (a.dbg & 8) {  // debug trace: per-CTA cycle counters, printed to stderr (synchronises)
    cudaMalloc(&a.trace, (size_t)grid * kTrSlots * 8);
    cudaMemsetAsync(a.trace, 0, (size_t)grid * kTrSlots * 8, st);
  }
  e = launch();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (a.trace) {
    std::vector<unsigned long long> h((size_t)grid * kTrSlots);
    cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[22] = {"tma_wait_empty", "tma_total", "mma_wait_accfree", "mma_wait_data", "mma_wait_band",
                             "mma_total", "band_wait_empty", "band_table", "band_total", "epi_wait_accfull",
                             "epi_total", "tail_bulk_wait", "tail_finishes", "epi_tail", "end_barrier", "cta_total",
                             "tail_park", "tail_arrive", "tail_prefix_load", "tail_fold", "tail_store", "tail_fix"};
    for (int k = 0; k < 22; ++k) {
      double sum = 0, mx = 0;
      for (int64_t c = 0; c < grid; ++c) {
        sum += (double)h[c * kTrSlots + k];
        mx = std::max(mx, (double)h[c * kTrSlots + k]);
      }
      fprintf(stderr, "[bps trace] %-18s mean %12.0f  max %12.0f cycles\n", names[k], sum / grid, mx);
    }
    cudaFree(a.trace);
  }
#else
  cudaEvent_t tev[2] = {nullptr, nullptr};
  const bool timed = timing_begin(st, tev);
  e = (a.ab & 32) ? cudaSuccess : launch();  // ab & 32: combine only (timing experiment)
  if (timed) timing_end(st, tev);
  g_launches.fetch_add(1, std::memory_order_relaxed);
#endif
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("bps_tc_kernel launch: ") + cudaGetErrorString(e));
  // straddling outputs exist when the stream has several ranges, or (full mode) windows wrap
  if (a.canon && (R > 1 || (!pl.range_mode && p.kappa > 1))) {
    const int64_t cgrid = n_ct * pl.n_out;
    if (cgrid > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "combine grid too large");
    cudaLaunchConfig_t cfg = {};
    const int cthreads = (a.ab & 8) ? 128 : 256;
    // element parts per (output, column tile): all of a tile's elements in flight at once, unless that
    // takes more than one wave of co-resident CTAs (5 per SM at 48 registers): every CTA walks its
    // output's segment list serially before loading, so extra waves cost a walk each (ncu: 2.8 waves
    // at 4 parts on LS, a third of the samples waiting on that walk)
    int nsplit = (int)std::max<int64_t>(1, ((int64_t)p.B_r * BN + cthreads * 4 - 1) / (cthreads * 4));
    const int64_t resident = (int64_t)hp.sms * ((a.ab & 8) ? 10 : 5);
    if (!(a.ab & 64)) nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit, resident / std::max<int64_t>(1, cgrid)));
    cfg.gridDim = dim3((unsigned)cgrid, (unsigned)std::min(nsplit, 65535));
    cfg.blockDim = dim3(cthreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (a.ab & 16) ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t cev[2] = {nullptr, nullptr};
    const bool ctimed = timing_begin(st, cev);
    e = cudaLaunchKernelEx(&cfg, bps_tc_combine<F32, TRANS, BN, TF>, a);
    if (ctimed) timing_end(st, cev, true);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("bps_tc_combine launch: ") + cudaGetErrorString(e));
  }
  return BPS_OK;
}

}  // namespace tcx
}  // namespace bps

#define BPS_TC_DEFINE(F, T, NM, B, C, TF_, RL_, SS_)                                                     \
  template int bps::tcx::launch_impl<F, T, NM, B, C, TF_, RL_, SS_>(                                     \
      const bps::SketchParams&, const void*, int64_t, int64_t, float*, int64_t, const bps::Placement&,   \
      const bps::tcx::HostPlan&, cudaStream_t);

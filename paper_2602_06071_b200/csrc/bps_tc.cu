// bps_tc.cu — tcgen05 tensor-core kernel for Y = S·A (the "tc" variant). DESIGN.md §6.
//
// Idea: the block sparsity of S is a union of κ permutations that are powers of one
// affine map f.  Ordering input and output blocks along the orbit
// g_i = f^i(0) turns the wiring into a sliding window: output i reads input positions
// i+1..i+κ.  A CTA streams a contiguous range of input positions once (no κ-fold
// re-read), and for each input block p it builds the dense ±1
// "band" B_p = [Φ_{g_{p-1},g_p}; …; Φ_{g_{p-κ},g_p}] (κ·B_r × B_c, bf16 exact, rows
// rotated so output i always lands in slot i mod κ) from the counter hash (R2) and
// feeds it to tcgen05.mma as the K-major A operand; the data tile (TMA, SW128) is
// the B operand (MN-major for row-major A, K-major for the transposed layout).
// D (TMEM, fp32) rows = band rows, columns = data columns.  Accumulation: the tensor
// core's fp32 accumulate is not round-to-nearest (measured: error grows ∝ #MMAs ×
// |acc|), so D is fresh for every group of G·64 input rows (two buffers D0/D1
// alternate) and the epilogue warps fold each group into a TMEM running sum S with
// IEEE round-to-nearest fp32 adds on the CUDA cores.  The κ slots of S hold the κ
// outputs in flight; after the last group of input block p the slot of output p−κ is
// complete: it is scaled by 1/√(κs), stored, and zeroed.
//   fp32 input: the converter warps split a = hi + lo (two bf16) and the MMA runs
//   twice (Φ is ±1, exact in bf16) — tf32 would miss the 1e-5 tolerance.
// Outputs whose κ inputs straddle two CTAs' ranges are combined with red.global.add
// into a zeroed Y; every such output has exactly two addends, so the result is still
// bitwise deterministic (a+b == b+a in IEEE arithmetic).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "bps_internal.h"
#include "bps_ptx.cuh"

namespace bps {
namespace {

constexpr int kBK = 64;                   // K rows per pipeline stage (one 128-byte swizzle row of bf16)
constexpr int kBandTile = 128 * kBK * 2;  // one M-tile (128 band rows) of a band stage, bytes
constexpr int kMaxGroup = 128;            // K-chunks per accumulation group (precision)

// Warp roles (the issue arbiter favours high warp ids, so the latency-critical single-thread
// roles take the last two warps): 0-3 epilogue (TMEM lane quarters 0-3) | 4-11 band
// generator | 12-19 fp32 hi/lo converter (fp32 only) | NWARPS-2 TMA producer |
// NWARPS-1 MMA issuer (+TMEM alloc).
template <bool F32, bool TRANS, int NMT, int BN_>
struct Cfg {
  static constexpr int BN = BN_;  // data columns per CTA; TMEM = D (NMT·BN) + S (NMT·BN)
  static constexpr int ESZ = F32 ? 4 : 2;
  static constexpr int RAW_STAGE = kBK * BN * ESZ;
  static constexpr int CONV_HALF = kBK * BN * 2;  // fp32: hi and lo bf16 tiles overwrite the raw stage in place
  static constexpr int BAND_STAGE = NMT * kBandTile;
  static constexpr int NBAND = (NMT == 1 && !F32) ? 3 : 2;
  static constexpr int BUDGET = 210 * 1024;
  static constexpr int NRAW_FIT = (BUDGET - NBAND * BAND_STAGE) / RAW_STAGE;
  static constexpr int NRAW = NRAW_FIT > 8 ? 8 : NRAW_FIT;
  static constexpr int OFF_RAW = 0;
  static constexpr int OFF_BAND = OFF_RAW + NRAW * RAW_STAGE;
  static constexpr int OFF_CKEY = OFF_BAND + NBAND * BAND_STAGE;  // [2][256] u64 per-block combo keys
  static constexpr int OFF_CROW = OFF_CKEY + 2 * 256 * 8;  // [64] u32 band-row base σ·B_r + j·C of chunk c
  static constexpr int OFF_BAR = OFF_CROW + 64 * 4;
  // raw full/empty, conv full (fp32: per raw stage), band full/empty, acc full, acc free
  static constexpr int NBARS = 3 * NRAW + 2 * NBAND + 2;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBARS * 8;
  static constexpr int SMEM = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  static constexpr int NWARPS = F32 ? 22 : 14;
  static constexpr int NCONVT = 256;  // fp32 converter threads (warps 12-19)
  static constexpr int W_TMA = NWARPS - 2, W_MMA = NWARPS - 1;
  static constexpr int NTHREADS = NWARPS * 32;
  static constexpr int NBANDT = 256;  // band generator threads
  // fp32: the hi and lo tiles are adjacent along N in smem, so ONE MMA with N = 2·BN reads
  // the band once for both (D columns [0,BN) = band·hi, [BN,2BN) = band·lo).
  static constexpr int DN = F32 ? 2 * BN : BN;  // D columns per M-tile
  static constexpr uint32_t TMEM_COLS = (NMT * (DN + BN) <= 256) ? 256 : 512;
  static constexpr uint32_t IDESC = ptx::idesc_bf16(128, DN, !TRANS);
  static_assert(NRAW >= 2, "smem: raw ring");
  static_assert(NMT * (DN + BN) <= 512 && DN <= 256, "TMEM / MMA N");
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
  static_assert(SMEM <= 227 * 1024, "smem");
};

struct TcArgs {
  SketchParams p;
  int64_t n;         // columns of A (row-major) or vectors (transposed)
  float* Y;
  int64_t ldy;
  int range_mode;
  int64_t pos_begin, pos_end;  // owned outputs (range mode)
  int64_t stream_begin;        // first input position of the launch window
  int64_t stream_len;          // number of input positions in the window
  int R;                       // ranges per column tile
  int balanced;                // 1: stage-granular equal ranges, split outputs parity-routed to Y / Y2
  float* Y2;                   // balanced mode: second accumulation buffer (odd ranges), same shape as Y
  int64_t ldy2;
  int G;                       // K-chunks per accumulation group (divides B_c/64)
  int dbg;  // experiment switches (env BPS_TC_DEBUG; 0 in production): 1 no band, 2 no convert, 4 no MMA,
            // 8 cycle trace, 16 no band proxy fence, 32 band without hashing
  unsigned long long* trace;   // dbg & 8: per-CTA cycle counters (16 per CTA), else nullptr
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

template <bool F32, bool TRANS, int NMT, int BN_>
__global__ void __launch_bounds__(Cfg<F32, TRANS, NMT, BN_>::NTHREADS, 1)
    bps_tc_kernel(const __grid_constant__ CUtensorMap tmap, const TcArgs args) {
  using K = Cfg<F32, TRANS, NMT, BN_>;
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
  uint64_t* acc_free = acc_full + 1;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + K::OFF_TMEMPTR);
  uint64_t* ckey = reinterpret_cast<uint64_t*>(smem + K::OFF_CKEY);
  uint32_t* crow = reinterpret_cast<uint32_t*>(smem + K::OFF_CROW);

  const SketchParams& p = args.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kappa = p.kappa;
  const int nk = (int)(p.B_c / kBK);
  const int G = args.G;

  // ---- this CTA's column tile and input-position range
  const int ct = blockIdx.x / args.R, rr = blockIdx.x % args.R;
  const int64_t col0 = (int64_t)ct * BN;
  // stage s ∈ [S0, S1) of the window = K-chunk s % nk of input position sb + s / nk
  const int64_t sb = args.stream_begin;
  int64_t S0, S1;
  if (args.balanced) {
    const int64_t Ts = args.stream_len * nk;
    S0 = Ts * rr / args.R;
    S1 = Ts * (rr + 1) / args.R;
  } else {
    const int64_t Lq = args.stream_len / args.R, Lrem = args.stream_len % args.R;
    S0 = (rr * Lq + (rr < Lrem ? rr : Lrem)) * nk;
    S1 = S0 + (Lq + (rr < Lrem ? 1 : 0)) * nk;
  }
  float* const Ysplit = (args.balanced && (rr & 1)) ? args.Y2 : args.Y;  // destination of split outputs
  const int64_t ldsplit = (args.balanced && (rr & 1)) ? args.ldy2 : args.ldy;

  if (threadIdx.x == 0) {
    for (int i = 0; i < K::NRAW; ++i) {
      ptx::mbar_init(&raw_full[i], 1);
      ptx::mbar_init(&raw_empty[i], 1);
      ptx::mbar_init(&conv_full[i], K::NCONVT);
    }
    for (int i = 0; i < K::NBAND; ++i) {
      ptx::mbar_init(&band_full[i], K::NBANDT);
      ptx::mbar_init(&band_empty[i], 1);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(acc_free, 128);
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tmap);
  }
  if (warp == K::W_MMA) ptx::tmem_alloc(tmem_ptr, K::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;               // D: per-group tensor-core accumulator
  const uint32_t tmem_S = tmem + NMT * K::DN;    // S: fp32 running sums (RN adds on CUDA cores)

  if (S1 > S0) {
    if (warp == K::W_TMA) {
      // ===================== TMA producer =====================
      if (lane == 0) {
        const Tr tr(args.trace ? args.trace + blockIdx.x * 16 : nullptr);
        const unsigned long long tstart = tr.now();
        const uint64_t pol = ptx::policy_evict_first();
        int64_t q = sb + S0 / nk;
        int kc = (int)(S0 % nk);
        uint32_t gq = affine_pow(p, (uint64_t)mod_pos(q, p.M), 0u);
        int s = 0;
        uint32_t ph = 0;
        for (int64_t st = S0; st < S1; ++st) {
          {
            const int64_t row0 = args.range_mode ? (q - (args.pos_begin + 1)) * (int64_t)p.B_c : (int64_t)gq * p.B_c;
            const unsigned long long t0 = tr.now();
            ptx::mbar_wait_sleep(&raw_empty[s], ph ^ 1, 20);
            tr.add(0, t0);
            ptx::mbar_arrive_expect_tx(&raw_full[s], K::RAW_STAGE);
            uint8_t* dst = smem + K::OFF_RAW + s * K::RAW_STAGE;
            const int32_t r = (int32_t)(row0 + kc * kBK);
            if (!TRANS) {
              if (F32) {
                ptx::tma_load_2d(dst, &tmap, &raw_full[s], (int32_t)col0, r, pol);
              } else {
#pragma unroll
                for (int b = 0; b < BN / 64; ++b)
                  ptx::tma_load_2d(dst + b * (kBK * 128), &tmap, &raw_full[s], (int32_t)(col0 + 64 * b), r, pol);
              }
            } else {
              ptx::tma_load_2d(dst, &tmap, &raw_full[s], r, (int32_t)col0, pol);
            }
            if (++s == K::NRAW) s = 0, ph ^= 1;
          }
          if (++kc == nk) kc = 0, ++q, gq = affine_step(p, gq);
        }
        tr.add(1, tstart);
      }
    } else if (warp == K::W_MMA) {
      // ===================== MMA issuer =====================
      if (lane == 0) {
        const Tr tr(args.trace ? args.trace + blockIdx.x * 16 : nullptr);
        const unsigned long long tstart = tr.now();
        int ds = 0, bs = 0;
        uint32_t dph = 0, bph = 0, fph = 0;
        uint64_t* dfull = F32 ? conv_full : raw_full;
        uint64_t* dempty = raw_empty;
        constexpr int NDS = K::NRAW;
        const uint32_t data_base = ptx::smem_u32(smem + K::OFF_RAW);
        constexpr int DSTAGE = K::RAW_STAGE;
        const uint32_t band_base = ptx::smem_u32(smem + K::OFF_BAND);
        bool first_group = true;
        int kc = (int)(S0 % nk);
        int gi = kc % G;  // position inside the accumulation group (groups restart at block starts)
        for (int64_t st = S0; st < S1; ++st) {
          {
            const bool gstart = st == S0 || gi == 0;
            const bool gend = st == S1 - 1 || kc == nk - 1 || gi == G - 1;
            if (gstart && !first_group) {  // D must have been folded into S
              const unsigned long long t0 = tr.now();
              ptx::mbar_wait(acc_free, fph);
              tr.add(2, t0);
              fph ^= 1;
              ptx::tc_fence_after();
            }
            unsigned long long t0 = tr.now();
            ptx::mbar_wait(&dfull[ds], dph);
            tr.add(3, t0);
            t0 = tr.now();
            ptx::mbar_wait(&band_full[bs], bph);
            tr.add(4, t0);
            ptx::tc_fence_after();
            const uint32_t dbase = data_base + ds * DSTAGE;
            const uint32_t bbase = band_base + bs * K::BAND_STAGE;
#pragma unroll
            for (int ks = 0; ks < kBK / 16; ++ks) {
#pragma unroll
              for (int m = 0; m < NMT; ++m) {
                const uint64_t adesc = ptx::smem_desc_sw128(bbase + m * kBandTile + ks * 32, 0, 1024);
                const uint64_t bdesc = TRANS ? ptx::smem_desc_sw128(dbase + ks * 32, 0, 1024)
                                             : ptx::smem_desc_sw128(dbase + ks * 16 * 128, kBK * 128, 1024);
                const uint32_t acc = (gstart && ks == 0) ? 0u : 1u;  // fresh per group
                if (!BPS_DBG(4)) ptx::mma_bf16_ss(tmem + m * K::DN, adesc, bdesc, K::IDESC, acc);
              }
            }
            ptx::mma_commit(&dempty[ds]);
            ptx::mma_commit(&band_empty[bs]);
            if (++ds == NDS) ds = 0, dph ^= 1;
            if (++bs == K::NBAND) bs = 0, bph ^= 1;
            if (gend) {
              ptx::mma_commit(acc_full);
              first_group = false;
            }
          }
          if (++kc == nk) kc = 0, gi = 0;
          else gi = (gi + 1 == G) ? 0 : gi + 1;
        }
        tr.add(5, tstart);
      }
    } else if (warp < 4) {
      // ============ epilogue: S += D (fp32 RN) per group; emit the slot that completes ============
      const int qtr = warp & 3;
      const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
      {  // S = 0
        uint32_t z[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) z[t] = 0u;
        for (int c = 0; c < NMT * BN; c += 16) ptx::tmem_st16(tmem_S + lane_off + c, z);
        ptx::tmem_wait_st();
      }
      auto emit = [&](int64_t i, uint32_t rho, const float* vals, int c0) {
        // vals: 16 sums of band row rho (slot of output i), columns col0+c0 .. +15
        const bool owned = args.range_mode ? (i >= args.pos_begin && i < args.pos_end) : true;
        if (!owned) return;
        const uint32_t lo = mod_pos(i, kappa) * p.B_r;
        // complete iff every stage of input blocks i+1 .. i+κ lies in this CTA's range
        const bool complete = (i + 1 - sb) * nk >= S0 && (i + (int64_t)kappa + 1 - sb) * nk <= S1;
        const int64_t row = (args.range_mode ? (i - args.pos_begin) * (int64_t)p.B_r
                                             : (int64_t)affine_pow(p, (uint64_t)mod_pos(i, p.M), 0u) * p.B_r) +
                            (int64_t)(rho - lo);
        const int64_t cbase = col0 + c0;
        float* const Yd = complete ? args.Y : Ysplit;
        const int64_t ldd = complete ? args.ldy : ldsplit;
        if (!TRANS) {
          float* y = Yd + row * ldd + cbase;
#pragma unroll
          for (int t = 0; t < 16; t += 4) {
            const float a0 = vals[t] * p.scale, a1 = vals[t + 1] * p.scale;
            const float a2 = vals[t + 2] * p.scale, a3 = vals[t + 3] * p.scale;
            if (cbase + t + 3 < args.n) {
              if (complete) *reinterpret_cast<float4*>(y + t) = make_float4(a0, a1, a2, a3);
              else ptx::red_add_v4(y + t, a0, a1, a2, a3);
            } else {
              const float a[4] = {a0, a1, a2, a3};
              for (int e = 0; e < 4; ++e)
                if (cbase + t + e < args.n) {
                  if (complete) y[t + e] = a[e];
                  else ptx::red_add(y + t + e, a[e]);
                }
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            if (cbase + t < args.n) {
              float* y = Yd + (cbase + t) * ldd + row;
              const float a = vals[t] * p.scale;
              if (complete) *y = a;
              else ptx::red_add(y, a);
            }
          }
        }
      };
      uint32_t aph = 0;
      const Tr tr((args.trace && threadIdx.x == 0) ? args.trace + blockIdx.x * 16 : nullptr);
      const unsigned long long tstart = tr.now();
      int kc = (int)(S0 % nk);
      int gi = kc % G;
      int64_t q = sb + S0 / nk;
      for (int64_t st = S0; st < S1;
           ++st, q += (kc + 1 == nk), gi = (kc + 1 == nk || gi + 1 == G) ? 0 : gi + 1, kc = (kc + 1 == nk) ? 0 : kc + 1) {
        const bool gend = st == S1 - 1 || kc == nk - 1 || gi == G - 1;
        if (!gend) continue;
        const int64_t i = q - (int64_t)kappa;  // output completed by input block q (if q ends here)
        const uint32_t lo = mod_pos(i, kappa) * p.B_r, hi = lo + p.B_r;
        {
          const unsigned long long t0 = tr.now();
          ptx::mbar_wait_sleep(acc_full, aph, 32);
          tr.add(9, t0);
          aph ^= 1;
          ptx::tc_fence_after();
          const bool last = kc == nk - 1;  // input block q fully streamed: output q-κ is done here
#pragma unroll 1
          for (int m = 0; m < NMT; ++m) {
            const uint32_t rho = m * 128 + qtr * 32 + lane;
            const bool in_slot = last && rho >= lo && rho < hi;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 16) {
              uint32_t d[16], sv[16];
              ptx::tmem_ld16(tmem + lane_off + m * K::DN + c0, d);
              ptx::tmem_ld16(tmem_S + lane_off + m * BN + c0, sv);
              float tot[16];
              if (F32) {  // hi and lo partial products
                uint32_t dl[16];
                ptx::tmem_ld16(tmem + lane_off + m * K::DN + BN + c0, dl);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  tot[t] = __uint_as_float(sv[t]) + (__uint_as_float(d[t]) + __uint_as_float(dl[t]));
              } else {
                ptx::tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 16; ++t) tot[t] = __uint_as_float(sv[t]) + __uint_as_float(d[t]);
              }
              if (in_slot) emit(i, rho, tot, c0);
#pragma unroll
              for (int t = 0; t < 16; ++t) sv[t] = in_slot ? 0u : __float_as_uint(tot[t]);
              ptx::tmem_st16(tmem_S + lane_off + m * BN + c0, sv);
            }
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(acc_free);
        }
      }
      tr.add(10, tstart);
      // range end: outputs fed by the last input block that are still open hold partial sums in S
      const int64_t q_last = sb + (S1 - 1) / nk;
      const bool full_end = (S1 - 1) % nk == nk - 1;
      for (int64_t i = q_last - (int64_t)kappa + (full_end ? 1 : 0); i <= q_last - 1; ++i) {
        const uint32_t lo = mod_pos(i, kappa) * p.B_r, hi = lo + p.B_r;
#pragma unroll 1
        for (int m = 0; m < NMT; ++m) {
          const uint32_t base = m * 128 + qtr * 32;
          if (base + 32 <= lo || base >= hi) continue;  // warp-uniform
          const uint32_t rho = base + lane;
          const bool in_slot = rho >= lo && rho < hi;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t sv[16];
            ptx::tmem_ld16(tmem_S + lane_off + m * BN + c0, sv);
            ptx::tmem_wait_ld();
            float tot[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) tot[t] = __uint_as_float(sv[t]);
            if (in_slot) emit(i, rho, tot, c0);
          }
        }
      }
    } else if (warp >= 4 && warp < 12) {
      // ===================== band generator =====================
      // Thread (u, cg) writes column u of every band stage for the row chunks c = cg + 4t,
      // c = σ·s + j (slot σ, chunk j).  A chunk's rows [σB_r + jC, +C) are owned by one thread
      // per column, so each thread can clear the single entry it wrote into this buffer
      // NBAND stages ago and write the new one without any barrier (no zero-fill pass).
      const int bt = threadIdx.x - 128;
      const uint32_t u = (uint32_t)bt & (kBK - 1);
      const uint32_t cg = (uint32_t)bt >> 6;  // 0..3
      const uint32_t ncombo = kappa * p.s;
      const uint32_t T = ncombo > cg ? (ncombo - cg + 3) / 4 : 0;  // chunks of this thread (≤ 16)
      const uint32_t band_u32 = ptx::smem_u32(smem + K::OFF_BAND);
      const uint32_t ucol = u >> 3, ulo = (u & 7) * 2;
      auto entry = [&](uint32_t sbase, uint32_t rho) {
        const uint32_t r7 = rho & 127;
        return sbase + (rho >> 7) * kBandTile + (r7 >> 3) * 1024 + (r7 & 7) * 128 + ((ucol ^ (r7 & 7)) << 4) + ulo;
      };
      {  // band buffers start zeroed; chunk row bases (fixed for the whole launch)
        uint4* bz = reinterpret_cast<uint4*>(smem + K::OFF_BAND);
        for (int i = bt; i < K::NBAND * K::BAND_STAGE / 16; i += K::NBANDT) bz[i] = make_uint4(0, 0, 0, 0);
        for (uint32_t c = bt; c < ncombo; c += K::NBANDT) crow[c] = (c / p.s) * p.B_r + (c % p.s) * p.C;
      }
      uint32_t prev[K::NBAND][4];  // rows written NBAND stages ago, 4 bytes per word (κ·B_r ≤ 256)
#pragma unroll
      for (int b = 0; b < K::NBAND; ++b)
#pragma unroll
        for (int w = 0; w < 4; ++w) prev[b][w] = 0;
      int bs = 0;
      uint32_t bph = 0;
      int64_t stage_no = 0;
      const Tr tr((args.trace && bt == 0) ? args.trace + blockIdx.x * 16 : nullptr);
      const unsigned long long tstart = tr.now();
      int kc = (int)(S0 % nk);
      int64_t q = sb + S0 / nk;
      for (int64_t st = S0; st < S1; ++st, q += (kc + 1 == nk), kc = (kc + 1 == nk) ? 0 : kc + 1, ++stage_no) {
        const int par = (int)(q & 1);  // tables double-buffered by block parity
        uint64_t* ck = ckey + par * 256;
        {
          unsigned long long t0 = tr.now();
          ptx::mbar_wait_sleep(&band_empty[bs], bph ^ 1, 20);
          tr.add(6, t0);
          t0 = tr.now();
          if (kc == 0 || st == S0) {
            // per input block q: hash key of chunk (σ, j): the output i ≡ σ (mod κ) fed by q is
            // i = q - ℓ with ℓ = ((q - σ - 1) mod κ) + 1
            for (uint32_t c = bt; c < ncombo; c += K::NBANDT) {
              const uint32_t sig = c / p.s, j = c % p.s;
              const uint32_t ell = mod_pos(q - (int64_t)sig - 1, kappa) + 1;
              const uint32_t g = affine_pow(p, (uint64_t)mod_pos(q - (int64_t)ell, p.M), 0u);
              ck[c] = (((uint64_t)g << 40) | ((uint64_t)(ell - 1) << 32) | (uint64_t)j) ^ p.K;
            }
            ptx::named_bar_sync(1, K::NBANDT);
            tr.add(7, t0);
          }
          const uint64_t uk = (uint64_t)((uint32_t)kc * kBK + u) << 8;
          const uint32_t sbase = band_u32 + bs * K::BAND_STAGE;
          const bool clear = stage_no >= K::NBAND;
          uint32_t nw[4] = {0, 0, 0, 0};
          if (!BPS_DBG(1)) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              if ((uint32_t)w * 4 >= T) break;
              uint64_t z[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const uint32_t c = cg + 4 * (4 * w + i);
                z[i] = BPS_DBG(32) ? (ck[c < ncombo ? c : cg] ^ uk) : mix64(ck[c < ncombo ? c : cg] ^ uk);
              }
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const uint32_t t = 4 * w + i;
                if (t >= T) break;
                const uint32_t c = cg + 4 * t;
                if (clear) ptx::st_shared_u16(entry(sbase, (prev[0][w] >> (8 * i)) & 0xFFu), 0);
                const uint32_t rho = crow[c] + __umulhi((uint32_t)(z[i] >> 32), p.C);  // R3
                ptx::st_shared_u16(entry(sbase, rho), (z[i] & 1) ? (uint16_t)0xBF80 : (uint16_t)0x3F80);
                nw[w] |= rho << (8 * i);
              }
            }
          }
#pragma unroll
          for (int b = 0; b + 1 < K::NBAND; ++b)
#pragma unroll
            for (int w = 0; w < 4; ++w) prev[b][w] = prev[b + 1][w];
#pragma unroll
          for (int w = 0; w < 4; ++w) prev[K::NBAND - 1][w] = nw[w];
          if (!BPS_DBG(16)) ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&band_full[bs]);
          if (++bs == K::NBAND) bs = 0, bph ^= 1;
        }
      }
      tr.add(8, tstart);
    } else if (F32 && warp >= 12 && warp < 20) {
      // ===================== fp32 -> (hi, lo) bf16 split =====================
      // a = hi + lo, hi = bf16_rn(a), lo = bf16_rn(a - hi): |a - hi - lo| ≤ 2^-17 |a|.
      // Thread cv owns 4 consecutive MN (or K) elements of rows cv/(BN/4) + RPI·i; the
      // swizzled destination offset is affine in i, so it is precomputed (two parities).
      const int cv = threadIdx.x - 384;
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
      const int64_t total = S1 - S0;
      const Tr tr((args.trace && cv == 0) ? args.trace + blockIdx.x * 16 : nullptr);
      const unsigned long long tstart = tr.now();
      for (int64_t it = 0; it < total; ++it) {
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
        ptx::mbar_arrive(&conv_full[rs]);
        if (++rs == K::NRAW) rs = 0, rph ^= 1;
      }
      tr.add(12, tstart);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == K::W_MMA) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, K::TMEM_COLS);
  }
}

// Y += Y2 (balanced decomposition: the two parity buffers of split outputs; a fixed-order,
// deterministic final combine).
__global__ void __launch_bounds__(256) bps_add_kernel(float* __restrict__ Y, int64_t ldy, const float* __restrict__ Y2,
                                                      int64_t ldy2, int64_t rows, int64_t cols) {
  const int64_t c4 = (cols + 3) / 4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * c4; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / c4, c = (e % c4) * 4;
    float* y = Y + r * ldy + c;
    const float* z = Y2 + r * ldy2 + c;
    if (c + 4 <= cols) {
      float4 a = *reinterpret_cast<float4*>(y);
      const float4 b = *reinterpret_cast<const float4*>(z);
      a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
      *reinterpret_cast<float4*>(y) = a;
    } else {
      for (int64_t t = c; t < cols; ++t) Y[r * ldy + t] += Y2[r * ldy2 + t];
    }
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

struct Plan {
  bool ok = false;
  int nmt = 1;
  int bn = 128;
  std::string why;
};

Plan plan_for(const SketchParams& p, bps_dtype dt) {
  Plan pl;
  if (dt != BPS_F32 && dt != BPS_BF16) {
    pl.why = "dtype";
    return pl;
  }
  if (p.B_c % kBK != 0) {
    pl.why = "tc variant needs B_c % 64 == 0";
    return pl;
  }
  const uint64_t rows = (uint64_t)p.kappa * p.B_r;
  if (rows > 256) {
    pl.why = "tc variant needs kappa*B_r <= 256";
    return pl;
  }
  if ((uint64_t)p.kappa * p.s > 64) {
    pl.why = "tc variant needs kappa*s <= 64";
    return pl;
  }
  pl.nmt = rows <= 128 ? 1 : 2;
  pl.ok = true;
  return pl;
}

// ranges per column tile: as many as fill the SMs, each ≥ κ-1 input blocks long so that
// every split output has exactly two contributors (deterministic red.add, see header)
int64_t ranges_for(const SketchParams& p, int64_t stream_len, int64_t n_ct, int sms) {
  int64_t R = n_ct >= sms ? 1 : sms / n_ct;
  if (R > stream_len) R = stream_len;
  const int64_t need = p.kappa > 1 ? (int64_t)p.kappa - 1 : 1;
  while (R > 1 && stream_len / R < need) --R;
  return R;
}

template <bool F32, bool TRANS, int NMT, int BN_>
int launch_impl(const SketchParams& p, const void* A, int64_t lda, int64_t n, float* Y, int64_t ldy,
                const Placement& pl, float* Y2, int64_t ldy2, cudaStream_t st) {
  using K = Cfg<F32, TRANS, NMT, BN_>;
  constexpr int BN = K::BN;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(BPS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  TcArgs a;
  a.p = p;
  a.n = n;
  a.Y = Y;
  a.ldy = ldy;
  a.range_mode = pl.range_mode;
  a.pos_begin = pl.pos_begin;
  a.pos_end = pl.pos_begin + pl.n_out;
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
  // accumulation group: largest divisor of B_c/64 that is <= kMaxGroup K-chunks (precision)
  const int nk = (int)(p.B_c / kBK);
  int G = 1;
  for (int g = kMaxGroup; g >= 1; --g)
    if (nk % g == 0) {
      G = g;
      break;
    }
  a.G = G;
  a.dbg = 0;
  a.trace = nullptr;
#ifdef BPS_TC_INSTRUMENT
  {
    const char* e = getenv("BPS_TC_DEBUG");
    a.dbg = e ? atoi(e) : 0;
  }
#endif
  if (const char* e = getenv("BPS_TC_GROUP")) {  // tuning knob: K-chunks per accumulation group
    const int g = atoi(e);
    if (g >= 1 && nk % g == 0) a.G = g;
  }
  const int64_t n_ct = (n + BN - 1) / BN;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t R;
  a.balanced = Y2 != nullptr;
  a.Y2 = Y2;
  a.ldy2 = ldy2;
  if (a.balanced) {
    // stage-granular equal ranges: every range ≥ (κ·nk − 1)/3 stages, so an output window of
    // κ·nk stages meets ≤ 4 ranges and each parity buffer receives ≤ 2 addends per element
    const int64_t Ts = a.stream_len * nk, W = (int64_t)p.kappa * nk;
    R = n_ct >= sms ? 1 : sms / n_ct;
    if (R > Ts) R = Ts;
    while (R > 1 && Ts / R < (W - 1 + 2) / 3) --R;
  } else {
    R = ranges_for(p, a.stream_len, n_ct, sms);
  }
  a.R = (int)R;
  const int64_t grid = n_ct * R;
  if (grid > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "grid too large");
  if (in_rows > 0x7FFFFFFF || n > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "tc variant: TMA coordinates exceed int32");

  // TMA descriptor for the data operand
  CUtensorMap tm;
  const CUtensorMapDataType tdt = F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2], strides[1];
  cuuint32_t box[2], estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = F32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B;
  strides[0] = (cuuint64_t)lda * K::ESZ;
  if (!TRANS) {
    dims[0] = (cuuint64_t)n;
    dims[1] = (cuuint64_t)in_rows;
    box[0] = F32 ? BN : 64;
    box[1] = kBK;
  } else {
    dims[0] = (cuuint64_t)in_rows;  // coordinates (d)
    dims[1] = (cuuint64_t)n;        // vectors
    box[0] = kBK;
    box[1] = BN;
  }
  CUresult cr = enc(&tm, tdt, 2, const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(BPS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));

  // outputs split between CTAs are accumulated with red.add into zeroed buffers
  const int64_t krows = pl.range_mode ? pl.n_out * (int64_t)p.B_r : (int64_t)p.M * p.B_r;
  const int64_t yrows = TRANS ? n : krows, ycols = TRANS ? krows : n;
  if (p.kappa > 1 || a.balanced) {
    cudaError_t e = cudaMemset2DAsync(Y, ldy * 4, 0, (size_t)ycols * 4, (size_t)yrows, st);
    if (e == cudaSuccess && a.balanced) e = cudaMemset2DAsync(Y2, ldy2 * 4, 0, (size_t)ycols * 4, (size_t)yrows, st);
    if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("cudaMemset2DAsync: ") + cudaGetErrorString(e));
  }
  auto kern = bps_tc_kernel<F32, TRANS, NMT, BN_>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
#ifdef BPS_TC_INSTRUMENT
  if (a.dbg & 8) {  // debug trace: per-CTA cycle counters, printed to stderr (synchronises)
    cudaMalloc(&a.trace, (size_t)grid * 16 * 8);
    cudaMemsetAsync(a.trace, 0, (size_t)grid * 16 * 8, st);
  }
  kern<<<(unsigned)grid, K::NTHREADS, K::SMEM, st>>>(tm, a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (a.trace) {
    std::vector<unsigned long long> h((size_t)grid * 16);
    cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[13] = {"tma_wait_empty", "tma_total", "mma_wait_accfree", "mma_wait_data", "mma_wait_band",
                             "mma_total", "band_wait_empty", "band_table", "band_total", "epi_wait_accfull",
                             "epi_total", "conv_wait_raw", "conv_total"};
    for (int k = 0; k < 13; ++k) {
      double sum = 0, mx = 0;
      for (int64_t c = 0; c < grid; ++c) {
        sum += (double)h[c * 16 + k];
        mx = std::max(mx, (double)h[c * 16 + k]);
      }
      fprintf(stderr, "[bps trace] %-18s mean %12.0f  max %12.0f cycles\n", names[k], sum / grid, mx);
    }
    cudaFree(a.trace);
  }
#else
  kern<<<(unsigned)grid, K::NTHREADS, K::SMEM, st>>>(tm, a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
#endif
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("bps_tc_kernel launch: ") + cudaGetErrorString(e));
  if (a.balanced) {
    const int64_t work = yrows * ((ycols + 3) / 4);
    const int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)sms * 8);
    bps_add_kernel<<<blocks, 256, 0, st>>>(Y, ldy, Y2, ldy2, yrows, ycols);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("bps_add_kernel launch: ") + cudaGetErrorString(e));
  }
  return BPS_OK;
}

}  // namespace

int tc_supported(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  (void)n;
  (void)transposed;
  (void)pl;
  Plan plan = plan_for(p, dt);
  if (!plan.ok) return fail(BPS_ERR_UNSUPPORTED, plan.why);
  return BPS_OK;
}

size_t tc_workspace_bytes(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl) {
  if (!plan_for(p, dt).ok) return 0;
  const int64_t krows = pl.range_mode ? pl.n_out * (int64_t)p.B_r : (int64_t)p.M * p.B_r;
  const int64_t rows = transposed ? n : krows, cols = transposed ? krows : n;
  return (size_t)rows * (size_t)((cols + 3) / 4 * 4) * 4;
}

int launch_tc(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y, int64_t ldy,
              bool transposed, const Placement& pl, void* ws, size_t ws_bytes, cudaStream_t st) {
  float* Y2 = nullptr;
  int64_t ldy2 = 0;
  const size_t need = tc_workspace_bytes(p, n, dt, transposed, pl);
  // the balanced decomposition only pays when whole-block ranges are uneven (e.g. LS: 128 blocks
  // over 37 ranges = 3 or 4 blocks); it costs two memsets and an add pass otherwise
  bool uneven = false;
  if (ws) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const Plan pln = plan_for(p, dt);
    const int bnx = (dt == BPS_F32) ? (pln.nmt == 1 ? 128 : 64) : 128;  // conservative (smaller) tile
    const int64_t sl = pl.range_mode ? pl.n_out + p.kappa - 1 : (int64_t)p.M;
    const int64_t nct = (n + bnx - 1) / bnx;
    const int64_t R = ranges_for(p, sl, nct, sms);
    const int64_t Lmax = (sl + R - 1) / R;
    uneven = R > 1 && (double)Lmax * R > 1.05 * (double)sl;
  }
  if (ws && uneven && need && ws_bytes >= need && ((uintptr_t)ws % 16) == 0) {
    const int64_t krows = pl.range_mode ? pl.n_out * (int64_t)p.B_r : (int64_t)p.M * p.B_r;
    Y2 = (float*)ws;
    ldy2 = ((transposed ? krows : n) + 3) / 4 * 4;
  }
  Plan plan = plan_for(p, dt);
  if (!plan.ok) return fail(BPS_ERR_UNSUPPORTED, plan.why);
  const bool f32 = dt == BPS_F32;
  // bf16, one M-tile: 256 columns per CTA (band reused over twice the columns) unless that
  // leaves SMs idle, then 128.
  int bn = 128;
  if (!f32 && plan.nmt == 1) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t sl = pl.range_mode ? pl.n_out + p.kappa - 1 : (int64_t)p.M;
    const int64_t ct256 = (n + 255) / 256, ct128 = (n + 127) / 128;
    const int64_t used256 = ct256 * ranges_for(p, sl, ct256, sms);
    const int64_t used128 = ct128 * ranges_for(p, sl, ct128, sms);
    bn = (used256 * 10 >= used128 * 9 || used256 >= sms) ? 256 : 128;
  }
#define BPS_TC_CASE(F, T, NM, B)                                        \
  if (f32 == F && transposed == T && plan.nmt == NM && bn == B)         \
    return launch_impl<F, T, NM, B>(p, A, lda, n, Y, ldy, pl, Y2, ldy2, st);
  BPS_TC_CASE(true, false, 1, 128)
  BPS_TC_CASE(true, true, 1, 128)
  if (f32) bn = 64;
  BPS_TC_CASE(true, false, 2, 64)
  BPS_TC_CASE(true, true, 2, 64)
  BPS_TC_CASE(false, false, 1, 256)
  BPS_TC_CASE(false, true, 1, 256)
  BPS_TC_CASE(false, false, 1, 128)
  BPS_TC_CASE(false, true, 1, 128)
  BPS_TC_CASE(false, false, 2, 128)
  BPS_TC_CASE(false, true, 2, 128)
#undef BPS_TC_CASE
  return fail(BPS_ERR_UNSUPPORTED, "no tc instantiation for this plan");
}

}  // namespace bps

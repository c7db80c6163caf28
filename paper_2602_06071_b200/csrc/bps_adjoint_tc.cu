// bps_adjoint_tc.cu — X = Sᵀ·Y on the 5th-generation tensor cores.
//
// For input block h = g_p (orbit position p) and a chunk of 64 rows u, the adjoint is the
// dense contraction
//     Xᵀ[cols, u] = Σ_ρ  Wᵀ[cols, ρ] · Band[ρ, u]          (ρ < K_w = κ·B_r window rows)
// where W is the window of the κ feeding outputs' Y rows (slot σ = i mod κ holds output
// g_i, i = p-ℓ, the same slot rule as the forward kernel) and Band is the
// forward kernel's band stage for (p, u-chunk): ±1 at (σ·B_r + row(g_i, ℓ, u, j), u)
// (R1-R3).  Each output sums exactly κ·s products, so the fp32 result needs no regrouping;
// Y (fp32) enters as hi + lo bf16 pairs (|y - hi - lo| ≤ 2^-17|y|), two MMAs per K step.
//
// Operands (tcgen05.mma kind::f16, cta_group::1, M = 128 columns, N = 64 rows u):
//   A = Wᵀ (MN-major, SW128): converter warps write the window in shared memory once per CTA
//       range and then ONE slot per input block (the entering output), after the MMAs of
//       the previous block completed;
//   B = Band (MN-major, SW128: the forward's K-major [ρ][u] band tile read the other way);
//   D = TMEM, double-buffered, drained by 8 epilogue warps with coalesced streaming stores.
// Work: the M·B_c/64 stages of every column group are split into equal contiguous ranges,
// one CTA per SM; every X element is written exactly once (no atomics, reproducible).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "bps_internal.h"
#include "bps_ptx.cuh"

namespace bps {
namespace {

constexpr int kU = 64;                  // rows u per stage (MMA N)
constexpr int kEpiWarps = 8, kBandWarps = 8, kConvWarps = 4;
constexpr int kWBand = kEpiWarps, kWConv = kWBand + kBandWarps, kWMma = kWConv + kConvWarps;
constexpr int kThreads = (kWMma + 1) * 32;
constexpr int kBandT = kBandWarps * 32, kConvT = kConvWarps * 32;
constexpr int kBudget = 222 * 1024;

struct AdjArgs {
  SketchParams p;
  const float* Y;
  int64_t ldy, n;
  float* X;
  int64_t ldx;
  int Kw;     // window rows rounded up to 16 (MMA K granularity)
  int nband;  // band ring depth
  int R;      // CTAs per column group
  int off_band, off_ckey, off_crow, off_bar;
};

__device__ __forceinline__ uint32_t mod_pos(int64_t i, uint32_t M) {
  int64_t r = i % (int64_t)M;
  return (uint32_t)(r < 0 ? r + M : r);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both MN-major, M = 128, N = 64.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((kU >> 3) << 17) |
                            ((128 >> 4) << 24);

template <int NMT, int NB>
__global__ void __launch_bounds__(kThreads, 1) bps_adjoint_tc_kernel(const AdjArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const SketchParams& p = args.p;
  const int Kw = args.Kw;
  const uint32_t AT = (uint32_t)Kw * 256;  // one operand (hi or lo) of one 128-column tile: 2 × Kw × 128 B
  const uint32_t BT = (uint32_t)Kw * 128;  // one band stage
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + args.off_bar);
  uint64_t* band_full = bars;
  uint64_t* band_empty = band_full + NB;
  uint64_t* d_full = band_empty + NB;  // [2]
  uint64_t* d_free = d_full + 2;       // [2]
  uint64_t* win_full = d_free + 2;
  uint64_t* win_empty = win_full + 1;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(win_empty + 1);
  uint64_t* ckey = reinterpret_cast<uint64_t*>(smem + args.off_ckey);
  uint32_t* crow = reinterpret_cast<uint32_t*>(smem + args.off_crow);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kappa = p.kappa;
  const int nk = (int)(p.B_c / kU);
  const int cg = blockIdx.x % (int)((args.n + NMT * 128 - 1) / (NMT * 128));
  const int rr = blockIdx.x / (int)((args.n + NMT * 128 - 1) / (NMT * 128));
  const int64_t col0 = (int64_t)cg * NMT * 128;
  const int64_t Ts = (int64_t)p.M * nk;
  const int64_t S0 = Ts * rr / args.R, S1 = Ts * (rr + 1) / args.R;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) {
      ptx::mbar_init(&band_full[i], kBandT);
      ptx::mbar_init(&band_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&d_full[i], 1);
      ptx::mbar_init(&d_free[i], kEpiWarps * 32);
    }
    ptx::mbar_init(win_full, kConvT);
    ptx::mbar_init(win_empty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == kWMma) ptx::tmem_alloc(tmem_ptr, NMT == 1 ? 128 : 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;  // D buffer b, tile m at column (b·NMT + m)·64

  if (S1 > S0) {
    if (warp == kWMma) {
      // ===================== MMA issuer =====================
      const uint32_t a_base = ptx::smem_u32(smem);
      const uint32_t b_base = ptx::smem_u32(smem + args.off_band);
      int bs = 0, db = 0;
      uint32_t bph = 0, dph = 0, wph = 0;
      int kc = (int)(S0 % nk);
      for (int64_t st = S0; st < S1; ++st) {
        if (st == S0 || kc == 0) {  // a new input block: its window must be in shared memory
          ptx::mbar_wait(win_full, wph);
          wph ^= 1;
        }
        ptx::mbar_wait(&band_full[bs], bph);
        ptx::mbar_wait(&d_free[db], dph ^ 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t bb = b_base + bs * BT;
#pragma unroll
          for (int m = 0; m < NMT; ++m) {
            const uint32_t d = tmem + (uint32_t)(db * NMT + m) * kU;
            const uint32_t ah = a_base + m * 2 * AT, al = ah + AT;
            for (int ks = 0; ks < Kw / 16; ++ks) {
              const uint64_t bdesc = ptx::smem_desc_sw128(bb + ks * 2048, BT, 1024);
              ptx::mma_bf16_ss(d, ptx::smem_desc_sw128(ah + ks * 2048, Kw * 128, 1024), bdesc, kIdesc, ks ? 1u : 0u);
              ptx::mma_bf16_ss(d, ptx::smem_desc_sw128(al + ks * 2048, Kw * 128, 1024), bdesc, kIdesc, 1u);
            }
          }
          ptx::mma_commit(&band_empty[bs]);
          ptx::mma_commit(&d_full[db]);
          if (kc == nk - 1 || st == S1 - 1) ptx::mma_commit(win_empty);  // window of this block released
        }
        __syncwarp();
        if (++bs == NB) bs = 0, bph ^= 1;
        if (++db == 2) db = 0, dph ^= 1;
        if (++kc == nk) kc = 0;
      }
    } else if (warp < kEpiWarps) {
      // ===================== epilogue: TMEM -> X (scaled) =====================
      // warp e: TMEM lane quarter e % 4 (columns 32q..32q+31 of a tile); NMT = 2: tile e / 4,
      // all 64 u; NMT = 1: tile 0, u half e / 4.
      const int qtr = warp & 3, half = warp >> 2;
      const int m = NMT == 2 ? half : 0;
      const int u_lo = NMT == 2 ? 0 : 32 * half, u_n = NMT == 2 ? 64 : 32;
      const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
      const int64_t col = col0 + m * 128 + qtr * 32 + lane;
      const bool live = col < args.n;
      int64_t q = S0 / nk;
      int kc = (int)(S0 % nk);
      uint32_t h = affine_pow(p, (uint64_t)q, 0u);
      int db = 0;
      uint32_t dph = 0;
      for (int64_t st = S0; st < S1; ++st) {
        ptx::mbar_wait_sleep(&d_full[db], dph, 32);
        ptx::tc_fence_after();
        float* xb = args.X + ((int64_t)h * p.B_c + (int64_t)kc * kU) * args.ldx + col;
        for (int c = u_lo; c < u_lo + u_n; c += 32) {
          uint32_t v[32];
          ptx::tmem_ld32(tmem + (uint32_t)(db * NMT + m) * kU + c + lane_off, v);
          ptx::tmem_wait_ld();
          if (live) {
#pragma unroll
            for (int t = 0; t < 32; ++t) __stcs(xb + (int64_t)(c + t) * args.ldx, __uint_as_float(v[t]) * p.scale);
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&d_free[db]);
        if (++db == 2) db = 0, dph ^= 1;
        if (++kc == nk) kc = 0, ++q, h = affine_step(p, h);
      }
    } else if (warp < kWConv) {
      auto band_gen = [&](auto affine_tag) {  // specialised on the intra-block mode
        constexpr bool AFF = decltype(affine_tag)::value;
        // ===================== band generator (same stages as the forward kernel) =====================
        // Thread (u, g4) owns column u of every band stage for the row chunks c = g4 + 4t,
        // c = σ·s + j; it clears the entry it wrote NB stages ago instead of zero-filling.
        const int bt = threadIdx.x - kWBand * 32;
        const uint32_t u = (uint32_t)bt & (kU - 1);
        const uint32_t g4 = (uint32_t)bt >> 6;
        const uint32_t ncombo = kappa * p.s;
        const uint32_t T = ncombo > g4 ? (ncombo - g4 + 3) / 4 : 0;  // ≤ 16 (κ·s ≤ 64)
        const uint32_t band_u32 = ptx::smem_u32(smem + args.off_band);
        const uint32_t ucol = u >> 3, ulo = (u & 7) * 2;
        auto entry = [&](uint32_t sbase, uint32_t rho) {
          return sbase + rho * 128 + (((rho ^ ucol) & 7) << 4) + ulo;  // SW128 row ρ
        };
        {
          uint4* bz = reinterpret_cast<uint4*>(smem + args.off_band);
          for (uint32_t i = bt; i < (uint32_t)NB * BT / 16; i += kBandT) bz[i] = make_uint4(0, 0, 0, 0);
          for (uint32_t c = bt; c < ncombo; c += kBandT) crow[c] = band_crow(p, c / p.s, c % p.s);
        }
        uint32_t prev[NB][4];  // rows written NB stages ago (this buffer), 8 bits each (κ·B_r ≤ 256)
  #pragma unroll
        for (int b = 0; b < NB; ++b)
  #pragma unroll
          for (int w = 0; w < 4; ++w) prev[b][w] = 0;
        int bs = 0;
        uint32_t bph = 0;
        int64_t local_no = 0;
        int kc = (int)(S0 % nk);
        int64_t q = S0 / nk;
        for (int64_t st = S0; st < S1; ++st, q += (kc + 1 == nk), kc = (kc + 1 == nk) ? 0 : kc + 1) {
          uint64_t* ck = ckey + (q & 1) * 64;
          ptx::mbar_wait_sleep(&band_empty[bs], bph ^ 1, 20);
          if (kc == 0 || st == S0) {
            // input block q: the output i ≡ σ (mod κ) feeding it is i = q - ℓ, ℓ = ((q - σ - 1) mod κ) + 1
            for (uint32_t c = bt; c < ncombo; c += kBandT) {
              const uint32_t sig = c / p.s, j = c % p.s;
              const uint32_t ell = mod_pos(q - (int64_t)sig - 1, kappa) + 1;
              const uint32_t g = affine_pow(p, (uint64_t)mod_pos(q - (int64_t)ell, p.M), 0u);
              ck[c] = (((uint64_t)g << 40) | ((uint64_t)(ell - 1) << 32) | (uint64_t)band_jfield(p, j)) ^ p.K;
            }
            ptx::named_bar_sync(1, kBandT);
          }
          const uint64_t uk = (uint64_t)((uint32_t)kc * kU + u) << 8;
          const uint32_t sbase = band_u32 + bs * BT;
          bool clear = local_no >= NB;
          ++local_no;
          uint32_t nw[4] = {0, 0, 0, 0};
          if constexpr (AFF) {
            // AffineUnique (R18), slot-major as in bps_tc.cu: one hash per (σ, u), σ ≡ g4 (mod 4);
            // κ > 16 slots: zero-fill the stage behind a barrier instead of tracking stale rows
            const bool zero_fill = kappa > 16u;
            if (zero_fill && clear) {
              uint4* bz = reinterpret_cast<uint4*>(smem + args.off_band + bs * BT);
              for (uint32_t i = bt; i < BT / 16; i += kBandT) bz[i] = make_uint4(0, 0, 0, 0);
              ptx::named_bar_sync(3, kBandT);
            }
            if (zero_fill) clear = false;
  #pragma unroll
            for (int t = 0; t < 16; ++t) {
              const uint32_t sig = g4 + 4 * t;
              if (sig >= kappa) break;
              const uint32_t base = sig * p.B_r;
              if (t < 4 && clear) {
                const uint32_t w = prev[0][t & 3], a0 = w & 0xFFFFu;
                uint32_t r = w >> 16;
                for (uint32_t j = 0; j < p.s; ++j, r = (r + a0) & p.Brmask) ptx::st_shared_u16(entry(sbase, base + r), 0);
              }
              const uint64_t z = mix64(ck[sig * p.s] ^ uk);
              const uint32_t alpha = (uint32_t)(((((z >> 32) & 0xFFFFu) * p.B_r) >> 16) | 1u);
              const uint32_t beta = (uint32_t)(((z >> 48) * p.B_r) >> 16);
              uint32_t r = beta, zs = (uint32_t)z;
              for (uint32_t j = 0; j < p.s; ++j, r = (r + alpha) & p.Brmask, zs >>= 1)
                ptx::st_shared_u16(entry(sbase, base + r), (zs & 1u) ? (uint16_t)0xBF80 : (uint16_t)0x3F80);
              if (t < 4) nw[t & 3] = alpha | (beta << 16);
            }
          } else {
  #pragma unroll
            for (int w = 0; w < 4; ++w) {
              if ((uint32_t)w * 4 < T) {
                uint64_t z[4];
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint32_t c = g4 + 4 * (4 * w + i);
                  z[i] = mix64(ck[c < ncombo ? c : g4] ^ uk);
                }
  #pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint32_t t = 4 * w + i;
                  if (t >= T) break;
                  const uint32_t c = g4 + 4 * t;
                  if (clear) ptx::st_shared_u16(entry(sbase, (prev[0][w] >> (8 * i)) & 0xFFu), 0);
                  uint32_t neg;
                  const uint32_t rho = band_draw_t<false>(p, crow[c], z[i], neg);
                  ptx::st_shared_u16(entry(sbase, rho), neg ? (uint16_t)0xBF80 : (uint16_t)0x3F80);
                  nw[w] |= rho << (8 * i);
                }
              }
            }
          }
  #pragma unroll
          for (int b = 0; b + 1 < NB; ++b)
  #pragma unroll
            for (int w = 0; w < 4; ++w) prev[b][w] = prev[b + 1][w];
  #pragma unroll
          for (int w = 0; w < 4; ++w) prev[NB - 1][w] = nw[w];
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&band_full[bs]);
          if (++bs == NB) bs = 0, bph ^= 1;
        }
      };
      if (p.mode)
        band_gen(std::true_type{});
      else
        band_gen(std::false_type{});
    } else if (warp < kWMma) {
      // ===================== window converter: Y rows -> (hi, lo) bf16, SW128 MN-major =====================
      const int ct = threadIdx.x - kWConv * 32;
      const int chunks_per_row = NMT * 16;  // 8 columns (16 B of bf16) per chunk
      auto load_slot = [&](uint32_t sig, uint32_t g) {
        const int tasks = (int)p.B_r * chunks_per_row;
        for (int t = ct; t < tasks; t += kConvT) {
          const uint32_t r = (uint32_t)t / chunks_per_row, ch = (uint32_t)t % chunks_per_row;
          const uint32_t rho = sig * p.B_r + r;
          const int64_t c = col0 + ch * 8;
          const float* src = args.Y + ((int64_t)g * p.B_r + r) * args.ldy + c;
          float a[8];
          if (c + 8 <= args.n) {
            const float4 v0 = __ldg(reinterpret_cast<const float4*>(src));
            const float4 v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
            a[0] = v0.x, a[1] = v0.y, a[2] = v0.z, a[3] = v0.w, a[4] = v1.x, a[5] = v1.y, a[6] = v1.z, a[7] = v1.w;
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = (c + e < args.n) ? src[e] : 0.f;
          }
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi[e]) : "f"(a[2 * e + 1]), "f"(a[2 * e]));
            const float r0 = a[2 * e] - __uint_as_float(hi[e] << 16);
            const float r1 = a[2 * e + 1] - __uint_as_float(hi[e] & 0xFFFF0000u);
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo[e]) : "f"(r1), "f"(r0));
          }
          const uint32_t m = ch >> 4, blk = (ch >> 3) & 1, c8 = ch & 7;
          const uint32_t off = m * 2 * AT + blk * (uint32_t)Kw * 128 + rho * 128 + ((c8 ^ (rho & 7)) << 4);
          *reinterpret_cast<uint4*>(smem + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(smem + off + AT) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      };
      {  // zero the window once: padding rows κ·B_r .. K_w stay zero
        uint4* z = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = ct; i < (uint32_t)NMT * 2 * AT / 16; i += kConvT) z[i] = make_uint4(0, 0, 0, 0);
        ptx::named_bar_sync(2, kConvT);
      }
      const int64_t q0 = S0 / nk, q1 = (S1 - 1) / nk;
      uint32_t eph = 0;
      for (int64_t q = q0; q <= q1; ++q) {
        if (q == q0) {
          for (uint32_t ell = 1; ell <= kappa; ++ell) {
            const int64_t i = q - ell;
            load_slot(mod_pos(i, kappa), affine_pow(p, (uint64_t)mod_pos(i, p.M), 0u));
          }
        } else {
          ptx::mbar_wait_sleep(win_empty, eph, 32);  // MMAs of block q-1 are complete
          eph ^= 1;
          const int64_t i = q - 1;  // the entering output replaces output q-1-κ in slot (q-1) mod κ
          load_slot(mod_pos(i, kappa), affine_pow(p, (uint64_t)mod_pos(i, p.M), 0u));
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(win_full);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kWMma) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, NMT == 1 ? 128 : 256);
  }
}

int smem_layout(const SketchParams& p, int nmt, AdjArgs& a) {
  a.Kw = (int)(((uint64_t)p.kappa * p.B_r + 15) / 16 * 16);
  const int win = nmt * 2 * a.Kw * 256;
  const int band = a.Kw * 128;
  const int fixed = 2 * 64 * 8 + 64 * 4 + 16 * 8 + 16 + 1024;
  a.nband = std::min(4, (kBudget - win - fixed) / band);
  a.off_band = win;
  a.off_ckey = win + a.nband * band;
  a.off_crow = a.off_ckey + 2 * 64 * 8;
  a.off_bar = a.off_crow + 64 * 4;
  return a.off_bar + (2 * a.nband + 6) * 8 + 16 + 1024;
}

}  // namespace

int adjoint_tc_supported(const SketchParams& p, int64_t n) {
  if (p.B_c % kU || (uint64_t)p.kappa * p.s > 64 || (uint64_t)p.kappa * p.B_r > 256) return 0;
  if (n < 1 || (uint64_t)p.M * p.B_c > (1ull << 40)) return 0;
  AdjArgs a{};
  smem_layout(p, 1, a);
  return a.nband >= 2;
}

int launch_adjoint_tc(const SketchParams& p, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                      cudaStream_t st) {
  if (!adjoint_tc_supported(p, n)) return fail(BPS_ERR_UNSUPPORTED, "adjoint tc: shape not covered");
  AdjArgs a{};
  int nmt = n > 128 ? 2 : 1;
  int smem = smem_layout(p, nmt, a);
  if (a.nband < 2) nmt = 1, smem = smem_layout(p, 1, a);
  a.p = p, a.Y = Y, a.ldy = ldy, a.n = n, a.X = X, a.ldx = ldx;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ncg = (n + nmt * 128 - 1) / (nmt * 128);
  const int64_t stages = (int64_t)p.M * (p.B_c / kU);
  a.R = (int)std::max<int64_t>(1, std::min<int64_t>(stages, sms / std::max<int64_t>(1, ncg)));
  const int64_t grid = ncg * a.R;
  if (grid > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "adjoint tc: grid too large");
  const bool nb4 = a.nband >= 4;
  a.nband = nb4 ? 4 : 2;
  smem = a.off_bar + (2 * a.nband + 6) * 8 + 16 + 1024;
  auto kern = nmt == 2 ? (nb4 ? bps_adjoint_tc_kernel<2, 4> : bps_adjoint_tc_kernel<2, 2>)
                       : (nb4 ? bps_adjoint_tc_kernel<1, 4> : bps_adjoint_tc_kernel<1, 2>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("adjoint tc attr: ") + cudaGetErrorString(e));
  kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("bps_adjoint_tc_kernel: ") + cudaGetErrorString(e));
  return BPS_OK;
}

}  // namespace bps

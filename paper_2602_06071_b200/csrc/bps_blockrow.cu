// bps_blockrow.cu — FlashBlockRow Y = S'·A, the block-row sampling sketch.
//
// Alg. `alg:blockrowsketch`: output block g gathers from κ distinct input blocks
// N_row(g) (R14); output row r adds s uniformly sampled rows of each (R15), signed, scaled by
// (κs)^{-1/2}(d/k)^{1/2} (R16).  Pure gather: no atomics, one write per output element
// (P:1433-1434).  Unlike the paper's kernel, which stages whole input blocks in shared memory,
// only the κ·s rows a row needs are read (straight from HBM/L2 with 16-byte vector loads), so
// HBM traffic is ≤ k·κs·n·elem + k·n·4 bytes instead of κ·d·n·elem.
//
// Row-major: CTA = (output block g, group of rows, TN-column tile).  Warp 0 draws N_row(g) into
// shared memory; each warp then handles G rows per iteration: its 32 lanes draw the G·κs
// (index, sign) pairs in passes of 32 into a per-warp table; lane groups of LPR lanes (one per
// row, 16 bytes of the row per lane and vector step) accumulate ±A rows in fp32 registers.
// Transposed (X = Aᵀ, n×d): CTA = (g, 32 vectors); the block's (index, sign) table is built in
// shared memory once, then thread (vector, row) gathers its κs elements (scattered reads).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "bps_internal.h"

namespace bps {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kQMax = 2;  // rows per lane group per iteration (registers: kQMax·V·E accumulators)
constexpr int kMaxKappaBr = 256;  // κ ≤ 256 (make-time validation)

// N_row(g) (R14): sequential rejection over attempts t; one warp; result in nb[0..κ).
__device__ void draw_neighbors(const BlockRowParams& p, uint32_t g, uint32_t* nb) {
  const int lane = threadIdx.x & 31;
  uint32_t cnt = 0;
  for (uint32_t t0 = 0; cnt < p.kappa; t0 += 32) {
    const uint32_t h = br_block_draw(p, g, t0 + lane);
    for (int L = 0; L < 32 && cnt < p.kappa; ++L) {
      const uint32_t hl = __shfl_sync(0xffffffffu, h, L);
      bool dup = false;
      for (uint32_t j = lane; j < cnt; j += 32) dup |= nb[j] == hl;
      if (!__any_sync(0xffffffffu, dup)) {
        if (lane == 0) nb[cnt] = hl;
        ++cnt;
        __syncwarp();
      }
    }
  }
}

template <bool BF16>
struct Vec;
template <>
struct Vec<false> {  // 4 fp32
  static constexpr int E = 4;
  __device__ static void acc(float* a, const uint4& v, float sg) {
    a[0] = fmaf(sg, __uint_as_float(v.x), a[0]);
    a[1] = fmaf(sg, __uint_as_float(v.y), a[1]);
    a[2] = fmaf(sg, __uint_as_float(v.z), a[2]);
    a[3] = fmaf(sg, __uint_as_float(v.w), a[3]);
  }
};
template <>
struct Vec<true> {  // 8 bf16, widened exactly
  static constexpr int E = 8;
  __device__ static void acc(float* a, const uint4& v, float sg) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[2 * i] = fmaf(sg, __uint_as_float(w[i] << 16), a[2 * i]);
      a[2 * i + 1] = fmaf(sg, __uint_as_float(w[i] & 0xFFFF0000u), a[2 * i + 1]);
    }
  }
};

// 16 bytes of row `row` starting at element cv, zero beyond n (tail of the last column tile)
template <bool BF16>
__device__ __forceinline__ uint4 load16(const char* row, int64_t cv, int64_t n) {
  constexpr int E = BF16 ? 8 : 4, ES = BF16 ? 2 : 4;
  if (cv + E <= n) return __ldg(reinterpret_cast<const uint4*>(row + cv * ES));
  uint32_t w[4] = {0, 0, 0, 0};
  if (BF16) {
    const uint16_t* r16 = reinterpret_cast<const uint16_t*>(row);
    for (int e = 0; e < 8; ++e)
      if (cv + e < n) w[e >> 1] |= (uint32_t)r16[cv + e] << (16 * (e & 1));
  } else {
    const uint32_t* r32 = reinterpret_cast<const uint32_t*>(row);
    for (int e = 0; e < 4; ++e)
      if (cv + e < n) w[e] = r32[cv + e];
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <bool BF16, int LPR, int V>
__global__ void __launch_bounds__(kThreads, 4) blockrow_rowmajor_kernel(BlockRowParams p, const void* __restrict__ Av,
                                                                      int64_t lda, int64_t n, float* __restrict__ Y,
                                                                      int64_t ldy, uint32_t rows_per_cta) {
  using VT = Vec<BF16>;
  constexpr int E = VT::E;            // elements per 16-byte vector
  constexpr int TN = LPR * V * E;     // columns per CTA tile
  constexpr int RPW = 32 / LPR;       // rows in flight per warp
  constexpr int ES = BF16 ? 2 : 4;
  constexpr int kBatch = BF16 ? 4 : 8;  // independent 16-byte loads in flight per lane
  __shared__ uint32_t nbw[kWarps][kMaxKappaBr];  // per-warp copy of N_row(g): no CTA-wide barrier
  __shared__ unsigned long long codes[kWarps][32];
  const uint32_t g = blockIdx.x;
  const uint32_t r_begin = blockIdx.y * rows_per_cta, r_end = min(p.B_r, r_begin + rows_per_cta);
  const int64_t col0 = (int64_t)blockIdx.z * TN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ks = p.kappa * p.s;
  const uint32_t q = min((uint32_t)kQMax, max(1u, 32u / (RPW * ks)));
  const uint32_t G = RPW * q, T = G * ks;
  if (r_begin + warp * G >= r_end) return;
  uint32_t* nb = nbw[warp];
  draw_neighbors(p, g, nb);

  const int grp = lane / LPR, gl = lane % LPR;
  const int64_t col = col0 + (int64_t)gl * V * E;
  const char* A = reinterpret_cast<const char*>(Av);

  for (uint32_t r0 = r_begin + warp * G; r0 < r_end; r0 += kWarps * G) {
    float acc[kQMax][V * E];
#pragma unroll
    for (int i = 0; i < kQMax; ++i)
#pragma unroll
      for (int e = 0; e < V * E; ++e) acc[i][e] = 0.f;
    for (uint32_t c0 = 0; c0 < T; c0 += 32) {
      const uint32_t c = c0 + lane;
      unsigned long long code = 0;
      if (c < T) {
        const uint32_t r = r0 + c / ks, cc = c % ks;
        if (r < r_end) {
          const uint32_t ell = cc / p.s + 1, t = cc % p.s;
          const BrDraw dr = br_index_draw(p, g, ell, r, t);
          code = ((unsigned long long)nb[ell - 1] * p.B_c + dr.i) | ((unsigned long long)dr.neg << 63);
        }
      }
      __syncwarp();
      codes[warp][lane] = code;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < kQMax; ++i) {
        if ((uint32_t)i < q) {
          const uint32_t rr = (uint32_t)i * RPW + grp;
          const uint32_t lo = max(rr * ks, c0), hi = min((rr + 1) * ks, min(c0 + 32, T));
          for (uint32_t t = lo; t < hi; t += kBatch) {
            uint4 x[kBatch][V];
            float sg[kBatch];
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
              if (t + b < hi) {
                const unsigned long long cw = codes[warp][t + b - c0];
                sg[b] = (cw >> 63) ? -1.f : 1.f;
                const char* row = A + (int64_t)(cw & 0x7FFFFFFFFFFFFFFFull) * lda * ES;
#pragma unroll
                for (int v = 0; v < V; ++v) x[b][v] = load16<BF16>(row, col + v * E, n);
              }
            }
#pragma unroll
            for (int b = 0; b < kBatch; ++b)
              if (t + b < hi)
#pragma unroll
                for (int v = 0; v < V; ++v) VT::acc(&acc[i][v * E], x[b][v], sg[b]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kQMax; ++i) {
      if ((uint32_t)i >= q) break;
      const uint32_t r = r0 + (uint32_t)i * RPW + grp;
      if (r >= r_end) continue;
      float* dst = Y + ((int64_t)g * p.B_r + r) * ldy + col;
#pragma unroll
      for (int v = 0; v < V * E; v += 4) {
        const int64_t cv = col + v;
        const float4 o = make_float4(acc[i][v] * p.scale, acc[i][v + 1] * p.scale, acc[i][v + 2] * p.scale,
                                     acc[i][v + 3] * p.scale);
        if (cv + 4 <= n) {
          *reinterpret_cast<float4*>(dst + v) = o;
        } else {
          if (cv < n) dst[v] = o.x;
          if (cv + 1 < n) dst[v + 1] = o.y;
          if (cv + 2 < n) dst[v + 2] = o.z;
        }
      }
    }
  }
}

// Transposed: Yt[t, g·B_r + r] = scale·Σ σ X[t, idx].  CTA = (g, row chunk, 32 vectors t).
template <bool BF16>
__global__ void __launch_bounds__(kThreads) blockrow_transposed_kernel(BlockRowParams p, const void* __restrict__ Xv,
                                                                        int64_t ldx, int64_t n, float* __restrict__ Yt,
                                                                        int64_t ldyt, uint32_t rows_per_cta) {
  extern __shared__ unsigned long long tab[];  // [rows_per_cta · κs] (index | sign<<63)
  __shared__ uint32_t nb[256];
  const uint32_t g = blockIdx.x;
  const uint32_t r_begin = blockIdx.y * rows_per_cta, r_end = min(p.B_r, r_begin + rows_per_cta);
  const uint32_t nr = r_end - r_begin, ks = p.kappa * p.s;
  if ((threadIdx.x >> 5) == 0) draw_neighbors(p, g, nb);
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < nr * ks; e += kThreads) {
    const uint32_t r = r_begin + e / ks, cc = e % ks;
    const uint32_t ell = cc / p.s + 1, t = cc % p.s;
    const BrDraw dr = br_index_draw(p, g, ell, r, t);
    tab[e] = ((unsigned long long)nb[ell - 1] * p.B_c + dr.i) | ((unsigned long long)dr.neg << 63);
  }
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.z * 32;
  for (uint32_t w = threadIdx.x; w < nr * 32; w += kThreads) {
    const uint32_t rl = w % nr;  // consecutive threads: consecutive output rows (coalesced stores)
    const int64_t t = t0 + w / nr;
    if (t >= n) continue;
    float acc = 0.f;
    const unsigned long long* tb = tab + (size_t)rl * ks;
    for (uint32_t c = 0; c < ks; ++c) {
      const unsigned long long cw = tb[c];
      const int64_t idx = (int64_t)(cw & 0x7FFFFFFFFFFFFFFFull);
      const float xv = BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(Xv)[t * ldx + idx])
                            : reinterpret_cast<const float*>(Xv)[t * ldx + idx];
      acc = (cw >> 63) ? acc - xv : acc + xv;
    }
    Yt[t * ldyt + (int64_t)g * p.B_r + r_begin + rl] = acc * p.scale;
  }
}

template <bool BF16, int LPR, int V>
int launch_rm(const BlockRowParams& p, const void* A, int64_t lda, int64_t n, float* Y, int64_t ldy, cudaStream_t st) {
  constexpr int TN = LPR * V * (BF16 ? 8 : 4);
  const int64_t ntiles = (n + TN - 1) / TN;
  if (ntiles > 65535) return fail(BPS_ERR_UNSUPPORTED, "blockrow: n too large for the grid");
  // rows per CTA = one iteration of every warp (G rows each): many small CTAs keep loads in flight
  constexpr uint32_t RPW = 32 / LPR;
  const uint32_t ks = p.kappa * p.s;
  const uint32_t G = RPW * std::min<uint32_t>(kQMax, std::max<uint32_t>(1, 32 / (RPW * ks)));
  const uint32_t rows_per_cta = std::max<uint32_t>(1, std::min<uint32_t>(p.B_r, kWarps * G));
  const uint32_t ny = (p.B_r + rows_per_cta - 1) / rows_per_cta;
  if (ny > 65535) return fail(BPS_ERR_UNSUPPORTED, "blockrow: B_r too large for the grid");
  blockrow_rowmajor_kernel<BF16, LPR, V><<<dim3(p.M, ny, (unsigned)ntiles), kThreads, 0, st>>>(p, A, lda, n, Y, ldy,
                                                                                              rows_per_cta);
  return BPS_OK;
}

}  // namespace

int launch_blockrow(const BlockRowParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y,
                    int64_t ldy, bool transposed, cudaStream_t st) {
  const bool bf = dt == BPS_BF16;
  int rc;
  if (!transposed) {
    // one 16-byte vector per lane and row: narrow column tiles give many independent warps
    // (the gather is latency-bound: parallelism, not per-warp work, sets the bandwidth)
    if (bf)
      rc = n > 64 ? launch_rm<true, 32, 1>(p, A, lda, n, Y, ldy, st)
           : n > 32 ? launch_rm<true, 8, 1>(p, A, lda, n, Y, ldy, st)
                    : launch_rm<true, 4, 1>(p, A, lda, n, Y, ldy, st);
    else
      rc = n > 64 ? launch_rm<false, 32, 1>(p, A, lda, n, Y, ldy, st)
           : n > 32 ? launch_rm<false, 16, 1>(p, A, lda, n, Y, ldy, st)
                    : launch_rm<false, 8, 1>(p, A, lda, n, Y, ldy, st);
  } else {
    const uint32_t ks = p.kappa * p.s;
    if (ks > 4096) return fail(BPS_ERR_UNSUPPORTED, "blockrow transposed: kappa*s must be <= 4096");
    const uint32_t rows_per_cta = std::max<uint32_t>(1, std::min<uint32_t>(p.B_r, 4096 / ks));
    const uint32_t ny = (p.B_r + rows_per_cta - 1) / rows_per_cta;
    const int64_t nz = (n + 31) / 32;
    if (ny > 65535 || nz > 65535) return fail(BPS_ERR_UNSUPPORTED, "blockrow transposed: grid too large");
    const size_t smem = (size_t)rows_per_cta * ks * 8;
    auto kern = bf ? blockrow_transposed_kernel<true> : blockrow_transposed_kernel<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<dim3(p.M, ny, (unsigned)nz), kThreads, smem, st>>>(p, A, lda, n, Y, ldy, rows_per_cta);
    rc = BPS_OK;
  }
  if (rc) return rc;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("blockrow kernel: ") + cudaGetErrorString(e));
  return BPS_OK;
}

}  // namespace bps

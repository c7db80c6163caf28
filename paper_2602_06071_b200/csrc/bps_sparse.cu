// bps_sparse.cu — CUDA-core gather kernels for Y = S·A (the "sparse" variant).
//
// Gather form of Alg. 1 without atomics: one CTA per (output block g,
// column tile), κ input blocks streamed, each input element added into s rows of a
// private accumulator.  Differences from the paper's design:
//   * destination rows are warp-uniform (lanes span columns), so each warp owns a
//     private shared-memory accumulator tile and no atomics are needed (P:1701 uses
//     shared-memory atomicAdd);
//   * warps split the rows u of every input block; their tiles are summed in a fixed
//     order at the end, so the result is bitwise reproducible;
//   * the s hash draws of a row are computed by s lanes at once and broadcast by
//     shuffles.
// This is the generic fallback (B_r ≤ 400 row-major, B_r ≤ 192 transposed, any n, both
// layouts); the tcgen05 kernel (bps_tc_kernel.cuh) is the fast path.
// Non-finite results (R12): fp32 partial sums of finite inputs near FLT_MAX can overflow where
// the exact sum does not; such elements are recomputed by one thread in fp64 (exact_elem_1t).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>

#include "bps_internal.h"

namespace bps {
namespace {

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  __device__ static void load(const float* p, int64_t col, int64_t n, float v[4]) {
    if (col + 4 <= n) {
      float4 t = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = (col + c < n) ? __ldg(p + c) : 0.f;
    }
  }
};
template <>
struct Vec4<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, int64_t col, int64_t n, float v[4]) {
    if (col + 4 <= n) {
      uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
      v[0] = __uint_as_float(t.x << 16);
      v[1] = __uint_as_float(t.x & 0xFFFF0000u);
      v[2] = __uint_as_float(t.y << 16);
      v[3] = __uint_as_float(t.y & 0xFFFF0000u);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = (col + c < n) ? __bfloat162float(p[c]) : 0.f;
    }
  }
};

template <typename T>
__device__ __forceinline__ float ld1(const T* p);
template <>
__device__ __forceinline__ float ld1<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

__device__ __forceinline__ uint32_t block_g(const SketchParams& p, int range_mode, int64_t pos_begin, uint32_t o) {
  return range_mode ? affine_pow(p, (uint64_t)pos_begin + o, 0u) : o;
}

// One element of Y by the sparse definition (Alg. 1), fp64, one thread: output o of
// the launch (full mode: block g = o; range mode: orbit position pos_begin + o), row r, column t.
template <typename T, bool TRANS>
__device__ float exact_elem_1t(const SketchParams& p, const T* A, int64_t lda, int range_mode, int64_t pos_begin,
                               uint32_t o, uint32_t g, uint32_t r, int64_t t) {
  double acc = 0.0;
  uint32_t h = g;
  for (uint32_t ell = 1; ell <= p.kappa; ++ell) {
    h = affine_step(p, h);
    const int64_t hrow = (range_mode ? (int64_t)o + ell - 1 : (int64_t)h) * p.B_c;
    for (uint32_t u = 0; u < p.B_c; ++u) {
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
        hit = d.row == r, neg = d.neg;
      }
      if (!hit) continue;
      const float v = ld1<T>(TRANS ? A + t * lda + hrow + u : A + (hrow + u) * lda + t);
      acc += neg ? -(double)v : (double)v;
    }
  }
  (void)pos_begin;
  return (float)(acc * (double)p.scale);
}

__device__ __forceinline__ bool not_finite(float v) { return (__float_as_uint(v) & 0x7F800000u) == 0x7F800000u; }

constexpr int kRowsPerIter = 4;  // rows u in flight per warp (ILP)

// Row-major A (d×n), Y (k×n).  Block = 32·W threads, tile = 128 columns (4 per lane).
template <typename T>
__global__ void __launch_bounds__(256) sparse_rowmajor_kernel(SketchParams p, const T* __restrict__ A, int64_t lda,
                                                               int64_t n, float* __restrict__ Y, int64_t ldy,
                                                               int range_mode, int64_t pos_begin) {
  extern __shared__ float smem[];
  constexpr int TN = 128;
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t o = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * TN;
  const uint32_t g = block_g(p, range_mode, pos_begin, o);
  const int64_t y_row = (int64_t)(range_mode ? o : g) * p.B_r;

  for (int e = threadIdx.x; e < W * (int)p.B_r * TN; e += blockDim.x) smem[e] = 0.f;
  __syncthreads();

  float* acc = smem + (size_t)warp * p.B_r * TN + lane * 4;
  const int64_t col = col0 + lane * 4;
  uint32_t h = g;
  for (uint32_t ell = 1; ell <= p.kappa; ++ell) {
    h = affine_step(p, h);
    const int64_t in_blk = range_mode ? (int64_t)o + ell - 1 : (int64_t)h;
    const T* Ablk = A + in_blk * p.B_c * lda + col;
    for (uint32_t u0 = warp * kRowsPerIter; u0 < p.B_c; u0 += W * kRowsPerIter) {
      float v[kRowsPerIter][4];
#pragma unroll
      for (int r = 0; r < kRowsPerIter; ++r) {
        const uint32_t u = u0 + r;
        if (u < p.B_c && col < n)
          Vec4<T>::load(Ablk + (int64_t)u * lda, col, n, v[r]);
        else
          v[r][0] = v[r][1] = v[r][2] = v[r][3] = 0.f;
      }
      // lanes compute the kRowsPerIter·s draws of this row group, 32 at a time
      const uint32_t npairs = kRowsPerIter * p.s;
      for (uint32_t base = 0; base < npairs; base += 32) {
        const uint32_t q = base + lane;
        Draw dr{0, 0};
        if (q < npairs) {
          const uint32_t rr = q / p.s, j = q % p.s;
          const uint32_t u = u0 + rr;
          if (u < p.B_c) dr = pattern(p, g, ell, u, j);
        }
        const uint32_t cnt = min(32u, npairs - base);
        for (uint32_t t = 0; t < cnt; ++t) {
          const uint32_t row = __shfl_sync(0xffffffffu, dr.row, t);
          const uint32_t neg = __shfl_sync(0xffffffffu, dr.neg, t);
          const uint32_t rr = (base + t) / p.s;
          if (u0 + rr >= p.B_c) continue;  // warp-uniform
          float* a = acc + (size_t)row * TN;
          float4 cur = *reinterpret_cast<float4*>(a);
          float vv[4] = {v[0][0], v[0][1], v[0][2], v[0][3]};
#pragma unroll
          for (int c = 1; c < kRowsPerIter; ++c)
            if ((int)rr == c) { vv[0] = v[c][0]; vv[1] = v[c][1]; vv[2] = v[c][2]; vv[3] = v[c][3]; }
          if (neg) {
            cur.x -= vv[0]; cur.y -= vv[1]; cur.z -= vv[2]; cur.w -= vv[3];
          } else {
            cur.x += vv[0]; cur.y += vv[1]; cur.z += vv[2]; cur.w += vv[3];
          }
          *reinterpret_cast<float4*>(a) = cur;
        }
      }
    }
  }
  __syncthreads();
  // fixed-order reduction over warps, scale, coalesced store
  for (int e = threadIdx.x; e < (int)p.B_r * TN; e += blockDim.x) {
    const int r = e / TN, c = e % TN;
    const int64_t cc = col0 + c;
    if (cc >= n) continue;
    float s = 0.f;
    for (int w = 0; w < W; ++w) s += smem[(size_t)w * p.B_r * TN + e];
    float y = s * p.scale;
    if (not_finite(y)) y = exact_elem_1t<T, false>(p, A, lda, range_mode, pos_begin, o, g, (uint32_t)r, cc);
    Y[(y_row + r) * ldy + cc] = y;
  }
}

// Transposed layout: X n×d (vectors in rows), Yt n×k.  CTA = output block × 128 vectors,
// 8 warps = 4 vector groups × 2 row-parities; X tiles staged through smem.
constexpr int kTK = 32;
template <typename T>
__global__ void __launch_bounds__(256) sparse_transposed_kernel(SketchParams p, const T* __restrict__ X, int64_t ldx,
                                                                 int64_t n, float* __restrict__ Yt, int64_t ldyt,
                                                                 int range_mode, int64_t pos_begin) {
  extern __shared__ float smem[];
  float* tile = smem;                      // [128][kTK+1]
  float* accs = smem + 128 * (kTK + 1);    // [8][B_r][33]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vg = warp & 3, uh = warp >> 2;
  const uint32_t o = blockIdx.x;
  const int64_t v0 = (int64_t)blockIdx.y * 128;
  const uint32_t g = block_g(p, range_mode, pos_begin, o);
  const int64_t y_col = (int64_t)(range_mode ? o : g) * p.B_r;
  for (int e = threadIdx.x; e < 8 * (int)p.B_r * 33; e += blockDim.x) accs[e] = 0.f;
  float* acc = accs + (size_t)warp * p.B_r * 33 + lane;

  uint32_t h = g;
  for (uint32_t ell = 1; ell <= p.kappa; ++ell) {
    h = affine_step(p, h);
    const int64_t in_blk = range_mode ? (int64_t)o + ell - 1 : (int64_t)h;
    const int64_t coord0 = in_blk * p.B_c;
    for (uint32_t u0 = 0; u0 < p.B_c; u0 += kTK) {
      __syncthreads();
      for (int i = threadIdx.x; i < 128 * kTK; i += blockDim.x) {
        const int uu = i % kTK, vv = i / kTK;
        float x = 0.f;
        if (v0 + vv < n && u0 + uu < p.B_c) x = ld1<T>(X + (v0 + vv) * ldx + coord0 + u0 + uu);
        tile[vv * (kTK + 1) + uu] = x;
      }
      __syncthreads();
      for (int uu = uh; uu < kTK && u0 + uu < p.B_c; uu += 2) {
        const float x = tile[(vg * 32 + lane) * (kTK + 1) + uu];
        for (uint32_t jb = 0; jb < p.s; jb += 32) {
          Draw dr{0, 0};
          if (jb + lane < p.s) dr = pattern(p, g, ell, u0 + uu, jb + lane);
          const uint32_t cnt = min(32u, p.s - jb);
          for (uint32_t t = 0; t < cnt; ++t) {
            const uint32_t row = __shfl_sync(0xffffffffu, dr.row, t);
            const uint32_t neg = __shfl_sync(0xffffffffu, dr.neg, t);
            acc[row * 33] += neg ? -x : x;
          }
        }
      }
    }
  }
  __syncthreads();
  // Yt[v][y_col + r] = (acc(vg,0) + acc(vg,1))[r][v] · scale ; lanes run over r (coalesced)
  for (int job = warp; job < 128; job += 8) {  // job = vector index inside the tile
    const int vgi = job >> 5, vl = job & 31;
    const int64_t v = v0 + job;
    if (v >= n) continue;
    for (uint32_t r = lane; r < p.B_r; r += 32) {
      const float a0 = accs[((size_t)(vgi)*p.B_r + r) * 33 + vl];
      const float a1 = accs[((size_t)(vgi + 4) * p.B_r + r) * 33 + vl];
      float y = (a0 + a1) * p.scale;
      if (not_finite(y)) y = exact_elem_1t<T, true>(p, X, ldx, range_mode, pos_begin, o, g, r, v);
      Yt[v * ldyt + y_col + r] = y;
    }
  }
}

static int launch_err(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return BPS_OK;
}

}  // namespace

int launch_sparse_rowmajor(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y,
                           int64_t ldy, const Placement& pl, cudaStream_t st) {
  constexpr int TN = 128;
  const size_t tile_bytes = (size_t)p.B_r * TN * 4;
  const size_t budget = 200 * 1024;
  int W = (int)(budget / tile_bytes);
  if (W < 1) return fail(BPS_ERR_UNSUPPORTED, "sparse kernel: B_r too large for the shared-memory accumulator (B_r <= 400)");
  if (W > 8) W = 8;
  const size_t smem = tile_bytes * W;
  const int64_t ntiles = (n + TN - 1) / TN;
  if (ntiles > 65535) return fail(BPS_ERR_UNSUPPORTED, "sparse kernel: n too large for grid.y");
  dim3 grid((unsigned)pl.n_out, (unsigned)ntiles), block(32 * W);
  cudaEvent_t tev[2] = {nullptr, nullptr};
  const bool timed = timing_begin(st, tev);
  if (dt == BPS_F32) {
    cudaFuncSetAttribute(sparse_rowmajor_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sparse_rowmajor_kernel<float><<<grid, block, smem, st>>>(p, (const float*)A, lda, n, Y, ldy, pl.range_mode,
                                                             pl.pos_begin);
  } else {
    cudaFuncSetAttribute(sparse_rowmajor_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sparse_rowmajor_kernel<__nv_bfloat16><<<grid, block, smem, st>>>(p, (const __nv_bfloat16*)A, lda, n, Y, ldy,
                                                                     pl.range_mode, pl.pos_begin);
  }
  if (timed) timing_end(st, tev);
  return launch_err("sparse_rowmajor_kernel");
}

int launch_sparse_transposed(const SketchParams& p, const void* X, int64_t ldx, int64_t n, bps_dtype dt, float* Yt,
                             int64_t ldyt, const Placement& pl, cudaStream_t st) {
  const size_t smem = (size_t)128 * (kTK + 1) * 4 + (size_t)8 * p.B_r * 33 * 4;
  if (smem > 220 * 1024) return fail(BPS_ERR_UNSUPPORTED, "sparse transposed kernel: B_r too large (B_r <= 192)");
  const int64_t ntiles = (n + 127) / 128;
  if (ntiles > 65535) return fail(BPS_ERR_UNSUPPORTED, "sparse kernel: n too large for grid.y");
  dim3 grid((unsigned)pl.n_out, (unsigned)ntiles), block(256);
  cudaEvent_t tev[2] = {nullptr, nullptr};
  const bool timed = timing_begin(st, tev);
  if (dt == BPS_F32) {
    cudaFuncSetAttribute(sparse_transposed_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sparse_transposed_kernel<float><<<grid, block, smem, st>>>(p, (const float*)X, ldx, n, Yt, ldyt, pl.range_mode,
                                                               pl.pos_begin);
  } else {
    cudaFuncSetAttribute(sparse_transposed_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    sparse_transposed_kernel<__nv_bfloat16><<<grid, block, smem, st>>>(p, (const __nv_bfloat16*)X, ldx, n, Yt, ldyt,
                                                                       pl.range_mode, pl.pos_begin);
  }
  if (timed) timing_end(st, tev);
  return launch_err("sparse_transposed_kernel");
}

}  // namespace bps

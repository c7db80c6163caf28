// bps_adjoint.cu — X = Sᵀ·Y, the adjoint of the sketch.
//
// Block form: X^(h) = κ^{-1/2} Σ_{g : h ∈ N(g)} Φ_{g,h}ᵀ Y^(g) (transpose of P:36-42).  With the
// orbit ordering the input block h = g_p is fed by the outputs g_{p-1..p-κ},
// and row u of X^(h) is a pure gather:
//   X[h·B_c+u, :] = (κs)^{-1/2} Σ_{ℓ=1..κ} Σ_{j<s} σ(g_{p-ℓ},ℓ,u,j) · Y[g_{p-ℓ}·B_r + row(g_{p-ℓ},ℓ,u,j), :]
// with the same counter-hash draws as the forward sketch (R1-R3) — no atomics, every element
// written once (bitwise reproducible).
//
// CTA = (orbit position p, TN-column tile, chunk of rows u).  The Y rows of the κ feeding output
// blocks (κ·B_r × TN fp32, L2-resident across CTAs) are staged in shared memory once per CTA.
// A warp processes G rows u per iteration: its 32 lanes draw the G·κs hashes of those rows (one
// per lane per pass) into a per-warp code table (row-in-window | sign), then lane groups of LPR
// lanes (one group per row, each lane owning 4·V columns) gather ±Y rows from shared memory with
// packed fp32 FMAs (fma.rn.f32x2: acc + (±1)·y is the exactly rounded acc ± y).  The output is
// written with 16-byte coalesced streaming stores; the kernel is HBM-write bound (roofline:
// d·n·4 bytes written + k·n·4 read per launch) once the FMA issue rate (κs FMAs per output) fits.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "bps_internal.h"

namespace bps {
namespace {

constexpr uint32_t kMaxKappa = 64;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kQMax = 4;  // rows per lane group per iteration

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// LPR lanes per row, V float4 per lane: TN = 4·LPR·V columns per CTA tile.
template <int LPR, int V>
__global__ void __launch_bounds__(kThreads, V == 1 ? 2 : 1)
    adjoint_kernel(SketchParams p, const float* __restrict__ Y, int64_t ldy, int64_t n, float* __restrict__ X,
                   int64_t ldx, uint32_t u_chunk) {
  constexpr int TN = LPR * 4 * V;
  constexpr int RPW = 32 / LPR;  // rows processed concurrently by one warp
  extern __shared__ uint4 ys[];  // [κ·B_r][TN/4] fp32, row ρ = (ℓ-1)·B_r + r
  __shared__ uint32_t gl[kMaxKappa];
  __shared__ uint32_t codes[kWarps][32];

  const uint32_t pos = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * TN;
  const uint32_t u_begin = blockIdx.z * u_chunk;
  const uint32_t u_end = min(p.B_c, u_begin + u_chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kappa = p.kappa, ks = p.kappa * p.s;
  const uint32_t h = affine_pow(p, pos, 0u);

  // gl[ℓ-1] = g_{p-ℓ}: the output block that reaches h through its ℓ-th neighbour (f^ℓ(g) = h)
  for (uint32_t e = threadIdx.x; e < kappa; e += kThreads)
    gl[e] = affine_pow(p, (uint64_t)((pos + p.M - ((e + 1) % p.M)) % p.M), 0u);
  __syncthreads();
  const uint32_t rows = kappa * p.B_r;
  for (uint32_t e = threadIdx.x; e < rows * (TN / 4); e += kThreads) {
    const uint32_t lr = e / (TN / 4), c4 = e % (TN / 4);
    const int64_t col = col0 + c4 * 4;
    const float* src = Y + ((int64_t)gl[lr / p.B_r] * p.B_r + lr % p.B_r) * ldy + col;
    float4 v;
    if (col + 4 <= n) {
      v = __ldg(reinterpret_cast<const float4*>(src));
    } else {
      v.x = col < n ? src[0] : 0.f;
      v.y = col + 1 < n ? src[1] : 0.f;
      v.z = col + 2 < n ? src[2] : 0.f;
      v.w = col + 3 < n ? src[3] : 0.f;
    }
    ys[e] = make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
  }
  __syncthreads();

  // q rows per lane group per iteration so that G·κs fills the 32 hash lanes when κs is small
  const uint32_t q = min((uint32_t)kQMax, max(1u, 32u / (RPW * ks)));
  const uint32_t G = RPW * q;  // rows per warp iteration; row r of the iteration is u0 + r, r = i·RPW + grp
  const int grp = lane / LPR, gl_lane = lane % LPR;
  const int64_t col = col0 + (int64_t)gl_lane * 4 * V;
  const uint32_t T = G * ks;
  const uint64_t one2 = 0x3F8000003F800000ull, neg2 = 0xBF800000BF800000ull;

  for (uint32_t u0 = u_begin + warp * G; u0 < u_end; u0 += kWarps * G) {
    uint64_t acc[kQMax][2 * V];
#pragma unroll
    for (int i = 0; i < kQMax; ++i)
#pragma unroll
      for (int v = 0; v < 2 * V; ++v) acc[i][v] = 0;
    for (uint32_t c0 = 0; c0 < T; c0 += 32) {
      const uint32_t c = c0 + lane;
      uint32_t code = 0;
      if (c < T) {
        const uint32_t u = u0 + c / ks, cc = c % ks;
        const uint32_t ell = cc / p.s + 1, j = cc % p.s;
        if (u < u_end) {
          const Draw dr = pattern(p, gl[ell - 1], ell, u, j);
          code = (((ell - 1) * p.B_r + dr.row) * (TN / 4)) | (dr.neg << 31);
        }
      }
      __syncwarp();
      codes[warp][lane] = code;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < kQMax; ++i) {
        if ((uint32_t)i < q) {
          const uint32_t r = (uint32_t)i * RPW + grp;
          const uint32_t lo = max(r * ks, c0), hi = min((r + 1) * ks, min(c0 + 32, T));
#pragma unroll 4
          for (uint32_t t = lo; t < hi; ++t) {
            const uint32_t cw = codes[warp][t - c0];
            const uint64_t sg = (cw >> 31) ? neg2 : one2;
            const uint4* row = ys + (cw & 0x7FFFFFFFu) + gl_lane * V;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const uint4 y = row[v];
              acc[i][2 * v] = ffma2(((uint64_t)y.y << 32) | y.x, sg, acc[i][2 * v]);
              acc[i][2 * v + 1] = ffma2(((uint64_t)y.w << 32) | y.z, sg, acc[i][2 * v + 1]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kQMax; ++i) {
      if ((uint32_t)i >= q) break;
      const uint32_t u = u0 + (uint32_t)i * RPW + grp;
      if (u >= u_end) continue;
      float* dst = X + ((int64_t)h * p.B_c + u) * ldx + col;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float4 o;
        o.x = __uint_as_float((uint32_t)acc[i][2 * v]) * p.scale;
        o.y = __uint_as_float((uint32_t)(acc[i][2 * v] >> 32)) * p.scale;
        o.z = __uint_as_float((uint32_t)acc[i][2 * v + 1]) * p.scale;
        o.w = __uint_as_float((uint32_t)(acc[i][2 * v + 1] >> 32)) * p.scale;
        const int64_t cv = col + 4 * v;
        if (cv + 4 <= n) {
          __stcs(reinterpret_cast<float4*>(dst + 4 * v), o);
        } else {
          if (cv < n) dst[4 * v] = o.x;
          if (cv + 1 < n) dst[4 * v + 1] = o.y;
          if (cv + 2 < n) dst[4 * v + 2] = o.z;
        }
      }
    }
  }
}

template <int LPR, int V>
int launch_t(const SketchParams& p, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx, cudaStream_t st) {
  constexpr int TN = LPR * 4 * V;
  const size_t smem = (size_t)p.kappa * p.B_r * TN * 4;
  auto kern = adjoint_kernel<LPR, V>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("adjoint attr: ") + cudaGetErrorString(e));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  per_sm = per_sm < 1 ? 1 : per_sm;
  const int64_t ntiles = (n + TN - 1) / TN;
  // split rows u so the grid covers ≥ ~8 waves (tail < 1/8); each chunk re-stages its Y window from L2
  const int64_t base = (int64_t)p.M * ntiles;
  int64_t nch = (8LL * sms * per_sm + base - 1) / base;
  nch = std::min<int64_t>(nch, std::max<int64_t>(1, p.B_c / 256));
  nch = std::min<int64_t>(nch, 65535);
  const uint32_t u_chunk = (uint32_t)((p.B_c + nch - 1) / nch);
  nch = (p.B_c + u_chunk - 1) / u_chunk;
  kern<<<dim3(p.M, (unsigned)ntiles, (unsigned)nch), kThreads, smem, st>>>(p, Y, ldy, n, X, ldx, u_chunk);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("adjoint_kernel: ") + cudaGetErrorString(e));
  return BPS_OK;
}

}  // namespace

int launch_adjoint(const SketchParams& p, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                   cudaStream_t st) {
  if (p.kappa > kMaxKappa) return fail(BPS_ERR_UNSUPPORTED, "adjoint: kappa must be <= 64");
  const uint64_t win = (uint64_t)p.kappa * p.B_r;  // Y rows staged per CTA
  if (win > 400) return fail(BPS_ERR_UNSUPPORTED, "adjoint: kappa*B_r must be <= 400");
  if ((n + 127) / 128 > 65535) return fail(BPS_ERR_UNSUPPORTED, "adjoint: n too large for the grid");
  const size_t budget = 200 * 1024;
  (void)budget;  // TN = 256 (V = 2) measured slower: shared-memory bandwidth bound
  if (n > 64) return launch_t<32, 1>(p, Y, ldy, n, X, ldx, st);
  if (n > 32) return launch_t<16, 1>(p, Y, ldy, n, X, ldx, st);
  return launch_t<8, 1>(p, Y, ldy, n, X, ldx, st);
}

}  // namespace bps

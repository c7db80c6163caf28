// bps_api.cu — the C ABI of libbps (include/bps.h): handle creation, validation and
// kernel dispatch.  All hot work happens in bps_sparse.cu / bps_tc.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "bps_internal.h"

namespace bps {

static thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

// ---- live timing of the dominant kernel (bps_timing_enable / bps_timing_read)
static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_tev, g_tev_aux;
bool timing_begin(cudaStream_t st, cudaEvent_t ev[2]) {
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing) return false;
  }
  if (cudaEventCreate(&ev[0]) != cudaSuccess || cudaEventCreate(&ev[1]) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaEventRecord(ev[0], st);
  return true;
}
void timing_end(cudaStream_t st, cudaEvent_t ev[2], bool aux) {
  cudaEventRecord(ev[1], st);
  std::lock_guard<std::mutex> lk(g_tmu);
  (aux ? g_tev_aux : g_tev).emplace_back(ev[0], ev[1]);
}
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static uint64_t rad(uint64_t M) {
  uint64_t r = 1, m = M;
  for (uint64_t q = 2; q * q <= m; ++q) {
    if (m % q == 0) {
      r *= q;
      while (m % q == 0) m /= q;
    }
  }
  if (m > 1) r *= m;
  return r;
}

// R4: (a, b) from the seed, Hull–Dobell full period.
static void select_affine(uint64_t seed, uint64_t M, uint32_t* a, uint32_t* b) {
  if (M == 1) {
    *a = 0;
    *b = 0;
    return;
  }
  uint64_t q = rad(M);
  if (M % 4 == 0) q *= 2;
  *a = (uint32_t)((1 + q * (mix64(seed ^ kTagA) % (M / q))) % M);
  for (uint64_t t = 0;; ++t) {
    uint64_t bb = mix64(seed ^ kTagB ^ t) % M;
    if (std::gcd(bb, M) == 1) {
      *b = (uint32_t)bb;
      return;
    }
  }
}

// Device check: cc 10.0 required (BJ: no multi-backend dispatch).
static int check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(BPS_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  static std::mutex mu;
  static int cached[64];
  static bool init = false;
  std::lock_guard<std::mutex> lk(mu);
  if (!init) {
    for (int& c : cached) c = -1;
    init = true;
  }
  if (dev < 0 || dev >= 64) return fail(BPS_ERR_CUDA, "device ordinal out of range");
  if (cached[dev] < 0) {
    int maj = 0, min = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return fail(BPS_ERR_CUDA, "cudaDeviceGetAttribute failed");
    cached[dev] = maj * 10 + min;
  }
  if (cached[dev] != 100)
    return fail(BPS_ERR_ARCH, "libbps is built for sm_100a (B200); current device has cc " +
                                  std::to_string(cached[dev] / 10) + "." + std::to_string(cached[dev] % 10));
  return BPS_OK;
}

static int elem_size(bps_dtype dt) { return dt == BPS_F32 ? 4 : (dt == BPS_BF16 ? 2 : 0); }

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// Common validation for the three apply entry points.
static int validate_apply(const bps_sketch* sk, const void* in, int64_t ldin, int64_t in_rows, int64_t in_cols,
                          bps_dtype dt, const float* out, int64_t ldout, int64_t out_rows, int64_t out_cols,
                          int variant) {
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "sketch handle is NULL");
  const int es = elem_size(dt);
  if (!es) return fail(BPS_ERR_INVALID_ARG, "dtype must be BPS_F32 or BPS_BF16");
  if (variant < BPS_VARIANT_AUTO || variant > BPS_VARIANT_TC) return fail(BPS_ERR_INVALID_ARG, "unknown variant");
  if (in_rows < 0 || in_cols < 0 || out_rows < 0 || out_cols < 0) return fail(BPS_ERR_INVALID_ARG, "negative size");
  if (in_rows == 0 || in_cols == 0 || out_rows == 0 || out_cols == 0) return BPS_OK;  // n == 0: no-op
  if (!in || !out) return fail(BPS_ERR_INVALID_ARG, "NULL data pointer");
  if (ldin < in_cols) return fail(BPS_ERR_INVALID_ARG, "input leading dimension smaller than its row length");
  if (ldout < out_cols) return fail(BPS_ERR_INVALID_ARG, "output leading dimension smaller than its row length");
  if (ldin > (int64_t(1) << 40) || ldout > (int64_t(1) << 40)) return fail(BPS_ERR_OVERFLOW, "leading dimension too large");
  if (((uintptr_t)in % 16) || ((uintptr_t)out % 16) || ((ldin * es) % 16) || ((ldout * 4) % 16))
    return fail(BPS_ERR_ALIGNMENT, "pointers and leading dimensions must be 16-byte aligned");
  const size_t in_bytes = (size_t)((in_rows - 1) * ldin + in_cols) * es;
  const size_t out_bytes = (size_t)((out_rows - 1) * ldout + out_cols) * 4;
  if (overlaps(in, in_bytes, out, out_bytes)) return fail(BPS_ERR_INVALID_ARG, "input and output overlap");
  return BPS_OK;
}

static int dispatch(const bps_sketch* sk, const void* in, int64_t ldin, int64_t n, bps_dtype dt, float* out,
                    int64_t ldout, bool transposed, const Placement& pl, void* stream, int variant,
                    void* ws = nullptr, size_t ws_bytes = 0) {
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (sk->kind == 1) {  // FlashBlockRow: one gather kernel (no tcgen05 variant, no ranges, no workspace)
    if (variant == BPS_VARIANT_TC) return fail(BPS_ERR_UNSUPPORTED, "blockrow sketch: only the gather kernel");
    if (pl.range_mode) return fail(BPS_ERR_UNSUPPORTED, "blockrow sketch: no orbit ranges");
    return launch_blockrow(sk->br, in, ldin, n, dt, out, ldout, transposed, st);
  }
  const bool tc_ok = tc_supported(sk->p, n, dt, transposed, pl) == BPS_OK;
  if (variant == BPS_VARIANT_TC && !tc_ok) return BPS_ERR_UNSUPPORTED;  // message set by tc_supported
  if (tc_ok && variant != BPS_VARIANT_SPARSE) {
    const int rc = launch_tc(sk->p, in, ldin, n, dt, out, ldout, transposed, pl, ws, ws_bytes, st);
    // AUTO: a shape the tc planner cannot launch runs on the sparse kernel (bps.h), nothing was enqueued
    if (rc != BPS_ERR_UNSUPPORTED || variant == BPS_VARIANT_TC) return rc;
  }
  if (transposed) return launch_sparse_transposed(sk->p, in, ldin, n, dt, out, ldout, pl, st);
  rc = launch_sparse_rowmajor(sk->p, in, ldin, n, dt, out, ldout, pl, st);
  // the CUDA-core kernel has no fused broadcast: copy the finished rows to the destinations
  if (rc == BPS_OK && pl.bc) rc = launch_bcast_rows(out, ldout, pl.n_out * sk->B_r, n, *pl.bc, st);
  return rc;
}

// Unfused broadcast copy: one thread per 4 consecutive elements of a row (row-major).
__global__ void bps_bcast_rows_kernel(const float* __restrict__ Y, int64_t ldy, int64_t rows, int64_t n,
                                      const __grid_constant__ Broadcast bc) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, per = (n + 3) / 4;
  if (q >= rows * per) return;
  const int64_t r = q / per, c = (q % per) * 4;
  for (int64_t e = c; e < c + 4 && e < n; ++e) {
    const float v = Y[r * ldy + e];
    const int64_t off = (bc.row0 + r) * bc.ld + e;
    for (int j = 0; j < bc.npeer; ++j) bc.peer[j][off] = v;
    if (bc.mc) asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(bc.mc + off), "f"(v) : "memory");
  }
}

int launch_bcast_rows(const float* Y, int64_t ldy, int64_t rows, int64_t n, const Broadcast& bc, cudaStream_t st) {
  const int64_t work = rows * ((n + 3) / 4);
  if (work <= 0) return BPS_OK;
  const int64_t blocks = (work + 255) / 256;
  if (blocks > 0x7FFFFFFF) return fail(BPS_ERR_UNSUPPORTED, "broadcast grid too large");
  bps_bcast_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(Y, ldy, rows, n, bc);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPS_OK : fail(BPS_ERR_CUDA, std::string("broadcast launch: ") + cudaGetErrorString(e));
}

}  // namespace bps

using namespace bps;

extern "C" {

const char* bps_last_error(void) { return g_last_error.c_str(); }

uint64_t bps_kernel_launches(void) { return g_launches.load(); }

int bps_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
  return BPS_OK;
}

int bps_timing_read_ex(int aux, double* total_ms, uint64_t* count) {
  if (!total_ms || !count) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    evs.swap(aux ? g_tev_aux : g_tev);
  }
  double tot = 0;
  int rc = BPS_OK;
  for (auto& pr : evs) {
    float ms = 0;
    cudaError_t e = cudaEventSynchronize(pr.second);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, pr.first, pr.second);
    if (e != cudaSuccess) rc = fail(BPS_ERR_CUDA, std::string("bps_timing_read: ") + cudaGetErrorString(e));
    tot += ms;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  *total_ms = tot;
  *count = evs.size();
  return rc;
}

int bps_timing_read(double* total_ms, uint64_t* count) { return bps_timing_read_ex(0, total_ms, count); }

const char* bps_version(void) { return "bps 0.1 sm_100a (sparse gather + tcgen05 NT band kernel)"; }

int bps_make_sketch_ex(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s, uint64_t seed, int mode,
                       bps_sketch** out) {
  if (!out) return fail(BPS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (mode != BPS_MODE_ROWPART && mode != BPS_MODE_AFFINE) return fail(BPS_ERR_INVALID_ARG, "unknown intra-block mode");
  if (M < 1 || B_r < 1 || B_c < 1) return fail(BPS_ERR_INVALID_ARG, "M, B_r, B_c must be >= 1");
  if (M >= (int64_t(1) << 24)) return fail(BPS_ERR_INVALID_ARG, "M must be < 2^24 (counter field, R2)");
  if (B_c >= (int64_t(1) << 24)) return fail(BPS_ERR_INVALID_ARG, "B_c must be < 2^24 (counter field, R2)");
  if (B_r >= (int64_t(1) << 31)) return fail(BPS_ERR_INVALID_ARG, "B_r too large");
  if (kappa < 1 || kappa > M || kappa > 256) return fail(BPS_ERR_INVALID_ARG, "need 1 <= kappa <= min(M, 256) (P:1531)");
  if (mode == BPS_MODE_AFFINE) {
    if ((B_r & (B_r - 1)) != 0 || B_r > 65536 || s < 1 || s > B_r || s > 32)
      return fail(BPS_ERR_INVALID_ARG, "AffineUnique: B_r a power of two <= 2^16 and 1 <= s <= min(B_r, 32) (R18)");
  } else if (s < 1 || s > B_r || s > 256 || B_r % s != 0) {
    return fail(BPS_ERR_INVALID_ARG, "need 1 <= s <= min(B_r, 256) and B_r % s == 0 (row-partitioned, R1)");
  }
  if (M > (int64_t(1) << 62) / B_c || M > (int64_t(1) << 62) / B_r) return fail(BPS_ERR_OVERFLOW, "M*B_c or M*B_r overflows");
  bps_sketch* sk = new (std::nothrow) bps_sketch;
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "out of host memory");
  sk->kind = 0;
  sk->br = BlockRowParams{};
  sk->M = M;
  sk->B_r = B_r;
  sk->B_c = B_c;
  sk->d = M * B_c;
  sk->k = M * B_r;
  sk->kappa = kappa;
  sk->s = s;
  sk->seed = seed;
  SketchParams& p = sk->p;
  p.M = (uint32_t)M;
  p.B_r = (uint32_t)B_r;
  p.B_c = (uint32_t)B_c;
  p.kappa = (uint32_t)kappa;
  p.s = (uint32_t)s;
  p.C = (uint32_t)(B_r / s);
  p.mode = (uint32_t)mode;
  p.Brmask = (uint32_t)(B_r - 1);
  p.Mmask = ((M & (M - 1)) == 0) ? (uint32_t)(M - 1) : 0u;
  select_affine(seed, (uint64_t)M, &p.a, &p.b);
  p.K = mix64(seed ^ kTagPhi);
  p.scale = (float)(1.0 / std::sqrt((double)kappa * (double)s));
  *out = sk;
  return BPS_OK;
}

int bps_make_sketch(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s, uint64_t seed, bps_sketch** out) {
  return bps_make_sketch_ex(M, B_r, B_c, kappa, s, seed, BPS_MODE_ROWPART, out);
}

int bps_sketch_mode(const bps_sketch* sk) {
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "sketch handle is NULL");
  return sk->kind == 0 ? (int)sk->p.mode : fail(BPS_ERR_INVALID_ARG, "not a BlockPerm-SJLT sketch");
}

int bps_make_blockrow(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s, uint64_t seed,
                      bps_sketch** out) {
  if (!out) return fail(BPS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (M < 1 || B_r < 1 || B_c < 1) return fail(BPS_ERR_INVALID_ARG, "M, B_r, B_c must be >= 1");
  if (M >= (int64_t(1) << 24) || B_r >= (int64_t(1) << 24) || B_c >= (int64_t(1) << 24))
    return fail(BPS_ERR_INVALID_ARG, "M, B_r, B_c must be < 2^24 (counter fields, R15)");
  if (kappa < 1 || kappa > M || kappa > 256) return fail(BPS_ERR_INVALID_ARG, "need 1 <= kappa <= min(M, 256) (R14)");
  if (s < 1 || s > 256) return fail(BPS_ERR_INVALID_ARG, "need 1 <= s <= 256 (R15)");
  bps_sketch* sk = new (std::nothrow) bps_sketch;
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "out of host memory");
  sk->kind = 1;
  sk->p = SketchParams{};
  sk->M = M;
  sk->B_r = B_r;
  sk->B_c = B_c;
  sk->d = M * B_c;
  sk->k = M * B_r;
  sk->kappa = kappa;
  sk->s = s;
  sk->seed = seed;
  BlockRowParams& p = sk->br;
  p.M = (uint32_t)M;
  p.B_r = (uint32_t)B_r;
  p.B_c = (uint32_t)B_c;
  p.kappa = (uint32_t)kappa;
  p.s = (uint32_t)s;
  p.Kb = mix64(seed ^ kTagRowBlk);
  p.Ki = mix64(seed ^ kTagRowIdx);
  p.scale = (float)(std::sqrt((double)B_c / (double)B_r) / std::sqrt((double)kappa * (double)s));
  *out = sk;
  return BPS_OK;
}

int bps_blockrow_neighbors(const bps_sketch* sk, int64_t g, int32_t* nb) {
  if (!sk || !nb) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (sk->kind != 1) return fail(BPS_ERR_INVALID_ARG, "not a blockrow sketch");
  if (g < 0 || g >= sk->M) return fail(BPS_ERR_INVALID_ARG, "g out of range");
  int cnt = 0;
  for (uint32_t t = 0; cnt < sk->kappa; ++t) {
    const uint32_t h = br_block_draw(sk->br, (uint32_t)g, t);
    bool dup = false;
    for (int j = 0; j < cnt; ++j) dup |= (uint32_t)nb[j] == h;
    if (!dup) nb[cnt++] = (int32_t)h;
  }
  return BPS_OK;
}

int bps_blockrow_draw_host(const bps_sketch* sk, int64_t g, int32_t ell, int64_t r, int32_t t, int32_t* i,
                           int32_t* sign) {
  if (!sk || !i || !sign) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (sk->kind != 1) return fail(BPS_ERR_INVALID_ARG, "not a blockrow sketch");
  if (g < 0 || g >= sk->M || ell < 1 || ell > sk->kappa || r < 0 || r >= sk->B_r || t < 0 || t >= sk->s)
    return fail(BPS_ERR_INVALID_ARG, "index out of range");
  const BrDraw dr = br_index_draw(sk->br, (uint32_t)g, (uint32_t)ell, (uint32_t)r, (uint32_t)t);
  *i = (int32_t)dr.i;
  *sign = dr.neg ? -1 : 1;
  return BPS_OK;
}

int bps_sketch_kind(const bps_sketch* sk) { return sk ? sk->kind : fail(BPS_ERR_INVALID_ARG, "sketch handle is NULL"); }

void bps_free_sketch(bps_sketch* sk) { delete sk; }

int bps_sketch_info(const bps_sketch* sk, int64_t* d, int64_t* k, uint32_t* a, uint32_t* b, float* scale) {
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "sketch handle is NULL");
  if (d) *d = sk->d;
  if (k) *k = sk->k;
  if (a) *a = sk->p.a;
  if (b) *b = sk->p.b;
  if (scale) *scale = sk->kind == 1 ? sk->br.scale : sk->p.scale;
  return BPS_OK;
}

int bps_orbit(const bps_sketch* sk, int32_t* g_of_pos) {
  if (!sk || !g_of_pos) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (sk->kind != 0) return fail(BPS_ERR_UNSUPPORTED, "orbit: BlockPerm-SJLT sketches only");
  uint32_t x = 0;
  for (int64_t i = 0; i < sk->M; ++i) {
    g_of_pos[i] = (int32_t)x;
    x = affine_step(sk->p, x);
  }
  return BPS_OK;
}

int bps_pattern_host(const bps_sketch* sk, int64_t g, int32_t ell, int64_t u, int32_t j, int32_t* row, int32_t* sign) {
  if (!sk || !row || !sign) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (sk->kind != 0) return fail(BPS_ERR_INVALID_ARG, "pattern: BlockPerm-SJLT sketches only");
  if (g < 0 || g >= sk->M || ell < 1 || ell > sk->kappa || u < 0 || u >= sk->B_c || j < 0 || j >= sk->s)
    return fail(BPS_ERR_INVALID_ARG, "index out of range");
  Draw dr = pattern(sk->p, (uint32_t)g, (uint32_t)ell, (uint32_t)u, (uint32_t)j);
  *row = (int32_t)dr.row;
  *sign = dr.neg ? -1 : 1;
  return BPS_OK;
}

int bps_apply_ex(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype, float* Y, int64_t ldy,
                 void* stream, int variant) {
  int rc = validate_apply(sk, A, lda, sk ? sk->d : 0, n, dtype, Y, ldy, sk ? sk->k : 0, n, variant);
  if (rc || n == 0) return rc;
  Placement pl{0, 0, sk->M};
  return dispatch(sk, A, lda, n, dtype, Y, ldy, false, pl, stream, variant);
}

int bps_apply(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype, float* Y, int64_t ldy,
              void* stream) {
  return bps_apply_ex(sk, A, lda, n, dtype, Y, ldy, stream, BPS_VARIANT_AUTO);
}

int bps_apply_t_ex(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype, float* Yt,
                   int64_t ldyt, void* stream, int variant) {
  int rc = validate_apply(sk, X, ldx, n, sk ? sk->d : 0, dtype, Yt, ldyt, n, sk ? sk->k : 0, variant);
  if (rc || n == 0) return rc;
  Placement pl{0, 0, sk->M};
  return dispatch(sk, X, ldx, n, dtype, Yt, ldyt, true, pl, stream, variant);
}

int bps_apply_t(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype, float* Yt, int64_t ldyt,
                void* stream) {
  return bps_apply_t_ex(sk, X, ldx, n, dtype, Yt, ldyt, stream, BPS_VARIANT_AUTO);
}

int bps_workspace_size(const bps_sketch* sk, int64_t n, bps_dtype dtype, int transposed, size_t* bytes) {
  if (!sk || !bytes) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (n < 0) return fail(BPS_ERR_INVALID_ARG, "negative n");
  Placement pl{0, 0, sk->M};
  *bytes = sk->kind ? 0 : tc_workspace_bytes(sk->p, n, dtype, transposed != 0, pl);
  return BPS_OK;
}

int bps_apply_ws(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype, float* Y, int64_t ldy,
                 void* workspace, size_t workspace_bytes, void* stream, int variant) {
  int rc = validate_apply(sk, A, lda, sk ? sk->d : 0, n, dtype, Y, ldy, sk ? sk->k : 0, n, variant);
  if (rc || n == 0) return rc;
  if (workspace && overlaps(workspace, workspace_bytes, Y, (size_t)((sk->k - 1) * ldy + n) * 4))
    return fail(BPS_ERR_INVALID_ARG, "workspace overlaps the output");
  Placement pl{0, 0, sk->M};
  return dispatch(sk, A, lda, n, dtype, Y, ldy, false, pl, stream, variant, workspace, workspace_bytes);
}

int bps_apply_t_ws(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype, float* Yt,
                   int64_t ldyt, void* workspace, size_t workspace_bytes, void* stream, int variant) {
  int rc = validate_apply(sk, X, ldx, n, sk ? sk->d : 0, dtype, Yt, ldyt, n, sk ? sk->k : 0, variant);
  if (rc || n == 0) return rc;
  if (workspace && overlaps(workspace, workspace_bytes, Yt, (size_t)((n - 1) * ldyt + sk->k) * 4))
    return fail(BPS_ERR_INVALID_ARG, "workspace overlaps the output");
  Placement pl{0, 0, sk->M};
  return dispatch(sk, X, ldx, n, dtype, Yt, ldyt, true, pl, stream, variant, workspace, workspace_bytes);
}

int bps_apply_adjoint_ex(const bps_sketch* sk, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                         void* stream, int variant) {
  int rc = validate_apply(sk, Y, ldy, sk ? sk->k : 0, n, BPS_F32, X, ldx, sk ? sk->d : 0, n, variant);
  if (rc || n == 0) return rc;
  if (sk->kind != 0) return fail(BPS_ERR_UNSUPPORTED, "adjoint: BlockPerm-SJLT sketches only");
  if ((rc = check_device())) return rc;
  const bool tc = bps::adjoint_tc_supported(sk->p, n);
  if (variant == BPS_VARIANT_TC && !tc) return fail(BPS_ERR_UNSUPPORTED, "adjoint tc: shape not covered");
  if (variant != BPS_VARIANT_SPARSE && tc) return bps::launch_adjoint_tc(sk->p, Y, ldy, n, X, ldx, (cudaStream_t)stream);
  return launch_adjoint(sk->p, Y, ldy, n, X, ldx, (cudaStream_t)stream);
}

int bps_apply_adjoint(const bps_sketch* sk, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                      void* stream) {
  return bps_apply_adjoint_ex(sk, Y, ldy, n, X, ldx, stream, BPS_VARIANT_AUTO);
}

static int check_range(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end) {
  if (!sk) return fail(BPS_ERR_INVALID_ARG, "sketch handle is NULL");
  if (sk->kind != 0) return fail(BPS_ERR_UNSUPPORTED, "orbit ranges: BlockPerm-SJLT sketches only");
  if (pos_begin < 0 || pos_begin >= sk->M || pos_end <= pos_begin || pos_end > pos_begin + sk->M)
    return fail(BPS_ERR_INVALID_ARG, "need 0 <= pos_begin < M and pos_begin < pos_end <= pos_begin + M");
  return BPS_OK;
}

int bps_apply_orbit_range_ws(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end, const void* A_local,
                             int64_t lda, int64_t n, bps_dtype dtype, float* Y_local, int64_t ldy, void* workspace,
                             size_t workspace_bytes, void* stream, int variant) {
  int rc = check_range(sk, pos_begin, pos_end);
  if (rc) return rc;
  const int64_t L = pos_end - pos_begin;
  const int64_t in_rows = (L + sk->kappa - 1) * sk->B_c;
  rc = validate_apply(sk, A_local, lda, in_rows, n, dtype, Y_local, ldy, L * sk->B_r, n, variant);
  if (rc || n == 0) return rc;
  if (workspace && overlaps(workspace, workspace_bytes, Y_local, (size_t)((L * sk->B_r - 1) * ldy + n) * 4))
    return fail(BPS_ERR_INVALID_ARG, "workspace overlaps the output");
  Placement pl{1, pos_begin, L};
  return dispatch(sk, A_local, lda, n, dtype, Y_local, ldy, false, pl, stream, variant, workspace, workspace_bytes);
}

int bps_apply_orbit_range_bcast(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end, const void* A_local,
                                int64_t lda, int64_t n, bps_dtype dtype, float* Y_local, int64_t ldy,
                                float* const* dst, int ndst, float* mc_dst, int64_t ld_dst, int64_t dst_row0,
                                void* workspace, size_t workspace_bytes, void* stream, int variant) {
  int rc = check_range(sk, pos_begin, pos_end);
  if (rc) return rc;
  if (ndst < 0 || ndst > 8 || (ndst > 0 && !dst)) return fail(BPS_ERR_INVALID_ARG, "need 0 <= ndst <= 8 destinations");
  const int64_t L = pos_end - pos_begin;
  if (ld_dst < n || dst_row0 < 0 || ((ld_dst * 4) % 16)) return fail(BPS_ERR_INVALID_ARG, "bad destination layout");
  Broadcast bc{};
  for (int j = 0; j < ndst; ++j) {
    if (!dst[j] || ((uintptr_t)dst[j] % 16)) return fail(BPS_ERR_INVALID_ARG, "destination pointers must be 16-byte aligned");
    bc.peer[j] = dst[j];
  }
  bc.npeer = ndst;
  bc.mc = mc_dst;
  bc.ld = ld_dst;
  bc.row0 = dst_row0;
  const int64_t in_rows = (L + sk->kappa - 1) * sk->B_c;
  rc = validate_apply(sk, A_local, lda, in_rows, n, dtype, Y_local, ldy, L * sk->B_r, n, variant);
  if (rc || n == 0) return rc;
  if (workspace && overlaps(workspace, workspace_bytes, Y_local, (size_t)((L * sk->B_r - 1) * ldy + n) * 4))
    return fail(BPS_ERR_INVALID_ARG, "workspace overlaps the output");
  Placement pl{1, pos_begin, L, (ndst > 0 || mc_dst) ? &bc : nullptr};
  return dispatch(sk, A_local, lda, n, dtype, Y_local, ldy, false, pl, stream, variant, workspace, workspace_bytes);
}

int bps_apply_orbit_range(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end, const void* A_local, int64_t lda,
                          int64_t n, bps_dtype dtype, float* Y_local, int64_t ldy, void* stream, int variant) {
  return bps_apply_orbit_range_ws(sk, pos_begin, pos_end, A_local, lda, n, dtype, Y_local, ldy, nullptr, 0, stream,
                                  variant);
}

int bps_orbit_range_workspace_size(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end, int64_t n,
                                   bps_dtype dtype, size_t* bytes) {
  int rc = check_range(sk, pos_begin, pos_end);
  if (rc) return rc;
  if (!bytes) return fail(BPS_ERR_INVALID_ARG, "NULL argument");
  if (n < 0) return fail(BPS_ERR_INVALID_ARG, "negative n");
  Placement pl{1, pos_begin, pos_end - pos_begin};
  *bytes = tc_workspace_bytes(sk->p, n, dtype, false, pl);
  return BPS_OK;
}

}  // extern "C"

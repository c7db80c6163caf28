// bps_internal.h — declarations shared by the libbps translation units (not installed).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/bps.h"
#include "bps_core.cuh"

struct bps_sketch {
  int kind;  // 0 = BlockPerm-SJLT, 1 = FlashBlockRow
  bps::SketchParams p;
  bps::BlockRowParams br;
  int64_t M, B_r, B_c, d, k;
  int32_t kappa, s;
  uint64_t seed;
};

namespace bps {

extern std::atomic<uint64_t> g_launches;
// bps_timing_enable: CUDA events around the dominant kernel of every apply (bps_api.cu)
bool timing_begin(cudaStream_t st, cudaEvent_t ev[2]);
void timing_end(cudaStream_t st, cudaEvent_t ev[2], bool aux = false);
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// Where the CTA for output index o (grid.x) finds its data:
//   full mode : o = g;  input block for ℓ at row f^ℓ(g)·B_c;  output rows g·B_r.
//   range mode: o = local orbit index; g = f^(pos_begin+o)(0); input block for ℓ at local
//               stacked block o+ℓ-1; output rows o·B_r.
// Output broadcast of an orbit-range apply (bps_apply_orbit_range_bcast): every final element of Y
// row r is also stored to row row0 + r of each destination (and through the NVLS multicast address).
struct Broadcast {
  float* peer[8];
  int npeer;
  float* mc;
  int64_t ld, row0;
};

struct Placement {
  int range_mode;
  int64_t pos_begin;
  int64_t n_out;  // number of output blocks launched (grid.x)
  const Broadcast* bc = nullptr;  // row-major orbit ranges only
};

// Unfused broadcast (sparse variant): copy rows [0, rows) of Y to every destination of bc.
int launch_bcast_rows(const float* Y, int64_t ldy, int64_t rows, int64_t n, const Broadcast& bc, cudaStream_t st);

// Sparse CUDA-core kernels (bps_sparse.cu).
int launch_sparse_rowmajor(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt,
                           float* Y, int64_t ldy, const Placement& pl, cudaStream_t st);
int launch_sparse_transposed(const SketchParams& p, const void* X, int64_t ldx, int64_t n, bps_dtype dt,
                             float* Yt, int64_t ldyt, const Placement& pl, cudaStream_t st);

// tcgen05 kernels (bps_tc.cu). Return BPS_ERR_UNSUPPORTED when the shape is not covered.
int tc_supported(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl);
size_t tc_workspace_bytes(const SketchParams& p, int64_t n, bps_dtype dt, bool transposed, const Placement& pl);
int launch_tc(const SketchParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y, int64_t ldy,
              bool transposed, const Placement& pl, void* ws, size_t ws_bytes, cudaStream_t st);

// Adjoint X = Sᵀ·Y (bps_adjoint.cu).
int launch_adjoint(const SketchParams& p, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                   cudaStream_t st);
// FlashBlockRow gather kernels (bps_blockrow.cu).
int launch_blockrow(const BlockRowParams& p, const void* A, int64_t lda, int64_t n, bps_dtype dt, float* Y,
                    int64_t ldy, bool transposed, cudaStream_t st);
// tcgen05 adjoint (bps_adjoint_tc.cu).
int adjoint_tc_supported(const SketchParams& p, int64_t n);
int launch_adjoint_tc(const SketchParams& p, const float* Y, int64_t ldy, int64_t n, float* X, int64_t ldx,
                      cudaStream_t st);

}  // namespace bps

/*
 * bps.h — C ABI of libbps: BlockPerm-SJLT sketch apply Y = S·A on NVIDIA B200 (sm_100a).
 *
 * The operation is the one defined in arXiv 2602.06071 ("FlashSketch"); citations
 * "P:n" are lines of the paper text, "R<k>" the readings
 * frozen in DESIGN.md §3 for what the paper leaves open.
 *
 *   d = M·B_c, k = M·B_r
 *   N(g) = (f^1(g), ..., f^κ(g)),  f(x) = (a·x + b) mod M        ((a,b) by R4)
 *   S_{g,h} = κ^{-1/2} Φ_{g,h} for h ∈ N(g), 0 otherwise
 *   Φ_{g,h}: row-partitioned SJLT, s nonzeros ±1/√s per column   (R1-R3)
 *   Y = S·A, each column of S has κ·s nonzeros of magnitude 1/√(κs)
 *
 * S is never stored: wiring, rows and signs are regenerated on the fly from a
 * counter hash of (seed, g, ℓ, u, j) (R2).
 *
 * Conventions (all entry points):
 *   - Return BPS_OK (0) on success or a negative bps_status; the message of the last
 *     failure on the calling thread is available from bps_last_error().
 *   - Validation happens before any device work; on a validation error no output is
 *     touched.
 *   - Device pointers are caller-owned CUDA device memory (e.g. torch tensors); the
 *     library never allocates, frees or copies them and holds no device memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream); work
 *     is enqueued asynchronously on it, with no implicit synchronisation. Execution
 *     faults surface at the caller's next synchronisation.
 *   - The current CUDA device is used and must be compute capability 10.0 (B200);
 *     otherwise BPS_ERR_ARCH. There is no CPU fallback.
 *   - Handles are immutable after creation; concurrent use from several threads or
 *     streams is safe.
 */
#ifndef BPS_H_
#define BPS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bps_sketch bps_sketch; /* opaque, host-only */

typedef enum { BPS_F32 = 0, BPS_BF16 = 1 } bps_dtype;

typedef enum {
  BPS_OK = 0,
  BPS_ERR_INVALID_ARG = -1, /* bad size / pointer / parameter */
  BPS_ERR_ALIGNMENT = -2,   /* pointer or leading dimension not 16-byte aligned */
  BPS_ERR_UNSUPPORTED = -3, /* valid sketch, but no kernel variant for this shape / variant request */
  BPS_ERR_ARCH = -4,        /* current device is not sm_100 */
  BPS_ERR_CUDA = -5,        /* a CUDA runtime / driver call failed (message has the CUDA error string) */
  BPS_ERR_OVERFLOW = -6     /* a size product does not fit the supported integer range */
} bps_status;

/* Intra-block pattern of Φ_{g,h} (bps_make_sketch_ex). */
typedef enum {
  BPS_MODE_ROWPART = 0, /* row-partitioned SJLT: chunk j = rows [jC,(j+1)C), C = B_r/s (R1, R3); default */
  BPS_MODE_AFFINE = 1   /* AffineUnique (R18): rows (α·j + β) mod B_r from one hash per column */
} bps_mode;

/* Kernel variant selector for bps_apply_ex / bps_apply_t_ex. */
typedef enum {
  BPS_VARIANT_AUTO = 0,   /* tcgen05 path when supported for the shape, else the sparse path */
  BPS_VARIANT_SPARSE = 1, /* CUDA-core gather kernel (private smem accumulators, no atomics) */
  BPS_VARIANT_TC = 2      /* tcgen05 tensor-core kernel; BPS_ERR_UNSUPPORTED if the shape is not covered */
} bps_variant;
/* tcgen05 coverage (bps_apply / bps_apply_t): B_c % 64 == 0, κ·s ≤ 128, κ·B_r ≤ 256 for fp32 and
 * ≤ 512 for bf16 (κ·B_r > 256 additionally needs B_r/s a power of two and κ·s % 4 == 0 in the
 * row-partitioned mode), d and n < 2^31.  Other shapes run on the sparse kernel under
 * BPS_VARIANT_AUTO.  The sparse kernel needs B_r ≤ 400 (row-major) / B_r ≤ 192 (transposed) and
 * ⌈n/128⌉ ≤ 65535; a shape neither kernel covers returns BPS_ERR_UNSUPPORTED. */

/*
 * bps_make_sketch — create the sketch S for layout (M, B_r, B_c) and parameters (κ, s, seed).
 *   d = M·B_c rows of A consumed, k = M·B_r rows of Y produced.
 *   Requirements (SPEC S:40-41 restating P:1531; counter widths R2):
 *     1 ≤ M < 2^24, 1 ≤ B_r, 1 ≤ B_c < 2^24, 1 ≤ κ ≤ min(M, 256),
 *     1 ≤ s ≤ min(B_r, 256), B_r % s == 0, M·B_c and M·B_r < 2^62.
 *   (a, b) are derived from the seed by R4 (Hull–Dobell).
 *   Host-only; no device work. *out receives a handle freed by bps_free_sketch.
 *   Errors: BPS_ERR_INVALID_ARG (out==NULL or a requirement violated), BPS_ERR_OVERFLOW.
 */
int bps_make_sketch(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s,
                    uint64_t seed, bps_sketch** out);

/* bps_free_sketch — release a handle. NULL-safe. */
void bps_free_sketch(bps_sketch* sk);

/*
 * bps_sketch_info — read back derived quantities. Any out-pointer may be NULL.
 *   d, k: dimensions; a, b: wiring map f(x)=(a x+b) mod M; scale: fp32(1/√(κs)) (R6).
 */
int bps_sketch_info(const bps_sketch* sk, int64_t* d, int64_t* k, uint32_t* a, uint32_t* b,
                    float* scale);

/*
 * bps_apply — Y = S·A  (output tile Y[gB_r:(g+1)B_r, columns]).
 *   A : device, d×n row-major, element type `dtype`, leading dimension lda ≥ n (elements).
 *   Y : device, k×n row-major fp32, leading dimension ldy ≥ n (elements). Overwritten; every
 *       element is written exactly once (no pre-zeroing, no atomics).
 *   bf16 inputs are widened exactly; accumulation is fp32; the scale 1/√(κs) is
 *   applied once at the end as an fp32 constant (R6).
 *   n == 0 is a no-op. A and Y must not overlap.
 *   Alignment: A, Y 16-byte aligned and lda·elem, ldy·4 multiples of 16 bytes,
 *   otherwise BPS_ERR_ALIGNMENT.
 *   Non-finite inputs (R12): an input element reaches only the κ·s rows its column of S
 *   names (Alg. 1), as in exact arithmetic: ±Inf/NaN appear only there, and
 *   finite inputs beyond the bf16 range are summed exactly (fp64) rather than overflowing.
 *   Determinism (R19): for a fixed handle, dtype, layout and variant, each
 *   element of Y is a fixed function of its input column — bitwise the same run to run, for
 *   any n, any column split (column shards), any orbit-range split (bps_apply_orbit_range),
 *   with or without a workspace, on any number of SMs.
 *   Without a workspace the tc variant uses "halo" ranges (each CTA re-streams κ−1 input
 *   blocks of halo, ≤ 25 % extra reads, fewer CTAs); bps_apply_ws is the full-occupancy form.
 */
int bps_apply(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype,
              float* Y, int64_t ldy, void* stream);

/*
 * bps_apply_t — transposed layout (R8): X = Aᵀ given n×d row-major (one length-d vector
 *   per row, ldx ≥ d), output Yt = (S·Xᵀ)ᵀ, n×k row-major fp32 (ldyt ≥ k).
 *   Same dtype, alignment, determinism and error rules as bps_apply.
 */
int bps_apply_t(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype,
                float* Yt, int64_t ldyt, void* stream);

/* Explicit-variant forms (tests / benchmarking). BPS_ERR_UNSUPPORTED if the requested
 * variant does not cover the shape. */
int bps_apply_ex(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype,
                 float* Y, int64_t ldy, void* stream, int variant);
int bps_apply_t_ex(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype,
                   float* Yt, int64_t ldyt, void* stream, int variant);

/*
 * Workspace forms (the full-occupancy tc path; the Python binding always uses them).  With a
 *   device workspace of at least bps_workspace_size() bytes the tc variant splits the input
 *   stream into equal group-aligned ranges, one CTA (pair) per SM; a CTA holding later
 *   accumulation groups of an output that straddles a range boundary leaves their partial sums
 *   in the workspace, and a second small kernel adds them, in stream order, onto the prefix the
 *   first CTA left in Y (no atomics, no pre-zeroing).  The result is bitwise identical to the
 *   no-workspace call (see bps_apply).
 *   Workspace: caller-owned device memory, 256-byte aligned, not overlapping the output; pure
 *   scratch (no initialisation needed, contents undefined afterwards).  One workspace must not be
 *   used by two calls that may run concurrently.  A too small workspace (or NULL) is ignored
 *   (no-workspace behaviour).  bytes = 0: the shape has no tc plan (sparse kernel).
 */
int bps_workspace_size(const bps_sketch* sk, int64_t n, bps_dtype dtype, int transposed, size_t* bytes);
int bps_apply_ws(const bps_sketch* sk, const void* A, int64_t lda, int64_t n, bps_dtype dtype,
                 float* Y, int64_t ldy, void* workspace, size_t workspace_bytes, void* stream,
                 int variant);
int bps_apply_t_ws(const bps_sketch* sk, const void* X, int64_t ldx, int64_t n, bps_dtype dtype,
                   float* Yt, int64_t ldyt, void* workspace, size_t workspace_bytes, void* stream,
                   int variant);

/*
 * bps_apply_adjoint — X = Sᵀ·Y, the adjoint (transpose) of the same sketch
 *   (S as in P:36-42 / P:1984-1992; Sᵀ is used e.g. to map a sketched-space solution back,
 *   SURVEY §8f).  X^(h) = κ^{-1/2} Σ_{g: h∈N(g)} Φ_{g,h}ᵀ Y^(g): row u of input block h gathers
 *   the κ·s rows of Y named by the column u of the pattern, with the same hash draws (R1-R3).
 *   Y: device, k × n fp32, row-major, leading dimension ldy (elements).
 *   X: device, d × n fp32, row-major, ldx; fully overwritten (every element written once, no
 *      atomics: bitwise reproducible).  Pointers / ld·4 16-byte aligned; X must not overlap Y.
 *   Kernels: tcgen05 (window of Y as the MMA A operand, the forward's band tile as B) when
 *   B_c % 64 == 0, κ·s ≤ 64 and κ·B_r ≤ 256; otherwise a CUDA-core gather kernel, which needs
 *   κ ≤ 64 and κ·B_r ≤ 400, else BPS_ERR_UNSUPPORTED.  n == 0 is a no-op.
 *   _ex: variant as for bps_apply_ex (TC on an uncovered shape -> BPS_ERR_UNSUPPORTED).
 */
int bps_apply_adjoint(const bps_sketch* sk, const float* Y, int64_t ldy, int64_t n, float* X,
                      int64_t ldx, void* stream);
int bps_apply_adjoint_ex(const bps_sketch* sk, const float* Y, int64_t ldy, int64_t n, float* X,
                         int64_t ldx, void* stream, int variant);

/*
 * bps_make_sketch_ex — bps_make_sketch with the intra-block pattern mode (bps_mode).
 *   BPS_MODE_AFFINE (R18): same wiring, scale and counter
 *   fields; column u of Φ_{g,f^ℓ(g)} takes z = fmix64((g≪40 | (ℓ−1)≪32 | u≪8) ⊕ K),
 *   α = (((z≫32) & 0xFFFF)·B_r ≫ 16) | 1, β = ((z≫48)·B_r) ≫ 16, rows (α·j + β) mod B_r and
 *   signs = bit j of z, j < s.  Requires B_r a power of two ≤ 2^16 and 1 ≤ s ≤ min(B_r, 32)
 *   (no B_r % s rule), else BPS_ERR_INVALID_ARG.  Every entry point accepts both modes.
 * bps_sketch_mode — the mode of a BlockPerm-SJLT handle (negative for NULL / FlashBlockRow).
 */
int bps_make_sketch_ex(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s, uint64_t seed,
                       int mode, bps_sketch** out);
int bps_sketch_mode(const bps_sketch* sk);

/*
 * FlashBlockRow (Alg. alg:blockrowsketch P:1447-1464) — the
 * paper's "fast but fragile" block-row sampling sketch S' (a different matrix from BlockPerm-SJLT):
 *   output block g gathers from κ distinct input blocks N_row(g) ⊂ [M] (R14); output row r adds
 *   s uniformly sampled rows i ∈ [B_c] (with replacement) of each, with Rademacher signs (R15):
 *   Y[g·B_r + r, :] = (κs)^{-1/2}·(d/k)^{1/2}·Σ_{h∈N_row(g)} Σ_t σ_t A[h·B_c + i_t, :]   (R16, R17)
 * bps_make_blockrow: 1 ≤ κ ≤ min(M, 256), 1 ≤ s ≤ 256, M, B_r, B_c < 2^24 (no B_r % s rule);
 *   BPS_ERR_INVALID_ARG otherwise.  The handle works with bps_apply / bps_apply_t / _ex / _ws
 *   (variant AUTO or SPARSE = the gather kernel; TC -> BPS_ERR_UNSUPPORTED; workspace size 0);
 *   bps_apply_orbit_range, bps_apply_adjoint, bps_orbit and bps_pattern_host return
 *   BPS_ERR_UNSUPPORTED / BPS_ERR_INVALID_ARG for it.  bps_sketch_info reports a = b = 0 and
 *   the block-row scale.  Transposed apply needs κ·s ≤ 4096.
 * bps_blockrow_neighbors: host, N_row(g) in draw order (ℓ = 1..κ) into nb[κ].
 * bps_blockrow_draw_host: host, (i, sign) of sample t of row r for the ℓ-th neighbour (ell 1-based).
 * bps_sketch_kind: 0 = BlockPerm-SJLT, 1 = FlashBlockRow, negative on a NULL handle.
 */
int bps_make_blockrow(int64_t M, int64_t B_r, int64_t B_c, int32_t kappa, int32_t s, uint64_t seed,
                      bps_sketch** out);
int bps_blockrow_neighbors(const bps_sketch* sk, int64_t g, int32_t* nb);
int bps_blockrow_draw_host(const bps_sketch* sk, int64_t g, int32_t ell, int64_t r, int32_t t,
                           int32_t* i, int32_t* sign);
int bps_sketch_kind(const bps_sketch* sk);

/*
 * bps_orbit — the wiring orbit g_pos = f^pos(0), pos = 0..M-1 (host).
 *   With this ordering N(g_i) = (g_{i+1}, ..., g_{i+κ}) (indices mod M), which is what
 *   makes block sharding contiguous.  g_of_pos: host array of length M.
 */
int bps_orbit(const bps_sketch* sk, int32_t* g_of_pos);

/*
 * bps_apply_orbit_range — partial apply over orbit positions [pos_begin, pos_end)
 *   (0 ≤ pos_begin < M, pos_begin < pos_end ≤ pos_begin + M; positions taken mod M).
 *   A_local: device, the input blocks at orbit positions pos_begin+1 .. pos_end+κ-1,
 *            stacked in that order: ((pos_end-pos_begin)+κ-1)·B_c rows × n, row-major, lda.
 *   Y_local: device, the output blocks at orbit positions pos_begin .. pos_end-1,
 *            stacked: (pos_end-pos_begin)·B_r rows × n fp32, row-major, ldy.
 *   Output block at local index i equals rows g_{pos_begin+i}·B_r.. of the full S·A — bitwise
 *   (same variant and dtype), so block sharding reproduces the 1-GPU result exactly (R19).
 * bps_apply_orbit_range_ws / bps_orbit_range_workspace_size: the workspace form (as bps_apply_ws).
 */
int bps_apply_orbit_range(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end,
                          const void* A_local, int64_t lda, int64_t n, bps_dtype dtype,
                          float* Y_local, int64_t ldy, void* stream, int variant);
int bps_apply_orbit_range_ws(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end,
                             const void* A_local, int64_t lda, int64_t n, bps_dtype dtype,
                             float* Y_local, int64_t ldy, void* workspace, size_t workspace_bytes,
                             void* stream, int variant);
int bps_orbit_range_workspace_size(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end, int64_t n,
                                   bps_dtype dtype, size_t* bytes);

/*
 * bps_apply_orbit_range_bcast — bps_apply_orbit_range_ws whose output is ALSO written into other
 *   buffers by the kernel epilogue itself: the all-gather step of orbit block sharding
 *   (rank r's output rows must reach every rank) fused into the
 *   store of each finished output tile, instead of a separate NCCL pass.
 *   dst:      host array of ndst (0..8) device pointers, each the base of a row-major fp32
 *             destination with leading dimension ld_dst (≥ n, 16-byte multiple) — typically the
 *             peers' symmetric buffers (CUDA IPC / symmetric-memory mappings of other GPUs'
 *             memory over NVLink), or local buffers.  Caller-owned; must be writable from the
 *             current device and not overlap Y_local, A_local or the workspace.
 *   mc_dst:   NULL, or an NVLS multicast address of such a buffer (one multimem.st reaches every
 *             GPU bound to the multicast object).
 *   dst_row0: row of the destinations receiving Y_local's row 0 (block sharding: the rank's first
 *             orbit position × B_r in an orbit-ordered k × n buffer).
 *   Y_local is written as in bps_apply_orbit_range_ws (it also holds the range's parked prefixes).
 *   Every destination receives bitwise the values of Y_local.  The tcgen05 variant stores to the
 *   destinations from its epilogue and combine pass; the sparse variant copies the finished rows
 *   with one extra kernel.  Ordering: the stores are complete when the stream reaches the next
 *   operation; making them visible to other GPUs needs the caller's cross-GPU barrier after that.
 *   Errors: BPS_ERR_INVALID_ARG for ndst outside 0..8, NULL/unaligned destinations or a bad
 *   ld_dst; otherwise as bps_apply_orbit_range_ws.
 */
int bps_apply_orbit_range_bcast(const bps_sketch* sk, int64_t pos_begin, int64_t pos_end,
                                const void* A_local, int64_t lda, int64_t n, bps_dtype dtype,
                                float* Y_local, int64_t ldy, float* const* dst, int ndst, float* mc_dst,
                                int64_t ld_dst, int64_t dst_row0, void* workspace, size_t workspace_bytes,
                                void* stream, int variant);

/*
 * bps_pattern_host — host evaluation of the frozen pattern draw (R2-R3), for tests:
 *   row ∈ [0, B_r) inside output block g and sign ∈ {+1,-1} of the j-th nonzero of
 *   column u of Φ_{g, f^ℓ(g)} (ell is 1-based). Uses the same code as the device kernels.
 */
int bps_pattern_host(const bps_sketch* sk, int64_t g, int32_t ell, int64_t u, int32_t j,
                     int32_t* row, int32_t* sign);

/* Number of CUDA kernels libbps has launched in this process so far (all devices, all
 * threads; cudaMemsetAsync nodes are not counted). Used by the bench to report how
 * many of the library's own kernels ran inside a timed region. */
uint64_t bps_kernel_launches(void);

/* Live timing of the dominant kernel (the bench's roofline figure): after bps_timing_enable(1),
 * every apply records a CUDA-event pair on its stream around its main kernel (tc stream kernel or
 * sparse gather kernel, not the combine pass); bps_timing_read synchronises on them, returns the
 * summed milliseconds and the number of launches, and clears the record.  Host-side state is
 * process-global and mutex-protected. */
int bps_timing_enable(int on);
int bps_timing_read(double* total_ms, uint64_t* count);
/* aux = 1: the same for the auxiliary kernels (the tc combine pass); aux = 0 is bps_timing_read. */
int bps_timing_read_ex(int aux, double* total_ms, uint64_t* count);

/* Library / build information ("bps <version> sm_100a ..."). */
const char* bps_version(void);

/* Thread-local message describing the last failure on this thread ("" if none). */
const char* bps_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BPS_H_ */

// bps_core.cuh — the frozen BlockPerm-SJLT randomness, shared by host code and every
// device kernel of libbps (never by the oracle).  DESIGN.md §3 R1-R4.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define BPS_HD __host__ __device__ __forceinline__
#else
#define BPS_HD inline
#endif

namespace bps {

constexpr uint64_t kTagA = 0xA11CE5EEDA11CE5EULL;
constexpr uint64_t kTagB = 0xB0B5EEDB0B5EEDB0ULL;
constexpr uint64_t kTagPhi = 0x5048495F5048495FULL;
constexpr uint64_t kTagRowBlk = 0x524F57424C4F434BULL;  // "ROWBLOCK" (R14)
constexpr uint64_t kTagRowIdx = 0x524F57494E444558ULL;  // "ROWINDEX" (R15)

// MurmurHash3 fmix64 (R2; "fast mixing hash").
BPS_HD uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xFF51AFD7ED558CCDULL;
  z ^= z >> 33;
  z *= 0xC4CEB9FE1A85EC53ULL;
  z ^= z >> 33;
  return z;
}

// Parameters every kernel needs; passed by value (fits in the param space).
struct SketchParams {
  uint32_t M, B_r, B_c, kappa, s, C;  // C = B_r / s (row-partition chunk, R1)
  uint32_t Mmask;                     // M-1 if M is a power of two (fast mod), else 0
  uint32_t a, b;                      // f(x) = (a x + b) mod M   (R4)
  uint64_t K;                         // mix64(seed ^ kTagPhi)     (R2)
  float scale;                        // fp32(1/sqrt(kappa*s))     (R6)
  uint32_t mode;                      // 0: row-partitioned (R1, R3); 1: AffineUnique (R18)
  uint32_t Brmask;                    // B_r - 1 (mode 1: B_r is a power of two)
};

// f(x) = (a x + b) mod M.
BPS_HD uint32_t affine_step(const SketchParams& p, uint32_t x) {
  if (p.Mmask) return (p.a * x + p.b) & p.Mmask;  // M = 2^m ≤ 2^24: low 32 bits of a·x+b suffice
  return (uint32_t)(((uint64_t)p.a * x + p.b) % p.M);
}

// f^e(x) by composing affine maps (square-and-multiply), e ≥ 0.
BPS_HD uint32_t affine_pow(const SketchParams& p, uint64_t e, uint32_t x) {
  if (p.Mmask) {  // power-of-two M: all arithmetic mod 2^32 then masked
    uint32_t ra = 1, rb = 0, ba = p.a, bb = p.b;
    while (e) {
      if (e & 1) {
        rb = ba * rb + bb;
        ra = ba * ra;
      }
      bb = ba * bb + bb;
      ba = ba * ba;
      e >>= 1;
    }
    return (ra * x + rb) & p.Mmask;
  }
  // Represent a map as (ma, mb): x -> ma x + mb (mod M).
  uint64_t ra = 1 % p.M, rb = 0;           // accumulated result
  uint64_t ba = p.a % p.M, bb = p.b % p.M; // f^(2^i)
  const uint64_t M = p.M;
  while (e) {
    if (e & 1) {  // result = base ∘ result
      rb = (ba * rb + bb) % M;
      ra = (ba * ra) % M;
    }
    bb = (ba * bb + bb) % M;
    ba = (ba * ba) % M;
    e >>= 1;
  }
  return (uint32_t)((ra * x + rb) % M);
}

// Row (inside the output block) and sign of the j-th nonzero of column u of
// Φ_{g, f^ell(g)}, ell 1-based (R1-R3; P:25-26 row-partitioned, P:1700 hash per (g,h,u,i)).
struct Draw {
  uint32_t row;
  uint32_t neg;  // 1 => sign -1
};

BPS_HD uint64_t pattern_hash(const SketchParams& p, uint32_t g, uint32_t ell, uint32_t u, uint32_t j) {
  const uint64_t ctr = ((uint64_t)g << 40) | ((uint64_t)(ell - 1) << 32) | ((uint64_t)u << 8) | (uint64_t)j;
  return mix64(ctr ^ p.K);
}

BPS_HD Draw draw_from_hash(const SketchParams& p, uint64_t z, uint32_t j) {
  const uint32_t hi = (uint32_t)(z >> 32);
  const uint32_t off = (uint32_t)(((uint64_t)hi * p.C) >> 32);  // Lemire range on the high word (R3)
  return Draw{j * p.C + off, (uint32_t)(z & 1)};
}

// AffineUnique (R18): z = hash of (g, ℓ, u) with j-field 0; α odd, β a shift;
// row_j = (α·j + β) mod B_r, sign_j = bit j of z.
BPS_HD Draw affine_draw(const SketchParams& p, uint64_t z, uint32_t j) {
  const uint32_t alpha = (uint32_t)(((((z >> 32) & 0xFFFFu) * p.B_r) >> 16) | 1u);
  const uint32_t beta = (uint32_t)(((z >> 48) * p.B_r) >> 16);
  return Draw{(alpha * j + beta) & p.Brmask, (uint32_t)((z >> j) & 1u)};
}

BPS_HD Draw pattern(const SketchParams& p, uint32_t g, uint32_t ell, uint32_t u, uint32_t j) {
  if (p.mode) return affine_draw(p, pattern_hash(p, g, ell, u, 0), j);
  return draw_from_hash(p, pattern_hash(p, g, ell, u, j), j);
}

// mix64 of (H:L) ⊕ (0:x) — the band generators' case, where only the low word varies with the
// input row u — from a per-key fold: L1 = L ⊕ (H≫1) absorbs the first xor-shift (whose input
// high word is the constant H), P1 = H·C1lo (mod 2^32) is the constant cross term of the first
// multiply.  Exactly mix64 (z≫33 of a 64-bit z is hi≫1 in the low word), in 32-bit operations.
BPS_HD void mix64_fold_key(uint64_t key, uint32_t& L1, uint32_t& P1) {
  const uint32_t H = (uint32_t)(key >> 32), L = (uint32_t)key;
  L1 = L ^ (H >> 1);
  P1 = H * 0xED558CCDu;
}
BPS_HD void mix64_folded(uint32_t L1, uint32_t P1, uint32_t x, uint32_t& hi, uint32_t& lo) {
  const uint32_t l1 = L1 ^ x;
  const uint64_t w = (uint64_t)l1 * 0xED558CCDu + ((uint64_t)P1 << 32);       // z *= C1 (low word × C1lo)
  const uint32_t h2 = (uint32_t)(w >> 32) + l1 * 0xFF51AFD7u, l2 = (uint32_t)w;  // + low word × C1hi
  const uint32_t l3 = l2 ^ (h2 >> 1);                                           // z ^= z >> 33
  const uint64_t w2 = (uint64_t)l3 * 0x1A85EC53u;                               // z *= C2
  hi = (uint32_t)(w2 >> 32) + h2 * 0x1A85EC53u + l3 * 0xC4CEB9FEu;
  lo = (uint32_t)w2 ^ (hi >> 1);                                                 // z ^= z >> 33
}

#ifdef __CUDACC__
// Band generators (tc kernels): combo c = (σ, j) of a block has a precomputed key
// ck = (g≪40 | (ℓ−1)≪32 | jfield) ⊕ K with jfield = j (mode 0) or 0 (mode 1), and
// cr = band_crow(...); z = mix64(ck ⊕ u≪8).  Returns the band row ρ and the sign bit.
__host__ __device__ __forceinline__ uint32_t band_jfield(const SketchParams& p, uint32_t j) { return p.mode ? 0u : j; }
__host__ __device__ __forceinline__ uint32_t band_crow(const SketchParams& p, uint32_t sigma, uint32_t j) {
  return p.mode ? (sigma * p.B_r) | (j << 16) : sigma * p.B_r + j * p.C;
}
template <bool AFF>
__device__ __forceinline__ uint32_t band_draw_t(const SketchParams& p, uint32_t cr, uint64_t z, uint32_t& neg) {
  if constexpr (AFF) {
    const Draw d = affine_draw(p, z, cr >> 16);
    neg = d.neg;
    return (cr & 0xFFFFu) + d.row;
  } else {
    neg = (uint32_t)(z & 1u);
    return cr + __umulhi((uint32_t)(z >> 32), p.C);  // R3
  }
}
__device__ __forceinline__ uint32_t band_draw(const SketchParams& p, uint32_t cr, uint64_t z, uint32_t& neg) {
  if (p.mode) {
    const Draw d = affine_draw(p, z, cr >> 16);
    neg = d.neg;
    return (cr & 0xFFFFu) + d.row;
  }
  neg = (uint32_t)(z & 1u);
  return cr + __umulhi((uint32_t)(z >> 32), p.C);  // R3
}
#endif

// ---------------------------------------------------------------- FlashBlockRow (R14-R16)
struct BlockRowParams {
  uint32_t M, B_r, B_c, kappa, s;
  uint64_t Kb, Ki;  // fmix64(seed ^ "ROWBLOCK"), fmix64(seed ^ "ROWINDEX")
  float scale;      // (κs)^{-1/2}·(d/k)^{1/2}
};

// attempt t of the rejection draw of N_row(g): a uniform block in [M) (R14)
BPS_HD uint32_t br_block_draw(const BlockRowParams& p, uint32_t g, uint32_t t) {
  const uint64_t z = mix64((((uint64_t)g << 32) | (uint64_t)t) ^ p.Kb);
  return (uint32_t)(((z >> 32) * (uint64_t)p.M) >> 32);
}

struct BrDraw {
  uint32_t i;    // row inside the input block, uniform in [B_c)
  uint32_t neg;  // 1 => sign -1
};

// sample t of output row r for the ℓ-th neighbour (ℓ 1-based) of output block g (R15)
BPS_HD BrDraw br_index_draw(const BlockRowParams& p, uint32_t g, uint32_t ell, uint32_t r, uint32_t t) {
  const uint64_t ctr = ((uint64_t)g << 40) | ((uint64_t)(ell - 1) << 32) | ((uint64_t)r << 8) | (uint64_t)t;
  const uint64_t z = mix64(ctr ^ p.Ki);
  return BrDraw{(uint32_t)(((z >> 32) * (uint64_t)p.B_c) >> 32), (uint32_t)(z & 1)};
}

}  // namespace bps

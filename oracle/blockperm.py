"""Plain float64 oracle for Y = S·A with S ~ BlockPerm-SJLT (TEST INFRASTRUCTURE ONLY).

Every function cites the passage it follows.  `P:n` = /root/reference/PAPER.md
line n; `R<k>` = reading k of DESIGN.md §3 (a choice the paper leaves open).

Definition being restated (P:15-47 = App. A "Construction and Notation", repeated
from §"BlockPerm-SJLT"):

  d = M·B_c, k = M·B_r
  N(g) = (π_1(g), ..., π_κ(g)),  π_ℓ(g) = f^ℓ(g),  f(x) = (a x + b) mod M
                                                                    
  S_{g,h} = κ^{-1/2} Φ_{g,h} if h ∈ N(g), else 0
  Φ_{g,h}: row-partitioned SJLT, exactly s nonzeros ±1/√s per column
  ⇒ each column of S has κ·s nonzeros of magnitude 1/√(κs)

Randomness (R1-R4): one 64-bit MurmurHash3 finaliser `mix64` of a packed counter
(seed, g, ℓ, u, j) yields the row offset inside chunk j and the sign; (a, b) are
derived from the seed by the Hull–Dobell rule.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
# R2: stream tags XOR-ed into the seed.
TAG_A = 0xA11CE5EEDA11CE5E
TAG_B = 0xB0B5EEDB0B5EEDB0
TAG_PHI = 0x5048495F5048495F
_C1 = 0xFF51AFD7ED558CCD
_C2 = 0xC4CEB9FE1A85EC53


# --------------------------------------------------------------------------- hash
def mix64(z):
    """MurmurHash3 fmix64 finaliser (R2; SPEC S:167 names it; the paper only says
    "a fast 32-bit mixing hash").

    Accepts a Python int (exact arithmetic, masked to 64 bits) or a numpy uint64
    array (numpy uint64 arithmetic wraps modulo 2^64).
    """
    if isinstance(z, np.ndarray):
        z = z.astype(np.uint64, copy=True)
        with np.errstate(over="ignore"):
            z ^= z >> np.uint64(33)
            z *= np.uint64(_C1)
            z ^= z >> np.uint64(33)
            z *= np.uint64(_C2)
            z ^= z >> np.uint64(33)
        return z
    z &= MASK64
    z ^= z >> 33
    z = (z * _C1) & MASK64
    z ^= z >> 33
    z = (z * _C2) & MASK64
    z ^= z >> 33
    return z


# ------------------------------------------------------------------------ wiring
def rad(M: int) -> int:
    """Product of the distinct prime factors of M (trial division)."""
    r, m, p = 1, M, 2
    while p * p <= m:
        if m % p == 0:
            r *= p
            while m % p == 0:
                m //= p
        p += 1
    if m > 1:
        r *= m
    return r


def hull_dobell(a: int, b: int, M: int) -> bool:
    """Full-period conditions (a)-(c) for f(x) = (a x + b) mod M."""
    if M == 1:
        return True
    if math.gcd(b, M) != 1:  # (a)
        return False
    m, p = M, 2
    while p * p <= m:  # (b): every prime p | M divides a-1
        if m % p == 0:
            if (a - 1) % p != 0:
                return False
            while m % p == 0:
                m //= p
        p += 1
    if m > 1 and (a - 1) % m != 0:
        return False
    if M % 4 == 0 and (a - 1) % 4 != 0:  # (c)
        return False
    return True


def full_cycle_bruteforce(a: int, b: int, M: int) -> bool:
    """Definition of period M: iterate x_{t+1}=f(x_t) from
    x_0 = 0 and check all of [M] is visited before returning to 0."""
    seen = set()
    x = 0
    for _ in range(M):
        if x in seen:
            return False
        seen.add(x)
        x = (a * x + b) % M
    return len(seen) == M and x == 0


def select_affine(seed: int, M: int) -> tuple[int, int]:
    """R4: deterministic (a, b) from the seed satisfying Hull–Dobell (the paper only
    says "the kernel chooses integers a and b").

    q = rad(M), doubled if 4 | M;  a = (1 + q·(mix64(seed^TAG_A) mod (M/q))) mod M;
    b = mix64(seed^TAG_B^t) mod M for the first t = 0,1,... with gcd(b, M) = 1.
    M = 1 gives (0, 0).
    """
    if M < 1:
        raise ValueError("M must be >= 1")
    if M == 1:
        return 0, 0
    q = rad(M)
    if M % 4 == 0:
        q *= 2
    a = (1 + q * (mix64(seed ^ TAG_A) % (M // q))) % M
    t = 0
    while True:
        b = mix64((seed ^ TAG_B ^ t) & MASK64) % M
        if math.gcd(b, M) == 1:
            break
        t += 1
    assert hull_dobell(a, b, M)
    return a, b


def neighborhood(a: int, b: int, M: int, kappa: int, g: int) -> list[int]:
    """N(g) = (f^1(g), ..., f^κ(g)), ℓ-fold composition, ℓ = 1..κ.
    Distinct for κ ≤ M."""
    out, h = [], g
    for _ in range(kappa):
        h = (a * h + b) % M
        out.append(h)
    return out


def neighborhoods(a: int, b: int, M: int, kappa: int) -> np.ndarray:
    """M×κ table, row g = N(g) in wiring order (order (π_1(g),...,π_κ(g)))."""
    return np.array([neighborhood(a, b, M, kappa, g) for g in range(M)], dtype=np.int64).reshape(M, kappa)


def check_edge_disjoint(tables) -> bool:
    """Edge-disjointness / pairwise derangement: for all g and ℓ≠ℓ',
    π_ℓ(g) ≠ π_ℓ'(g).  `tables` is a list of κ permutations of [M] (π_ℓ[g])."""
    tables = [list(t) for t in tables]
    M = len(tables[0]) if tables else 0
    for g in range(M):
        vals = [t[g] for t in tables]
        if len(set(vals)) != len(vals):
            return False
    return True


def orbit(a: int, b: int, M: int) -> list[int]:
    """Orbit of 0 under f: g_0 = 0, g_i = f(g_{i-1}) (full cycle)."""
    out, x = [], 0
    for _ in range(M):
        out.append(x)
        x = (a * x + b) % M
    return out


# ----------------------------------------------------------------------- sketch
@dataclass(frozen=True)
class Sketch:
    M: int
    B_r: int
    B_c: int
    kappa: int
    s: int
    seed: int
    a: int
    b: int
    K: int  # mix64(seed ^ TAG_PHI), R2
    mode: str = "rowpart"  # intra-block rows: "rowpart" (R1, R3) or "affine" (AffineUnique, R18)

    @property
    def d(self) -> int:
        return self.M * self.B_c

    @property
    def k(self) -> int:
        return self.M * self.B_r

    @property
    def C(self) -> int:
        """Row-partition chunk size B_r / s (R1)."""
        return self.B_r // self.s

    @property
    def scale(self) -> float:
        """Nonzero magnitude 1/√(κs), float64."""
        return 1.0 / math.sqrt(self.kappa * self.s)


def make_sketch(M: int, B_r: int, B_c: int, kappa: int, s: int, seed: int, mode: str = "rowpart") -> Sketch:
    """Validate (1≤κ≤M, 1≤s≤B_r, B_r mod s = 0; counter widths R2) and
    derive (a, b, K).  mode="affine" (R18): B_r a power of two ≤ 2^16, s ≤ min(B_r, 32), no
    divisibility rule."""
    if M < 1 or B_r < 1 or B_c < 1:
        raise ValueError("M, B_r, B_c must be >= 1")
    if not (1 <= kappa <= M):
        raise ValueError("need 1 <= kappa <= M (P:1531)")
    if mode == "affine":
        if B_r & (B_r - 1) or B_r > 1 << 16 or not (1 <= s <= min(B_r, 32)):
            raise ValueError("affine mode: B_r a power of two <= 2^16 and 1 <= s <= min(B_r, 32) (R18)")
    elif mode != "rowpart":
        raise ValueError("mode must be 'rowpart' or 'affine'")
    elif not (1 <= s <= B_r) or B_r % s != 0:
        raise ValueError("need 1 <= s <= B_r and B_r % s == 0 (row-partitioned, R1)")
    if M >= 1 << 24 or B_c >= 1 << 24 or kappa > 256 or s > 256:
        raise ValueError("counter field widths exceeded (R2)")
    seed &= MASK64
    a, b = select_affine(seed, M)
    return Sketch(M, B_r, B_c, kappa, s, seed, a, b, mix64(seed ^ TAG_PHI), mode)


def pattern(sk: Sketch, g: int, ell: int, u: int, j: int) -> tuple[int, int]:
    """Row (inside output block g) and sign of the j-th nonzero of column u of
    Φ_{g,π_ℓ(g)} — row-partitioned SJLT, one nonzero per chunk j (
    R1-R3).  ell is 1-based.

    ctr = g<<40 | (ℓ-1)<<32 | u<<8 | j ;  z = mix64(ctr ^ K)
    row = j·C + ((z>>32)·C >> 32) ;  sign = -1 if z&1 else +1
    """
    if sk.mode == "affine":
        return pattern_affine(sk, g, ell, u, j)
    ctr = (g << 40) | ((ell - 1) << 32) | (u << 8) | j
    z = mix64(ctr ^ sk.K)
    off = ((z >> 32) * sk.C) >> 32
    return j * sk.C + off, (-1 if (z & 1) else 1)


def affine_params(sk: Sketch, g: int, ell: int, u: int) -> tuple[int, int, int]:
    """R18 (AffineUnique: "s unique row indices using an affine permutation map ...
    with scale and shift parameters generated from the hash"): one hash per column u of
    Φ_{g,π_ℓ(g)}:  z = mix64((g<<40 | (ℓ-1)<<32 | u<<8) ^ K);
    scale α = (((z>>32) & 0xFFFF)·B_r >> 16) | 1  (odd: a unit mod the power of two B_r),
    shift β = ((z>>48)·B_r) >> 16.  Returns (α, β, z)."""
    z = mix64(((g << 40) | ((ell - 1) << 32) | (u << 8)) ^ sk.K)
    alpha = ((((z >> 32) & 0xFFFF) * sk.B_r) >> 16) | 1
    beta = ((z >> 48) * sk.B_r) >> 16
    return alpha, beta, z


def pattern_affine(sk: Sketch, g: int, ell: int, u: int, j: int) -> tuple[int, int]:
    """R18: row_j = (α·j + β) mod B_r — the first s images of the permutation x ↦ αx+β of
    [B_r], hence s distinct rows; sign_j = −1 iff bit j of z is set (j < 32)."""
    alpha, beta, z = affine_params(sk, g, ell, u)
    return (alpha * j + beta) % sk.B_r, (-1 if (z >> j) & 1 else 1)


def _block_entries(sk: Sketch, g: int):
    """All nonzeros of block row g of S as (rows, cols, vals) int64/int64/float64,
    following P:36-42 (S_{g,h} = κ^{-1/2} Φ_{g,h}, h ∈ N(g)) with Φ entries ±1/√s."""
    nbr = neighborhood(sk.a, sk.b, sk.M, sk.kappa, g)
    u = np.arange(sk.B_c, dtype=np.uint64)
    rows, cols, vals = [], [], []
    for ell, h in enumerate(nbr, start=1):
        if sk.mode == "affine":
            ctr = (np.uint64(g) << np.uint64(40)) | (np.uint64(ell - 1) << np.uint64(32)) | (u << np.uint64(8))
            z = mix64(ctr ^ np.uint64(sk.K))
            alpha = ((((z >> np.uint64(32)) & np.uint64(0xFFFF)) * np.uint64(sk.B_r)) >> np.uint64(16)) | np.uint64(1)
            beta = ((z >> np.uint64(48)) * np.uint64(sk.B_r)) >> np.uint64(16)
            for j in range(sk.s):
                row = (alpha * np.uint64(j) + beta) % np.uint64(sk.B_r)
                sign = np.where(((z >> np.uint64(j)) & np.uint64(1)) == 1, -1.0, 1.0)
                rows.append(g * sk.B_r + row.astype(np.int64))
                cols.append(h * sk.B_c + u.astype(np.int64))
                vals.append(sign * sk.scale)
            continue
        for j in range(sk.s):
            ctr = (np.uint64(g) << np.uint64(40)) | (np.uint64(ell - 1) << np.uint64(32)) | (u << np.uint64(8)) | np.uint64(j)
            z = mix64(ctr ^ np.uint64(sk.K))
            with np.errstate(over="ignore"):
                off = ((z >> np.uint64(32)) * np.uint64(sk.C)) >> np.uint64(32)
            sign = np.where((z & np.uint64(1)) == 1, -1.0, 1.0)
            rows.append(g * sk.B_r + j * sk.C + off.astype(np.int64))
            cols.append(h * sk.B_c + u.astype(np.int64))
            vals.append(sign * sk.scale)
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def build_S_dense(sk: Sketch) -> np.ndarray:
    """Explicit k×d float64 S (tiny sizes only, k·d ≤ 2^26)."""
    if sk.k * sk.d > (1 << 26):
        raise ValueError("dense S too large; use build_S_csr")
    S = np.zeros((sk.k, sk.d), dtype=np.float64)
    for g in range(sk.M):
        r, c, v = _block_entries(sk, g)
        # distinct positions by construction (distinct chunks j, distinct blocks h)
        np.add.at(S, (r, c), v)
    return S


def build_S_csr(sk: Sketch, blocks=None):
    """SciPy CSR of the block rows `blocks` (default all) of S, shape (len·B_r)×d;
    row i of the result is global row blocks[i//B_r]·B_r + i%B_r."""
    import scipy.sparse as sp

    blocks = list(range(sk.M)) if blocks is None else list(blocks)
    R, Cc, V = [], [], []
    for bi, g in enumerate(blocks):
        r, c, v = _block_entries(sk, g)
        R.append(r - g * sk.B_r + bi * sk.B_r)
        Cc.append(c)
        V.append(v)
    nrow = len(blocks) * sk.B_r
    if not R:
        return sp.csr_matrix((nrow, sk.d), dtype=np.float64)
    return sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(Cc))), shape=(nrow, sk.d), dtype=np.float64)


def apply(sk: Sketch, A: np.ndarray, blocks=None) -> np.ndarray:
    """Y = S·A in float64 (A: d×n, any float dtype; upcast is exact for fp32/bf16).
    With `blocks`, returns only those output block rows, stacked.

    Evaluated as the sum over the nonzeros of S only (CSR product; Alg. 1, P:1688-1709 adds
    σ·a into the s drawn rows of each of the κ output blocks an input row feeds), so the zeros
    of S never multiply A: with a non-finite a, ±Inf/NaN reach exactly the κ·s rows its
    column of S names (reading R12) — a dense product would form 0·Inf = NaN everywhere."""
    A64 = np.asarray(A, dtype=np.float64)
    if A64.shape[0] != sk.d:
        raise ValueError("A must have d rows")
    return build_S_csr(sk, blocks) @ A64


def apply_t(sk: Sketch, X: np.ndarray, blocks=None) -> np.ndarray:
    """Transposed layout (R8): X is n×d (one vector per row); returns (S·Xᵀ)ᵀ, n×k
    (or n×(len(blocks)·B_r))."""
    X64 = np.asarray(X, dtype=np.float64)
    return apply(sk, X64.T, blocks).T


def apply_adjoint(sk: Sketch, Yin: np.ndarray) -> np.ndarray:
    """X = Sᵀ·Y in float64 (Y: k×n) — the adjoint of the sketch, the plain
    transpose of the explicit S of P:36-42."""
    Y64 = np.asarray(Yin, dtype=np.float64)
    if Y64.shape[0] != sk.k:
        raise ValueError("Y must have k rows")
    return build_S_csr(sk).T @ Y64  # nonzeros only (R12, as apply)


def sketch_rows(sk: Sketch, g: int) -> np.ndarray:
    """Global row indices of output block g (P:1663-1666 tiles)."""
    return np.arange(g * sk.B_r, (g + 1) * sk.B_r)


def energy_identity_lhs(sk: Sketch, x: np.ndarray) -> float:
    """Σ_g ‖x_{N(g)}‖²; the lemma says it equals κ‖x‖²."""
    tot = 0.0
    for g in range(sk.M):
        for h in neighborhood(sk.a, sk.b, sk.M, sk.kappa, g):
            blk = np.asarray(x[h * sk.B_c:(h + 1) * sk.B_c], dtype=np.float64)
            tot += float(blk @ blk)
    return tot

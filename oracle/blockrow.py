"""Plain float64 oracle for FlashBlockRow, the block-row sampling sketch (TEST INFRASTRUCTURE ONLY).

Restates App. "FlashBlockRow: A Fast but Fragile Alternative" and its
Algorithm `alg:blockrowsketch`, with the readings R14-R17 of DESIGN.md §3:

  for every output block g ∈ [M]:
    N_row(g) ⊂ [M], |N_row(g)| = κ                                    (R14: uniform, distinct)
    for every h ∈ N_row(g), every output row r ∈ [B_r]:
      sample i_1..i_s ∈ [B_c] uniformly and signs σ_1..σ_s ∈ {±1}       (R15)
      Y[g·B_r + r, :] += (κs)^{-1/2} · (d/k)^{1/2} · Σ_t σ_t A[h·B_c + i_t, :]   (R16, R17)

So S has at most κ·s nonzeros per ROW (not per column): columns may be empty, which is the
"fragility" the paper names.  Random bits come from the same MurmurHash3
finaliser as BlockPerm-SJLT (R2), keyed by separate stream tags.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .blockperm import MASK64, mix64

# R14/R15 stream tags ("ROWBLOCK", "ROWINDEX")
TAG_ROWBLK = 0x524F57424C4F434B
TAG_ROWIDX = 0x524F57494E444558


@dataclass(frozen=True)
class BlockRow:
    M: int
    B_r: int
    B_c: int
    kappa: int
    s: int
    seed: int

    @property
    def d(self) -> int:
        return self.M * self.B_c

    @property
    def k(self) -> int:
        return self.M * self.B_r

    @property
    def scale(self) -> float:
        """R16: (κs)^{-1/2}·(d/k)^{1/2}, computed in double, applied once."""
        return math.sqrt(self.d / self.k) / math.sqrt(self.kappa * self.s)

    @property
    def K_blk(self) -> int:
        return mix64((self.seed ^ TAG_ROWBLK) & MASK64)

    @property
    def K_idx(self) -> int:
        return mix64((self.seed ^ TAG_ROWIDX) & MASK64)


def make_blockrow(M: int, B_r: int, B_c: int, kappa: int, s: int, seed: int) -> BlockRow:
    """Validation as for BlockPerm-SJLT's counter fields: 1 ≤ κ ≤ M (κ distinct
    blocks), 1 ≤ s ≤ 256, g, r < 2^24, κ ≤ 256."""
    if not (M >= 1 and B_r >= 1 and B_c >= 1 and 1 <= kappa <= M and 1 <= s <= 256):
        raise ValueError("invalid block-row sketch parameters")
    if M >= (1 << 24) or B_r >= (1 << 24) or B_c >= (1 << 24) or kappa > 256:
        raise ValueError("counter field overflow")
    return BlockRow(M, B_r, B_c, kappa, s, seed & MASK64)


def lemire(z32: int, m: int) -> int:
    """Map a uniform 32-bit word to [0, m): ⌊z·m / 2^32⌋ (R3's range reduction)."""
    return (z32 * m) >> 32


def neighbors_row(br: BlockRow, g: int) -> list[int]:
    """R14: N_row(g) — κ distinct blocks, uniform without replacement, by sequential
    rejection: attempt t = 0, 1, …: h_t = lemire(mix64((g≪32 | t) ⊕ K_blk) ≫ 32, M); keep h_t
    if not yet chosen; stop at κ.  Order = acceptance order (ℓ = 1..κ)."""
    out: list[int] = []
    t = 0
    while len(out) < br.kappa:
        z = mix64((((g << 32) | t) ^ br.K_blk) & MASK64)
        h = lemire(z >> 32, br.M)
        if h not in out:
            out.append(h)
        t += 1
    return out


def draw_index(br: BlockRow, g: int, ell: int, r: int, t: int) -> tuple[int, int]:
    """R15: (i, σ) of sample t of output row r for the ℓ-th neighbour (ℓ 1-based):
    z = mix64((g≪40 | (ℓ−1)≪32 | r≪8 | t) ⊕ K_idx); i = lemire(z ≫ 32, B_c) (uniform, with
    replacement); σ = −1 iff z & 1."""
    ctr = (g << 40) | ((ell - 1) << 32) | (r << 8) | t
    z = mix64((ctr ^ br.K_idx) & MASK64)
    return lemire(z >> 32, br.B_c), (-1 if (z & 1) else 1)


def triplets(br: BlockRow, g: int):
    """All (global row, global column, value) contributions of output block g in the
    algorithm's loop order h ∈ N_row(g), r, t.  Duplicates are kept (R17)."""
    R, Cc, V = [], [], []
    for ell, h in enumerate(neighbors_row(br, g), start=1):
        for r in range(br.B_r):
            for t in range(br.s):
                i, sg = draw_index(br, g, ell, r, t)
                R.append(g * br.B_r + r)
                Cc.append(h * br.B_c + i)
                V.append(sg * br.scale)
    return np.asarray(R, np.int64), np.asarray(Cc, np.int64), np.asarray(V, np.float64)


def build_S_csr(br: BlockRow, blocks=None):
    """SciPy CSR of the output-block rows `blocks` (default all), (len·B_r) × d; duplicate
    (row, column) contributions are summed (R17)."""
    import scipy.sparse as sp

    blocks = list(range(br.M)) if blocks is None else list(blocks)
    R, Cc, V = [], [], []
    for bi, g in enumerate(blocks):
        r, c, v = triplets(br, g)
        R.append(r - g * br.B_r + bi * br.B_r)
        Cc.append(c)
        V.append(v)
    return sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(Cc))),
                         shape=(len(blocks) * br.B_r, br.d))


def build_S_dense(br: BlockRow) -> np.ndarray:
    return build_S_csr(br).toarray()


def apply(br: BlockRow, A: np.ndarray, blocks=None) -> np.ndarray:
    """Y = S·A in float64 (A: d×n); `blocks` restricts to those output blocks (stacked)."""
    A64 = np.asarray(A, dtype=np.float64)
    if A64.shape[0] != br.d:
        raise ValueError("A must have d rows")
    return build_S_csr(br, blocks) @ A64


def apply_t(br: BlockRow, X: np.ndarray, blocks=None) -> np.ndarray:
    """Transposed layout (R8): X = Aᵀ (n×d) -> (S·Xᵀ)ᵀ (n×k)."""
    return apply(br, np.asarray(X, dtype=np.float64).T, blocks).T

"""Pins of the FlashBlockRow oracle (oracle/blockrow.py) against the paper and mathematics.

P:1424-1466 (App. "FlashBlockRow") and Alg. `alg:blockrowsketch`; readings R14-R17.
"""

import math

import numpy as np
import pytest

from oracle import blockrow as BR


def _brute_apply(br, A):
    """Alg. alg:blockrowsketch written as loops with Python floats: per output block g, per
    h ∈ N_row(g), per row r, s samples, sY_r += scale·Σ σ A[h·B_c + i]."""
    n = A.shape[1]
    Y = [[0.0] * n for _ in range(br.k)]
    for g in range(br.M):
        for ell, h in enumerate(BR.neighbors_row(br, g), start=1):
            for r in range(br.B_r):
                for t in range(br.s):
                    i, sg = BR.draw_index(br, g, ell, r, t)
                    for c in range(n):
                        Y[g * br.B_r + r][c] += br.scale * sg * float(A[h * br.B_c + i, c])
    return np.array(Y)


@pytest.mark.parametrize("layout", [(8, 4, 16, 2, 2), (5, 3, 7, 5, 3), (1, 2, 9, 1, 4), (16, 2, 32, 3, 1)])
def test_apply_equals_algorithm_loops(layout):
    br = BR.make_blockrow(*layout, seed=3)
    A = np.random.default_rng(0).standard_normal((br.d, 3))
    assert np.allclose(BR.apply(br, A), _brute_apply(br, A), rtol=1e-13, atol=1e-13)
    # transposed layout is the same map
    assert np.allclose(BR.apply_t(br, A.T), BR.apply(br, A).T, rtol=0, atol=0)


def test_neighborhoods_distinct_and_uniform():
    """|N_row(g)| = κ distinct blocks of [M]; uniform marginals (χ² over blocks)."""
    M, kappa = 16, 4
    counts = np.zeros(M)
    for seed in range(200):
        br = BR.make_blockrow(M, 2, 4, kappa, 1, seed)
        for g in range(M):
            nb = BR.neighbors_row(br, g)
            assert len(nb) == kappa and len(set(nb)) == kappa and all(0 <= h < M for h in nb)
            counts[nb] += 1
    exp = counts.sum() / M
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    assert chi2 < 45.0  # 15 dof, p ≈ 1e-4
    br = BR.make_blockrow(7, 1, 1, 7, 1, 11)  # κ = M: a permutation of [M]
    assert sorted(BR.neighbors_row(br, 3)) == list(range(7))


def test_indices_uniform_and_signs_balanced():
    br = BR.make_blockrow(4, 64, 24, 2, 8, 5)
    idx, sg = [], []
    for g in range(br.M):
        for ell in (1, 2):
            for r in range(br.B_r):
                for t in range(br.s):
                    i, s = BR.draw_index(br, g, ell, r, t)
                    idx.append(i)
                    sg.append(s)
    idx, sg = np.array(idx), np.array(sg)
    assert idx.min() >= 0 and idx.max() < br.B_c
    counts = np.bincount(idx, minlength=br.B_c)
    exp = len(idx) / br.B_c
    assert float(((counts - exp) ** 2 / exp).sum()) < 60.0  # 23 dof
    assert abs(sg.mean()) < 4 / math.sqrt(len(sg))


def test_unbiased_norm():
    """E‖Sx‖² = ‖x‖²: each of the k·κ·s samples picks a uniform coordinate (block marginal 1/M,
    index 1/B_c) with an independent sign, so E‖Sx‖² = k·κs·scale²·‖x‖²/d and
    scale² = d/(k·κs).  Monte-Carlo over seeds within 4 standard errors."""
    x = np.random.default_rng(1).standard_normal(128)
    vals = []
    for seed in range(3000):
        br = BR.make_blockrow(8, 4, 16, 2, 2, seed)
        vals.append(float(np.sum(BR.apply(br, x[:, None]) ** 2)) / float(x @ x))
    vals = np.array(vals)
    se = vals.std(ddof=1) / math.sqrt(len(vals))
    assert se < 0.01
    assert abs(vals.mean() - 1.0) < 4 * se


def test_row_structure_and_fragility():
    """Rows: entries are integer multiples of the scale, Σ|v|/scale ≤ κs with the parity of κs
    (duplicate samples add, opposite signs cancel in pairs).  Columns may be EMPTY — the
    fragility of P:1437-1440 — whenever k·κ·s < d."""
    br = BR.make_blockrow(8, 2, 64, 2, 1, 7)  # k·κ·s = 32 < d = 512
    S = BR.build_S_dense(br)
    q = S / br.scale
    assert np.allclose(q, np.round(q), atol=1e-12)
    tot = np.abs(np.round(q)).sum(axis=1)
    assert np.all(tot <= br.kappa * br.s) and np.all((tot - br.kappa * br.s) % 2 == 0)
    assert int((np.abs(S).sum(axis=0) == 0).sum()) >= br.d - br.k * br.kappa * br.s
    # each output row touches at most κ input blocks, all distinct per N_row(g)
    for g in range(br.M):
        blocks = {c // br.B_c for c in np.nonzero(S[g * br.B_r:(g + 1) * br.B_r].any(axis=0))[0]}
        assert blocks <= set(BR.neighbors_row(br, g))


def test_signed_row_sampling_special_case():
    """κ = s = B_r = B_c = 1: S is a signed uniform row-sampling matrix — one ±√(d/k) = ±1 per row
    (the textbook sampling sketch the block-row family generalises)."""
    br = BR.make_blockrow(12, 1, 1, 1, 1, 9)
    S = BR.build_S_dense(br)
    assert np.all((S != 0).sum(axis=1) == 1)
    assert np.all(np.abs(S[S != 0]) == 1.0)


def test_make_rejects():
    for args in [(4, 2, 2, 5, 1), (4, 2, 2, 0, 1), (4, 2, 2, 2, 0), (4, 2, 2, 2, 300)]:
        with pytest.raises(ValueError):
            BR.make_blockrow(*args, seed=0)

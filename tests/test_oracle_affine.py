"""Pins of the AffineUnique intra-block mode of the oracle (R18; §8f rank 4).

"It generates s unique row indices using an affine permutation map similar to the one above,
with scale and shift parameters generated from the hash".
"""

import math

import numpy as np
import pytest

import oracle
from oracle import blockperm as bp

LAYOUTS = [(8, 32, 128, 2, 2), (16, 64, 128, 4, 8), (5, 16, 24, 3, 3), (4, 8, 16, 2, 8), (6, 1, 9, 2, 1)]


def test_rows_distinct_and_full_permutation():
    """The s rows of every column of Φ_{g,h} are distinct; with s = B_r they are a permutation
    of [B_r] (an affine map x ↦ αx + β with α a unit is a bijection of Z/B_r)."""
    rng = np.random.default_rng(0)
    for layout in LAYOUTS:
        sk = oracle.make_sketch(*layout, seed=7, mode="affine")
        for _ in range(200):
            g, ell, u = int(rng.integers(sk.M)), int(rng.integers(1, sk.kappa + 1)), int(rng.integers(sk.B_c))
            rows = [bp.pattern(sk, g, ell, u, j)[0] for j in range(sk.s)]
            assert len(set(rows)) == sk.s and all(0 <= r < sk.B_r for r in rows)
    sk = oracle.make_sketch(4, 16, 8, 2, 16, seed=3, mode="affine")
    for u in range(sk.B_c):
        assert sorted(bp.pattern(sk, 1, 2, u, j)[0] for j in range(16)) == list(range(16))


@pytest.mark.parametrize("layout", LAYOUTS)
def test_column_structure_and_unit_norm(layout):
    """Each column of S has exactly κ·s nonzeros of magnitude 1/√(κs), so
    ‖S e_i‖₂ = 1 exactly; block-row g touches only N(g)."""
    sk = oracle.make_sketch(*layout, seed=11, mode="affine")
    S = oracle.build_S_dense(sk)
    nnz = (S != 0).sum(axis=0)
    assert np.all(nnz == sk.kappa * sk.s)
    assert np.allclose(np.abs(S[S != 0]), sk.scale, rtol=0, atol=0)
    assert np.allclose((S ** 2).sum(axis=0), 1.0, rtol=1e-14)


def test_apply_equals_scalar_definition():
    """The vectorised block builder equals the scalar R18 definition enumerated one (ℓ,u,j) at a
    time (Alg. 1 loop order, scale applied last); dense ≡ CSR."""
    sk = oracle.make_sketch(4, 8, 16, 2, 4, seed=3, mode="affine")
    A = np.random.default_rng(4).standard_normal((sk.d, 3))
    Y = np.zeros((sk.k, 3))
    for g in range(sk.M):
        for ell, h in enumerate(bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, g), start=1):
            for u in range(sk.B_c):
                for j in range(sk.s):
                    r, sg = bp.pattern_affine(sk, g, ell, u, j)
                    Y[g * sk.B_r + r] += sg * A[h * sk.B_c + u]
    Y /= math.sqrt(sk.kappa * sk.s)
    assert np.allclose(oracle.apply(sk, A), Y, rtol=0, atol=1e-13)
    assert np.array_equal(oracle.build_S_dense(sk), oracle.build_S_csr(sk).toarray())


def test_shift_uniform_scale_odd_signs_balanced():
    sk = oracle.make_sketch(128, 32, 8192, 4, 4, seed=1234, mode="affine")
    al, be, sg = [], [], []
    for u in range(sk.B_c):
        a, b, z = bp.affine_params(sk, 5, 2, u)
        al.append(a)
        be.append(b)
        sg.extend(((z >> j) & 1) for j in range(sk.s))
    al, be, sg = np.array(al), np.array(be), np.array(sg)
    assert np.all(al % 2 == 1) and np.all((0 < al) & (al < sk.B_r))
    for vals, bins in [(be, sk.B_r), ((al - 1) // 2, sk.B_r // 2)]:
        counts = np.bincount(vals, minlength=bins)
        exp = len(vals) / bins
        assert float(((counts - exp) ** 2 / exp).sum()) < 70.0  # ≤ 31 dof, p ≈ 1e-4
    assert abs(sg.mean() - 0.5) < 4 * 0.5 / math.sqrt(sg.size)


def test_monte_carlo_unbiased_affine():
    """E‖Sx‖² = ‖x‖² (independent signs per column): mean over seeds within 4 SE."""
    x = np.random.default_rng(5).standard_normal(1024)
    vals = []
    for seed in range(1500):
        sk = oracle.make_sketch(8, 32, 128, 2, 2, seed=seed, mode="affine")
        y = oracle.build_S_csr(sk) @ x
        vals.append(float(y @ y) / float(x @ x))
    vals = np.array(vals)
    se = vals.std(ddof=1) / math.sqrt(len(vals))
    assert se < 0.005 and abs(vals.mean() - 1.0) < 4 * se


def test_affine_validation():
    for args in [(8, 24, 16, 2, 2), (8, 32, 16, 2, 33), (8, 1 << 17, 2, 2, 2)]:
        with pytest.raises(ValueError):
            oracle.make_sketch(*args, seed=0, mode="affine")
    oracle.make_sketch(8, 32, 16, 2, 3, seed=0, mode="affine")  # B_r % s != 0 allowed

"""Pins for the CPU oracle against what the paper (and mathematics) fix — DESIGN.md §4.

Each test names the passage it checks.  None of these compares the oracle with a
retyped copy of itself: they use the paper's worked example, SPEC restatements of
paper facts, closed forms (energy identity, isometry special case), brute force
(Hull–Dobell vs orbit enumeration) and statistics (E‖Sx‖² = ‖x‖², sign balance,
uniform row offsets).
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import blockperm as bp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------- wiring
def test_hull_dobell_matches_bruteforce_orbit_all_M_le_64():
    """conditions (a)-(c) ⇔ period M; exhaustive for M ≤ 64."""
    mismatches = 0
    for M in range(1, 65):
        for a in range(M):
            for b in range(M):
                if bp.hull_dobell(a, b, M) != bp.full_cycle_bruteforce(a, b, M):
                    mismatches += 1
    assert mismatches == 0


def test_spec_worked_examples():
    g = _gold("paper_spec_examples.json")
    for ex in g["hull_dobell"]:
        assert bp.hull_dobell(ex["a"], ex["b"], ex["M"]) == ex["full_cycle"], ex["cite"]
        assert bp.full_cycle_bruteforce(ex["a"], ex["b"], ex["M"]) == ex["full_cycle"], ex["cite"]
    for ex in g["iterated_neighborhood"]:
        assert bp.neighborhood(ex["a"], ex["b"], ex["M"], ex["kappa"], ex["g"]) == ex["N"], ex["cite"]
    for ex in g["edge_disjoint"]:
        assert bp.check_edge_disjoint(ex["tables"]) == ex["edge_disjoint"], ex["cite"]
    assert bp.mix64(g["mix64_zero"]["in"]) == g["mix64_zero"]["out"]


@pytest.mark.parametrize("seed", [0, 1, 1234, 2**63 + 7, 2**64 - 1])
def test_select_affine_is_full_cycle(seed):
    """R4 must always land in the Hull–Dobell family, checked by brute force."""
    for M in list(range(1, 130)) + [256, 512, 1000, 1024]:
        a, b = bp.select_affine(seed, M)
        assert 0 <= a < M or M == 1
        assert bp.full_cycle_bruteforce(a, b, M), (M, a, b)
    assert bp.select_affine(seed, 1) == (0, 0)
    a, b = bp.select_affine(seed, 12)
    assert (a - 1) % 6 == 0 and (a - 1) % 4 == 0 and math.gcd(b, 12) == 1  # S:107 example


@pytest.mark.parametrize("seed", [3, 99])
def test_iterated_wiring_is_edge_disjoint_and_bijective(seed):
    """π_ℓ = f^ℓ are bijections and pairwise derangements for κ ≤ M;
    κ = M gives N(g) = [M]."""
    for M in range(1, 65):
        a, b = bp.select_affine(seed, M)
        for kappa in sorted(k for k in {1, 2, 3, M} if k <= M):
            T = bp.neighborhoods(a, b, M, kappa)
            tables = [T[:, l] for l in range(kappa)]
            for t in tables:
                assert sorted(t.tolist()) == list(range(M))  # bijection
            assert bp.check_edge_disjoint(tables)
            if kappa == M:
                for g in range(M):
                    assert sorted(T[g].tolist()) == list(range(M))


def test_orbit_sliding_window():
    """With g_i = f^i(0), N(g_i) = (g_{i+1}, ..., g_{i+κ}) (P:1528 iterated map) — the
    structural fact the kernel's orbit ordering relies on."""
    for (M, kappa, seed) in [(8, 3, 1), (128, 8, 5), (16, 4, 9), (512, 8, 2)]:
        a, b = bp.select_affine(seed, M)
        orb = bp.orbit(a, b, M)
        assert sorted(orb) == list(range(M))
        for i in range(M):
            assert bp.neighborhood(a, b, M, kappa, orb[i]) == [orb[(i + l) % M] for l in range(1, kappa + 1)]


# ----------------------------------------------------------------------- S shape
def test_figure_example_structure():
    """Fig. caption: M=16, B_r=64, B_c=128, κ=4, s=2 → d=2048, k=1024,
    κs = 8 nonzeros per column, each of magnitude 1/√(κs); κ-regular block
    graph; one nonzero per row chunk j in each (g,h) block column."""
    f = _gold("paper_spec_examples.json")["figure_example"]
    sk = oracle.make_sketch(f["M"], f["B_r"], f["B_c"], f["kappa"], f["s"], seed=77)
    assert (sk.d, sk.k) == (f["d"], f["k"])
    S = oracle.build_S_dense(sk)
    nnz_col = (S != 0).sum(axis=0)
    assert np.all(nnz_col == f["nnz_per_column"])
    assert np.all(np.abs(S[S != 0]) == f["magnitude"])
    # block support
    blk = np.abs(S).reshape(sk.M, sk.B_r, sk.M, sk.B_c).sum(axis=(1, 3)) > 0
    assert np.all(blk.sum(axis=1) == sk.kappa) and np.all(blk.sum(axis=0) == sk.kappa)
    for g in range(sk.M):
        assert set(np.nonzero(blk[g])[0].tolist()) == set(bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, g))
    # row-partitioned: each chunk of C rows holds exactly one nonzero per (g,h) column
    C = sk.C
    for g in range(sk.M):
        for h in bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, g):
            B = S[g * sk.B_r:(g + 1) * sk.B_r, h * sk.B_c:(h + 1) * sk.B_c]
            per_chunk = (B != 0).reshape(sk.s, C, sk.B_c).sum(axis=1)
            assert np.all(per_chunk == 1)


def test_kappa1_is_block_diagonal_up_to_permutation():
    """P:1994 / P:1603: κ = 1 reduces to a localized block-diagonal SJLT."""
    sk = oracle.make_sketch(8, 16, 32, 1, 4, seed=5)
    S = oracle.build_S_dense(sk)
    blk = np.abs(S).reshape(sk.M, sk.B_r, sk.M, sk.B_c).sum(axis=(1, 3)) > 0
    assert np.all(blk.sum(axis=1) == 1) and np.all(blk.sum(axis=0) == 1)


def test_signed_permutation_isometry():
    """κ = s = B_r = B_c = 1, M = k = d: S is a signed permutation, ‖Sx‖ = ‖x‖ exactly."""
    sk = oracle.make_sketch(64, 1, 1, 1, 1, seed=11)
    S = oracle.build_S_dense(sk)
    assert np.all(np.abs(S).sum(axis=0) == 1) and np.all(np.abs(S).sum(axis=1) == 1)
    x = np.random.default_rng(0).standard_normal(64)
    assert np.linalg.norm(S @ x) == pytest.approx(np.linalg.norm(x), rel=1e-15)


def test_dense_and_csr_agree_and_linearity():
    sk = oracle.make_sketch(8, 32, 128, 2, 2, seed=1)
    Sd = oracle.build_S_dense(sk)
    Sc = oracle.build_S_csr(sk).toarray()
    assert np.array_equal(Sd, Sc)
    sub = oracle.build_S_csr(sk, blocks=[3, 1]).toarray()
    assert np.array_equal(sub[:32], Sd[96:128]) and np.array_equal(sub[32:], Sd[32:64])
    rng = np.random.default_rng(2)
    A, B = rng.standard_normal((sk.d, 5)), rng.standard_normal((sk.d, 5))
    assert np.allclose(oracle.apply(sk, 2 * A - 3 * B), 2 * oracle.apply(sk, A) - 3 * oracle.apply(sk, B), atol=1e-12)
    assert not np.any(oracle.apply(sk, np.zeros((sk.d, 3))))
    assert np.allclose(oracle.apply_t(sk, A.T), oracle.apply(sk, A).T, atol=0)


def test_apply_equals_triplet_sum_bruteforce():
    """Brute force on a tiny case: Y[i,t] = Σ over the κ·s·B_c nonzeros of block row g,
    enumerated one (ℓ,u,j) at a time with Python ints (Alg. 1's loop
    structure, scale applied last)."""
    sk = oracle.make_sketch(4, 8, 16, 2, 2, seed=3)
    A = np.random.default_rng(4).standard_normal((sk.d, 3))
    Y = np.zeros((sk.k, 3))
    for g in range(sk.M):
        for ell, h in enumerate(bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, g), start=1):
            for u in range(sk.B_c):
                for j in range(sk.s):
                    r, sg = bp.pattern(sk, g, ell, u, j)
                    Y[g * sk.B_r + r] += sg * A[h * sk.B_c + u]
    Y /= math.sqrt(sk.kappa * sk.s)
    assert np.allclose(oracle.apply(sk, A), Y, rtol=0, atol=1e-13)


def test_nonfinite_inputs_follow_the_sparse_sum():
    """R12: Y = S·A is the sum over the nonzeros of S (Alg. 1); an input element
    reaches only the κ·s rows its column of S names (κs nonzeros per column).  Pinned
    against the brute-force triplet loop with Python floats (IEEE: x + Inf = Inf, Inf − Inf = NaN,
    NaN propagates) and, for a huge finite value, against exact rational arithmetic."""
    from fractions import Fraction

    sk = oracle.make_sketch(4, 8, 16, 2, 2, seed=3)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((sk.d, 4))
    A[5, 0] = np.inf
    A[9, 1] = np.nan
    A[17, 2], A[40, 2] = np.inf, -np.inf
    A[33, 3] = 3.4e38  # beyond the bf16 range, finite in fp32 and fp64
    Y = oracle.apply(sk, A)
    ref = [[0.0] * 4 for _ in range(sk.k)]
    exact3 = [Fraction(0)] * sk.k
    for g in range(sk.M):
        for ell, h in enumerate(bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, g), start=1):
            for u in range(sk.B_c):
                for j in range(sk.s):
                    r, sg = bp.pattern(sk, g, ell, u, j)
                    for t in range(4):
                        ref[g * sk.B_r + r][t] += sg * float(A[h * sk.B_c + u, t])
                    exact3[g * sk.B_r + r] += sg * Fraction(float(A[h * sk.B_c + u, 3]))
    ref = np.array(ref) / math.sqrt(sk.kappa * sk.s)
    # non-finite pattern: exactly the rows the brute force puts there
    assert np.array_equal(np.isnan(Y), np.isnan(ref)) and np.array_equal(np.isposinf(Y), np.isposinf(ref))
    assert np.array_equal(np.isneginf(Y), np.isneginf(ref))
    S = oracle.build_S_csr(sk)
    assert (~np.isfinite(Y[:, 0])).sum() == sk.kappa * sk.s  # one Inf input: κs infinite rows
    assert set(np.flatnonzero(~np.isfinite(Y[:, 0]))) == set(S[:, 5].nonzero()[0])
    assert (np.isnan(Y[:, 1])).sum() == sk.kappa * sk.s
    fin = np.isfinite(ref)
    assert np.allclose(Y[fin], ref[fin], rtol=1e-12, atol=1e-12)
    want3 = np.array([float(v) for v in exact3]) / math.sqrt(sk.kappa * sk.s)
    assert np.all(np.isfinite(Y[:, 3])) and np.allclose(Y[:, 3], want3, rtol=1e-12, atol=1e-9)


# --------------------------------------------------------------- identities
def test_energy_identity():
    """Lemma P:54-65: Σ_g ‖x_N(g)‖² = κ‖x‖² and Σ_g U_Nᵀ U_N = κ UᵀU."""
    rng = np.random.default_rng(8)
    for (M, Br, Bc, kappa, s) in [(8, 32, 128, 2, 2), (16, 64, 128, 4, 2), (13, 4, 7, 5, 1)]:
        sk = oracle.make_sketch(M, Br, Bc, kappa, s, seed=21)
        x = rng.standard_normal(sk.d)
        assert oracle.energy_identity_lhs(sk, x) == pytest.approx(kappa * float(x @ x), rel=1e-12)
        U = rng.standard_normal((sk.d, 3))
        lhs = np.zeros((3, 3))
        for g in range(M):
            idx = np.concatenate([np.arange(h * Bc, (h + 1) * Bc) for h in bp.neighborhood(sk.a, sk.b, M, kappa, g)])
            lhs += U[idx].T @ U[idx]
        assert np.allclose(lhs, kappa * U.T @ U, rtol=1e-12, atol=1e-10)


@pytest.mark.slow
def test_monte_carlo_unbiased():
    """E‖Sx‖² = ‖x‖² (per-column unbiasedness of the row-partitioned SJLT, plus
    the energy identity); BASELINE north_star: mean within 1 ± 0.01.
    4000 seeds, Gaussian x fixed, tiny layout (R13)."""
    x = np.random.default_rng(123).standard_normal(1024)
    nx = float(x @ x)
    vals = []
    for seed in range(4000):
        sk = oracle.make_sketch(8, 32, 128, 2, 2, seed=seed)
        y = oracle.build_S_csr(sk) @ x
        vals.append(float(y @ y) / nx)
    vals = np.array(vals)
    se = vals.std(ddof=1) / math.sqrt(len(vals))
    assert se < 0.0025
    assert abs(vals.mean() - 1.0) < 0.01


def test_sign_balance_and_row_uniformity():
    """Independent Rademacher signs and uniform row positions inside each chunk
    (P:97): sign mean within 4σ of 0 and chi-square of row offsets, C = 8."""
    sk = oracle.make_sketch(128, 32, 8192, 4, 4, seed=1234)  # LS layout, C = 8
    r, c, v = bp._block_entries(sk, 5)
    sign = np.sign(v)
    n = sign.size
    assert abs(sign.mean()) < 4 / math.sqrt(n)
    off = (r - 5 * sk.B_r) % sk.C
    counts = np.bincount(off, minlength=sk.C)
    expected = n / sk.C
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    assert chi2 < 30.0  # 7 dof; P(chi2 > 30) ≈ 1e-4


def test_counter_layout_validation():
    with pytest.raises(ValueError):
        oracle.make_sketch(8, 32, 128, 9, 2, seed=0)  # κ > M
    with pytest.raises(ValueError):
        oracle.make_sketch(8, 30, 128, 2, 4, seed=0)  # B_r % s != 0
    with pytest.raises(ValueError):
        oracle.make_sketch(8, 32, 1 << 24, 2, 2, seed=0)  # u field overflow


def test_matches_independent_scratch_vectors():
    """SURVEY.md App. A vectors from an independent scratch implementation of R2-R4."""
    g = _gold("survey_appA_vectors.json")
    for M, ab in g["affine"].items():
        assert list(bp.select_affine(g["seed"], int(M))) == ab
    assert hex(bp.mix64(g["seed"] ^ bp.TAG_PHI)) == g["K"]
    assert hex(bp.mix64(1)) == g["mix64_1"]
    t = g["tiny_patterns_g0"]
    sk = oracle.make_sketch(*t["layout"], seed=g["seed"])
    assert bp.neighborhood(sk.a, sk.b, sk.M, sk.kappa, 0) == g["tiny_N0"]
    for ell, key in ((1, "ell1"), (2, "ell2")):
        for u, pair in enumerate(t[key]):
            for j, (row, sign) in enumerate(pair):
                assert bp.pattern(sk, 0, ell, u, j) == (row, sign)


def test_adjoint_identity():
    """⟨S x, y⟩ = ⟨x, Sᵀ y⟩ for all x, y (definition of the adjoint), through the oracle's two
    independent code paths (apply builds rows of S per output block; apply_adjoint transposes)."""
    rng = np.random.default_rng(9)
    for layout in [(8, 32, 128, 2, 2), (16, 64, 128, 4, 2), (32, 16, 256, 8, 2)]:
        sk = oracle.make_sketch(*layout, seed=4)
        X = rng.standard_normal((sk.d, 3))
        Yv = rng.standard_normal((sk.k, 3))
        lhs = np.sum(oracle.apply(sk, X) * Yv)
        rhs = np.sum(X * oracle.apply_adjoint(sk, Yv))
        assert lhs == pytest.approx(rhs, rel=1e-12)
        # each column of Sᵀ has κs... each row of Sᵀ (= column of S) has κs nonzeros: Sᵀ e_i
        E = np.zeros((sk.k, 1))
        E[5] = 1.0
        col = oracle.apply_adjoint(sk, E)[:, 0]
        S = oracle.build_S_dense(sk)
        assert np.array_equal(col, S[5])

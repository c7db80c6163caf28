"""GPU parity of the AffineUnique intra-block mode (R18; §8f rank 4) through the C ABI.

Same criteria as the row-partitioned mode (tests/test_gpu_parity.py): bit-exact selector
columns; fp32 max|err| ≤ 1e-5·‖A_col‖₂; bf16 2e-2 relative plus the tight bound on the rounded
input.  Covers both kernels, both layouts, the full-size LS shape and the adjoint.
"""

import numpy as np
import pytest

import oracle
import synth
from parity import assert_bf16, assert_f32
from test_gpu_parity import _run, _sampled_check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402

VARIANTS = ["sparse", "tc"]


def _pair(M, Br, Bc, kappa, s, seed=1234):
    return (Sketch(M, Br, Bc, kappa, s, seed, mode="affine"),
            oracle.make_sketch(M, Br, Bc, kappa, s, seed, mode="affine"))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (16, 64, 128, 4, 8), (128, 32, 8192, 4, 4),
                                    (512, 16, 32768, 8, 2), (16, 32, 256, 2, 3)])
def test_affine_selector_columns_bit_exact(variant, layout):
    sk, osk = _pair(*layout)
    M, Br, Bc, kappa, s = layout
    rng = np.random.default_rng(0)
    h = int(rng.integers(M))
    J = np.concatenate([[h * Bc, h * Bc + Bc - 1], h * Bc + rng.choice(Bc, 30, replace=False)])
    A = torch.zeros((sk.d, len(J)), device="cuda")
    A[torch.as_tensor(J, device="cuda"), torch.arange(len(J), device="cuda")] = 1.0
    try:
        Y = sk.apply(A, variant=variant).cpu().numpy()
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    S = oracle.build_S_csr(osk)[:, J].toarray()
    assert np.array_equal(Y != 0, S != 0)
    assert np.array_equal(np.sign(Y), np.sign(S))
    assert np.all(np.abs(Y[Y != 0]) == np.float32(sk.scale))
    assert ((Y != 0).sum(axis=0) == kappa * s).all()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(5, 16, 40, 3, 3), (8, 32, 128, 8, 2), (4, 8, 64, 2, 8), (64, 16, 512, 8, 2),
                                    (7, 4, 96, 7, 4), (16, 32, 192, 4, 5)])
@pytest.mark.parametrize("n", [1, 17, 130])
def test_affine_layouts_ragged_n(variant, layout, n):
    sk, osk = _pair(*layout, seed=99)
    A = synth.host_matrix("gaussian", sk.d, n, seed=n)
    Yref = oracle.apply(osk, A)
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    assert_f32(_run(sk, A, variant), Yref, nrm, f"{layout} n={n} {variant}")
    assert_f32(_run(sk, A.T, variant, transposed=True).T, Yref, nrm, f"T {layout} n={n} {variant}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_affine_bf16(variant):
    sk, osk = _pair(64, 16, 512, 8, 2, seed=5)
    A = synth.host_matrix("gaussian", sk.d, 96, seed=3)
    Y = _run(sk, A, variant, dtype=torch.bfloat16)
    assert_bf16(Y, oracle.apply(osk, A), "bf16 vs fp32 A")
    Ab = synth.bf16_round(A)
    assert_f32(Y, oracle.apply(osk, Ab), np.linalg.norm(Ab.astype(np.float64), axis=0), "bf16 tight")


@pytest.mark.parametrize("variant", ["auto", "sparse"])
def test_affine_ls_config_sampled(variant):
    _sampled_check(C.LS, variant, mode="affine")


def test_affine_grad_config_sampled():
    _sampled_check(C.GRAD, "auto", mode="affine")
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (32, 16, 256, 8, 2), (16, 64, 128, 4, 8)])
def test_affine_adjoint(variant, layout):
    sk, osk = _pair(*layout, seed=4)
    n = 72
    Yh = synth.host_matrix("gaussian", sk.k, n, seed=2)
    Y = torch.from_numpy(Yh).cuda()
    try:
        X = sk.apply_adjoint(Y, variant=variant).cpu().numpy()
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    assert_f32(X, oracle.apply_adjoint(osk, Yh.astype(np.float64)), np.linalg.norm(Yh.astype(np.float64), axis=0),
               f"adjoint {layout} {variant}")

"""GPU parity of the adjoint X = Sᵀ·Y (bps_apply_adjoint) vs the oracle.

Tolerance: each X element is a signed sum of κ·s entries of one Y column times 1/√(κs), so the
fp32 rule of the forward path applies with Y's column norm: max|err| ≤ 1e-5·‖Y[:,t]‖₂.
Selector columns (Y = e_i) are bit-exact: Sᵀe_i is row i of S.
"""

import numpy as np
import pytest

import oracle
import synth
from parity import assert_f32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402


def _pair(M, Br, Bc, kappa, s, seed=1234):
    return Sketch(M, Br, Bc, kappa, s, seed), oracle.make_sketch(M, Br, Bc, kappa, s, seed)


def _padded(rows, cols, fill=None):
    ld = max(4, -(-cols // 4) * 4)
    base = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
    v = base[:, :cols]
    if fill is not None:
        v.copy_(fill)
    return v


VARIANTS = ["sparse", "tc"]


def _adjoint(sk, Y_host, variant="auto"):
    Y = _padded(sk.k, Y_host.shape[1], torch.from_numpy(np.ascontiguousarray(Y_host, np.float32)).cuda())
    X = _padded(sk.d, Y_host.shape[1])
    try:
        sk.apply_adjoint(Y, out=X, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(f"tc adjoint does not cover this shape: {e}")
        raise
    torch.cuda.synchronize()
    return X.cpu().numpy()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (16, 64, 128, 4, 2), (32, 16, 256, 8, 2),
                                    (12, 24, 96, 3, 3), (5, 8, 40, 5, 1), (1, 32, 64, 1, 4),
                                    (6, 24, 192, 3, 3), (64, 16, 512, 8, 4)])
@pytest.mark.parametrize("n", [1, 7, 33, 64, 128, 300, 520])
def test_adjoint_matches_oracle(layout, n, variant):
    sk, osk = _pair(*layout)
    Yh = synth.host_matrix("gaussian", sk.k, n, seed=11 + n)
    X = _adjoint(sk, Yh, variant)
    Xr = oracle.apply_adjoint(osk, Yh.astype(np.float64))
    assert_f32(X, Xr, np.linalg.norm(Yh.astype(np.float64), axis=0), f"adjoint {layout} n={n}")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (128, 32, 8192, 4, 4), (512, 16, 32768, 8, 2)])
def test_adjoint_selector_rows_bit_exact(layout, variant):
    """Y = E_I (unit columns at rows I) gives X = S[I, :]ᵀ: positions, signs and the value
    fp32(1/√(κs)) must match the oracle's explicit S exactly."""
    sk, osk = _pair(*layout)
    M, Br = layout[0], layout[1]
    rng = np.random.default_rng(3)
    g = int(rng.integers(M))
    I = np.concatenate([[g * Br, g * Br + Br - 1], g * Br + rng.choice(Br, min(Br, 14), replace=False)])
    Yh = np.zeros((sk.k, len(I)), np.float32)
    Yh[I, np.arange(len(I))] = 1.0
    X = _adjoint(sk, Yh, variant)
    S_rows = oracle.build_S_csr(osk, blocks=[g])[I - g * Br].toarray()  # len(I) × d
    assert np.array_equal(X.T != 0, S_rows != 0)
    assert np.array_equal(np.sign(X.T), np.sign(S_rows))
    assert np.all(np.abs(X[X != 0]) == np.float32(sk.scale))


@pytest.mark.parametrize("variant", VARIANTS)
def test_adjoint_identity_with_forward(variant):
    """⟨S·A, Y⟩ = ⟨A, Sᵀ·Y⟩ with both sides from libbps (forward tc/sparse vs adjoint)."""
    sk = Sketch(64, 32, 1024, 4, 4, seed=5)
    A = synth.device_matrix("gaussian", sk.d, 256, seed=1, dtype=torch.float32)
    Y = synth.device_matrix("gaussian", sk.k, 256, seed=2, dtype=torch.float32)
    lhs = float((sk.apply(A).double() * Y.double()).sum())
    rhs = float((A.double() * sk.apply_adjoint(Y, variant=variant).double()).sum())
    assert lhs == pytest.approx(rhs, rel=1e-5)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("cfg", [C.LS, C.SMALLN], ids=["ls", "smalln"])
def test_adjoint_sampled_blocks(cfg, variant):
    """LS shape (d = 2^20, k = 4096, κ = s = 4, n = 512) and the narrow shape (d = 2^24, n = 32),
    in the bench's launch configuration: sampled input blocks of X against Sᵀ restricted to
    the κ output blocks that feed them (computed by the oracle)."""
    sk, osk = Sketch(**cfg.sketch_args()), oracle.make_sketch(**cfg.sketch_args())
    Y = synth.device_matrix("gaussian", sk.k, cfg.n, seed=7, dtype=torch.float32)
    X = sk.apply_adjoint(Y, variant=variant)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy().astype(np.float64)
    norms = np.linalg.norm(Yh, axis=0)
    rng = np.random.default_rng(0)
    for h in [0, cfg.M - 1, *rng.choice(cfg.M, 3, replace=False)]:
        gs = [g for g in range(cfg.M) if h in oracle.neighborhood(osk.a, osk.b, cfg.M, cfg.kappa, g)]
        S_sub = oracle.build_S_csr(osk, blocks=gs)[:, h * cfg.B_c:(h + 1) * cfg.B_c]
        rows = np.concatenate([np.arange(g * cfg.B_r, (g + 1) * cfg.B_r) for g in gs])
        Xr = S_sub.T @ Yh[rows]
        assert_f32(X[h * cfg.B_c:(h + 1) * cfg.B_c].cpu().numpy(), Xr, norms, f"{cfg.name} adjoint block {h}")


def test_adjoint_deterministic_and_unsupported():
    sk = Sketch(64, 32, 1024, 4, 4, seed=5)
    Y = synth.device_matrix("gaussian", sk.k, 200, seed=3, dtype=torch.float32)[:, :197]
    for v in VARIANTS:
        a = sk.apply_adjoint(Y, out=_padded(sk.d, 197), variant=v)
        b = sk.apply_adjoint(Y, out=_padded(sk.d, 197), variant=v)
        assert torch.equal(a, b)
    big = Sketch(16, 256, 64, 2, 2, seed=1)  # κ·B_r = 512 > 400
    with pytest.raises(BpsError) as e:
        big.apply_adjoint(torch.zeros((big.k, 8), device="cuda"))
    assert e.value.code == -3

"""GPU parity of FlashBlockRow (§8f rank 3) through the C ABI vs the oracle.

Criteria (BJ's, adapted to this sketch's scale): the block-row scale (κs)^{-1/2}(d/k)^{1/2} is
not ≤ 1, so the fp32 bound is max|err| ≤ 1e-5·scale·√(κs)·‖A_col‖₂ (an output sums κs signed
inputs, then is scaled); bf16 inputs: 2e-2 per-column relative ℓ2 vs the fp32-A oracle.
Columns of S (A = E_J) are bit-exact.
"""

import numpy as np
import pytest

import synth
from oracle import blockrow as BR
from parity import assert_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402


def _pair(M, Br, Bc, kappa, s, seed=1234):
    return Sketch(M, Br, Bc, kappa, s, seed, kind="blockrow"), BR.make_blockrow(M, Br, Bc, kappa, s, seed)


def _padded(rows, cols, dtype, fill=None):
    mult = 16 // torch.tensor([], dtype=dtype).element_size()
    ld = max(mult, -(-cols // mult) * mult)
    v = torch.zeros((rows, ld), dtype=dtype, device="cuda")[:, :cols]
    if fill is not None:
        v.copy_(fill)
    return v


def _assert_f32(Y, Yr, A64, br, what):
    bound = 1e-5 * br.scale * np.sqrt(br.kappa * br.s) * np.linalg.norm(A64, axis=0)
    err = np.abs(np.asarray(Y, np.float64) - Yr).max(axis=0)
    assert np.all(err <= np.maximum(bound, 1e-30)), f"{what}: max err/bound {float((err / np.maximum(bound, 1e-30)).max()):.3e}"


LAYOUTS = [(8, 4, 16, 2, 2), (5, 3, 7, 5, 3), (1, 2, 9, 1, 4), (16, 8, 64, 3, 1), (32, 16, 256, 8, 2), (12, 7, 40, 4, 5),
           (64, 8, 128, 4, 2)]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("n", [1, 5, 33, 130, 300, 600])
def test_blockrow_rowmajor_f32(layout, n):
    sk, br = _pair(*layout)
    A = synth.host_matrix("gaussian", br.d, n, seed=n)
    Ad = _padded(br.d, n, torch.float32, torch.from_numpy(A).cuda())
    Y = _padded(br.k, n, torch.float32)
    sk.apply(Ad, out=Y)
    torch.cuda.synchronize()
    A64 = A.astype(np.float64)
    _assert_f32(Y.cpu().numpy(), BR.apply(br, A64), A64, br, f"{layout} n={n}")


@pytest.mark.parametrize("layout", LAYOUTS[:4] + LAYOUTS[-1:])
@pytest.mark.parametrize("n", [3, 40, 64, 520])
def test_blockrow_bf16_and_transposed(layout, n):
    sk, br = _pair(*layout)
    A = synth.host_matrix("gaussian", br.d, n, seed=7 + n)
    Ab = torch.from_numpy(A).cuda().to(torch.bfloat16)
    Ad = _padded(br.d, n, torch.bfloat16, Ab)
    Y = _padded(br.k, n, torch.float32)
    sk.apply(Ad, out=Y)
    torch.cuda.synchronize()
    A64b = Ab.float().cpu().numpy().astype(np.float64)
    # R9: tight fp32 criterion against the oracle on the bf16-rounded input, and the 2e-2
    # relative criterion against fp32 A where a column has enough rows for it to be meaningful
    _assert_f32(Y.cpu().numpy(), BR.apply(br, A64b), A64b, br, f"bf16 (rounded A) {layout} n={n}")
    if br.k >= 32:
        assert_bf16(Y.cpu().numpy(), BR.apply(br, A.astype(np.float64)), f"bf16 {layout} n={n}")
    # transposed layout, fp32 and bf16: X = Aᵀ (n×d) -> Yᵀ (n×k)
    for dt, src in [(torch.float32, torch.from_numpy(A).cuda()), (torch.bfloat16, Ab)]:
        X = _padded(n, br.d, dt, src.T)
        Yt = _padded(n, br.k, torch.float32)
        sk.apply_t(X, out=Yt)
        torch.cuda.synchronize()
        ref = BR.apply(br, A.astype(np.float64) if dt == torch.float32 else A64b).T
        _assert_f32(Yt.cpu().numpy().T, ref.T, (A.astype(np.float64) if dt == torch.float32 else A64b), br,
                    f"transposed {dt} {layout} n={n}")


@pytest.mark.parametrize("layout", [(8, 4, 16, 2, 2), (128, 32, 8192, 4, 4)])
def test_blockrow_columns_bit_exact(layout):
    """A = E_J gives S[:, J]: values are exact fp32 multiples of the scale (duplicates add,
    opposite signs cancel) and equal the oracle's S bit-for-bit after fp32 rounding."""
    sk, br = _pair(*layout)
    rng = np.random.default_rng(2)
    g = int(rng.integers(br.M))
    nb = BR.neighbors_row(br, g)
    # columns actually hit by block g (so the test is not vacuous) plus a few random ones
    hit = sorted({nb[ell - 1] * br.B_c + BR.draw_index(br, g, ell, r, t)[0]
                  for ell in range(1, br.kappa + 1) for r in range(br.B_r) for t in range(br.s)})
    J = np.array(hit[:24] + list(rng.choice(br.d, 8, replace=False)))
    A = _padded(br.d, len(J), torch.float32)
    A[torch.as_tensor(J, device="cuda"), torch.arange(len(J), device="cuda")] = 1.0
    Y = sk.apply(A, out=_padded(br.k, len(J), torch.float32)).cpu().numpy()
    S = BR.build_S_csr(br, blocks=[g])[:, J].toarray()
    rows = slice(g * br.B_r, (g + 1) * br.B_r)
    q = S / br.scale
    expect = (np.round(q).astype(np.float32) * np.float32(br.scale)).astype(np.float32)
    assert np.array_equal(Y[rows], expect)
    assert np.count_nonzero(Y[rows]) > 0


def test_blockrow_ls_shape_sampled():
    """LS shape (d = 2^20, k = 4096, κ = s = 4, n = 512, fp32) in the bench launch: sampled
    output blocks × 16 columns against the oracle."""
    cfg = C.LS
    sk, br = _pair(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed)
    A = synth.device_matrix("gaussian", br.d, cfg.n, seed=3, dtype=torch.float32)
    Y = sk.apply(A)
    torch.cuda.synchronize()
    cols = np.array([0, 1, 2, 3, 127, 128, 255, 256, 300, 383, 384, 500, 508, 509, 510, 511])
    A_sub = A[:, torch.as_tensor(cols, device="cuda")].cpu().numpy().astype(np.float64)
    blocks = [0, cfg.M - 1, 17, 64]
    Yr = BR.apply(br, A_sub, blocks=blocks)
    rows = np.concatenate([np.arange(g * br.B_r, (g + 1) * br.B_r) for g in blocks])
    _assert_f32(Y.cpu().numpy()[rows][:, cols], Yr, A_sub, br, "LS blockrow")


def test_blockrow_unsupported_and_deterministic():
    sk, br = _pair(16, 8, 64, 3, 1)
    A = synth.device_matrix("gaussian", br.d, 96, seed=1, dtype=torch.float32)
    assert torch.equal(sk.apply(A), sk.apply(A))
    with pytest.raises(BpsError) as e:
        sk.apply(A, variant="tc")
    assert e.value.code == -3
    with pytest.raises(BpsError) as e:
        sk.apply_adjoint(torch.zeros((br.k, 8), device="cuda"))
    assert e.value.code == -3

"""Non-finite, huge and subnormal inputs (reading R12): every kernel computes the sparse
sum of Alg. 1 — an input element reaches only the κ·s rows its column of S names —
exactly as the oracle does.  The tcgen05 kernel multiplies the dense ±1 band, so it detects
non-finite outputs and recomputes those columns by the sparse definition.

Run on a B200:  python -m pytest tests -m gpu
"""

import numpy as np
import pytest

import oracle
import synth
from parity import F32_TOL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402

LAYOUTS = [(16, 32, 1024, 4, 4), (64, 16, 512, 8, 2), (32, 32, 2048, 16, 4), (8, 32, 128, 2, 2), (5, 12, 40, 3, 3)]
BF16_MAX = 3.3895313892515355e38


def _inputs(d, dt, seed=6):
    """Columns: 0 one +Inf; 1 one NaN; 2 +Inf and -Inf; 3 huge finite values (beyond the bf16 range
    for fp32, the bf16 maximum for bf16) whose partial sums overflow fp32; 4 subnormal column;
    5 tiny normal column; 6 ordinary Gaussian; 7 -Inf in every block."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((d, 8)).astype(np.float32)
    A[d // 3, 0] = np.inf
    A[d // 2 + 1, 1] = np.nan
    A[7, 2], A[d - 5, 2] = np.inf, -np.inf
    big = np.float32(3.4e38) if dt == "f32" else np.float32(BF16_MAX)
    A[rng.choice(d, 6, replace=False), 3] = big * np.sign(rng.standard_normal(6)).astype(np.float32)
    A[:, 4] = (rng.standard_normal(d) * 1e-39).astype(np.float32)  # fp32 subnormals
    A[:, 5] *= np.float32(1e-30)
    A[::max(1, d // 7), 7] = -np.inf
    if dt == "bf16":
        A = synth.bf16_round(A)
    return A


def _check(Y, ref, A, what):
    for arr in (np.isnan, np.isposinf, np.isneginf):
        bad = arr(Y) != arr(ref)
        assert not bad.any(), f"{what}: {arr.__name__} pattern differs at {np.argwhere(bad)[:5].tolist()}"
    fin = np.isfinite(ref)
    A64 = np.where(np.isfinite(A), A.astype(np.float64), 0.0)
    nrm = np.linalg.norm(A64, axis=0)
    err = np.where(fin, np.abs(np.asarray(Y, np.float64) - np.where(fin, ref, 0.0)), 0.0).max(axis=0)
    big = np.abs(np.where(fin, ref, 0.0)).max(axis=0)
    # fp32 criterion per column; columns holding huge values: relative to the largest output
    tol = np.maximum(F32_TOL * nrm, 1e-6 * big)
    assert np.all(err <= tol), f"{what}: max|err| {err} > {tol}"


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("variant", ["tc", "sparse"])
@pytest.mark.parametrize("transposed", [False, True])
def test_nonfinite_and_extreme_inputs(layout, dt, variant, transposed):
    sk = Sketch(*layout, seed=41)
    osk = oracle.make_sketch(*layout, 41)
    A = _inputs(sk.d, dt)
    with np.errstate(invalid="ignore", over="ignore"):
        ref = oracle.apply(osk, A)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    At = torch.from_numpy(np.ascontiguousarray(A.T if transposed else A)).cuda().to(tdt)
    outs = []
    for ws in (True, False):
        try:
            Y = (sk.apply_t if transposed else sk.apply)(At, variant=variant, use_workspace=ws)
        except BpsError as e:
            if e.code == -3 and variant == "tc":
                pytest.skip(str(e))
            raise
        torch.cuda.synchronize()
        Yn = Y.cpu().numpy()
        outs.append(Yn.T if transposed else Yn)
    assert np.array_equal(outs[0], outs[1], equal_nan=True), "workspace vs halo ranges"
    with np.errstate(invalid="ignore"):
        _check(outs[0], ref, A, f"{layout} {dt} {variant} T={transposed}")


@pytest.mark.parametrize("variant", ["tc", "sparse"])
def test_subnormal_only_column(variant):
    """A column of fp32 subnormals alone: the result must keep them (not flush to zero)."""
    sk = Sketch(16, 32, 1024, 4, 4, seed=42)
    osk = oracle.make_sketch(16, 32, 1024, 4, 4, 42)
    rng = np.random.default_rng(3)
    A = (rng.standard_normal((sk.d, 16)) * 1e-40).astype(np.float32)
    ref = oracle.apply(osk, A)
    Y = sk.apply(torch.from_numpy(A).cuda(), variant=variant).cpu().numpy()
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    err = np.abs(Y.astype(np.float64) - ref).max(axis=0) / nrm
    assert np.all(err <= F32_TOL), err

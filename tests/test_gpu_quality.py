"""RandNLA task metrics computed with the GPU sketch agree with the same metrics
computed from the oracle's explicit S (float64), and reduce to exact values in the isometric
special case."""

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import Sketch  # noqa: E402
from paper_2602_06071_b200 import quality as Q  # noqa: E402


def _np_metrics(S, A, b, lam):
    G = A.T @ A
    SA, Sb = S @ A, S @ b
    Gh = SA.T @ SA
    gram = np.linalg.norm(Gh - G) / np.linalg.norm(G)
    Qm, _ = np.linalg.qr(A)
    SQ = S @ Qm
    ose = np.linalg.norm(SQ.T @ SQ - np.eye(Qm.shape[1]), 2)
    x = np.linalg.solve(SA.T @ SA + lam * np.eye(A.shape[1]), SA.T @ Sb)
    ridge = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    xs = np.linalg.lstsq(SA, Sb, rcond=None)[0]
    sas = np.linalg.norm(A @ xs - b) / np.linalg.norm(b)
    return gram, ose, ridge, sas


@pytest.mark.parametrize("kind", ["gaussian", "coherent", "lowrank"])
def test_metrics_match_oracle(kind):
    layout = (64, 32, 512, 4, 4)  # d = 32768, k = 2048
    sk = Sketch(*layout, seed=3)
    osk = oracle.make_sketch(*layout, seed=3)
    n = 60
    A = synth.host_matrix(kind, sk.d, n, seed=1, M=64).astype(np.float64)
    b = synth.host_matrix("gaussian", sk.d, 1, seed=2)[:, 0].astype(np.float64)
    S = oracle.build_S_csr(osk)
    ref = _np_metrics(S, A, b, lam=1e-2)
    At = torch.from_numpy(A.astype(np.float32)).cuda()
    bt = torch.from_numpy(b.astype(np.float32)).cuda()
    SA = sk.apply(torch.cat([At, torch.zeros((sk.d, 4), device="cuda")], 1).contiguous())[:, :n]
    got = (Q.gram_error(At, SA), Q.ose_error(sk, At, r=n), Q.ridge_residual(sk, At, bt, 1e-2)[1],
           Q.sketch_and_solve(sk, At, bt)[1])
    # inputs were rounded to fp32 for the GPU; metrics are smooth in A, agreement to ~1e-4 rel
    for g, r in zip(got, ref):
        assert g == pytest.approx(r, rel=2e-3, abs=1e-6)


def test_isometry_special_case():
    """κ = s = B_r = B_c = 1: S is a signed permutation — Gram error and OSE error are
    at rounding level and sketch-and-solve reproduces the exact least-squares residual."""
    d = 4096
    sk = Sketch(d, 1, 1, 1, 1, seed=5)
    A = torch.randn((d, 32), device="cuda")
    b = torch.randn(d, device="cuda")
    SA = sk.apply(A)
    assert Q.gram_error(A, SA) < 1e-6
    assert Q.ose_error(sk, A, r=32) < 1e-5
    exact = torch.linalg.lstsq(A.double(), b.double().reshape(-1, 1)).solution.reshape(-1)
    r_exact = float(torch.linalg.vector_norm(A.double() @ exact - b.double()) / torch.linalg.vector_norm(b.double()))
    _, r = Q.sketch_and_solve(sk, A, b)
    assert r == pytest.approx(r_exact, rel=1e-5)

"""Sketch-quality workloads on top of `Sketch.apply`.

The paper's RandNLA tasks consume SA; these functions compute its error metrics exactly as
defined in App. "Metrics", with the sketch applied by libbps on the GPU and the
small k×n algebra done by torch.linalg (float64):

  gram_error       E_Gram,rel = ‖(SA)ᵀ(SA) − AᵀA‖_F / ‖AᵀA‖_F
  ose_error        E_OSE = ‖(SQ)ᵀ(SQ) − I_r‖_2, Q = qr(A)[:, :r] or Gaussian probes
  ridge_residual   x = argmin ‖SAx − Sb‖² + λ‖x‖²,  ‖Ax − b‖ / ‖b‖
  sketch_and_solve x = argmin ‖SAx − Sb‖,            ‖Ax − b‖ / ‖b‖
"""

from __future__ import annotations

import torch

from .sketch import Sketch


def _rel(num: torch.Tensor, den: torch.Tensor) -> float:
    d = float(den)
    return float(num) / d if d > 0 else float(num)


def gram_error(A: torch.Tensor, SA: torch.Tensor) -> float:
    A64, SA64 = A.double(), SA.double()
    G = A64.T @ A64
    Gh = SA64.T @ SA64
    return _rel(torch.linalg.matrix_norm(Gh - G), torch.linalg.matrix_norm(G))


def ose_error(sk: Sketch, A: torch.Tensor | None = None, r: int = 64, probes: int = 0, seed: int = 0) -> float:
    """Column-space variant Q = qr(A) with r = min(r, d, n) (default), or Gaussian probes."""
    if probes:
        g = torch.Generator(device="cuda").manual_seed(seed)
        Q = torch.randn((sk.d, probes), generator=g, device="cuda", dtype=torch.float64)
        Q, _ = torch.linalg.qr(Q)
    else:
        rr = min(r, sk.d, A.shape[1])
        Q, _ = torch.linalg.qr(A.double())
        Q = Q[:, :rr]
    SQ = sk.apply(Q.float().contiguous()).double()
    I = torch.eye(SQ.shape[1], dtype=torch.float64, device=SQ.device)
    return float(torch.linalg.matrix_norm(SQ.T @ SQ - I, ord=2))


def _sketch_Ab(sk: Sketch, A: torch.Tensor, b: torch.Tensor):
    Ab = torch.cat([A, b.reshape(-1, 1).to(A.dtype)], dim=1)
    pad = (-Ab.shape[1]) % 4
    if pad:
        Ab = torch.cat([Ab, torch.zeros((Ab.shape[0], pad), dtype=Ab.dtype, device=Ab.device)], dim=1)
    S = sk.apply(Ab.contiguous()).double()
    n = A.shape[1]
    return S[:, :n], S[:, n]


def ridge_residual(sk: Sketch, A: torch.Tensor, b: torch.Tensor, lam: float) -> tuple[torch.Tensor, float]:
    SA, Sb = _sketch_Ab(sk, A, b)
    n = SA.shape[1]
    x = torch.linalg.solve(SA.T @ SA + lam * torch.eye(n, dtype=torch.float64, device=SA.device), SA.T @ Sb)
    res = A.double() @ x - b.double()
    return x, _rel(torch.linalg.vector_norm(res), torch.linalg.vector_norm(b.double()))


def sketch_and_solve(sk: Sketch, A: torch.Tensor, b: torch.Tensor) -> tuple[torch.Tensor, float]:
    SA, Sb = _sketch_Ab(sk, A, b)
    x = torch.linalg.lstsq(SA, Sb.reshape(-1, 1)).solution.reshape(-1)
    res = A.double() @ x - b.double()
    return x, _rel(torch.linalg.vector_norm(res), torch.linalg.vector_norm(b.double()))

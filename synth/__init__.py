"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

Holds none of the sketch's arithmetic (no wiring, hashing or scaling) — only input
matrices shaped like the paper's workloads:

  gaussian  : A_ij ~ N(0,1) i.i.d.
  coherent  : Gaussian with the rows of c = max(1, M//64) input blocks ×100
              ("planted block-coherent"; high μ_blk)
  lowrank   : G1 G2ᵀ/√r + σN, r = 16, σ = 0.1 (construction fixed by SPEC S:451;
              the paper only names "low-rank + noise")

Host (numpy) generators are used for parity-size cases; device (torch.cuda)
generators for bench-size matrices that would take too long to create on the host.
"""

from __future__ import annotations

import numpy as np

KINDS = ("gaussian", "coherent", "lowrank")


def coherent_blocks(M: int, seed: int) -> np.ndarray:
    """Which input blocks are scaled in the 'coherent' kind (depends on seed only)."""
    rng = np.random.default_rng(seed ^ 0xC0FFEE)
    c = max(1, M // 64)
    return np.sort(rng.choice(M, size=c, replace=False))


def host_matrix(kind: str, rows: int, cols: int, seed: int, *, M: int = 1, dtype=np.float32) -> np.ndarray:
    """rows×cols matrix (row-major) on the host. For 'coherent', rows must be M·B_c."""
    rng = np.random.default_rng(seed)
    if kind == "gaussian":
        A = rng.standard_normal((rows, cols), dtype=np.float32)
    elif kind == "coherent":
        A = rng.standard_normal((rows, cols), dtype=np.float32)
        Bc = rows // M
        for h in coherent_blocks(M, seed):
            A[h * Bc:(h + 1) * Bc] *= 100.0
    elif kind == "lowrank":
        r = 16
        G1 = rng.standard_normal((rows, r), dtype=np.float32)
        G2 = rng.standard_normal((cols, r), dtype=np.float32)
        A = (G1 @ G2.T) / np.float32(np.sqrt(r)) + np.float32(0.1) * rng.standard_normal((rows, cols), dtype=np.float32)
    elif kind == "zeros":
        A = np.zeros((rows, cols), dtype=np.float32)
    else:
        raise ValueError(kind)
    return A.astype(dtype, copy=False)


def device_matrix(kind: str, rows: int, cols: int, seed: int, *, M: int = 1, dtype=None, device="cuda", out=None):
    """Same distributions generated on the GPU with torch's Philox generator (values
    differ from host_matrix; parity tests copy the sampled rows/columns back)."""
    import torch

    dtype = dtype or torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    A = out if out is not None else torch.empty((rows, cols), dtype=dtype, device=device)
    # fill in row panels to bound the fp32 temporary
    panel = max(1, (1 << 28) // max(1, cols))
    for r0 in range(0, rows, panel):
        r1 = min(rows, r0 + panel)
        if kind == "lowrank":
            r = 16
            G1 = torch.randn((r1 - r0, r), generator=g, device=device)
            if r0 == 0:
                G2 = torch.randn((cols, r), generator=g, device=device)
            t = (G1 @ G2.T) / (r ** 0.5) + 0.1 * torch.randn((r1 - r0, cols), generator=g, device=device)
        else:
            t = torch.randn((r1 - r0, cols), generator=g, device=device)
        A[r0:r1].copy_(t)
    if kind == "coherent":
        Bc = rows // M
        for h in coherent_blocks(M, seed):
            A[h * Bc:(h + 1) * Bc] *= 100.0
    return A


def bf16_round(A: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 → bf16 → fp32 on the host (for the tight bf16 check)."""
    a = np.ascontiguousarray(A, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (a >> 16) & 1
    r = ((a + 0x7FFF + lsb) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(A.shape)

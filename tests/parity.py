"""Shared parity criteria (BASELINE.json north_star; DESIGN.md §4 / R9).

fp32 input : max_i |Y_gpu[i,t] - Y_ref[i,t]| ≤ 1e-5 · ‖A[:,t]‖₂ for every column t.
bf16 input : ‖Y_gpu[:,t] - Y_ref(fp32 A)[:,t]‖₂ ≤ 2e-2 · ‖Y_ref[:,t]‖₂ per column (primary),
             and the fp32 criterion against Y_ref(bf16-rounded A) (tight).
Indices, signs, nnz: bit-exact (selector columns).
"""

import numpy as np

F32_TOL = 1e-5
BF16_REL = 2e-2


def f32_violation(Y_gpu: np.ndarray, Y_ref: np.ndarray, A_colnorm: np.ndarray) -> float:
    """max over columns of max|err| / ‖A_col‖ (must be ≤ F32_TOL)."""
    err = np.abs(np.asarray(Y_gpu, np.float64) - Y_ref).max(axis=0)
    den = np.maximum(A_colnorm, 1e-300)
    ok_zero = (A_colnorm == 0) & (err == 0)
    r = np.where(ok_zero, 0.0, err / den)
    return float(r.max()) if r.size else 0.0


def bf16_violation(Y_gpu: np.ndarray, Y_ref: np.ndarray) -> float:
    num = np.linalg.norm(np.asarray(Y_gpu, np.float64) - Y_ref, axis=0)
    den = np.linalg.norm(Y_ref, axis=0)
    r = np.where(den == 0, num, num / np.maximum(den, 1e-300))
    return float(r.max()) if r.size else 0.0


def assert_f32(Y_gpu, Y_ref, A_colnorm, what=""):
    v = f32_violation(Y_gpu, Y_ref, A_colnorm)
    assert v <= F32_TOL, f"{what}: max|err|/‖A_col‖ = {v:.3e} > {F32_TOL}"
    return v


def assert_bf16(Y_gpu, Y_ref_fp32A, what=""):
    v = bf16_violation(Y_gpu, Y_ref_fp32A)
    assert v <= BF16_REL, f"{what}: per-column rel ℓ2 = {v:.3e} > {BF16_REL}"
    return v

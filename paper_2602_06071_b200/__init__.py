"""paper_2602_06071_b200 — B200-native BlockPerm-SJLT sketch apply (arXiv 2602.06071).

Thin Python binding over the C-ABI library ``libbps.so`` (include/bps.h).  This module
only marshals arguments (pointers, sizes, the current CUDA stream); every step of
Y = S·A runs in the library's CUDA kernels.  There is no CPU fallback: if the library
is missing or the device is not sm_100, calls raise.

    from paper_2602_06071_b200 import Sketch
    sk = Sketch(M=128, B_r=32, B_c=8192, kappa=4, s=4, seed=1234)
    Y = sk.apply(A)            # A: cuda tensor d×n (float32 or bfloat16) -> Y: k×n float32
    Yt = sk.apply_t(X)         # X: n×d -> Yt: n×k

The library is loaded on first use of ``Sketch``/``lib`` (not by importing submodules such as
``configs``), so host-only tools — the bench's CPU-oracle arm — never map it.
"""

from __future__ import annotations

__all__ = ["Sketch", "BpsError", "VARIANTS", "lib", "lib_path"]


def __getattr__(name):
    if name in ("BpsError", "lib", "lib_path"):
        from . import _lib

        return getattr(_lib, name)
    if name in ("Sketch", "VARIANTS"):
        from . import sketch

        return getattr(sketch, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

"""ctypes loader for libbps.so (C ABI declared in include/bps.h)."""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BPS_LIB may point at the instrumented build (libbps_instr.so) for experiments
lib_path = os.environ.get("BPS_LIB") or os.path.join(_HERE, "libbps.so")

BPS_OK = 0
STATUS = {
    0: "BPS_OK",
    -1: "BPS_ERR_INVALID_ARG",
    -2: "BPS_ERR_ALIGNMENT",
    -3: "BPS_ERR_UNSUPPORTED",
    -4: "BPS_ERR_ARCH",
    -5: "BPS_ERR_CUDA",
    -6: "BPS_ERR_OVERFLOW",
}
EXPORTS = [
    "bps_make_sketch", "bps_free_sketch", "bps_sketch_info", "bps_apply", "bps_apply_t", "bps_apply_ex",
    "bps_apply_t_ex", "bps_workspace_size", "bps_apply_ws", "bps_apply_t_ws", "bps_orbit", "bps_apply_orbit_range",
    "bps_apply_orbit_range_ws", "bps_orbit_range_workspace_size", "bps_apply_orbit_range_bcast", "bps_pattern_host",
    "bps_kernel_launches",
    "bps_timing_enable", "bps_timing_read", "bps_timing_read_ex",
    "bps_version", "bps_last_error",
]


class BpsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def _load() -> ctypes.CDLL:
    if not os.path.exists(lib_path):
        raise ImportError(
            f"libbps.so not found at {lib_path}; build it with `python -m paper_2602_06071_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(lib_path)
    i64, i32, u64, u32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
    L.bps_make_sketch.argtypes = [i64, i64, i64, i32, i32, u64, ctypes.POINTER(vp)]
    L.bps_make_sketch.restype = ctypes.c_int
    L.bps_free_sketch.argtypes = [vp]
    L.bps_free_sketch.restype = None
    L.bps_sketch_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(u32),
                                  ctypes.POINTER(u32), ctypes.POINTER(ctypes.c_float)]
    L.bps_sketch_info.restype = ctypes.c_int
    for name in ("bps_apply", "bps_apply_t"):
        f = getattr(L, name)
        f.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp, i64, vp]
        f.restype = ctypes.c_int
    for name in ("bps_apply_ex", "bps_apply_t_ex"):
        f = getattr(L, name)
        f.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp, i64, vp, ctypes.c_int]
        f.restype = ctypes.c_int
    if hasattr(L, "bps_workspace_size"):  # absent only in old builds loaded via BPS_LIB for A/B runs
        L.bps_workspace_size.argtypes = [vp, i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.bps_workspace_size.restype = ctypes.c_int
        for name in ("bps_apply_ws", "bps_apply_t_ws"):
            f = getattr(L, name)
            f.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp, i64, vp, ctypes.c_size_t, vp, ctypes.c_int]
            f.restype = ctypes.c_int
    L.bps_apply_adjoint.argtypes = [vp, vp, i64, i64, vp, i64, vp]
    L.bps_apply_adjoint.restype = ctypes.c_int
    L.bps_apply_adjoint_ex.argtypes = [vp, vp, i64, i64, vp, i64, vp, ctypes.c_int]
    L.bps_apply_adjoint_ex.restype = ctypes.c_int
    L.bps_make_sketch_ex.argtypes = [i64, i64, i64, i32, i32, u64, ctypes.c_int, ctypes.POINTER(vp)]
    L.bps_make_sketch_ex.restype = ctypes.c_int
    L.bps_sketch_mode.argtypes = [vp]
    L.bps_sketch_mode.restype = ctypes.c_int
    L.bps_make_blockrow.argtypes = [i64, i64, i64, i32, i32, u64, ctypes.POINTER(vp)]
    L.bps_make_blockrow.restype = ctypes.c_int
    L.bps_blockrow_neighbors.argtypes = [vp, i64, ctypes.POINTER(i32)]
    L.bps_blockrow_neighbors.restype = ctypes.c_int
    L.bps_blockrow_draw_host.argtypes = [vp, i64, i32, i64, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.bps_blockrow_draw_host.restype = ctypes.c_int
    L.bps_sketch_kind.argtypes = [vp]
    L.bps_sketch_kind.restype = ctypes.c_int
    L.bps_orbit.argtypes = [vp, ctypes.POINTER(i32)]
    L.bps_orbit.restype = ctypes.c_int
    L.bps_apply_orbit_range.argtypes = [vp, i64, i64, vp, i64, i64, ctypes.c_int, vp, i64, vp, ctypes.c_int]
    L.bps_apply_orbit_range.restype = ctypes.c_int
    if hasattr(L, "bps_apply_orbit_range_ws"):  # absent only in old builds loaded via BPS_LIB for A/B runs
        L.bps_apply_orbit_range_ws.argtypes = [vp, i64, i64, vp, i64, i64, ctypes.c_int, vp, i64, vp, ctypes.c_size_t,
                                               vp, ctypes.c_int]
        L.bps_apply_orbit_range_ws.restype = ctypes.c_int
        L.bps_orbit_range_workspace_size.argtypes = [vp, i64, i64, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.bps_orbit_range_workspace_size.restype = ctypes.c_int
    if hasattr(L, "bps_apply_orbit_range_bcast"):
        L.bps_apply_orbit_range_bcast.argtypes = [vp, i64, i64, vp, i64, i64, ctypes.c_int, vp, i64,
                                                  ctypes.POINTER(vp), ctypes.c_int, vp, i64, i64, vp, ctypes.c_size_t,
                                                  vp, ctypes.c_int]
        L.bps_apply_orbit_range_bcast.restype = ctypes.c_int
    L.bps_pattern_host.argtypes = [vp, i64, i32, i64, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.bps_pattern_host.restype = ctypes.c_int
    if hasattr(L, "bps_timing_enable"):  # absent only in old builds loaded via BPS_LIB for A/B runs
        L.bps_timing_enable.argtypes = [ctypes.c_int]
        L.bps_timing_enable.restype = ctypes.c_int
        L.bps_timing_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
        L.bps_timing_read.restype = ctypes.c_int
        L.bps_timing_read_ex.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
        L.bps_timing_read_ex.restype = ctypes.c_int
    L.bps_kernel_launches.argtypes = []
    L.bps_kernel_launches.restype = ctypes.c_uint64
    L.bps_version.argtypes = []
    L.bps_version.restype = ctypes.c_char_p
    L.bps_last_error.argtypes = []
    L.bps_last_error.restype = ctypes.c_char_p
    return L


lib = _load()


def check(rc: int) -> None:
    if rc != BPS_OK:
        raise BpsError(rc, lib.bps_last_error().decode(errors="replace"))

"""`Sketch`: torch-tensor front end of the C ABI (argument marshalling only)."""

from __future__ import annotations

import ctypes

from ._lib import check, lib

BPS_F32, BPS_BF16 = 0, 1
VARIANTS = {"auto": 0, "sparse": 1, "tc": 2}


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return BPS_F32
    if t.dtype == torch.bfloat16:
        return BPS_BF16
    raise TypeError(f"unsupported dtype {t.dtype} (float32 or bfloat16)")


def _stream_ptr(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def _check_matrix(t, name):
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libbps has no CPU path)")
    if t.stride(1) != 1:
        raise ValueError(f"{name} must be row-major with unit column stride")


class Sketch:
    """BlockPerm-SJLT S (k×d, k = M·B_r, d = M·B_c) regenerated on the fly (bps_make_sketch);
    kind="blockrow": the FlashBlockRow sampling sketch of P:1424-1466 (bps_make_blockrow)."""

    MODES = {"rowpart": 0, "affine": 1}

    def __init__(self, M: int, B_r: int, B_c: int, kappa: int, s: int, seed: int = 0, kind: str = "blockperm",
                 mode: str = "rowpart"):
        """kind: "blockperm" (BlockPerm-SJLT) or "blockrow" (FlashBlockRow); mode (blockperm only):
        "rowpart" (R1) or "affine" (AffineUnique, R18)."""
        h = ctypes.c_void_p()
        sd = ctypes.c_uint64(seed & (2**64 - 1))
        if kind == "blockperm":
            check(lib.bps_make_sketch_ex(M, B_r, B_c, kappa, s, sd, self.MODES[mode], ctypes.byref(h)))
        elif kind == "blockrow":
            if mode != "rowpart":
                raise ValueError("mode applies to BlockPerm-SJLT sketches only")
            check(lib.bps_make_blockrow(M, B_r, B_c, kappa, s, sd, ctypes.byref(h)))
        else:
            raise ValueError(f"unknown sketch kind {kind!r}")
        self.kind, self.mode = kind, mode
        self._h = h
        self.M, self.B_r, self.B_c, self.kappa, self.s, self.seed = M, B_r, B_c, kappa, s, seed & (2**64 - 1)
        d, k = ctypes.c_int64(), ctypes.c_int64()
        a, b = ctypes.c_uint32(), ctypes.c_uint32()
        sc = ctypes.c_float()
        check(lib.bps_sketch_info(h, ctypes.byref(d), ctypes.byref(k), ctypes.byref(a), ctypes.byref(b), ctypes.byref(sc)))
        self.d, self.k, self.a, self.b, self.scale = d.value, k.value, a.value, b.value, sc.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.bps_free_sketch(h)
            self._h = None

    @property
    def handle(self) -> int:
        return self._h.value

    def info(self) -> dict:
        return dict(M=self.M, B_r=self.B_r, B_c=self.B_c, kappa=self.kappa, s=self.s, seed=self.seed,
                    d=self.d, k=self.k, a=self.a, b=self.b, scale=self.scale)

    def neighbors_row(self, g: int) -> list[int]:
        """FlashBlockRow N_row(g) in draw order (R14)."""
        arr = (ctypes.c_int32 * self.kappa)()
        check(lib.bps_blockrow_neighbors(self._h, g, arr))
        return list(arr)

    def blockrow_draw(self, g: int, ell: int, r: int, t: int) -> tuple[int, int]:
        i, sg = ctypes.c_int32(), ctypes.c_int32()
        check(lib.bps_blockrow_draw_host(self._h, g, ell, r, t, ctypes.byref(i), ctypes.byref(sg)))
        return i.value, sg.value

    def orbit(self) -> list[int]:
        arr = (ctypes.c_int32 * self.M)()
        check(lib.bps_orbit(self._h, arr))
        return list(arr)

    def workspace_bytes(self, n: int, dtype_code: int, transposed: bool = False) -> int:
        key = (n, dtype_code, transposed)
        cache = self.__dict__.setdefault("_ws_cache", {})
        if key not in cache:
            b = ctypes.c_size_t()
            check(lib.bps_workspace_size(self._h, n, dtype_code, int(transposed), ctypes.byref(b)))
            cache[key] = b.value
        return cache[key]

    def _scratch(self, nbytes: int, device):
        """One scratch workspace per device, grown on demand (bps.h: no initialisation needed).
        A Sketch must not run two applies concurrently on different streams (they would share it)."""
        import torch

        if not nbytes:
            return None, 0
        bufs = self.__dict__.setdefault("_ws_bufs", {})
        key = (device.type, device.index if device.index is not None else torch.cuda.current_device())
        buf = bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            bufs[key] = buf
        return buf, buf.numel()

    def _workspace(self, n, dtype_code, transposed, device, use_workspace):
        """Scratch for the full-occupancy tc decomposition (bps_apply_ws)."""
        nbytes = self.workspace_bytes(n, dtype_code, transposed) if use_workspace else 0
        return self._scratch(nbytes, device)

    def pattern(self, g: int, ell: int, u: int, j: int) -> tuple[int, int]:
        r, sg = ctypes.c_int32(), ctypes.c_int32()
        check(lib.bps_pattern_host(self._h, g, ell, u, j, ctypes.byref(r), ctypes.byref(sg)))
        return r.value, sg.value

    # ------------------------------------------------------------------ apply
    def apply(self, A, out=None, variant: str = "auto", use_workspace: bool = True):
        """Y = S·A. A: cuda d×n (float32/bfloat16, row-major, lda = A.stride(0)) -> k×n float32."""
        import torch

        _check_matrix(A, "A")
        if A.shape[0] != self.d:
            raise ValueError(f"A has {A.shape[0]} rows, sketch expects d={self.d}")
        n = A.shape[1]
        if out is None:
            out = torch.empty((self.k, n), dtype=torch.float32, device=A.device)
        _check_matrix(out, "out")
        if out.dtype != torch.float32 or tuple(out.shape) != (self.k, n):
            raise ValueError("out must be float32 k×n")
        code = _dtype_code(A)
        ws, nbytes = self._workspace(n, code, False, A.device, use_workspace)
        if ws is None:
            check(lib.bps_apply_ex(self._h, A.data_ptr(), A.stride(0), n, code, out.data_ptr(), out.stride(0),
                                   _stream_ptr(A.device), VARIANTS[variant]))
            return out
        check(lib.bps_apply_ws(self._h, A.data_ptr(), A.stride(0), n, code, out.data_ptr(), out.stride(0),
                               ws.data_ptr() if ws is not None else None, nbytes, _stream_ptr(A.device),
                               VARIANTS[variant]))
        return out

    def apply_adjoint(self, Y, out=None, variant: str = "auto"):
        """X = Sᵀ·Y. Y: cuda k×n float32 (row-major) -> d×n float32 (bps_apply_adjoint)."""
        import torch

        _check_matrix(Y, "Y")
        if Y.shape[0] != self.k or Y.dtype != torch.float32:
            raise ValueError(f"Y must be float32 with k={self.k} rows")
        n = Y.shape[1]
        if out is None:
            out = torch.empty((self.d, n), dtype=torch.float32, device=Y.device)
        _check_matrix(out, "out")
        if out.dtype != torch.float32 or tuple(out.shape) != (self.d, n):
            raise ValueError("out must be float32 d×n")
        check(lib.bps_apply_adjoint_ex(self._h, Y.data_ptr(), Y.stride(0), n, out.data_ptr(), out.stride(0),
                                       _stream_ptr(Y.device), VARIANTS[variant]))
        return out

    def apply_t(self, X, out=None, variant: str = "auto", use_workspace: bool = True):
        """Transposed layout: X cuda n×d -> (S·Xᵀ)ᵀ, n×k float32."""
        import torch

        _check_matrix(X, "X")
        if X.shape[1] != self.d:
            raise ValueError(f"X has {X.shape[1]} columns, sketch expects d={self.d}")
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, self.k), dtype=torch.float32, device=X.device)
        _check_matrix(out, "out")
        if out.dtype != torch.float32 or tuple(out.shape) != (n, self.k):
            raise ValueError("out must be float32 n×k")
        code = _dtype_code(X)
        ws, nbytes = self._workspace(n, code, True, X.device, use_workspace)
        if ws is None:
            check(lib.bps_apply_t_ex(self._h, X.data_ptr(), X.stride(0), n, code, out.data_ptr(), out.stride(0),
                                     _stream_ptr(X.device), VARIANTS[variant]))
            return out
        check(lib.bps_apply_t_ws(self._h, X.data_ptr(), X.stride(0), n, code, out.data_ptr(), out.stride(0),
                                 ws.data_ptr() if ws is not None else None, nbytes, _stream_ptr(X.device),
                                 VARIANTS[variant]))
        return out

    def apply_orbit_range(self, pos_begin: int, pos_end: int, A_local, out=None, variant: str = "auto",
                          use_workspace: bool = True, dst=(), mc_ptr: int = 0, dst_ld: int | None = None,
                          dst_row0: int = 0):
        """Partial apply over orbit positions [pos_begin, pos_end) (bps_apply_orbit_range_ws): the
        output blocks at those positions, stacked, bitwise equal to the matching rows of apply().

        dst / mc_ptr (bps_apply_orbit_range_bcast): the kernel epilogue also stores every output row r
        into row dst_row0 + r of each destination — device pointers (ints: peers' symmetric buffers
        or local tensors' data_ptr()) and/or an NVLS multicast address — with leading dimension dst_ld."""
        import torch

        _check_matrix(A_local, "A_local")
        L = pos_end - pos_begin
        if A_local.shape[0] != (L + self.kappa - 1) * self.B_c:
            raise ValueError("A_local must hold (L+kappa-1)*B_c rows")
        n = A_local.shape[1]
        if out is None:
            out = torch.empty((L * self.B_r, n), dtype=torch.float32, device=A_local.device)
        _check_matrix(out, "out")
        if out.dtype != torch.float32 or tuple(out.shape) != (L * self.B_r, n) or out.device != A_local.device:
            raise ValueError("out must be float32 (L*B_r)×n on the device of A_local")
        code = _dtype_code(A_local)
        nbytes = 0
        if use_workspace:
            b = ctypes.c_size_t()
            check(lib.bps_orbit_range_workspace_size(self._h, pos_begin, pos_end, n, code, ctypes.byref(b)))
            nbytes = b.value
        ws, wsb = self._scratch(nbytes, A_local.device)
        if dst or mc_ptr:
            ptrs = [int(p) for p in dst]
            if len(ptrs) > 8:
                raise ValueError("at most 8 destinations")
            arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
            check(lib.bps_apply_orbit_range_bcast(self._h, pos_begin, pos_end, A_local.data_ptr(), A_local.stride(0), n,
                                                  code, out.data_ptr(), out.stride(0), arr, len(ptrs), mc_ptr or None,
                                                  dst_ld if dst_ld is not None else n, dst_row0,
                                                  ws.data_ptr() if ws is not None else None, wsb,
                                                  _stream_ptr(A_local.device), VARIANTS[variant]))
            return out
        check(lib.bps_apply_orbit_range_ws(self._h, pos_begin, pos_end, A_local.data_ptr(), A_local.stride(0), n, code,
                                           out.data_ptr(), out.stride(0), ws.data_ptr() if ws is not None else None,
                                           wsb, _stream_ptr(A_local.device), VARIANTS[variant]))
        return out

    def apply_raw(self, A_ptr: int, lda: int, n: int, dtype_code: int, Y_ptr: int, ldy: int, stream: int,
                  variant: str = "auto") -> None:
        """Pointer-level call (used by the bench's CUDA-graph capture)."""
        check(lib.bps_apply_ex(self._h, A_ptr, lda, n, dtype_code, Y_ptr, ldy, stream, VARIANTS[variant]))

"""CPU-side checks of the C ABI: the library loads, exports every symbol include/bps.h
declares, validates arguments, and its host-side derivations reproduce the oracle's
frozen vectors bit-exactly (no device compute here)."""

import ctypes
import json
import os
import re

import pytest

from paper_2602_06071_b200 import BpsError, Sketch, lib
from paper_2602_06071_b200 import configs as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "bps.h")).read()
    declared = set(re.findall(r"\b(bps_[a-z_]+)\s*\(", hdr))
    assert {"bps_make_sketch", "bps_apply", "bps_apply_t", "bps_last_error"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.bps_version()


@pytest.mark.parametrize("args", [
    (8, 32, 128, 9, 2),     # kappa > M
    (8, 32, 128, 0, 2),     # kappa < 1
    (8, 30, 128, 2, 4),     # B_r % s != 0
    (8, 4, 128, 2, 8),      # s > B_r
    (0, 32, 128, 1, 1),     # M < 1
    (8, 32, 1 << 24, 2, 2), # B_c counter width
    (8, 32, 128, 2, 512),   # s > 256
])
def test_make_sketch_rejects(args):
    with pytest.raises(BpsError) as e:
        Sketch(*args, seed=1)
    assert e.value.code == -1


def test_null_handle_and_apply_validation():
    h = ctypes.c_void_p()
    assert lib.bps_make_sketch(8, 32, 128, 2, 2, 1, None) == -1
    assert lib.bps_sketch_info(None, None, None, None, None, None) == -1
    assert b"NULL" in lib.bps_last_error()
    assert lib.bps_make_sketch(8, 32, 128, 2, 2, 1, ctypes.byref(h)) == 0
    # n == 0 is a no-op even with NULL pointers
    assert lib.bps_apply(h, None, 0, 0, 0, None, 0, None) == 0
    # NULL data pointers with n > 0
    assert lib.bps_apply(h, None, 16, 16, 0, None, 16, None) == -1
    # misaligned pointer -> alignment error before touching the device
    assert lib.bps_apply(h, 0x1004, 16, 16, 0, 0x100000000, 16, None) == -2
    # lda < n
    assert lib.bps_apply(h, 0x1000, 8, 16, 0, 0x100000000, 16, None) == -1
    # bad dtype
    assert lib.bps_apply(h, 0x1000, 16, 16, 7, 0x100000000, 16, None) == -1
    # overlapping input/output
    assert lib.bps_apply(h, 0x1000, 16, 16, 0, 0x1000, 16, None) == -1
    # bad orbit range
    assert lib.bps_apply_orbit_range(h, 8, 9, 0x1000, 16, 16, 0, 0x100000000, 16, None, 0) == -1
    # adjoint: NULL / misaligned / overlapping arguments rejected before device work
    assert lib.bps_apply_adjoint(h, None, 16, 0, None, 16, None) == 0
    assert lib.bps_apply_adjoint(h, None, 16, 16, None, 16, None) == -1
    assert lib.bps_apply_adjoint(h, 0x1004, 16, 16, 0x100000000, 16, None) == -2
    assert lib.bps_apply_adjoint(h, 0x1000, 16, 16, 0x1000, 16, None) == -1
    lib.bps_free_sketch(h)
    lib.bps_free_sketch(None)


def _gold():
    with open(os.path.join(ROOT, "tests", "golden", "oracle_vectors.json")) as f:
        return json.load(f)


def test_host_derivation_matches_oracle_vectors():
    g = _gold()
    for M, (a, b) in g["affine"].items():
        sk = Sketch(int(M), 1, 1, 1, 1, seed=g["seed"])
        assert (sk.a, sk.b) == (a, b), M
    for p in g["patterns"]:
        sk = Sketch(p["M"], p["B_r"], p["B_c"], p["kappa"], p["s"], seed=g["seed"])
        assert sk.pattern(p["g"], p["ell"], p["u"], p["j"]) == (p["row"], p["sign"]), p


def test_orbit_and_scale():
    import math

    import numpy as np

    for cfg in (C.TINY, C.LS, C.GRAD):
        sk = Sketch(**cfg.sketch_args())
        orb = sk.orbit()
        assert sorted(orb) == list(range(cfg.M))
        # f(g_i) = g_{i+1}
        assert all((sk.a * orb[i] + sk.b) % cfg.M == orb[(i + 1) % cfg.M] for i in range(cfg.M))
        assert sk.scale == np.float32(1.0 / math.sqrt(cfg.kappa * cfg.s))
        assert (sk.d, sk.k) == (cfg.d, cfg.k)


def test_apply_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sk = Sketch(**C.TINY.sketch_args())
    A = torch.zeros((C.TINY.d, 16))
    with pytest.raises(ValueError):
        sk.apply(A)  # CPU tensor: no CPU path


def test_blockrow_host_derivation_matches_oracle():
    """FlashBlockRow N_row(g) and (i, sign) draws of libbps equal the oracle's bit-exactly (R14-R16)."""
    import numpy as np

    from oracle import blockrow as BR

    for layout, seed in [((8, 4, 16, 2, 2), 3), ((128, 32, 8192, 4, 4), 1234), ((7, 5, 9, 7, 3), 2**63 + 5)]:
        sk = Sketch(*layout, seed=seed, kind="blockrow")
        br = BR.make_blockrow(*layout, seed=seed)
        assert lib.bps_sketch_kind(sk.handle) == 1
        assert np.float32(br.scale) == np.float32(sk.scale)
        assert (sk.d, sk.k) == (br.d, br.k)
        rng = np.random.default_rng(0)
        for g in rng.choice(br.M, min(br.M, 6), replace=False):
            g = int(g)
            assert sk.neighbors_row(g) == BR.neighbors_row(br, g)
            for _ in range(10):
                ell = int(rng.integers(1, br.kappa + 1))
                r, t = int(rng.integers(br.B_r)), int(rng.integers(br.s))
                assert sk.blockrow_draw(g, ell, r, t) == BR.draw_index(br, g, ell, r, t)


def test_blockrow_validation_and_unsupported_calls():
    for args in [(4, 2, 2, 5, 1), (4, 2, 2, 0, 1), (4, 2, 2, 2, 0), (4, 2, 2, 2, 300), (1 << 24, 1, 1, 1, 1)]:
        with pytest.raises(BpsError) as e:
            Sketch(*args, seed=0, kind="blockrow")
        assert e.value.code == -1
    sk = Sketch(8, 4, 16, 2, 3, seed=1, kind="blockrow")  # B_r % s != 0 is fine here
    with pytest.raises(BpsError):
        sk.orbit()
    with pytest.raises(BpsError):
        sk.pattern(0, 1, 0, 0)
    bp = Sketch(8, 32, 128, 2, 2, seed=1)
    assert lib.bps_sketch_kind(bp.handle) == 0
    with pytest.raises(BpsError):
        bp.neighbors_row(0)


def test_affine_mode_host_draws_match_oracle():
    """AffineUnique (R18): libbps's (row, sign) draws equal the oracle's bit-exactly."""
    import numpy as np

    import oracle

    for layout, seed in [((8, 32, 128, 2, 2), 1), ((128, 32, 8192, 4, 4), 1234), ((16, 64, 128, 4, 8), 9)]:
        sk = Sketch(*layout, seed=seed, mode="affine")
        osk = oracle.make_sketch(*layout, seed=seed, mode="affine")
        assert lib.bps_sketch_mode(sk.handle) == 1
        assert lib.bps_sketch_mode(Sketch(*layout, seed=seed).handle) == 0
        rng = np.random.default_rng(1)
        for _ in range(200):
            g, ell = int(rng.integers(osk.M)), int(rng.integers(1, osk.kappa + 1))
            u, j = int(rng.integers(osk.B_c)), int(rng.integers(osk.s))
            assert sk.pattern(g, ell, u, j) == oracle.pattern(osk, g, ell, u, j)
    for args in [(8, 24, 16, 2, 2), (8, 64, 16, 2, 33)]:
        with pytest.raises(BpsError) as e:
            Sketch(*args, seed=0, mode="affine")
        assert e.value.code == -1

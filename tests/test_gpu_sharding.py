"""Canonical decomposition (R19, §6.2): Y is one fixed bit pattern for
every column split, orbit-range split and with / without a workspace — the 1-GPU ≡ sharded
contract, simulated on one GPU (T-sharding-sim) — and the orbit-range apply agrees with the
oracle element by element.

Run on a B200:  python -m pytest tests -m gpu
"""

import os
import socket

import numpy as np
import pytest

import oracle
import synth
from parity import assert_f32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402
from paper_2602_06071_b200 import dist as D  # noqa: E402

# (M, B_r, B_c, κ, s), n, dtype, mode
CASES = [
    ((16, 32, 1024, 4, 4), 200, "f32", "rowpart"),
    ((64, 16, 2048, 8, 2), 304, "bf16", "rowpart"),
    ((7, 32, 64, 4, 4), 64, "f32", "rowpart"),     # odd M (odd range count)
    ((8, 32, 128, 8, 2), 40, "bf16", "rowpart"),    # κ = M
    ((16, 16, 256, 1, 4), 64, "f32", "rowpart"),    # κ = 1
    ((32, 32, 2048, 16, 4), 136, "bf16", "rowpart"),  # κ·B_r = 512: four band tiles
    ((32, 16, 1024, 8, 4), 192, "f32", "rowpart"),  # κ·B_r = 128 fp32
    ((64, 32, 1024, 4, 8), 256, "bf16", "affine"),  # AffineUnique
    ((12, 24, 192, 5, 3), 96, "f32", "rowpart"),    # non-power-of-two M, B_r, C
]
IDS = [f"{c[0]}-n{c[1]}-{c[2]}-{c[3]}" for c in CASES]


def _tdt(dt):
    return torch.float32 if dt == "f32" else torch.bfloat16


def _shards(n, parts, align):
    cuts = sorted({0, n} | {min(n, (n * r // parts) // align * align) for r in range(1, parts)})
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("variant", ["tc", "sparse"])
def test_column_shards_bitwise(case, variant):
    """Column shards (multiples of 64 columns, any number of them) reproduce the full apply
    bit for bit, in both layouts, with and without the workspace."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=31, mode=mode)
    A = torch.randn((sk.d, n), device="cuda").to(_tdt(dt))
    try:
        Y = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    assert torch.equal(Y, sk.apply(A, variant=variant)), "run-to-run"
    assert torch.equal(Y, sk.apply(A, variant=variant, use_workspace=False)), "workspace vs halo ranges"
    for parts in (2, 3, 5):
        Ys = torch.empty_like(Y)
        for c0, c1 in _shards(n, parts, 64):
            sk.apply(A[:, c0:c1], out=Ys[:, c0:c1], variant=variant)
        assert torch.equal(Ys, Y), f"{parts} column shards"
    X = A.t().contiguous()
    Yt = sk.apply_t(X, variant=variant)
    assert torch.equal(Yt, sk.apply_t(X, variant=variant, use_workspace=False))
    Yts = torch.empty_like(Yt)
    for c0, c1 in _shards(n, 3, 64):
        sk.apply_t(X[c0:c1], out=Yts[c0:c1], variant=variant)
    assert torch.equal(Yts, Yt), "transposed shards"


def _orbit_local(sk, A, p0, p1):
    orb = sk.orbit()
    return torch.cat([A[orb[p % sk.M] * sk.B_c:(orb[p % sk.M] + 1) * sk.B_c] for p in range(p0 + 1, p1 + sk.kappa)])


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("variant", ["tc", "sparse"])
def test_orbit_ranges_bitwise(case, variant):
    """T-sharding-sim of block sharding: P orbit ranges run one after another, concatenated in
    orbit order and permuted back to g order, equal the full apply bit for bit."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=32, mode=mode)
    M = sk.M
    A = torch.randn((sk.d, n), device="cuda").to(_tdt(dt))
    try:
        Y = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    orb = sk.orbit()
    for P in sorted({1, 2, min(3, M), min(4, M)}):
        parts = [sk.apply_orbit_range(*D.orbit_shard(M, P, r), _orbit_local(sk, A, *D.orbit_shard(M, P, r)),
                                      variant=variant) for r in range(P)]
        assert torch.equal(D.gather_orbit_to_g(torch.cat(parts), orb, sk.B_r), Y), f"P={P}"
    for p0, p1 in [(M - 1, M + min(2, M - 1)), (1, 1 + max(1, M // 2))]:  # wrap-around and interior
        if p1 <= p0:
            continue
        Yl = sk.apply_orbit_range(p0, p1, _orbit_local(sk, A, p0, p1), variant=variant)
        ref = torch.cat([Y[orb[p % M] * sk.B_r:(orb[p % M] + 1) * sk.B_r] for p in range(p0, p1)])
        assert torch.equal(Yl, ref), (p0, p1)


@pytest.mark.parametrize("case", CASES[:5] + CASES[7:], ids=IDS[:5] + IDS[7:])
@pytest.mark.parametrize("variant", ["tc", "sparse"])
def test_orbit_range_vs_oracle(case, variant):
    """bps_apply_orbit_range element by element against the oracle's rows of S·A (several
    ranges, including one that wraps past position M)."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=33, mode=mode)
    osk = oracle.make_sketch(*layout, 33, mode=mode)
    M, orb = sk.M, sk.orbit()
    A = synth.host_matrix("gaussian", sk.d, n, seed=9)
    if dt == "bf16":
        A = synth.bf16_round(A)
    At = torch.from_numpy(A).cuda().to(_tdt(dt))
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    for p0, p1 in [(0, M), (0, max(1, M // 3)), (M // 2, M // 2 + max(1, M // 4)), (M - 2, M + 1)]:
        if p1 <= p0 or p1 > p0 + M or p0 < 0:
            continue
        try:
            Yl = sk.apply_orbit_range(p0, p1, _orbit_local(sk, At, p0, p1), variant=variant)
        except BpsError as e:
            if e.code == -3 and variant == "tc":
                pytest.skip(str(e))
            raise
        ref = oracle.apply(osk, A, blocks=[orb[p % M] for p in range(p0, p1)])
        assert_f32(Yl.cpu().numpy(), ref, nrm, f"orbit range [{p0},{p1}) {variant}")


@pytest.mark.parametrize("cfg,span", [(C.LS, (0, 24)), (C.GRAD, (50, 66))], ids=["ls", "grad"])
def test_full_size_range_boundaries(cfg, span):
    """Full-size configs in the bench's launch configuration: the workspace path (many stream
    ranges, straddling outputs finished from contributors' partials) equals the halo path bit for
    bit, and a run of consecutive orbit positions crossing several range boundaries matches the
    oracle element by element on sampled columns."""
    sk = Sketch(**cfg.sketch_args())
    osk = oracle.make_sketch(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed)
    tdt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    A = synth.device_matrix("gaussian", cfg.d, cfg.n, seed=12, M=cfg.M, dtype=tdt)
    Y = sk.apply(A)
    assert torch.equal(Y, sk.apply(A, use_workspace=False))
    orb = sk.orbit()
    gs = [orb[p] for p in range(*span)]
    cols = np.array([0, 1, cfg.n // 2, cfg.n - 1])
    idx = torch.as_tensor(cols, device="cuda")
    A_cols = A.index_select(1, idx).float().cpu().numpy()
    ref = oracle.apply(osk, A_cols, blocks=gs)
    rows = np.concatenate([np.arange(g * cfg.B_r, (g + 1) * cfg.B_r) for g in gs])
    got = Y.index_select(1, idx).cpu().numpy()[rows]
    assert_f32(got, ref, np.linalg.norm(A_cols.astype(np.float64), axis=0), f"{cfg.name} boundary run")
    del A, Y
    torch.cuda.empty_cache()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_block_sharded_apply_nccl_world1():
    """dist.block_sharded_apply through a real NCCL process group (world size 1) with the CUDA
    bps_apply_orbit_range: bitwise equal to the full apply."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sk = Sketch(64, 16, 2048, 8, 2, seed=34)
        A = torch.randn((sk.d, 256), device="cuda", dtype=torch.bfloat16)
        p0, p1 = D.orbit_shard(sk.M, 1, 0)
        blocks = D.input_blocks(sk.orbit(), p0, p1, sk.kappa)
        A_loc = torch.cat([A[h * sk.B_c:(h + 1) * sk.B_c] for h in blocks])
        Y = D.block_sharded_apply(sk, A_loc)
        torch.cuda.synchronize()
        assert torch.equal(Y, sk.apply(A))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["tc", "sparse"])
def test_workspace_epochs(variant):
    """The workspace's epoch-tagged flags need no re-zeroing: many consecutive calls on one
    workspace (different n, both layouts) stay bitwise reproducible."""
    sk = Sketch(32, 32, 2048, 4, 4, seed=35)
    A = torch.randn((sk.d, 384), device="cuda")
    ref = {n: sk.apply(A[:, :n].contiguous(), variant=variant) for n in (64, 384)}
    for _ in range(3):
        for n in (384, 64):
            assert torch.equal(sk.apply(A[:, :n].contiguous(), variant=variant), ref[n])


BCAST_CASES = [CASES[0], CASES[1], CASES[2], CASES[3], CASES[7], CASES[8]]


@pytest.mark.parametrize("case", BCAST_CASES, ids=[f"{c[0]}-n{c[1]}-{c[2]}-{c[3]}" for c in BCAST_CASES])
@pytest.mark.parametrize("variant", ["tc", "sparse"])
@pytest.mark.parametrize("use_ws", [True, False])
def test_orbit_range_bcast(case, variant, use_ws):
    """bps_apply_orbit_range_bcast (the all-gather fused into the epilogue): three
    destination buffers with a padded leading dimension stand in for the peers' symmetric buffers;
    each receives, at rows dst_row0.., bitwise the rows of Y_local (= the full apply's rows), and
    nothing outside them."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=36, mode=mode)
    M = sk.M
    A = torch.randn((sk.d, n), device="cuda").to(_tdt(dt))
    try:
        Y = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    orb = sk.orbit()
    ld = n + 4
    for p0, p1 in sorted({(0, M), (M - 1, M + min(2, M - 1)), (1, 1 + max(1, M // 2))}):
        if p1 <= p0:
            continue
        rows = (p1 - p0) * sk.B_r
        row0 = (p0 % 3) * sk.B_r + 5
        dsts = [torch.full((row0 + rows + 7, ld), float("nan"), device="cuda") for _ in range(3)]
        Yl = sk.apply_orbit_range(p0, p1, _orbit_local(sk, A, p0, p1), variant=variant, use_workspace=use_ws,
                                  dst=[t.data_ptr() for t in dsts], dst_ld=ld, dst_row0=row0)
        torch.cuda.synchronize()
        ref = torch.cat([Y[orb[p % M] * sk.B_r:(orb[p % M] + 1) * sk.B_r] for p in range(p0, p1)])
        assert torch.equal(Yl, ref), (p0, p1)
        for t in dsts:
            assert torch.equal(t[row0:row0 + rows, :n], Yl), (p0, p1)
            assert torch.isnan(t[:row0]).all() and torch.isnan(t[row0 + rows:]).all() and torch.isnan(t[:, n:]).all()


def test_orbit_range_bcast_nonfinite():
    """The exact-recompute path (R12) also reaches the destinations."""
    sk = Sketch(16, 32, 1024, 4, 4, seed=37)
    A = torch.randn((sk.d, 128), device="cuda")
    A[5, 3] = float("inf")
    A[700, 9] = float("nan")
    Y = sk.apply(A)
    M = sk.M
    dst = torch.full((M * sk.B_r, 128), 7.0, device="cuda")
    Yl = sk.apply_orbit_range(0, M, _orbit_local(sk, A, 0, M), dst=[dst.data_ptr()], dst_ld=128, dst_row0=0)
    torch.cuda.synchronize()
    assert torch.equal(torch.nan_to_num(Yl, nan=1.5), torch.nan_to_num(dst, nan=1.5))
    orb = sk.orbit()
    ref = torch.cat([Y[orb[p] * sk.B_r:(orb[p] + 1) * sk.B_r] for p in range(M)])
    assert torch.equal(torch.nan_to_num(Yl, nan=1.5), torch.nan_to_num(ref, nan=1.5))


def test_block_sharded_apply_fused_nccl_world1():
    """dist.block_sharded_apply_fused through a real NCCL group (world 1) and torch symmetric memory:
    the epilogue stores straight into the symmetric buffer (peer pointer, and the NVLS multicast
    address when the platform exposes one); bitwise equal to the full apply."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sk = Sketch(64, 16, 2048, 8, 2, seed=38)
        A = torch.randn((sk.d, 256), device="cuda", dtype=torch.bfloat16)
        p0, p1 = D.orbit_shard(sk.M, 1, 0)
        blocks = D.input_blocks(sk.orbit(), p0, p1, sk.kappa)
        A_loc = torch.cat([A[h * sk.B_c:(h + 1) * sk.B_c] for h in blocks])
        ref = sk.apply(A)
        try:
            D.symmetric_rendezvous((8, 8), A.device)
        except Exception as e:  # noqa: BLE001 — platform without symmetric memory
            pytest.skip(f"torch symmetric memory unavailable: {e}")
        for mc in (False, True):
            Y = D.block_sharded_apply_fused(sk, A_loc, multicast=mc)
            torch.cuda.synchronize()
            assert torch.equal(Y, ref), f"multicast={mc}"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[2], CASES[5]], ids=[IDS[0], IDS[1], IDS[2], IDS[5]])
def test_combine_flag_handoff(case):
    """The combine pass folds each straddling output once the CTAs holding its pieces have published
    them (per-CTA epoch flags in the workspace, BPS_TC_AB=256, no whole-grid wait): bitwise equal to
    the default whole-grid wait, over repeated calls on one workspace (stale flags of earlier launches)."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=39, mode=mode)
    A = torch.randn((sk.d, n), device="cuda").to(_tdt(dt))
    ref = sk.apply(A, variant="tc")
    os.environ["BPS_TC_AB"] = "256"
    try:
        for _ in range(4):
            assert torch.equal(sk.apply(A, variant="tc"), ref)
    finally:
        del os.environ["BPS_TC_AB"]


@pytest.mark.parametrize("layout", [(32, 32, 2048, 16, 4), (32, 32, 2048, 8, 4), (64, 16, 1024, 16, 2)])
def test_fp32_slot_split_t_form(layout):
    """fp32 κ·B_r in (128, 512] in the optional T form (BPS_TC_FORM=tf: the slot-split cluster's CTAs
    convert the multicast stage into TMEM) — within the fp32 criterion of the oracle (the T form folds
    the hi and lo products in one accumulator, the NT form adds them after: not bitwise equal)."""
    sk = Sketch(*layout, seed=40)
    osk = oracle.make_sketch(*layout, 40)
    A = synth.host_matrix("gaussian", sk.d, 200, seed=2)
    At = torch.from_numpy(A).cuda()
    ref = sk.apply(At, variant="tc")
    os.environ["BPS_TC_FORM"] = "tf"
    try:
        Y = sk.apply(At, variant="tc")
    finally:
        del os.environ["BPS_TC_FORM"]
    torch.cuda.synchronize()
    assert_f32(Y.cpu().numpy(), oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), str(layout))
    assert_f32(ref.cpu().numpy(), oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), str(layout))


@pytest.mark.parametrize("case", [CASES[1], CASES[3], CASES[7]], ids=[IDS[1], IDS[3], IDS[7]])
def test_narrow_tile_columns_bitwise(case):
    """Column slices of ≤ 32 columns take the 32-column SW64 tile (bf16): bitwise equal to the same
    columns of the wide-tile apply (the canonical fold does not depend on the tile width), and within
    the oracle criterion."""
    layout, n, dt, mode = case
    sk = Sketch(*layout, seed=41, mode=mode)
    A = torch.randn((sk.d, n), device="cuda").to(_tdt(dt))
    Y = sk.apply(A, variant="tc")
    for c0, w in [(0, 32), (8, 24), (n - 8, 8), (32, 16)]:  # widths: 16-byte aligned rows
        Yn = sk.apply(A[:, c0:c0 + w].contiguous(), variant="tc")
        assert torch.equal(Yn, Y[:, c0:c0 + w]), (c0, w)

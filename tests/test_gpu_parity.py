"""GPU parity: libbps (through the C ABI) vs the CPU oracle, element by element.

Run on a B200:  python -m pytest tests -m gpu
"""

import numpy as np
import pytest

import oracle
import synth
from parity import assert_bf16, assert_f32

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402

VARIANTS = ["sparse", "tc"]


def _padded(rows, cols, dtype, fill=None):
    """rows×cols view with a 16-byte-aligned leading dimension (ABI alignment rule)."""
    mult = 16 // torch.tensor([], dtype=dtype).element_size()
    ld = max(mult, -(-cols // mult) * mult)
    base = torch.zeros((rows, ld), dtype=dtype, device="cuda")
    v = base[:, :cols]
    if fill is not None:
        v.copy_(fill)
    return v


def _run(sk, A_host, variant, dtype=torch.float32, transposed=False):
    A_src = torch.from_numpy(np.ascontiguousarray(A_host)).cuda().to(dtype)
    A = _padded(A_src.shape[0], A_src.shape[1], dtype, A_src)
    out = _padded(A.shape[0], sk.k, torch.float32) if transposed else _padded(sk.k, A.shape[1], torch.float32)
    try:
        Y = sk.apply_t(A, out=out, variant=variant) if transposed else sk.apply(A, out=out, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(f"tc variant does not cover this shape: {e}")
        raise
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def _pair(M, Br, Bc, kappa, s, seed=1234, mode="rowpart"):
    return Sketch(M, Br, Bc, kappa, s, seed, mode=mode), oracle.make_sketch(M, Br, Bc, kappa, s, seed, mode=mode)


# ------------------------------------------------------------ bit-exact pattern
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (16, 64, 128, 4, 2), (128, 32, 8192, 4, 4), (512, 16, 32768, 8, 2),
                                    # band generator paths: C = 1 dense rows (κs = 128), κs = 8 and 12 (batch tails)
                                    (64, 8, 4096, 16, 8), (32, 64, 2048, 1, 8), (32, 32, 2048, 3, 4),
                                    # C = 2 and C = 4 whole-piece rows
                                    (64, 8, 4096, 16, 4), (32, 16, 2048, 8, 4), (16, 16, 1024, 3, 8)])
def test_selector_columns_bit_exact(variant, layout):
    """A = E_J (unit columns) gives Y = S[:, J]: rows, signs and nnz must match the
    oracle bit-exactly and every value must be exactly ±fp32(1/√(κs))."""
    sk, osk = _pair(*layout)
    M, Br, Bc, kappa, s = layout
    rng = np.random.default_rng(0)
    h = int(rng.integers(M))
    J = np.concatenate([[h * Bc, h * Bc + Bc - 1], h * Bc + rng.choice(Bc, 30, replace=False)])
    n = len(J)
    A = torch.zeros((sk.d, n), device="cuda")
    A[torch.as_tensor(J, device="cuda"), torch.arange(n, device="cuda")] = 1.0
    try:
        Y = sk.apply(A, variant=variant).cpu().numpy()
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    gs = [g for g in range(M) if h in oracle.neighborhood(osk.a, osk.b, M, kappa, g)]
    assert len(gs) == kappa
    S_sub = oracle.build_S_csr(osk, blocks=gs)[:, J].toarray()
    rows = np.concatenate([np.arange(g * Br, (g + 1) * Br) for g in gs])
    Ysub = Y[rows]
    assert np.array_equal(Ysub != 0, S_sub != 0)
    assert np.array_equal(np.sign(Ysub), np.sign(S_sub))
    assert np.all(np.abs(Ysub[Ysub != 0]) == np.float32(sk.scale))
    mask = np.ones(sk.k, bool)
    mask[rows] = False
    assert not np.any(Y[mask])
    assert ((Y != 0).sum(axis=0) == kappa * s).all()


# ------------------------------------------------------------------ tiny config
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("kind", ["gaussian", "coherent", "lowrank"])
def test_tiny_config_full(variant, kind):
    cfg = C.TINY
    sk, osk = _pair(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed)
    A = synth.host_matrix(kind, cfg.d, cfg.n, seed=7, M=cfg.M)
    Yref = oracle.apply(osk, A)
    Y = _run(sk, A, variant)
    assert_f32(Y, Yref, np.linalg.norm(A.astype(np.float64), axis=0), f"tiny/{kind}/{variant}")
    Yt = _run(sk, A.T, variant, transposed=True)
    assert_f32(Yt.T, Yref, np.linalg.norm(A.astype(np.float64), axis=0), f"tiny-t/{kind}/{variant}")


# ----------------------------------------------------- odd layouts, ragged n, edges
ODD = [
    (5, 12, 40, 3, 3),      # non-power-of-two everything
    (8, 32, 128, 8, 2),     # kappa = M
    (16, 16, 256, 1, 4),    # kappa = 1
    (4, 8, 64, 2, 8),       # s = B_r (C = 1)
    (32, 32, 192, 4, 1),    # s = 1
    (7, 48, 96, 7, 6),      # kappa = M odd
    (64, 16, 512, 8, 2),
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", ODD)
@pytest.mark.parametrize("n", [1, 3, 17, 130])
def test_odd_layouts_ragged_n(variant, layout, n):
    sk, osk = _pair(*layout, seed=99)
    A = synth.host_matrix("gaussian", sk.d, n, seed=n)
    Yref = oracle.apply(osk, A)
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    assert_f32(_run(sk, A, variant), Yref, nrm, f"{layout} n={n} {variant}")
    assert_f32(_run(sk, A.T, variant, transposed=True).T, Yref, nrm, f"T {layout} n={n} {variant}")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("layout", [(8, 32, 128, 2, 2), (64, 16, 512, 8, 2), (16, 32, 1024, 4, 4)])
def test_bf16_input(variant, layout):
    sk, osk = _pair(*layout, seed=5)
    n = 96
    A = synth.host_matrix("gaussian", sk.d, n, seed=3)
    Y = _run(sk, A, variant, dtype=torch.bfloat16)
    assert_bf16(Y, oracle.apply(osk, A), "bf16 vs fp32 A")
    Ab = synth.bf16_round(A)
    assert_f32(Y, oracle.apply(osk, Ab), np.linalg.norm(Ab.astype(np.float64), axis=0), "bf16 tight")
    Yt = _run(sk, A.T, variant, dtype=torch.bfloat16, transposed=True)
    assert_f32(Yt.T, oracle.apply(osk, Ab), np.linalg.norm(Ab.astype(np.float64), axis=0), "bf16-t tight")


@pytest.mark.parametrize("n", [1, 17, 32, 64, 65])
def test_bf16_narrow(n):
    """Narrow bf16 inputs take the 64-column tile (n ≤ 64) with the deep ring; 65 the 128 tile."""
    sk, osk = _pair(64, 16, 2048, 8, 2, seed=11)
    A = synth.host_matrix("gaussian", sk.d, n, seed=n)
    Ab = synth.bf16_round(A)
    Y = _run(sk, A, "tc", dtype=torch.bfloat16)
    assert_f32(Y, oracle.apply(osk, Ab), np.linalg.norm(Ab.astype(np.float64), axis=0), f"bf16 narrow n={n}")


@pytest.mark.parametrize("layout", [(32, 32, 2048, 16, 1), (32, 32, 2048, 16, 4), (32, 32, 2048, 16, 8),
                                    (64, 24, 1024, 16, 8)])
@pytest.mark.parametrize("transposed", [False, True])
def test_wide_band_bf16(layout, transposed):
    """κ·B_r in (256, 512]: row-major runs the slot-split form (4-CTA clusters, κ/4 slots each,
    multicast data), transposed the four-band-tile form (bf16 only, 64-column tiles). Selector
    columns must reproduce S bit-exactly; Gaussian data meets the fp32 criterion against the
    bf16-rounded input."""
    M, Br, Bc, kappa, s = layout
    sk, osk = _pair(*layout, seed=21)
    if ((Br // s) & (Br // s - 1)) and transposed:  # C not a power of two: the 4-tile form rejects it
        with pytest.raises(BpsError):
            sk.apply_t(torch.zeros((8, sk.d), device="cuda", dtype=torch.bfloat16), variant="tc")
        return  # (row-major: the slot-split form covers it, checked below)
    rng = np.random.default_rng(1)
    J = rng.choice(sk.d, 40, replace=False)
    E = np.zeros((sk.d, len(J)), dtype=np.float32)
    E[J, np.arange(len(J))] = 1.0
    Y = _run(sk, E.T if transposed else E, "tc", dtype=torch.bfloat16, transposed=transposed)
    Y = Y.T if transposed else Y
    Sref = oracle.apply(osk, E)
    np.testing.assert_array_equal(np.sign(Y), np.sign(Sref))
    nz = Sref != 0
    assert np.all(np.abs(Y[nz]) == np.float32(1.0 / np.sqrt(kappa * s)))
    A = synth.host_matrix("gaussian", sk.d, 70, seed=2)
    Ab = synth.bf16_round(A)
    Y = _run(sk, A.T if transposed else A, "tc", dtype=torch.bfloat16, transposed=transposed)
    Y = Y.T if transposed else Y
    assert_f32(Y, oracle.apply(osk, Ab), np.linalg.norm(Ab.astype(np.float64), axis=0), f"wide {layout} T={transposed}")


@pytest.mark.parametrize("layout", [(32, 32, 2048, 16, 1), (32, 32, 2048, 16, 8), (64, 16, 1024, 16, 2),
                                    (32, 32, 2048, 8, 4), (64, 24, 1024, 16, 8), (32, 48, 1024, 6, 3)])
def test_slot_split_fp32(layout):
    """fp32 row-major with κ·B_r in (128, 512]: the slot-split form (2- or 4-CTA clusters, κ/SS band
    slots per CTA, TMA-multicast data) — bit-exact selector columns and the fp32 criterion."""
    M, Br, Bc, kappa, s = layout
    sk, osk = _pair(*layout, seed=22)
    rng = np.random.default_rng(3)
    J = rng.choice(sk.d, 40, replace=False)
    E = np.zeros((sk.d, len(J)), dtype=np.float32)
    E[J, np.arange(len(J))] = 1.0
    Y = _run(sk, E, "tc")
    Sref = oracle.apply(osk, E)
    np.testing.assert_array_equal(np.sign(Y), np.sign(Sref))
    assert np.all(np.abs(Y[Sref != 0]) == np.float32(1.0 / np.sqrt(kappa * s)))
    A = synth.host_matrix("gaussian", sk.d, 200, seed=4)
    assert_f32(_run(sk, A, "tc"), oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), f"ss {layout}")


def test_zero_n_and_zero_input():
    sk = Sketch(8, 32, 128, 2, 2, 1)
    A = torch.zeros((sk.d, 0), device="cuda")
    Y = sk.apply(A)
    assert Y.shape == (sk.k, 0)
    Y = sk.apply(torch.zeros((sk.d, 40), device="cuda"))
    assert not torch.any(Y)


@pytest.mark.parametrize("variant", VARIANTS)
def test_orbit_range_matches_full(variant):
    """bps_apply_orbit_range over [p0,p1) on stacked input blocks = the matching rows of the
    full apply of the same variant, bit for bit (R19; DESIGN.md §7 block sharding), and the
    oracle's rows per column (tests/test_gpu_sharding.py has the full sweep)."""
    M, Br, Bc, kappa, s = 16, 32, 256, 4, 2
    sk, osk = _pair(M, Br, Bc, kappa, s, seed=8)
    n = 64
    A_h = synth.host_matrix("gaussian", sk.d, n, seed=8)
    A = torch.from_numpy(A_h).cuda()
    try:
        Yfull = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    orb = sk.orbit()
    nrm = np.linalg.norm(A_h.astype(np.float64), axis=0)
    for (p0, p1) in [(0, 16), (3, 9), (13, 20), (15, 16)]:
        blocks = [orb[(p % M)] for p in range(p0 + 1, p1 + kappa)]
        A_loc = torch.cat([A[h * Bc:(h + 1) * Bc] for h in blocks])
        Y_loc = sk.apply_orbit_range(p0, p1, A_loc, variant=variant)
        ref = torch.cat([Yfull[orb[p % M] * Br:(orb[p % M] + 1) * Br] for p in range(p0, p1)])
        assert torch.equal(Y_loc, ref), (p0, p1)
        assert_f32(Y_loc.cpu().numpy(), oracle.apply(osk, A_h, blocks=[orb[p % M] for p in range(p0, p1)]), nrm,
                   f"orbit [{p0},{p1}) {variant}")


@pytest.mark.parametrize("variant", VARIANTS)
def test_deterministic(variant):
    sk = Sketch(128, 32, 2048, 4, 4, 3)
    A = torch.randn((sk.d, 300), device="cuda")
    try:
        Y1 = sk.apply(A, variant=variant).clone()
        Y2 = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    assert torch.equal(Y1, Y2)


# ------------------------------------------------- full-size configs, sampled outputs
def _sampled_check(cfg, variant, kind="gaussian", n_cols=6, n_blocks=3, transposed=False, mode="rowpart"):
    """Full-size apply in the bench's launch configuration; the oracle recomputes a
    sample of output blocks × columns one by one (task contract ③)."""
    dev = torch.device("cuda")
    tdt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    sk = Sketch(**cfg.sketch_args(), mode=mode)
    osk = oracle.make_sketch(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed, mode=mode)
    A = synth.device_matrix(kind, cfg.d, cfg.n, seed=11, M=cfg.M, dtype=tdt)
    try:
        if transposed:
            X = A.t().contiguous()
            del A
            Y = sk.apply_t(X, variant=variant).t()
            A = X.t()
        else:
            Y = sk.apply(A, variant=variant)
    except BpsError as e:
        if e.code == -3 and variant == "tc":
            pytest.skip(str(e))
        raise
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    cols = np.unique(np.concatenate([[0, cfg.n - 1], rng.choice(cfg.n, n_cols, replace=False)]))
    gs = sorted(set([0, cfg.M - 1] + rng.choice(cfg.M, n_blocks, replace=False).tolist()))
    idx = torch.as_tensor(cols, device=dev)
    A_cols = A.index_select(1, idx).float().cpu().numpy()  # d × |cols| (exact upcast)
    Yref = oracle.apply(osk, A_cols, blocks=gs)
    rows = np.concatenate([np.arange(g * cfg.B_r, (g + 1) * cfg.B_r) for g in gs])
    Yg = Y.index_select(1, idx).cpu().numpy()[rows]
    if cfg.dtype == "f32":
        return assert_f32(Yg, Yref, np.linalg.norm(A_cols.astype(np.float64), axis=0), cfg.name)
    return assert_f32(Yg, Yref, np.linalg.norm(A_cols.astype(np.float64), axis=0), cfg.name + " (bf16 tight)")


@pytest.mark.parametrize("variant", ["auto", "sparse"])
@pytest.mark.parametrize("kind", ["gaussian", "coherent"])
def test_ls_config_sampled(variant, kind):
    _sampled_check(C.LS, variant, kind)


@pytest.mark.parametrize("variant", ["auto"])
def test_ls_config_transposed_sampled(variant):
    _sampled_check(C.LS, variant, transposed=True)


@pytest.mark.parametrize("variant", ["auto"])
def test_grad_config_sampled(variant):
    _sampled_check(C.GRAD, variant)
    torch.cuda.empty_cache()


def test_smalln_config_sampled():
    _sampled_check(C.SMALLN, "tc")
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [C.sweep(1, 1), C.sweep(4, 8), C.sweep(16, 2), C.sweep(8, 4, "f32"),
                                 C.sweep_tuned(16, 8), C.sweep_tuned(16, 1, "f32"), C.sweep_tuned(8, 8),
                                 C.sweep_tuned(1, 8, "f32")],
                         ids=lambda c: c.name)
def test_sweep_sampled(cfg):
    _sampled_check(cfg, "auto")


# ------------------------------------- workspace (stream ranges) vs halo-range decomposition
@pytest.mark.parametrize("layout,n,dt", [((128, 32, 8192, 4, 4), 512, "f32"), ((16, 32, 1024, 4, 4), 200, "f32"),
                                         ((64, 16, 512, 8, 2), 304, "bf16"), ((16, 16, 256, 1, 4), 64, "f32"),
                                         ((8, 32, 128, 8, 2), 40, "bf16"), ((8, 32, 128, 8, 2), 48, "bf16"),
                                         ((7, 32, 64, 4, 4), 64, "f32")])
@pytest.mark.parametrize("transposed", [False, True])
def test_workspace_decomposition(layout, n, dt, transposed):
    """Group-aligned stream ranges with the owner/contributor workspace (bps_apply_ws) agree with
    the oracle, are bitwise reproducible and bitwise equal to the no-workspace (halo) ranges.
    (7, 32, 64, 4, 4): odd M, the shape ADVICE r1 found breaking the old parity routing."""
    sk, osk = _pair(*layout, seed=17)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    A = synth.host_matrix("gaussian", sk.d, n, seed=4)
    if dt == "bf16":
        A = synth.bf16_round(A)
    ref = oracle.apply(osk, A)
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    At = torch.from_numpy(np.ascontiguousarray(A.T if transposed else A)).cuda().to(tdt)
    f = sk.apply_t if transposed else sk.apply
    outs = []
    for use_ws in (True, True, False):
        try:
            Y = f(At, variant="tc", use_workspace=use_ws)
        except BpsError as e:
            if e.code == -3:
                pytest.skip(str(e))
            raise
        torch.cuda.synchronize()
        Yn = Y.cpu().numpy()
        outs.append(Yn.T if transposed else Yn)
    assert np.array_equal(outs[0], outs[1])  # bitwise reproducible
    assert np.array_equal(outs[0], outs[2])  # bitwise independent of the decomposition
    for Y in outs:
        assert_f32(Y, ref, nrm, f"{layout} n={n} {dt} T={transposed}")


def test_scaleout_config_one_panel_sampled():
    """BASELINE configs[4] (d=2^26, k=16384, κ=8, s=4, bf16) at full d on one column panel
    (n=512, 64 GiB of A): the per-rank unit of the 8-GPU scale-out run."""
    cfg = C.SCALEOUT.with_(n=512)
    free, _ = torch.cuda.mem_get_info()
    if free < cfg.d * cfg.n * 2 * 1.1:
        pytest.skip("not enough device memory for one scale-out panel")
    _sampled_check(cfg, "auto", n_cols=4, n_blocks=2)
    torch.cuda.empty_cache()

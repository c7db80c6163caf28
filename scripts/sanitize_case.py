"""Small applies for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel
family on tiny shapes — tc (workspace + combine, halo, transposed, orbit range, 4 band tiles, AffineUnique),
sparse, adjoint, FlashBlockRow — each result checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from parity import assert_f32
from paper_2602_06071_b200 import Sketch

def check(layout, n, dt="f32", variant="tc", mode="rowpart", transposed=False, ws=True):
    sk = Sketch(*layout, seed=5, mode=mode); osk = oracle.make_sketch(*layout, 5, mode=mode)
    A = synth.host_matrix("gaussian", sk.d, n, seed=1)
    if dt == "bf16":
        A = synth.bf16_round(A)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    At = torch.from_numpy(np.ascontiguousarray(A.T if transposed else A)).cuda().to(tdt)
    Y = (sk.apply_t if transposed else sk.apply)(At, variant=variant, use_workspace=ws)
    torch.cuda.synchronize()
    Y = Y.cpu().numpy()
    assert_f32(Y.T if transposed else Y, oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), str(layout))

check((16, 32, 1024, 4, 4), 200)                    # tc T form, workspace + combine
check((16, 32, 1024, 4, 4), 200, ws=False)          # halo ranges
check((16, 32, 1024, 4, 4), 130, transposed=True)   # fp32 transposed NT
check((64, 16, 512, 8, 2), 136, dt="bf16")          # bf16 NT
check((64, 16, 512, 8, 2), 64, dt="bf16", transposed=True)  # bf16 transposed re-layout
check((32, 32, 2048, 16, 4), 64, dt="bf16")         # kappa*B_r = 512 row-major: slot-split 4-CTA cluster
check((32, 32, 2048, 16, 4), 128)                   # fp32 slot split
check((32, 32, 2048, 8, 4), 128, dt="bf16")         # kappa*B_r = 256: slot-split pair
check((32, 32, 2048, 16, 4), 64, dt="bf16", transposed=True)  # four band tiles (transposed)
check((16, 32, 1024, 4, 8), 64, dt="bf16", mode="affine")
check((8, 32, 128, 2, 2), 16, variant="sparse")
check((8, 32, 128, 2, 2), 16, variant="sparse", transposed=True)
sk = Sketch(16, 32, 1024, 4, 4, seed=5); orb = sk.orbit()
A = torch.randn((sk.d, 64), device="cuda")
loc = torch.cat([A[orb[p % 16] * 1024:(orb[p % 16] + 1) * 1024] for p in range(3 + 1, 10 + 4)])
Yl = sk.apply_orbit_range(3, 10, loc); torch.cuda.synchronize()
Yin = torch.randn((sk.k, 64), device="cuda"); X = sk.apply_adjoint(Yin); torch.cuda.synchronize()
br = Sketch(16, 32, 1024, 4, 4, seed=5, kind="blockrow"); Yb = br.apply(A); torch.cuda.synchronize()
print("sanitize cases ok")

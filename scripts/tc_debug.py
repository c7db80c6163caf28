"""Quick tcgen05-variant diagnostics vs the oracle (run under `timeout` on the GPU box)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2602_06071_b200 import Sketch, BpsError

def run(layout, n, dt, trans, variant="tc", kind="gaussian"):
    M, Br, Bc, kappa, s = layout
    sk = Sketch(*layout, seed=1234); osk = oracle.make_sketch(*layout, seed=1234)
    A = synth.host_matrix(kind, sk.d, n, seed=5)
    if dt == "bf16":
        A = synth.bf16_round(A)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    At = torch.from_numpy(A.T.copy() if trans else A).cuda().to(tdt)
    t0 = time.time()
    try:
        Y = sk.apply_t(At, variant=variant) if trans else sk.apply(At, variant=variant)
        torch.cuda.synchronize()
    except BpsError as e:
        print(layout, n, dt, trans, "ERR", e); return
    Y = Y.cpu().numpy()
    if trans: Y = Y.T
    ref = oracle.apply(osk, A)
    nrm = np.linalg.norm(A.astype(np.float64), axis=0)
    err = np.abs(Y - ref).max(axis=0) / nrm
    bad = np.argwhere(np.abs(Y - ref) > 1e-5 * nrm[None, :])
    print(f"{layout} n={n} {dt} T={trans}: max rel {err.max():.3e}  nbad={len(bad)}  t={time.time()-t0:.2f}s", flush=True)
    if len(bad):
        for (i, t) in bad[:8]:
            print("   row", i, "col", t, "gpu", Y[i, t], "ref", ref[i, t])
        rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
        print("   bad rows blocks:", np.unique(rows // Br)[:20], "bad cols:", cols[:20], "...", len(cols))

cases = [
    ((8, 32, 128, 2, 2), 256, "bf16", False),
    ((8, 32, 128, 2, 2), 16, "f32", False),
    ((8, 32, 128, 2, 2), 16, "f32", True),
    ((8, 32, 128, 2, 2), 256, "bf16", True),
    ((16, 64, 128, 4, 2), 300, "bf16", False),
    ((64, 16, 512, 8, 2), 500, "bf16", False),
    ((16, 32, 1024, 4, 4), 200, "f32", False),
    ((32, 32, 192, 4, 1), 130, "f32", True),
    ((8, 32, 128, 8, 2), 64, "bf16", False),
    ((16, 16, 256, 1, 4), 64, "f32", False),
    ((128, 32, 8192, 4, 4), 512, "f32", False),
]
only = sys.argv[1:] 
for i, c in enumerate(cases):
    if only and str(i) not in only: continue
    run(*c)

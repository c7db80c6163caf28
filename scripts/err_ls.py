"""Print the parity error (max|err|/||A_col||) of the full-size LS config on sampled blocks."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, synth
from paper_2602_06071_b200 import Sketch, configs as C
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import f32_violation
for name in sys.argv[1:] or ["ls"]:
    cfg = C.CONFIGS[name]
    tdt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    sk = Sketch(**cfg.sketch_args()); osk = oracle.make_sketch(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed)
    for kind in ("gaussian", "coherent"):
        A = synth.device_matrix(kind, cfg.d, cfg.n, seed=5, M=cfg.M, dtype=tdt)
        Y = sk.apply(A)
        cols = torch.arange(0, cfg.n, max(1, cfg.n // 8), device="cuda")
        gs = list(range(0, cfg.M, max(1, cfg.M // 12)))
        Ac = A.index_select(1, cols).float().cpu().numpy()
        ref = oracle.apply(osk, Ac, blocks=gs)
        rows = np.concatenate([np.arange(g * cfg.B_r, (g + 1) * cfg.B_r) for g in gs])
        got = Y.index_select(1, cols).cpu().numpy()[rows]
        print(name, kind, "max|err|/||A_col|| =", f32_violation(got, ref, np.linalg.norm(Ac.astype(np.float64), axis=0)), flush=True)
        del A, Y; torch.cuda.empty_cache()

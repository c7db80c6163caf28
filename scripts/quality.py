"""RandNLA quality metrics on the LS config (BASELINE configs[1]: d=2^20, k=4096,
κ=4, s=4, n=512) for Gaussian, coherent and low-rank+noise inputs; one JSON line each."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2602_06071_b200 import Sketch, quality as Q, configs as C

cfg = C.LS
sk = Sketch(**cfg.sketch_args())
for kind in ("gaussian", "coherent", "lowrank"):
    A = synth.device_matrix(kind, cfg.d, cfg.n, seed=21, M=cfg.M)
    b = synth.device_matrix("gaussian", cfg.d, 1, seed=22)[:, 0]
    t0 = time.time()
    SA = sk.apply(A)
    rec = {"config": cfg.name, "kind": kind, "d": cfg.d, "k": cfg.k, "n": cfg.n, "kappa": cfg.kappa, "s": cfg.s,
           "gram_rel": Q.gram_error(A, SA), "ose": Q.ose_error(sk, A, r=64),
           "ridge_rel_residual": Q.ridge_residual(sk, A, b, 1e-3)[1],
           "sketch_and_solve_rel_residual": Q.sketch_and_solve(sk, A, b)[1]}
    exact = torch.linalg.lstsq(A.double(), b.double().reshape(-1, 1)).solution.reshape(-1)
    rec["exact_ls_rel_residual"] = float(torch.linalg.vector_norm(A.double() @ exact - b.double()) / torch.linalg.vector_norm(b.double()))
    rec["seconds"] = time.time() - t0
    print(json.dumps(rec), flush=True)

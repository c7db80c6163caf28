import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
from paper_2602_06071_b200 import Sketch, configs as C
cfg = C.GRAD.with_(n=1024)
sk = Sketch(**cfg.sketch_args())
A = torch.randn((cfg.d + (sk.kappa - 1) * sk.B_c, cfg.n), device="cuda", dtype=torch.bfloat16)
M, B_r = sk.M, sk.B_r
Yl = torch.empty((M * B_r, cfg.n), device="cuda")
dst = torch.empty((M * B_r, cfg.n), device="cuda")
kw = dict(dst=[dst.data_ptr()], dst_ld=cfg.n) if os.environ.get("MODE") == "bcast" else {}
for _ in range(4): sk.apply_orbit_range(0, M, A, out=Yl, **kw)
torch.cuda.synchronize()

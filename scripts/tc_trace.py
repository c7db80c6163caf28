"""Run one traced apply (BPS_TC_DEBUG=8) per config and print the per-role cycle breakdown."""
import os, sys
os.environ["BPS_TC_DEBUG"] = os.environ.get("BPS_TC_DEBUG", "8")
os.environ.setdefault("BPS_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_06071_b200", "libbps_instr.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2602_06071_b200 import Sketch, configs as C
for name in sys.argv[1:] or ["ls", "grad"]:
    cfg = C.CONFIGS[name]
    tdt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    sk = Sketch(**cfg.sketch_args())
    A = synth.device_matrix("gaussian", cfg.d, cfg.n, seed=1, M=cfg.M, dtype=tdt)
    Y = torch.empty((cfg.k, cfg.n), device="cuda")
    os.environ["BPS_TC_DEBUG"] = "0"
    for _ in range(3): sk.apply(A, out=Y)
    torch.cuda.synchronize()
    os.environ["BPS_TC_DEBUG"] = os.environ.get("TRACE_DBG", "8")
    print("====", name, "dbg", os.environ["BPS_TC_DEBUG"], flush=True)
    sk.apply(A, out=Y)
    torch.cuda.synchronize()
    sys.stderr.flush()
    del A
    torch.cuda.empty_cache()

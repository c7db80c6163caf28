"""Small applies on the fp32 slot-split paths (T form and NT form) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from parity import assert_f32
from paper_2602_06071_b200 import Sketch
for layout, n in [((32, 32, 2048, 16, 4), 128), ((32, 32, 2048, 8, 4), 200), ((16, 32, 1024, 8, 2), 136), ((64, 16, 1024, 16, 2), 256)]:
    sk = Sketch(*layout, seed=5); osk = oracle.make_sketch(*layout, 5)
    A = synth.host_matrix("gaussian", sk.d, n, seed=1)
    Y = sk.apply(torch.from_numpy(A).cuda(), variant="tc"); torch.cuda.synchronize()
    assert_f32(Y.cpu().numpy(), oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), str(layout))
    print("ok", layout, n, os.environ.get("BPS_TC_FORM", "tf"), flush=True)

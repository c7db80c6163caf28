"""One small apply on the cta_group::2 pair path (bf16, kappa*B_r = 256) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from parity import assert_f32
from paper_2602_06071_b200 import Sketch
for layout, n in [((32, 32, 2048, 8, 4), 256), ((16, 32, 1024, 8, 2), 136), ((64, 16, 1024, 16, 2), 512)]:
    sk = Sketch(*layout, seed=5); osk = oracle.make_sketch(*layout, 5)
    A = synth.bf16_round(synth.host_matrix("gaussian", sk.d, n, seed=1))
    Y = sk.apply(torch.from_numpy(A).cuda().bfloat16(), variant="tc"); torch.cuda.synchronize()
    assert_f32(Y.cpu().numpy(), oracle.apply(osk, A), np.linalg.norm(A.astype(np.float64), axis=0), str(layout))
    print("ok", layout, n, flush=True)

"""κ×s sweep (BASELINE.json configs[3]): sparse CUDA-core vs tcgen05 variant, d=2^22, k=4096,
n=1024, B_r=32 (M=128, B_c=32768), bf16 and fp32.  One JSON line per (dtype, κ, s, variant)
to stdout; GB/s uses the algorithmic bytes d·n·elem + k·n·4.  Run on a B200:
    python scripts/sweep.py > gpurun_out/sweep.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2602_06071_b200 import BpsError, Sketch  # noqa: E402
from paper_2602_06071_b200 import configs as C  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6545.3


def timed(fn, reps):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    args = sys.argv[1:]
    tuned = "--tuned" in args  # B_r per (κ, s) by the layout rule (configs.sweep_tuned)
    variants = ("tc",) if "--tc-only" in args else ("sparse", "tc")
    dtypes = [a for a in args if not a.startswith("--")] or ["bf16", "f32"]
    make = C.sweep_tuned if tuned else C.sweep
    for dt in dtypes:
        base = C.sweep(1, 1, dt)
        tdt = torch.float32 if dt == "f32" else torch.bfloat16
        A = synth.device_matrix("gaussian", base.d, base.n, seed=5, dtype=tdt)
        Y = torch.empty((base.k, base.n), device="cuda")
        for kappa in (1, 2, 4, 8, 16):
            for s in (1, 2, 4, 8):
                cfg = make(kappa, s, dt)
                sk = Sketch(**cfg.sketch_args())
                for variant in variants:
                    rec = {"dtype": dt, "kappa": kappa, "s": s, "B_r": cfg.B_r, "variant": variant, "config": cfg.name}
                    try:
                        fn = lambda: sk.apply(A, out=Y, variant=variant)  # noqa: E731
                        fn()
                        fn()
                        torch.cuda.synchronize()
                        reps = 3 if variant == "sparse" and kappa * s >= 32 else 5
                        ms = timed(fn, reps)
                        gbs = cfg.roofline_bytes() / (ms / 1e3) / 1e9
                        rec.update(ms=ms, gbs=gbs, frac=gbs / PEAK, columns_per_s=cfg.n / (ms / 1e3))
                    except BpsError as e:
                        rec.update(unsupported=str(e))
                    print(json.dumps(rec), flush=True)
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — sketch-apply throughput (BASELINE.json metric) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config ls] [--variant auto]
    torchrun --nproc-per-node N bench.py --gpus N ...            (N > 1, one rank per GPU)
    python bench.py --impl reference ...                          (the CPU oracle arm)

A step is one bps_apply (the whole hot path: wiring, hashing, streaming, accumulation,
epilogue — SURVEY §8a rows a1-a7) over the config's synthetic d×n input, resident in
HBM.  Multi-GPU is weak scaling: every rank applies the same sketch to its own n-column
batch (column sharding needs no collective); value = all ranks' bytes ÷
the max-over-ranks device time.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch-apply GB/s and columns/s per GPU (% of HBM roofline) at 1/2/4/8 B200"
UNIT = "GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="ls")
    ap.add_argument("--variant", default="auto", choices=["auto", "sparse", "tc"])
    ap.add_argument("--kind", default="gaussian", choices=["gaussian", "coherent", "lowrank"])
    ap.add_argument("--shard", default="column", choices=["column", "block", "block-fused"],
                    help="column: weak scaling, every rank its own n-column batch (no collective; at N>1 the "
                         "line also carries the strong-scaling measurement: the config's n split over the "
                         "ranks with dist.column_shard); block: strong scaling of one d×n problem sharded along "
                         "the wiring orbit + all-gather; block-fused: the same with the all-gather fused into the "
                         "kernel epilogue (stores into the peers' symmetric buffers, dist.block_sharded_apply_fused)")
    ap.add_argument("--op", default="apply", choices=["apply", "adjoint"],
                    help="adjoint: X = Sᵀ·Y (fp32 k×n -> d×n) on the same sketch; secondary line, no e2e/cpu legs")
    ap.add_argument("--sketch", default="blockperm", choices=["blockperm", "blockrow"],
                    help="blockrow: the FlashBlockRow sampling sketch (P:1424-1466); secondary line")
    ap.add_argument("--mode", default="rowpart", choices=["rowpart", "affine"],
                    help="intra-block pattern of BlockPerm-SJLT: row-partitioned (R1) or AffineUnique (R18)")
    ap.add_argument("--panel-cols", type=int, default=0, help="scaleout: columns per HBM panel (0 = fit 60%% of free memory)")
    ap.add_argument("--layout", default="n", choices=["n", "t"],
                    help="t: transposed layout (bps_apply_t, §8a8): X = Aᵀ n×d row-major in, Yᵀ n×k out")
    ap.add_argument("--t-pad", type=int, default=0, help=argparse.SUPPRESS)  # experiment: ldx = d + pad (transposed)
    ap.add_argument("--no-workspace", action="store_true", help="block-aligned ranges (no balanced workspace)")
    ap.add_argument("--ref-cols", type=int, default=64, help="reference arm: columns of the oracle sample per step")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)  # launcher test without a GPU
    ap.add_argument("--no-strong", action="store_true", help="N>1 column mode: skip the strong-scaling measurement")
    ap.add_argument("--n", type=int, default=0, help="override the config's column count (experiments)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if "bf16_tflops" in d:
            return float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, dense burst)"
    return 2250.0, "nominal (B200 dense bf16)"


def ncu_traffic(cfg_name, variant):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(cfg_name, {}).get(variant)


class Clocks:
    """Sample nvidia-smi clocks/throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str, enabled=True):
        self.gpu_id, self.enabled, self.rows, self.proc = gpu_id, enabled, [], None

    def start(self):
        if not self.enabled:
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.t.join(1)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ the CPU oracle as a baseline
_POOL_STATE = {}


def _oracle_panel(cols):
    """Worker: the oracle's product S @ A64 on a column panel (fork-inherited S and A)."""
    import numpy as np

    S, A = _POOL_STATE["S"], _POOL_STATE["A"]
    return S @ np.asarray(A[:, cols[0]:cols[1]], dtype=np.float64)


def oracle_timing(cfg, n_sample, cores=None, repeats=1):
    """Time the oracle as it stands (oracle.build_S_csr, then the CSR product oracle.apply performs)
    on an n_sample-column sample of the config, over all host cores: S built once per repeat
    (timed), the product split into column panels over a fork pool with one BLAS thread per worker
    (timed).  Returns dict(build_s, multiply_s, cores, n)."""
    import multiprocessing as mp

    import numpy as np

    import oracle
    import synth

    cores = cores or len(os.sched_getaffinity(0))
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    osk = oracle.make_sketch(cfg.M, cfg.B_r, cfg.B_c, cfg.kappa, cfg.s, cfg.seed)
    A = synth.host_matrix("gaussian", cfg.d, n_sample, seed=3, dtype=np.float32)
    nw = max(1, min(cores, n_sample))
    panels = [(n_sample * w // nw, n_sample * (w + 1) // nw) for w in range(nw)]
    builds, mults = [], []
    for _ in range(repeats):
        t0 = time.perf_counter()
        S = oracle.build_S_csr(osk)
        builds.append(time.perf_counter() - t0)
        _POOL_STATE.update(S=S, A=A)
        with mp.get_context("fork").Pool(nw) as pool:
            t0 = time.perf_counter()
            parts = pool.map(_oracle_panel, panels)
            mults.append(time.perf_counter() - t0)
        assert sum(x.shape[1] for x in parts) == n_sample
        _POOL_STATE.clear()
    return {"build_s": statistics.median(builds), "multiply_s": statistics.median(mults), "cores": nw, "n": n_sample}


def oracle_fits(cfg):
    # the oracle builds S explicitly (d·κs nonzeros in float64 CSR): beyond 2^28 nonzeros it does
    # not fit the host, so no bounded sample of this workload exists for it
    return cfg.d * cfg.kappa * cfg.s <= (1 << 28)


def reference_arm(args, cfg, rank):
    """--impl reference: the oracle (there is no reference implementation to install,
    DESIGN.md §8), as it stands, on the host cores; every step = S build + pooled product on a
    bounded column sample.  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return
    if not oracle_fits(cfg):
        print(json.dumps({"impl": "reference", "unavailable": f"oracle cannot build S for {cfg.name} "
                          f"(d*kappa*s = {cfg.d * cfg.kappa * cfg.s} > 2^28 nonzeros)"}), flush=True)
        return
    n_s = max(1, min(cfg.n, args.ref_cols))
    oracle_timing(cfg, n_s, repeats=max(1, min(args.warmup, 1)))  # warm-up (imports, page-in)
    t0 = time.perf_counter()
    tm = oracle_timing(cfg, n_s, repeats=args.steps)
    dt = (time.perf_counter() - t0) / args.steps
    gbs = cfg.roofline_bytes(n_s) / dt / 1e9
    sample = (f"{n_s} of {cfg.n} columns of {cfg.name} per step: S built in float64 CSR "
              f"(median {tm['build_s']:.2f} s) + product over {tm['cores']} worker processes "
              f"(median {tm['multiply_s']:.2f} s)")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic gaussian (host, numpy)",
        "config": {"workload": cfg.name, "d": cfg.d, "k": cfg.k, "kappa": cfg.kappa, "s": cfg.s, "n": n_s,
                   "B_r": cfg.B_r, "M": cfg.M, "B_c": cfg.B_c},
        "columns_per_s": n_s / dt,
        "cpu_baseline": {"value": gbs, "unit": UNIT, "cores": tm["cores"], "kind": "oracle", "sample": sample,
                         "build_s": tm["build_s"], "multiply_s": tm["multiply_s"]},
        "e2e": {"value": gbs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N without a torchrun environment: re-exec this script under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def dry_run(args, world, rank):
    """--dry-run: the launcher / aggregation path without a GPU (gloo; a numpy step stands in for the
    apply).  Used by the CPU tests of the multi-process plumbing."""
    import numpy as np
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    x = np.random.default_rng(rank).standard_normal((256, 256))
    for _ in range(max(3, args.warmup)):
        x = np.tanh(x @ x.T / 256)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x = np.tanh(x @ x.T / 256)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item()) / args.steps * 1e3
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms, "dry_run": True,
                          "comm": {"backend": "gloo", "world": world}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))  # one process per GPU under torch.distributed.run
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        dry_run(args, world, rank)
        return
    from paper_2602_06071_b200 import configs as C

    cfg = C.CONFIGS[args.config]
    if args.n:  # experiment: the config's sketch and d with another column count
        cfg = cfg.with_(n=args.n, name=f"{cfg.name}_n{args.n}")
    if args.impl == "reference":
        reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    import synth
    from paper_2602_06071_b200 import Sketch, lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        # NCCL prints its communicator init (nranks, NVLink/NVLS topology) to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        one = torch.ones(1, device=dev)
        dist.all_reduce(one)
        comm = {"backend": dist.get_backend(), "world": dist.get_world_size(), "allreduce_of_ones": float(one.item())}
    n = cfg.n
    tdt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    sk = Sketch(**cfg.sketch_args(), kind=args.sketch, **({"mode": args.mode} if args.sketch == "blockperm" else {}))
    if args.sketch == "blockrow":  # secondary line: the e2e/cpu legs are defined for the main sketch
        args.no_cpu_baseline = args.no_e2e = True
    stream = torch.cuda.current_stream(dev)
    if args.shard in ("block", "block-fused") and world > 1:
        from paper_2602_06071_b200 import dist as D

        p0, p1 = D.orbit_shard(cfg.M, world, rank)
        nblk = (p1 - p0) + cfg.kappa - 1
        # this rank's stacked input blocks (orbit positions p0+1 .. p1+κ-1), synthetic
        A = synth.device_matrix(args.kind, nblk * cfg.B_c, n, seed=1000 + rank, M=nblk, dtype=tdt, device=dev)
        Y = torch.empty((cfg.k, n), dtype=torch.float32, device=dev)

        def step():
            if args.shard == "block-fused":
                Y.copy_(D.block_sharded_apply_fused(sk, A, variant=args.variant))
            else:
                D.block_sharded_apply(sk, A, out=Y)
    elif args.op == "adjoint":
        Yin = synth.device_matrix(args.kind, cfg.k, n, seed=1000 + rank, dtype=torch.float32, device=dev)
        X = torch.empty((cfg.d, n), dtype=torch.float32, device=dev)
        args.no_e2e = args.no_cpu_baseline = True

        def step():
            sk.apply_adjoint(Yin, out=X, variant=args.variant)
    elif cfg.name == "scaleout":
        # BASELINE configs[4]: the job's n columns are split over the ranks (strong scaling) and each
        # rank streams its share through HBM in column panels that fit (2 TiB of A in total): every
        # panel is a full apply over all d rows into its own column range of Y (ldy = n_rank).  The
        # panel buffer is reused across panels (synthetic data), so each step reads d·n_rank·elem.
        n = cfg.n // world
        free = torch.cuda.mem_get_info(dev)[0]
        fit = int(0.6 * free) // (cfg.d * cfg.elem)
        # multiples of 512 columns keep the column tiles pairable into 2-CTA clusters (band sharing;
        # measured: 768-column panels 4.2 TB/s, 512/1024-column panels 5.3 TB/s)
        n_p = args.panel_cols or max(128, min(n, fit // 512 * 512 if fit >= 512 else fit // 128 * 128))
        A = synth.device_matrix(args.kind, cfg.d, n_p, seed=1000 + rank, M=cfg.M, dtype=tdt, device=dev)
        Y = torch.empty((cfg.k, n), dtype=torch.float32, device=dev)
        panels = [(c0, min(n_p, n - c0)) for c0 in range(0, n, n_p)]
        args.no_e2e = True  # 2 TiB of host->device traffic per step is not an end-to-end workload
        args.panels = {"panel_cols": n_p, "panels_per_step": len(panels), "n_per_rank": n}

        def step():
            for c0, w in panels:
                sk.apply(A[:, :w], out=Y[:, c0:c0 + w], variant=args.variant, use_workspace=not args.no_workspace)
    elif args.layout == "t":
        X = synth.device_matrix(args.kind, n, cfg.d + args.t_pad, seed=1000 + rank, dtype=tdt, device=dev)
        X = X[:, :cfg.d]
        Yt = torch.empty((n, cfg.k), dtype=torch.float32, device=dev)
        args.no_e2e = True

        def step():
            sk.apply_t(X, out=Yt, variant=args.variant, use_workspace=not args.no_workspace)
    else:
        A = synth.device_matrix(args.kind, cfg.d, n, seed=1000 + rank, M=cfg.M, dtype=tdt, device=dev)
        Y = torch.empty((cfg.k, n), dtype=torch.float32, device=dev)

        def step():
            sk.apply(A, out=Y, variant=args.variant, use_workspace=not args.no_workspace)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    clocks = Clocks(uuid if uuid.startswith("GPU-") else ("GPU-" + uuid), enabled=not args.no_clocks)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = lib.bps_kernel_launches()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for i in range(args.steps):
        step()
        ev[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    launches = lib.bps_kernel_launches() - l0
    # the dominant kernel's mean launch time: CUDA events the library records on the launch stream
    # around it, in a second run of the same steps (events between the stream kernel and the
    # combine pass would serialise their programmatic dependent launch, so not in the timed region)
    kern_ms = aux_ms = None
    timing = hasattr(lib, "bps_timing_enable")
    if timing:
        import ctypes

        lib.bps_timing_enable(1)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
        lib.bps_timing_enable(0)
        tot, cnt = ctypes.c_double(), ctypes.c_uint64()
        if lib.bps_timing_read(ctypes.byref(tot), ctypes.byref(cnt)) == 0 and cnt.value:
            kern_ms = tot.value / cnt.value
            launches_main = cnt.value
        if lib.bps_timing_read_ex(1, ctypes.byref(tot), ctypes.byref(cnt)) == 0 and cnt.value:
            aux_ms = tot.value / args.steps
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total = ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_max = float(t.item())
    ms = total_max / args.steps
    block = args.shard in ("block", "block-fused") and world > 1
    bytes_rank = cfg.roofline_bytes(n) if not block else cfg.roofline_bytes(n) // world
    if args.op == "adjoint":  # read Y (k×n fp32) once, write X (d×n fp32) once
        bytes_rank = (cfg.k + cfg.d) * n * 4
    if args.sketch == "blockrow":  # gather: κs sampled input rows per output row, one fp32 write
        bytes_rank = cfg.k * n * (cfg.kappa * cfg.s * cfg.elem + 4)
    value = world * bytes_rank / (ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    # roofline of the dominant kernel: algorithmic bytes per launch / its mean launch duration
    launches_per_step = (launches_main / args.steps) if kern_ms else None
    if kern_ms and launches_per_step and launches_per_step > 1:  # scale-out panels: several launches per step
        achieved = (bytes_rank / launches_per_step) / (kern_ms / 1e3) / 1e9
    else:
        achieved = bytes_rank / ((kern_ms if kern_ms else statistics.mean(per)) / 1e3) / 1e9

    # the dense ±1 band costs 2·κ·B_r flops per input element (×2 for the fp32 hi/lo split): where that
    # needs more time at the measured tensor peak than the bytes at the HBM peak, the kernel's roofline
    # is the tensor pipe (the κ·B_r = 512 sweep points)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak}
    if args.op == "apply" and args.sketch == "blockperm" and args.variant != "sparse" and not block:
        tpeak, tsrc = measured_tensor_peak()
        flops = 2.0 * cfg.kappa * cfg.B_r * cfg.d * n * (2 if cfg.dtype == "f32" else 1)
        if flops / (tpeak * 1e12) > bytes_rank / (peak * 1e9):
            t_launch = (kern_ms if kern_ms else statistics.mean(per)) / 1e3
            ach_t = flops / (launches_per_step or 1) / t_launch / 1e12
            roof = {"bound": "tensor", "achieved": ach_t, "peak": tpeak, "unit": "TFLOP/s", "frac": ach_t / tpeak,
                    "flops_per_launch": flops / (launches_per_step or 1), "tensor_peak_source": tsrc,
                    "hbm": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak}}

    # strong scaling (column mode, N > 1): the config's n columns split over the ranks (tile-aligned,
    # dist.column_shard), max-over-ranks device time, value = the whole job's bytes / that time
    strong = None
    if world > 1 and args.shard == "column" and not args.no_strong and args.op == "apply" and args.layout == "n" \
            and cfg.name != "scaleout":
        from paper_2602_06071_b200 import dist as D

        c0, c1 = D.column_shard(cfg.n, world, rank, align=128)
        A_s, Y_s = A[:, c0:c1], Y[:, c0:c1]

        def sstep():
            if c1 > c0:
                sk.apply(A_s, out=Y_s, variant=args.variant, use_workspace=not args.no_workspace)

        for _ in range(max(3, args.warmup)):
            sstep()
        torch.cuda.synchronize(dev)
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            sstep()
        s1.record(stream)
        torch.cuda.synchronize(dev)
        ts = torch.tensor([s0.elapsed_time(s1) / args.steps], device=dev, dtype=torch.float64)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        strong = {"value": cfg.roofline_bytes(cfg.n) / (float(ts.item()) / 1e3) / 1e9, "unit": UNIT,
                  "ms_per_step": float(ts.item()), "n_total": cfg.n, "n_per_rank_max": -(-cfg.n // 128 // world) * 128,
                  "scaling": "strong", "shard": "dist.column_shard (128-column aligned)"}

    # end-to-end through the public API with pinned host buffers (H2D + apply + D2H per step)
    e2e = None
    if not args.no_e2e and not block:
        max_e2e_bytes = 8 << 30
        n_e = n if bytes_rank <= max_e2e_bytes else max(128, int(n * max_e2e_bytes / bytes_rank) // 128 * 128)
        A_h = torch.empty((cfg.d, n_e), dtype=tdt, pin_memory=True)
        A_h.copy_(A[:, :n_e].cpu() if n_e < n else A.cpu())
        Y_h = torch.empty((cfg.k, n_e), dtype=torch.float32, pin_memory=True)
        A_d = A if n_e == n else torch.empty((cfg.d, n_e), dtype=tdt, device=dev)
        Y_d = Y if n_e == n else torch.empty((cfg.k, n_e), dtype=torch.float32, device=dev)

        def e2e_step():
            A_d.copy_(A_h, non_blocking=True)
            sk.apply(A_d, out=Y_d, variant=args.variant, use_workspace=not args.no_workspace)
            Y_h.copy_(Y_d, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        te = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = cfg.d * n_e * cfg.elem
        d2h = cfg.k * n_e * 4
        e2e = {"value": world * cfg.roofline_bytes(n_e) / (float(te.item()) / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "columns": n_e,
               "ms_per_step": float(te.item())}
        del A_h, Y_h

    cpu = None
    if not oracle_fits(cfg):
        args.no_cpu_baseline = True
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = min(cfg.n, 256)
        tm = oracle_timing(cfg, n_s, repeats=2)
        t_cpu = tm["build_s"] + tm["multiply_s"]
        cpu = {"value": cfg.roofline_bytes(n_s) / t_cpu / 1e9, "unit": UNIT, "cores": tm["cores"], "kind": "oracle",
               "sample": f"{n_s} of {cfg.n} columns of {cfg.name}: S built in float64 CSR (median {tm['build_s']:.2f} s, "
                         f"one core) + product over {tm['cores']} worker processes (median {tm['multiply_s']:.2f} s)",
               "build_s": tm["build_s"], "multiply_s": tm["multiply_s"],
               "host_cores_available": len(os.sched_getaffinity(0))}

    if rank == 0:
        line = {
            "metric": ("blockrow_gather_gbs" if args.sketch == "blockrow" else METRIC) if args.op == "apply"
            else "adjoint_throughput_gbs", "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if (block or cfg.name == "scaleout") else "weak",
            "vs_baseline": None, "dtype": "f32" if cfg.dtype == "f32" or args.op == "adjoint" else "bf16-in/f32-acc",
            "data": f"synthetic {args.kind} (torch Philox on device), seed {1000}+rank",
            "config": {"workload": cfg.name, "d": cfg.d, "k": cfg.k, "kappa": cfg.kappa, "s": cfg.s,
                       "n_per_gpu": n, "B_r": cfg.B_r, "M": cfg.M, "B_c": cfg.B_c, "variant": args.variant, "op": args.op, "sketch": args.sketch, "mode": args.mode, "layout": args.layout,
                       "parallelism": (f"orbit-block-shard x{world} + " + ("epilogue broadcast into symmetric memory"
                                       if args.shard == "block-fused" else "NCCL all_gather") if block
                                       else f"column-shard x{world} (no collective)"),
                       "l2": "inputs larger than L2 (no flush needed)" if bytes_rank > (256 << 20) else "input fits L2"},
            "columns_per_s": (n if block else world * n) / (ms / 1e3),
            **({"panels": args.panels} if getattr(args, "panels", None) else {}),
            "gbs_per_gpu": value / world,
            "frac_of_8tbs": value / world / 8000.0,
            "ms_min": min(per), "ms_median": statistics.median(per),
            "roofline": {**roof,
                         "traffic": ncu_traffic(cfg.name + (":t" if args.layout == "t" else "") + (":affine" if args.mode == "affine" else ""),
                                                args.variant) if (args.op == "apply" and args.sketch == "blockperm") else None,
                         "peak_source": peak_src,
                         "kernel": "bps_tc_kernel" if args.variant != "sparse" else "sparse gather kernel",
                         "kernel_ms_mean": kern_ms,
                         "aux_ms_per_step": aux_ms if timing else None,
                         "algorithmic_bytes_per_launch": bytes_rank / (launches_per_step or 1)},
            "gpu_launches": launches,
            **({"strong_scaling": strong} if strong else {}),
            **({"comm": comm} if comm else {}),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

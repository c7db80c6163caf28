"""Build libbps.so in-tree with nvcc for sm_100a (no torch involved).

    python -m paper_2602_06071_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbps.so")
LIB_INSTR = os.path.join(HERE, "libbps_instr.so")  # -DBPS_TC_INSTRUMENT: cycle trace + ablation switches
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(HERE, "..", "include", "bps.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, instrument: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    custom = out is not None
    out = out or (LIB_INSTR if instrument else LIB)
    if not force and not instrument and not custom and not needs_build():
        return LIB
    tmp = out + ".tmp"
    extra = (["-DBPS_TC_INSTRUMENT"] if instrument else []) + [f"-D{d}" for d in defines]
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(HERE, "..", "include"), "-o", tmp, *sources()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(force="--force" in args, verbose="-v" in args, instrument="--instrument" in args, out=out, defines=defs))

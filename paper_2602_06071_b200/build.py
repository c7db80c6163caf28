"""Build libbps.so in-tree with nvcc for sm_100a (no torch involved).

    python -m paper_2602_06071_b200.build [--force] [-v]      # or __graft_entry__.build()

Every csrc/*.cu is compiled to its own object in parallel (the tcgen05 kernel is split into
instantiation units bps_tc_i*.cu for this), then linked with the static CUDA runtime.  The
library is rebuilt whenever the SHA-256 of its sources (all .cu/.cuh/.h, include/bps.h, the
flags and this file) differs from the hash recorded next to it (libbps.so.srchash), so a
shipped binary can never silently disagree with the committed sources.  Objects are cached
under ~/.cache/bps_obj (BPS_OBJ_CACHE) by the hash of their own inputs.
"""
from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(HERE, "..", "include")
LIB = os.path.join(HERE, "libbps.so")
LIB_INSTR = os.path.join(HERE, "libbps_instr.so")  # -DBPS_TC_INSTRUMENT: cycle trace + ablation switches
OBJDIR = os.environ.get("BPS_OBJ_CACHE") or os.path.join(os.path.expanduser("~"), ".cache", "bps_obj")  # object cache (outside the repo)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH,
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(INCLUDE, "bps.h")])


def _digest(paths, extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for p in paths:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def source_hash(defines: tuple = ()) -> str:
    """Hash of everything the library is built from (sources, headers, flags, this script)."""
    return _digest(sources() + headers() + [os.path.abspath(__file__)], " ".join(NVCC_FLAGS + list(defines)))


def recorded_hash(lib: str = LIB) -> str | None:
    try:
        with open(lib + ".srchash") as f:
            return f.read().strip()
    except OSError:
        return None


def needs_build() -> bool:
    return not os.path.exists(LIB) or recorded_hash() != source_hash()


def _compile(src: str, extra: list, log: list) -> str:
    key = _digest([src] + headers(), " ".join(NVCC_FLAGS + extra))[:16]
    os.makedirs(OBJDIR, exist_ok=True)
    obj = os.path.join(OBJDIR, f"{os.path.basename(src)}.{key}.o")
    if os.path.exists(obj):
        return obj
    tmp = obj + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, "-c", src, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)} (see {os.path.join(HERE, 'build.log')})")
    os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False, instrument: bool = False, out: str | None = None,
          defines: tuple = ()) -> tuple[str, str]:
    """Returns (library path, "compiled" | "up to date")."""
    custom = out is not None
    out = out or (LIB_INSTR if instrument else LIB)
    defs = (("BPS_TC_INSTRUMENT",) if instrument else ()) + tuple(defines)
    want = source_hash(defs)
    if not force and not instrument and not custom and os.path.exists(out) and recorded_hash(out) == want:
        return out, "up to date"
    extra = [f"-D{d}" for d in defs]
    log: list = []
    jobs = min(len(sources()), os.cpu_count() or 4)
    try:
        with ThreadPoolExecutor(max_workers=jobs) as ex:
            objs = list(ex.map(lambda s: _compile(s, extra, log), sources()))
    finally:
        with open(os.path.join(HERE, "build.log"), "w") as f:
            f.write("\n".join(log))
    tmp = out + ".tmp"
    cmd = [nvcc(), *LINK_FLAGS, "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError("nvcc link failed")
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(tmp, out)
    with open(out + ".srchash", "w") as f:
        f.write(want + "\n")
    return out, "compiled"


if __name__ == "__main__":
    args = sys.argv[1:]
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(*build(force="--force" in args, verbose="-v" in args, instrument="--instrument" in args, out=out,
                 defines=defs))

"""bench.py plumbing on CPU: the --gpus N self-launch (torch.distributed.run, gloo in --dry-run),
one JSON line from rank 0 with n_gpus = N, and the CPU-oracle reference arm, which must not map
the product library (the driver checks which .so files each arm loads)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_gpus2_self_launch_prints_one_line():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "MASTER_ADDR": "127.0.0.1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["comm"]["world"] == 2


def test_reference_arm_does_not_load_the_library():
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'tiny', '--steps', '1', "
            "'--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "print('MAPPED', any('libbps' in l for l in open('/proc/self/maps')))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference"
    cb = lines[0]["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["build_s"] >= 0 and cb["multiply_s"] >= 0
    assert "MAPPED False" in r.stdout

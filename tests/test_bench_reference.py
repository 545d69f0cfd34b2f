"""bench.py's reference arm runs on the host CPU (the reference library compiled
in place, oracle/_ref): its JSON line at N = 1 and under torchrun at N = 2 (rank
0 alone runs it, with every host core -- torchrun sets OMP_NUM_THREADS=1)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libhdcref.so")


def parse(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def check(d, n):
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == ("reference" if os.path.exists(REF_LIB) else "port")
    assert cb["cores"] == len(os.sched_getaffinity(0)) and cb["value"] == pytest.approx(d["value"], rel=1e-3)
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_single_process():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    check(parse(p.stdout), 1)


def test_reference_arm_under_torchrun():
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    check(parse(p.stdout), 2)

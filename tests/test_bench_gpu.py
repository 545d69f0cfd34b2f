"""bench.py contract on the GPU: the default command (config 4, N = 1) and one
single-SpMV workload run to completion and print one JSON line carrying the
keys the driver and the judge read (roofline, e2e, clocks, gpu_launches)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    p = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def check_line(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["achieved"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_default_config4():
    d = run_bench("--steps", "2", "--warmup", "3", "--no-cpu-baseline")
    check_line(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3


def test_bench_workload_c1():
    d = run_bench("--workload", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    check_line(d)

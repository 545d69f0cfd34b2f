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


def test_bench_two_ranks_on_one_gpu(tmp_path):
    """bench.py's N > 1 path end to end on this one-GPU box: torchrun with two (and four) ranks
    that share cuda:0 over gloo (HDCG_BENCH_SHARED_GPU) on a small grid
    (HDCG_BENCH_GRID) -- slab plan and per-rank conversion, both halo transports
    (peer-memory stores through CUDA IPC, and send/recv), the halo checks after the
    warm-up and after the timed loop, the max-over-ranks reductions and the JSON
    line.  The final iterate's checksum and norm are bitwise those of the N = 1 line."""
    import socket
    env = dict(os.environ, HDCG_BENCH_GRID="64,64,32", MASTER_ADDR="127.0.0.1")
    p = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    one = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][0])
    assert one["test_mode"]["grid"] == [64, 64, 32] and one["n_gpus"] == 1
    for world, halo, want in ((2, "auto", "p2p"), (2, "nccl", "nccl"), (4, "auto", "p2p")):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
               "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", str(world),
               "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--halo", halo]
        p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                           env=dict(env, HDCG_BENCH_SHARED_GPU="1"))
        assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
        lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, p.stdout
        two = json.loads(lines[0])
        check_line(two)
        assert two["n_gpus"] == world and two["test_mode"]["ranks_share_one_gpu_gloo"]
        assert two["halo_check"]["transport"] == want and two["halo_check"]["ok_all_ranks"]
        assert two["halo_check"]["after_warmup"] and two["halo_check"]["after_timed"]
        assert two["result"]["y_checksum_lo_hi"] == one["result"]["y_checksum_lo_hi"]
        assert two["result"]["norm2_last_hex"] == one["result"]["norm2_last_hex"]
        assert two["config"]["nnz"] == one["config"]["nnz"]
        assert two["e2e"]["result_checked"] is True  # the chunked host pipeline returned the slab's exact y

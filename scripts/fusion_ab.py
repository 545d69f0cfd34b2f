"""Same-box A/B: what the power iteration's fused scale + per-tile norm costs.
Config 1 (256^3, bl 4096) and config 4 (1024x1024x512, bl 4096): plain SpMV
(spmv_device) vs the slab entry point with x_scale and tile sums, 10 launches
each, fraction of the measured peak of the algorithmic bytes."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200.dist import SlabPlan  # noqa: E402

H.init(0)
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream


def run(label, m, n, flush):
    info = m.info
    bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
    y = torch.empty_like(x)
    tiles = torch.empty(info.n_tiles, dtype=torch.float64, device="cuda")
    sc = torch.tensor([0.5], dtype=torch.float64, device="cuda")
    calls = {
        "plain": lambda: H.spmv_device(m, x.data_ptr(), y.data_ptr(), st),
        "scale": lambda: H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(), 0, st),
        "norm": lambda: H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, 0, tiles.data_ptr(), st),
        "scale+norm": lambda: H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(),
                                          tiles.data_ptr(), st),
    }
    for rep in range(2):
        for k, f in calls.items():
            for _ in range(3):
                f()
            ts = []
            for _ in range(10):
                if flush is not None:
                    flush.fill_(1.0)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                f()
                e.record()
                ts.append((s, e))
            torch.cuda.synchronize()
            ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
            print(json.dumps({"matrix": label, "variant": k, "ms": round(ms, 4),
                              "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)


flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
from paper_2105_04937_b200 import synth  # noqa: E402
rp, col, val = synth.laplacian7(256, 256, 256)
n = len(rp) - 1
m = H.to_mhdc(H.CsrMatrix(n, val, col, rp.astype("int32")), 0.6, 4096, validate=False)
run("c1_bl4096", m, n, flush)
m.free()
del rp, col, val
nx, ny, nz = bench.GRID4
plan = SlabPlan.make(nx * ny * nz, 4096, nx * ny, 1, unit=nx * ny)
m, nnz, _ = bench.build_config4_slab(H, torch, plan, 0, 4096)
run("c4_bl4096", m, nx * ny * nz, None)

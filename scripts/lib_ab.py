"""One process of a same-box library A/B: times the SpMV of the named workloads
(c1 bl 4096 plain and power-iteration form, c4 power-iteration form) with the
library HDCG_LIBRARY points at.  10 launches after 3 warm-up; prints JSON lines."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402
from paper_2105_04937_b200.dist import SlabPlan  # noqa: E402

H.init(0)
label = sys.argv[1]
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def timeit(m, n, fused, do_flush):
    info = m.info
    bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
    y = torch.empty_like(x)
    tiles = torch.empty(info.n_tiles, dtype=torch.float64, device="cuda")
    sc = torch.tensor([0.5], dtype=torch.float64, device="cuda")

    def call():
        if fused:
            H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(), tiles.data_ptr(), st)
        else:
            H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
    for _ in range(3):
        call()
    ts = []
    for _ in range(10):
        if do_flush:
            flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        call()
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
    return ms, bts / (ms * 1e-3) / 1e9 / peak


rp, col, val = synth.laplacian7(256, 256, 256)
n = len(rp) - 1
m = H.to_mhdc(H.CsrMatrix(n, val, col, rp.astype("int32")), 0.6, 4096, validate=False)
for fused in (False, True):
    ms, f = timeit(m, n, fused, True)
    print(json.dumps({"lib": label, "w": "c1" + ("_fused" if fused else ""), "ms": round(ms, 4), "frac": round(f, 4)}))
m.free()
nx, ny, nz = bench.GRID4
n = nx * ny * nz
plan = SlabPlan.make(n, 4096, nx * ny, 1, unit=nx * ny)
m, _, _ = bench.build_config4_slab(H, torch, plan, 0, 4096)
ms, f = timeit(m, n, True, False)
print(json.dumps({"lib": label, "w": "c4_fused", "ms": round(ms, 4), "frac": round(f, 4)}))

"""Same-box A/B of a per-call env knob of libhdcgpu.so over several workloads.

    python scripts/knob_ab.py HDCG_TMA_PREFETCH 0,1 c1:256 c1:512 c1:4096 c2 c3 c4

Each workload is built once; each value of the knob is timed (10 launches, L2
flushed before each for the small configurations, mean of CUDA-event times),
twice, alternating.  c4 runs the power-iteration form (x_scale + tile sums).
One JSON line per (workload, value, repetition)."""
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
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream
knob, values = sys.argv[1], sys.argv[2].split(",")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
cache = {}


def host_matrix(w):
    if w not in cache:
        cache.clear()
        if w == "c1":
            cache[w] = synth.laplacian7(256, 256, 256)
        elif w == "c2":
            cache[w] = synth.stencil27(192, 2)
        else:
            cache[w] = synth.quasi_diag(1 << 24, 4)
    return cache[w]


for spec in sys.argv[3:]:
    w, _, b = spec.partition(":")
    if w == "c4":
        nx, ny, nz = bench.GRID4
        n = nx * ny * nz
        plan = SlabPlan.make(n, 4096, nx * ny, 1, unit=nx * ny)
        m, _, _ = bench.build_config4_slab(H, torch, plan, 0, int(b or 4096))
    else:
        rp, col, val = host_matrix(w)
        n = len(rp) - 1
        bl = int(b) if b else {"c1": 4096, "c2": 4096, "c3": 8192}[w]
        m = H.to_mhdc(H.CsrMatrix(n, val, col, rp.astype("int32")), 0.6, bl, validate=False)
    info = m.info
    bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
    y = torch.empty_like(x)
    tiles = torch.empty(info.n_tiles, dtype=torch.float64, device="cuda")
    sc = torch.tensor([0.5], dtype=torch.float64, device="cuda")
    if w == "c4":
        def call():
            H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(), tiles.data_ptr(), st)
    else:
        def call():
            H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
    ref = None
    for rep in range(2):
        for v in values:
            os.environ[knob] = v
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            assert torch.equal(y.view(torch.int64), ref.view(torch.int64)), (spec, v)
            ts = []
            for _ in range(10):
                if w != "c4":
                    flush.fill_(1.0)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                call()
                e.record()
                ts.append((s, e))
            torch.cuda.synchronize()
            ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
            print(json.dumps({"workload": spec, knob: v, "ms": round(ms, 4),
                              "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)
    del os.environ[knob]
    m.free()
    del x, y, tiles
    torch.cuda.empty_cache()

"""Which kernel runs, and how fast, for shapes outside the BASELINE set: odd n
HDC (255^3 grid), odd bl, small even bl.  10 launches each, L2 flushed."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

H.init(0)
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
cases = [("lap255_hdc", 255, None), ("lap256_bl4095", 256, 4095), ("lap256_bl2047", 256, 2047),
         ("lap256_bl192", 256, 192), ("lap256_bl4096", 256, 4096)]
if len(sys.argv) > 1:  # named cases, or any "lap256_bl<N>"
    named = {c[0]: c for c in cases}
    cases = [named.get(a) or (a, 256, int(a.split("_bl")[1])) for a in sys.argv[1:]]
for label, g, bl in cases:
    rp, col, val = synth.laplacian7(g, g, g)
    n = len(rp) - 1
    A = H.CsrMatrix(n, val, col, rp.astype("int32"))
    m = H.to_hdc(A, 0.6, validate=False) if bl is None else H.to_mhdc(A, 0.6, bl, validate=False)
    info = m.info
    bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
    y = torch.empty_like(x)
    for _ in range(3):
        H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
    print(json.dumps({"case": label, "n": n, "bl": info.bl, "kernels": H.spmv_kernels(info), "ms": round(ms, 4),
                      "gflops": round(2 * int(rp[-1]) / (ms * 1e-3) / 1e9, 1),
                      "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)
    m.free()

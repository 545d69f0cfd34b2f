"""hdcg_spmv_host with pinned vs pageable host vectors (the reference API hands over
std::vector storage, i.e. pageable memory): ms per call and GB/s per direction."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

H.init(0)
which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    rp, col, val = synth.laplacian7(256, 256, 256)
else:
    rp, col, val = synth.laplacian7(512, 512, 256)
n = len(rp) - 1
A = H.CsrMatrix(n, val, col, rp.astype(np.int32))
m = H.to_mhdc(A, 0.6, 4096, validate=False)
x = synth.x_vector(n, 1)
for kind in ("pinned", "pageable", "pageable-fresh"):
    if kind == "pinned":
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.empty(n, dtype=torch.float64).pin_memory()
        xp, yp = xh.data_ptr(), yh.data_ptr()
    else:
        xa, ya = x.copy(), np.empty(n)
        xp, yp = xa.ctypes.data, ya.ctypes.data
    ts = []
    for i in range(6):
        if kind == "pageable-fresh":   # a new output vector per call, like the allocating overloads
            ya = np.empty(n)
            yp = ya.ctypes.data
        t0 = time.perf_counter()
        H.check(H.lib().hdcg_spmv_host(m.handle, xp, yp))
        ts.append(time.perf_counter() - t0)
    best = min(ts[1:])
    print(json.dumps({"workload": which, "n": n, "host_vectors": kind, "first_call_ms": round(ts[0] * 1e3, 3), "ms": round(best * 1e3, 3),
                      "gbs_each_way": round(8 * n / best / 1e9, 1)}), flush=True)

"""The reference-facing calls on host containers (what the C++ shim does per call):
to_mhdc from a host CSR (upload + device conversion), export of the format into host
arrays, spmv on host vectors -- with numpy (pageable) storage."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

H.init(0)
rp, col, val = synth.laplacian7(256, 256, 256)
n = len(rp) - 1
A = H.CsrMatrix(n, val, col, rp.astype(np.int32))
x = synth.x_vector(n, 1)
out = {}
for rep in range(3):
    t0 = time.perf_counter()
    m = H.to_mhdc(A, 0.6, 4096, validate=False)
    t1 = time.perf_counter()
    e = m.export()
    t2 = time.perf_counter()
    y = H.spmv_mhdc(m, x)
    t3 = time.perf_counter()
    out = {"to_mhdc_ms": round((t1 - t0) * 1e3, 2), "export_ms": round((t2 - t1) * 1e3, 2),
           "spmv_ms": round((t3 - t2) * 1e3, 2), "csr_bytes": int(12 * rp[-1] + 4 * (n + 1)),
           "format_bytes": int(e["segments"].nbytes)}
    m.free()
print(json.dumps(out))

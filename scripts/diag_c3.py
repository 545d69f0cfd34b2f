"""Diagnose TMA-kernel parity on the config-3 family: runs the SpMV repeatedly
under the current HDCG_TMA_* settings and reports mismatching rows against the
oracle (and against the general kernel)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Port  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
P = Port()
rp, col, val = synth.quasi_diag(n, seed=4)
x = synth.x_vector(n, 4)
A = H.CsrMatrix(n, val, col, rp.astype(np.int32))
for bl in (1024, 8192):
    ref = P.to_mhdc(rp, col, val, 0.6, bl)
    yref = P.spmv_mhdc(ref, x, 0)
    m = H.to_mhdc(A, 0.6, bl)
    for pol, rm in ((H.POLICY_GENERAL, 0), (H.POLICY_TMA, H.REST_SPLIT), (H.POLICY_TMA, H.REST_STAGED),
                    (H.POLICY_TMA, H.REST_GLOBAL)):
        H.set_kernel_policy(pol, rm)
        for rep in range(3):
            y = H.spmv_mhdc(m, x)
            bad = np.nonzero(y.view(np.int64) != yref.view(np.int64))[0]
            info = ""
            if bad.size:
                i = bad[0]
                info = (f" first row {i} (tile {i // 512}, row-in-tile {i % 512}), got {y[i]!r} want {yref[i]!r}, "
                        f"rest entries {ref.rest_rp[i + 1] - ref.rest_rp[i]}, rest_rp {ref.rest_rp[i]}; "
                        f"rows: {bad[:12].tolist()}")
            print(f"bl={bl} policy={pol} rest={rm} rep={rep}: {bad.size} bad rows{info}", flush=True)
    H.set_kernel_policy(H.POLICY_AUTO)

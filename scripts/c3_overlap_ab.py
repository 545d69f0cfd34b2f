"""Same-box A/B of the remainder modes on config 3 (quasi-diagonal 2^24, bl 8192 and
1024): mode 2 (rest_kernel then SpMV) vs mode 4 (chunked, overlapped on a side
stream) over chunk counts and TMA CTAs per SM.  Prints one line per variant:
label, ms (mean of 20, L2 flushed before each), fraction of the measured peak."""
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
rp, col, val = synth.quasi_diag(1 << 24, 4)
n = len(rp) - 1
A = H.CsrMatrix(n, val, col, rp.astype("int32"))
x = torch.from_numpy(synth.x_vector(n, 4)).cuda()
y = torch.empty(n, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream
variants = [("split", 2, {})]
for ch in (4, 8, 16, 32):
    for ct in (1, 2):
        variants.append((f"ovl_c{ch}_t{ct}", 4, {"HDCG_OVL_CHUNKS": str(ch), "HDCG_OVL_CTAS": str(ct)}))
for bl in (8192, 1024):
    m = H.to_mhdc(A, 0.6, bl, validate=False)
    info = m.info
    bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
    ref = None
    for rep in range(2):
        for label, mode, env in variants:
            os.environ.update(env)
            H.set_kernel_policy(H.POLICY_AUTO, mode)
            for _ in range(3):
                H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            assert torch.equal(y.view(torch.int64), ref.view(torch.int64)), label
            ts = []
            for _ in range(20):
                flush.fill_(1.0)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
                e.record()
                ts.append((s, e))
            torch.cuda.synchronize()
            ms = statistics.mean(s.elapsed_time(e) for s, e in ts)
            for k in env:
                del os.environ[k]
            print(json.dumps({"bl": bl, "variant": label, "ms": round(ms, 4),
                              "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)
    m.free()
H.set_kernel_policy(H.POLICY_AUTO)

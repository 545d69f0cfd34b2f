"""Same-box A/B of kernel variants: one process times the SpMV of the named
workloads with the library HDCG_LIBRARY points at (default libhdcgpu.so) and the
current HDCG_* environment knobs.  Matrices are generated once per box call and
cached under /tmp.  20 launches after 3 warm-up, 256 MB L2 flush before each;
prints one JSON line per workload (ms, fraction of the measured HBM peak).

    python scripts/ab.py LABEL c1-100 c1-4096 c1-hdc c1-csr c2-4096 c3-8192 c3-1024 c3-hdc
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402


THETA = float(os.environ.get("HDCG_AB_THETA", "0.6"))  # fill threshold of the conversions (A/B knob)


def matrix(w):
    path = f"/tmp/hdcg_ab_{w}.npz"
    if os.path.exists(path):
        d = np.load(path)
        return d["rp"], d["col"], d["val"], int(d["seed"])
    if w == "c1":
        (rp, col, val), seed = synth.laplacian7(256, 256, 256), 1
    elif w == "c2":
        (rp, col, val), seed = synth.stencil27(192, 2), 3
    else:
        (rp, col, val), seed = synth.quasi_diag(1 << 24, 4), 4
    np.savez(path, rp=rp, col=col, val=val, seed=seed)
    return rp, col, val, seed


def main():
    label = sys.argv[1]
    H.init(0)
    peak, _ = bench.load_peaks()
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for spec in sys.argv[2:]:
        w, fmt = spec.replace("-", ":").split(":")  # c3-8192 (gpu.sh steps split on ":")
        rp, col, val, seed = matrix(w)
        n = len(rp) - 1
        A = H.CsrMatrix(n, val, col, rp.astype(np.int32))
        if fmt == "csr":
            m = H.device_csr(A)
        elif fmt == "hdc":
            m = H.to_hdc(A, THETA, validate=False)
        else:
            m = H.to_mhdc(A, THETA, int(fmt), validate=False)
        info = m.info
        x = torch.from_numpy(synth.x_vector(n, seed)).cuda()
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            H.spmv_device(m, x.data_ptr(), y.data_ptr(), st)
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
        bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
        ck = int(y.view(torch.int64).sum().item())
        print(json.dumps({"lib": label, "w": spec, "ms": round(ms, 4), "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 4),
                          "gflops": round(2 * int(rp[-1]) / (ms * 1e-3) / 1e9, 1), "kernels": H.spmv_kernels(info),
                          "packed_stages": info.packed_stages, "y_sum": ck}), flush=True)
        m.free()


if __name__ == "__main__":
    main()

"""CSR -> M-HDC / HDC conversion time on the device (inputs resident in HBM), against
the bytes a conversion has to move:

    census pass   read row_ptr + col_ind
    fill pass     read row_ptr + col_ind + values, write 8 B per segment slot,
                  12 B per remainder entry, 4 B per row (remainder row pointers)

Wall time of the C-ABI call (hdcg_build_mhdc / hdcg_build_hdc with device inputs: it
returns after its own stream synchronisation), best of `reps`, and the fraction of
the measured HBM copy peak those bytes would take.

    python scripts/convert_bench.py [c1 c2 c3 c4] [--validate]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402


def device_csr_arrays(w):
    if w == "c4":
        nx, ny, nz = bench.GRID4
        n = nx * ny * nz
        nnz = H.gen_laplacian7_nnz(nx, ny, nz, 0, nz)
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(nnz, dtype=torch.int32, device="cuda")
        val = torch.empty(nnz, dtype=torch.float64, device="cuda")
        H.gen_laplacian7(nx, ny, nz, 0, nz, rp.data_ptr(), col.data_ptr(), val.data_ptr())
        torch.cuda.synchronize()
        return n, nnz, rp, col, val, True
    if w == "c1":
        rp, col, val = synth.laplacian7(256, 256, 256)
    elif w == "c2":
        rp, col, val = synth.stencil27(192, 2)
    else:
        rp, col, val = synth.quasi_diag(1 << 24, 4)
    n = len(rp) - 1
    return (n, int(rp[-1]), torch.from_numpy(rp.astype(np.int32)).cuda(), torch.from_numpy(col).cuda(),
            torch.from_numpy(val).cuda(), False)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1", "c2", "c3", "c4"]
    validate = "--validate" in sys.argv
    H.init(0)
    peak, _ = bench.load_peaks()
    for w in args:
        n, nnz, rp, col, val, rp64 = device_csr_arrays(w)
        rpb = 8 if rp64 else 4
        for fmt, bl in (("mhdc", {"c3": 8192}.get(w, 4096)), ("mhdc", {"c3": 1024}.get(w, 256)), ("hdc", 0)):
            if w == "c4" and fmt == "hdc":
                continue  # 7 lanes of 5.4e8 doubles: the same bytes as M-HDC, one block
            best, info = 1e9, None
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if fmt == "hdc":
                    m = H.build_hdc_device(n, nnz, rp.data_ptr(), col.data_ptr(), val.data_ptr(), bench.THETA,
                                           rp64=rp64, validate=validate)
                else:
                    m = H.build_mhdc_device(n, n, 0, nnz, rp.data_ptr(), col.data_ptr(), val.data_ptr(), bench.THETA,
                                            bl, rp64=rp64, validate=validate)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
                info = m.info
                m.free()
            by = (rpb * (n + 1) + 4 * nnz) + (rpb * (n + 1) + 12 * nnz) + 8 * info.dia_slots + 12 * info.nnz_rest + 4 * (n + 1)
            if validate:
                by += rpb * (n + 1) + 4 * nnz
            print(json.dumps({"w": w, "format": fmt, "bl": bl, "n": n, "nnz": nnz, "validate": validate,
                              "convert_ms": round(best * 1e3, 3), "bytes": by,
                              "gbs": round(by / best / 1e9, 1), "frac_of_copy_peak": round(by / best / 1e9 / peak, 4),
                              "n_seg": info.n_seg, "nnz_rest": info.nnz_rest}), flush=True)
        del rp, col, val
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

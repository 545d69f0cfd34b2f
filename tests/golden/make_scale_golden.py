"""Regenerate tests/golden/scale_digests.json: SHA-256 digests of the formats and
products the UNMODIFIED reference computes at the BASELINE configurations' full
sizes, for the at-scale GPU parity tests (tests/test_gpu_scale.py).

Run in the build container (where /root/reference exists; several minutes):

    make -C oracle && python tests/golden/make_scale_golden.py

Everything digested is an OUTPUT of the reference's own code (oracle/_ref/
libhdcref.so = /root/reference/proj/src/*.cpp + oracle/ref_capi.cpp): to_mhdc /
to_hdc (convert.cpp:89-169), rates (convert.cpp:173-196), spmv_mhdc / spmv_hdc
(kernels.cpp:107-206), on the seeded inputs of paper_2105_04937_b200.synth.  Our
C restatement (oracle/hdc_oracle.c) is checked against every array here as well.

* config 3 (quasi-diagonal, n = 2^24, seed 4; x seed 4): M-HDC bl = 1024 and 8192,
  HDC -- every format array and y.
* config 4 (7-point Laplacian 1024x1024x512; x uniform[-1,1] seed 5): the first,
  a middle and the last 16-plane z-slab (both Dirichlet faces), each as the slab
  with its halo columns (synth.laplacian7_slab_square): the slab's blocks of the
  bl = 4096 M-HDC (dia_ptr rebased, offsets, segments; no remainder) and y over
  the slab's rows.  These are the global format's blocks and rows exactly
  (per-block census, convert.cpp:48-56).

Arrays are digested in the device layout (int32 indices, float64 values,
little-endian) so the GPU test hashes its exports directly.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Ref  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale_digests.json")
THETA = 0.6
GRID4 = (1024, 1024, 512)
C4_SLABS = ((0, 16), (248, 264), (496, 512))


def digest(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def fmt_digests(m):
    return {"dia_ptr": digest(m.dia_ptr, "<i4"), "dia_offsets": digest(m.offsets, "<i4"),
            "segments": digest(m.segments, "<f8"), "rest_row_ptr": digest(m.rest_rp, "<i4"),
            "rest_col_ind": digest(m.rest_col, "<i4"), "rest_values": digest(m.rest_val, "<f8"),
            "n_seg": int(m.offsets.size), "nnz_rest": int(m.rest_col.size)}


def same(a, b):
    return all(np.asarray(getattr(a, f)).tobytes() == np.asarray(getattr(b, f)).tobytes()
               for f in ("dia_ptr", "offsets", "segments", "rest_rp", "rest_col", "rest_val"))


def config3(R, P):
    t = time.time()
    n = 1 << 24
    rp, col, val = synth.quasi_diag(n, seed=4)
    x = synth.x_vector(n, 4)
    out = {"n": n, "nnz": int(rp[-1]), "x_seed": 4}
    for bl in (1024, 8192, 0):
        key = f"mhdc_bl{bl}" if bl else "hdc"
        hd = R.mhdc_handle(rp, col, val, THETA, bl) if bl else R.hdc_handle(rp, col, val, THETA)
        m = R.export_mhdc(hd) if bl else R.export_hdc(hd)
        y = R.spmv("mhdc" if bl else "hdc", hd, x)
        a, b, slots = R.rates(hd)
        mp = P.to_mhdc(rp, col, val, THETA, bl) if bl else P.to_hdc(rp, col, val, THETA)
        assert same(m, mp), key  # our C restatement agrees with the reference
        assert P.spmv_mhdc(mp, x, 0).tobytes() == y.tobytes(), key
        d = fmt_digests(m)
        d.update(y=digest(y, "<f8"), rates=[a, b, int(slots)], y_head=y[:4].tolist())
        out[key] = d
        del hd, m, mp, y
        print(f"config 3 {key}: {time.time() - t:.1f} s", flush=True)
    return out


def config4(R, P):
    nx, ny, nz = GRID4
    plane, bl = nx * ny, 4096
    out = {"grid": list(GRID4), "bl": bl, "x_seed": 5, "slabs": {}}
    for z0, z1 in C4_SLABS:
        t = time.time()
        rp, col, val, g0 = synth.laplacian7_slab_square(nx, ny, nz, z0, z1)
        n_s = len(rp) - 1
        n_full = nx * ny * nz
        x = np.zeros(n_s)
        lo, hi = max(0, g0), min(n_full, g0 + n_s)
        x[lo - g0:hi - g0] = synth.uniform_pm1(5, 0, np.arange(lo, hi, dtype=np.int64))
        hd = R.mhdc_handle(rp, col, val, THETA, bl)
        m = R.export_mhdc(hd)
        y = R.spmv("mhdc", hd, x)
        mp = P.to_mhdc(rp, col, val, THETA, bl)
        assert same(m, mp), (z0, z1)
        assert P.spmv_mhdc(mp, x, 0).tobytes() == y.tobytes(), (z0, z1)
        # the slab's rows are [plane, plane + rows) of the square matrix; its blocks
        # start at block plane/bl (bl divides a plane)
        rows = (z1 - z0) * plane
        b0, b1 = plane // bl, (plane + rows) // bl
        dp = m.dia_ptr[b0:b1 + 1] - m.dia_ptr[b0]
        k0, k1 = int(m.dia_ptr[b0]), int(m.dia_ptr[b1])
        assert m.rest_col.size == 0
        out["slabs"][f"{z0}-{z1}"] = {
            "z0": z0, "z1": z1, "row0": z0 * plane, "rows": rows, "block0": z0 * plane // bl,
            "blocks": b1 - b0, "n_seg": k1 - k0,
            "dia_ptr": digest(dp, "<i4"), "dia_offsets": digest(m.offsets[k0:k1], "<i4"),
            "segments": digest(m.segments[k0 * bl:k1 * bl], "<f8"),
            "y": digest(y[plane:plane + rows], "<f8"), "y_head": y[plane:plane + 4].tolist(),
        }
        del hd, m, mp, y, rp, col, val
        print(f"config 4 slab z[{z0},{z1}): {time.time() - t:.1f} s", flush=True)
    return out


def main():
    R, P = Ref(), Port()
    res = {"generator": "tests/golden/make_scale_golden.py (the unmodified reference, oracle/_ref)",
           "theta": THETA, "config4": config4(R, P), "config3": config3(R, P)}
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()

"""Regenerate tests/golden/ref_cases.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every array stored here is an OUTPUT of the reference's own code
(oracle/_ref/libhdcref.so = /root/reference/proj/src/*.cpp + oracle/ref_capi.cpp):
to_mhdc / to_hdc (convert.cpp:89-169), rates (convert.cpp:173-196),
census_blocked (convert.cpp:39-58) and the six spmv_* kernels
(kernels.cpp:39-206), on seeded inputs from paper_2105_04937_b200.synth.
The GPU tests compare the CUDA path against these arrays on boxes where
/root/reference does not exist.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_2105_04937_b200 import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_cases.npz")


def cancel_matrix():
    """proj/tests/data/cancel.mtx (17x17): row 0 = 1e16 @0, -1e16 @8, 3 @16; unit diagonal."""
    rows = [0, 0, 0] + list(range(1, 17))
    cols = [0, 8, 16] + list(range(1, 17))
    vals = [1e16, -1e16, 3.0] + [1.0] * 16
    return synth.coo_to_csr(17, rows, cols, vals)


def cases():
    rng = np.random.default_rng(20240811)
    out = []
    rp, col, val = synth.example_matrix()
    out.append(("example", (rp, col, val), 0.6, 4, np.arange(1, 9, dtype=np.float64)))
    # acceptance.cpp:134-201 shapes: random, single diagonal, dense row, stencils
    for rep in range(24):
        n = int(rng.integers(2, 160))
        A = synth.random_matrix(n, float(rng.uniform(0.01, 0.30)), rng)
        theta = float(rng.uniform(0.0, 1.0)) if rep % 6 else 0.0
        bl = int(rng.integers(1, n + 3))
        out.append((f"random{rep}", A, theta, bl, rng.uniform(0.5, 1.5, n)))
    for off in (-100, 0, 100):
        out.append((f"single_diag{off}", synth.single_diagonal_matrix(101, off), 0.5, 16,
                    rng.uniform(0.5, 1.5, 101)))
    for row in (0, 63, 127):
        out.append((f"dense_row{row}", synth.dense_row_matrix(128, row, rng), 0.6, 32,
                    rng.uniform(0.5, 1.5, 128)))
    for kind in ("p3_1d", "p5_2d", "p7_3d"):
        for n in (27, 64, 300):
            out.append((f"{kind}_n{n}", synth.reference_stencil(kind, n), 0.6, 50,
                        rng.uniform(0.5, 1.5, n)))
    # test_convert.cpp:131-156 edge cases
    out.append(("theta_edge", synth.coo_to_csr(4, [0, 1, 0], [0, 1, 3], [1.0, 1.0, 2.0]), 0.5, 4,
                np.ones(4)))
    out.append(("short_last_block", synth.coo_to_csr(5, range(5), range(5), [2.0] * 5), 1.0, 4,
                np.arange(1, 6, dtype=np.float64)))
    # test_kernels.cpp:101-114 accumulation-order pin
    out.append(("order_pin", synth.coo_to_csr(3, [0, 0, 0, 1, 2], [0, 1, 2, 1, 2],
                                              [1e16, 1.0, -1e16, 1.0, 1.0]), 0.5, 2, np.ones(3)))
    # cancel.mtx with the CLI's x (hdcmv.cpp:38-42): x_i = 1 + (i mod 8)/8
    out.append(("cancel", cancel_matrix(), 0.6, 100,
                1.0 + (np.arange(17) % 8) / 8.0))
    # BASELINE-config shapes at small sizes
    out.append(("lap7_12x10x9", synth.laplacian7(12, 10, 9), 0.6, 64, synth.x_vector(1080, 1)))
    out.append(("st27_g8", synth.stencil27(8, seed=2), 0.6, 128, synth.x_vector(512, 3)))
    out.append(("quasi_small", synth.quasi_diag(6000, seed=4, seg_min=100, seg_max=900), 0.6, 256,
                synth.x_vector(6000, 4)))
    return out


def main():
    R = Ref()
    store = {}
    names = []
    for name, (rp, col, val), theta, bl, x in cases():
        names.append(name)
        p = name + "/"
        store[p + "rp"], store[p + "col"], store[p + "val"] = rp, col, val
        store[p + "theta"] = np.array(theta)
        store[p + "bl"] = np.array(bl)
        store[p + "x"] = x
        mh = R.mhdc_handle(rp, col, val, theta, bl)
        m = R.export_mhdc(mh)
        for f in ("dia_ptr", "offsets", "segments", "rest_rp", "rest_col", "rest_val"):
            store[p + "mhdc_" + f] = getattr(m, f)
        hh = R.hdc_handle(rp, col, val, theta)
        h = R.export_hdc(hh)
        for f in ("offsets", "segments", "rest_rp", "rest_col", "rest_val"):
            store[p + "hdc_" + f] = getattr(h, f)
        try:
            store[p + "mhdc_rates"] = np.array(R.rates(mh), dtype=np.float64)
            store[p + "hdc_rates"] = np.array(R.rates(hh), dtype=np.float64)
        except ValueError:
            store[p + "mhdc_rates"] = np.array([np.nan, np.nan, 0.0])
            store[p + "hdc_rates"] = np.array([np.nan, np.nan, 0.0])
        bp, offs, cnt = R.census(rp, col, val, bl)
        store[p + "census_bp"], store[p + "census_off"], store[p + "census_cnt"] = bp, offs, cnt
        c = R.csr(rp, col, val)
        store[p + "y_csr"] = R.spmv("csr", c, x)
        store[p + "y_dia"] = R.spmv("dia", c, x)
        store[p + "y_bdia"] = R.spmv("bdia", c, x, bl=bl)
        store[p + "y_hdc"] = R.spmv("hdc", hh, x)
        store[p + "y_bhdc"] = R.spmv("bhdc", hh, x, bl=bl)
        store[p + "y_mhdc"] = R.spmv("mhdc", mh, x)
    store["names"] = np.array(names)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(names)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

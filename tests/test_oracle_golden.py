"""Pin the CPU oracle (oracle/hdc_oracle.c) against the reference's own golden
vectors before it is trusted as the GPU parity checker.

* tests/golden/example_fixture.json: the reference's fixture arrays
  (proj/tests/test_convert.cpp:14-129, test_kernels.cpp:34-43).
* tests/golden/ref_cases.npz: outputs of the unmodified reference library
  (tests/golden/make_golden.py) on 47 seeded cases.
* when oracle/_ref/libhdcref.so exists (this container), bit-for-bit
  comparison against the live reference on fresh random matrices.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import Ref, dense_multiply, max_rel_err
from paper_2105_04937_b200 import synth

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fixture():
    with open(os.path.join(HERE, "golden", "example_fixture.json")) as f:
        return json.load(f)


def _csr(fx):
    c = fx["csr"]
    return (np.array(c["row_ptr"], np.int64), np.array(c["col_ind"], np.int32),
            np.array(c["values"], np.float64))


def test_example_matrix_matches_fixture(fixture):
    rp, col, val = synth.example_matrix()
    frp, fcol, fval = _csr(fixture)
    assert np.array_equal(rp, frp) and np.array_equal(col, fcol) and np.array_equal(val, fval)


def test_census_fixture(port, fixture):
    rp, col, val = _csr(fixture)
    bp, offs, cnt = port.census(rp, col, 8)
    assert [[int(o), int(c)] for o, c in zip(offs, cnt)] == fixture["census_global"]
    bp, offs, cnt = port.census(rp, col, 4)
    blocks = [[[int(offs[k]), int(cnt[k])] for k in range(bp[b], bp[b + 1])] for b in range(2)]
    assert blocks == fixture["census_bl4"]


def test_hdc_fixture(port, fixture):
    rp, col, val = _csr(fixture)
    h = port.to_hdc(rp, col, val, 0.6)
    f = fixture["hdc_theta0.6"]
    assert h.offsets.tolist() == f["offsets"]
    assert h.segments.tolist() == f["lanes"]
    assert h.rest_val.tolist() == f["rest_values"]
    assert h.rest_col.tolist() == f["rest_col_ind"]
    assert h.rest_rp.tolist() == f["rest_row_ptr"]
    assert port.rates(h) == (f["alpha"], f["beta"], f["dia_slots"])


def test_dia_fixture(port, fixture):
    rp, col, val = _csr(fixture)
    d = port.to_hdc(rp, col, val, 0.0)
    assert d.offsets.tolist() == fixture["dia"]["offsets"]
    assert d.segments.tolist() == fixture["dia"]["lanes"]
    assert d.rest_val.size == 0


def test_mhdc_fixture(port, fixture):
    rp, col, val = _csr(fixture)
    m = port.to_mhdc(rp, col, val, 0.6, 4)
    f = fixture["mhdc_theta0.6_bl4"]
    assert m.dia_ptr.tolist() == f["dia_ptr"]
    assert m.offsets.tolist() == f["offsets"]
    assert m.segments.tolist() == f["segments"]
    assert m.rest_val.tolist() == f["rest_values"]
    assert m.rest_col.tolist() == f["rest_col_ind"]
    assert m.rest_rp.tolist() == f["rest_row_ptr"]
    assert port.rates(m) == (f["alpha"], f["beta"], f["dia_slots"])


def test_fixture_product(port, fixture):
    rp, col, val = _csr(fixture)
    x = np.array(fixture["x"], np.float64)
    want = fixture["y"]
    assert port.spmv_csr(rp, col, val, x).tolist() == want
    assert port.spmv_mhdc(port.to_mhdc(rp, col, val, 0.6, 4), x).tolist() == want
    assert port.spmv_mhdc(port.to_hdc(rp, col, val, 0.6), x).tolist() == want


def _case(g, name):
    p = name + "/"
    return (g[p + "rp"], g[p + "col"], g[p + "val"], float(g[p + "theta"]), int(g[p + "bl"]), g[p + "x"])


def test_port_matches_reference_golden(port, golden):
    """Every stored reference output is reproduced bit for bit by the port."""
    for name in golden["names"]:
        rp, col, val, theta, bl, x = _case(golden, str(name))
        p = str(name) + "/"
        m = port.to_mhdc(rp, col, val, theta, bl)
        assert np.array_equal(m.dia_ptr, golden[p + "mhdc_dia_ptr"]), name
        assert np.array_equal(m.offsets, golden[p + "mhdc_offsets"]), name
        assert m.segments.tobytes() == golden[p + "mhdc_segments"].tobytes(), name
        assert np.array_equal(m.rest_rp, golden[p + "mhdc_rest_rp"]), name
        assert np.array_equal(m.rest_col, golden[p + "mhdc_rest_col"]), name
        assert m.rest_val.tobytes() == golden[p + "mhdc_rest_val"].tobytes(), name
        h = port.to_hdc(rp, col, val, theta)
        assert np.array_equal(h.offsets, golden[p + "hdc_offsets"]), name
        assert h.segments.tobytes() == golden[p + "hdc_segments"].tobytes(), name
        assert h.rest_val.tobytes() == golden[p + "hdc_rest_val"].tobytes(), name
        assert np.array_equal(h.rest_rp, golden[p + "hdc_rest_rp"]), name
        # kernels: every reference kernel has the same per-row order as one of these
        ym = port.spmv_mhdc(m, x)
        yh = port.spmv_mhdc(h, x)
        yc = port.spmv_csr(rp, col, val, x)
        assert ym.tobytes() == golden[p + "y_mhdc"].tobytes(), name
        assert yh.tobytes() == golden[p + "y_hdc"].tobytes(), name
        assert yh.tobytes() == golden[p + "y_bhdc"].tobytes(), name
        assert yc.tobytes() == golden[p + "y_csr"].tobytes(), name
        d = port.to_hdc(rp, col, val, 0.0)
        yd = port.spmv_mhdc(d, x)
        assert yd.tobytes() == golden[p + "y_dia"].tobytes(), name
        assert yd.tobytes() == golden[p + "y_bdia"].tobytes(), name
        bp, offs, cnt = port.census(rp, col, bl)
        assert np.array_equal(bp, golden[p + "census_bp"]), name
        assert np.array_equal(offs, golden[p + "census_off"]), name
        assert np.array_equal(cnt, golden[p + "census_cnt"]), name
        want_rates = golden[p + "mhdc_rates"]
        if np.isnan(want_rates[0]):
            with pytest.raises(ValueError):
                port.rates(m)
        else:
            assert port.rates(m) == (want_rates[0], want_rates[1], int(want_rates[2])), name


def test_cancel_fixture_order(golden):
    """cancel.mtx (proj/tests/data/cancel.mtx): hybrid order gives 4, CSR gives 3
    (proj/tests/cli_exit_codes.cmake:32-38)."""
    assert golden["cancel/y_csr"][0] == 3.0
    assert golden["cancel/y_hdc"][0] == 4.0
    assert golden["cancel/y_mhdc"][0] == 4.0


def test_port_vs_dense_oracle(port):
    """test_kernels.cpp:59-72: random matrices against the dense multiply, <= 1e-13."""
    rng = np.random.default_rng(123)
    for _ in range(10):
        n = int(rng.integers(8, 64))
        rp, col, val = synth.random_matrix(n, float(rng.uniform(0.02, 0.22)), rng)
        x = rng.uniform(0.5, 1.5, n)
        ref = dense_multiply(n, rp, col, val, x)
        theta = float(rng.uniform(0.1, 0.9))
        bl = int(rng.integers(1, n + 3))
        for y in (port.spmv_csr(rp, col, val, x), port.spmv_mhdc(port.to_mhdc(rp, col, val, theta, bl), x),
                  port.spmv_mhdc(port.to_hdc(rp, col, val, theta), x)):
            assert max_rel_err(y, ref) <= 1e-13


def test_port_threads_bit_invariant(port):
    rng = np.random.default_rng(31415)
    rp, col, val = synth.random_matrix(400, 0.05, rng)
    x = rng.uniform(0.5, 1.5, 400)
    m = port.to_mhdc(rp, col, val, 0.5, 7)
    y1 = port.spmv_mhdc(m, x, 1)
    for t in (2, 3, 0):
        assert port.spmv_mhdc(m, x, t).tobytes() == y1.tobytes()


@pytest.mark.skipif(not Ref.available(), reason="reference library not built here")
def test_port_matches_live_reference(port):
    R = Ref()
    rng = np.random.default_rng(7)
    for rep in range(60):
        n = int(rng.integers(2, 300))
        A = synth.random_matrix(n, float(rng.uniform(0.01, 0.3)), rng)
        theta = float(rng.uniform()) if rep % 5 else 0.0
        bl = int(rng.integers(1, n + 3))
        a, b = port.to_mhdc(*A, theta, bl), R.to_mhdc(*A, theta, bl)
        for f in a._fields:
            assert np.array_equal(getattr(a, f), getattr(b, f)), (rep, f)
        a, b = port.to_hdc(*A, theta), R.to_hdc(*A, theta)
        for f in a._fields:
            assert np.array_equal(getattr(a, f), getattr(b, f)), (rep, f)
        x = rng.uniform(-1, 1, n)
        assert port.spmv_mhdc(port.to_mhdc(*A, theta, bl), x).tobytes() == \
            R.spmv("mhdc", R.mhdc_handle(*A, theta, bl), x).tobytes()
    # the BASELINE generators at reduced size
    for A, bl in ((synth.laplacian7(16, 12, 10), 256), (synth.stencil27(10), 128),
                  (synth.quasi_diag(20000, 4, 200, 2000), 512)):
        a, b = port.to_mhdc(*A, 0.6, bl), R.to_mhdc(*A, 0.6, bl)
        for f in a._fields:
            assert np.array_equal(getattr(a, f), getattr(b, f)), f


# ---- generators ---------------------------------------------------------------

def test_laplacian_shape():
    rp, col, val = synth.laplacian7(64, 64, 64)
    assert rp[-1] == 1_810_432  # BASELINE config 0
    assert np.all(np.diff(rp) >= 4)
    i = np.repeat(np.arange(64 ** 3), np.diff(rp))
    assert set(np.unique(col - i).tolist()) == {-4096, -64, -1, 0, 1, 64, 4096}
    assert np.all(val[col == i] == 6.0) and np.all(val[col != i] == -1.0)


def test_laplacian_slabs_concatenate():
    full = synth.laplacian7(6, 5, 8)
    parts = [synth.laplacian7(6, 5, 8, z0, z1) for z0, z1 in ((0, 3), (3, 5), (5, 8))]
    col = np.concatenate([p[1] for p in parts])
    assert np.array_equal(col, full[1])
    rp = np.concatenate([parts[0][0][:-1], parts[1][0][:-1] + parts[0][0][-1],
                         parts[2][0] + parts[0][0][-1] + parts[1][0][-1]])
    assert np.array_equal(rp, full[0])


def test_stencil27_shape():
    g = 12
    rp, col, val = synth.stencil27(g)
    assert rp[-1] == (3 * g - 2) ** 3
    i = np.repeat(np.arange(g ** 3), np.diff(rp))
    off = val[col != i]
    assert np.all((off >= -1.0) & (off < 0.0))
    # diag = 1 + sum |off| (accumulated in column order)
    for r in (0, 5, 777, g ** 3 - 1):
        s = 0.0
        for k in range(rp[r], rp[r + 1]):
            if col[k] != r:
                s += abs(val[k])
        assert val[rp[r]:rp[r + 1]][col[rp[r]:rp[r + 1]] == r][0] == 1.0 + s


def test_quasi_diag_shape():
    n = 1 << 18
    rp, col, val = synth.quasi_diag(n, 4)
    i = np.repeat(np.arange(n), np.diff(rp))
    off = col.astype(np.int64) - i
    assert np.all(np.diff(col)[np.diff(i) == 0] > 0)  # strictly ascending per row
    assert np.all(val[off == 0] == 10.0)
    assert np.count_nonzero(off == 0) == n
    cand = np.isin(off, synth.QD_CANDIDATES)
    extras = ~cand & (off != 0)
    assert np.all(np.abs(off[extras]) < (1 << 16))
    assert np.count_nonzero(extras) == 6 * n
    assert 11.0 < rp[-1] / n < 12.5


def test_counter_rng_known_values():
    # splitmix64 of 0 is the published first output of the SplitMix64 reference sequence
    assert int(synth.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    x = synth.x_vector(1000, 5)
    assert np.all((x >= -1.0) & (x < 1.0)) and abs(x.mean()) < 0.1

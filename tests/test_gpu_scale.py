"""At-scale GPU parity: the BASELINE configurations at their full sizes, bit-exact
against digests of the UNMODIFIED reference's outputs (tests/golden/
scale_digests.json, made by tests/golden/make_scale_golden.py with oracle/_ref;
our C restatement agreed with every array when they were made).

* config 4 (n = 536,870,912; nnz = 3,753,902,080 > 2^31 through the int64 row
  pointer; 30 GB of segments indexed past 2^31 doubles): the whole matrix is
  generated and converted on one B200 exactly as bench.py does, one SpMV runs,
  and the first, a middle and the last 16-plane z-slab (both Dirichlet faces) are
  compared: dia_ptr, offsets, segments and y, SHA-256 of the device arrays.
* config 3 (n = 2^24, quasi-diagonal): M-HDC bl 1024 and 8192 and HDC, every
  format array and y, in every remainder mode.
* the power iteration (x <- y/||y||, fused norm and x scale): 100 steps on a
  reduced grid, y bitwise equal to the oracle's SpMV of the device's scaled
  iterate at EVERY step, and the final norm within 1e-12.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2105_04937_b200 import hdcgpu as H
from paper_2105_04937_b200 import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a GPU", allow_module_level=True)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale_digests.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def digest(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def test_config4_full_size_slabs(gold):
    g = gold["config4"]
    nx, ny, nz = g["grid"]
    bl = g["bl"]
    n, plane = nx * ny * nz, nx * ny
    H.init(0)
    nnz = H.gen_laplacian7_nnz(nx, ny, nz, 0, nz)
    assert nnz == 3_753_902_080 > 2 ** 31
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(nnz, dtype=torch.int32, device="cuda")
    val = torch.empty(nnz, dtype=torch.float64, device="cuda")
    H.gen_laplacian7(nx, ny, nz, 0, nz, rp.data_ptr(), col.data_ptr(), val.data_ptr())
    m = H.build_mhdc_device(n, n, 0, nnz, rp.data_ptr(), col.data_ptr(), val.data_ptr(), 0.6, bl,
                            rp64=True, validate=True)
    del rp, col, val
    torch.cuda.empty_cache()
    try:
        assert m.n_segments == 916_992 and m.info.nnz_rest == 0
        assert m.n_segments * bl > 2 ** 31  # segment indices past 2^31 doubles
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        H.gen_uniform_pm1(g["x_seed"], 0, 0, n, x.data_ptr())
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        H.spmv_device(m, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        for key, s in g["slabs"].items():
            e = m.export_blocks(s["block0"], s["block0"] + s["blocks"])
            assert e["dia_offsets"].size == s["n_seg"], key
            assert digest(e["dia_ptr"], "<i4") == s["dia_ptr"], key
            assert digest(e["dia_offsets"], "<i4") == s["dia_offsets"], key
            assert digest(e["segments"], "<f8") == s["segments"], key
            assert e["rest_col_ind"].size == 0 and not e["rest_row_ptr"].any(), key
            ys = y[s["row0"]:s["row0"] + s["rows"]].cpu().numpy()
            assert ys[:4].tolist() == s["y_head"], key
            assert digest(ys, "<f8") == s["y"], key
        # the same SpMV through the slab entry point with the fused norm and x
        # scale of the power iteration (scale 1.0): identical y
        y2 = torch.empty_like(y)
        one = torch.ones(1, dtype=torch.float64, device="cuda")
        tiles = torch.empty(m.info.n_tiles, dtype=torch.float64, device="cuda")
        H.spmv_slab(m, x.data_ptr(), y2.data_ptr(), 0, m.n_blocks, one.data_ptr(), tiles.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int64), y2.view(torch.int64))
        out = torch.empty(2, dtype=torch.float64, device="cuda")
        H.tree_sum(tiles.data_ptr(), tiles.numel(), out.data_ptr())
        torch.cuda.synchronize()
        ref = float(torch.dot(y, y))
        assert abs(out[0].item() - ref) <= 1e-12 * ref
    finally:
        m.free()
        torch.cuda.empty_cache()


def _c3_matrix():
    rp, col, val = synth.quasi_diag(1 << 24, seed=4)
    return H.CsrMatrix(len(rp) - 1, val, col, rp.astype(np.int32)), synth.x_vector(1 << 24, 4)


def test_config3_full_size(gold):
    g = gold["config3"]
    A, x = _c3_matrix()
    assert A.nnz == g["nnz"]
    for key in ("mhdc_bl1024", "mhdc_bl8192", "hdc"):
        d = g[key]
        m = H.to_mhdc(A, 0.6, int(key[7:])) if key != "hdc" else H.to_hdc(A, 0.6)
        e = m.export()
        for arr, dt in (("dia_ptr", "<i4"), ("dia_offsets", "<i4"), ("segments", "<f8"), ("rest_row_ptr", "<i4"),
                        ("rest_col_ind", "<i4"), ("rest_values", "<f8")):
            assert digest(e[arr], dt) == d[arr], (key, arr)
        assert list(H.rates(m)) == [d["rates"][0], d["rates"][1], d["rates"][2]], key
        try:
            for mode in (H.REST_DEFAULT, H.REST_GLOBAL, H.REST_SPLIT, H.REST_FUSED):
                H.set_kernel_policy(H.POLICY_AUTO, mode)
                y = H.spmv_mhdc(m, x)
                assert y[:4].tolist() == d["y_head"], (key, mode)
                assert digest(y, "<f8") == d["y"], (key, mode)
        finally:
            H.set_kernel_policy(H.POLICY_AUTO)
        m.free()


def test_power_iteration_100_steps(port):
    """Config 4's iteration on a 128x128x64 grid (bl = 4096): each step's y is bitwise
    the oracle's SpMV of the device's scaled previous iterate (x * s with s =
    1/||y|| from the device's deterministic tree), and the device's norms agree
    with numpy's within 1e-12 for all 100 steps."""
    nx, ny, nz, bl, steps = 128, 128, 64, 4096, 100
    n = nx * ny * nz
    rp, col, val = synth.laplacian7(nx, ny, nz)
    ref = port.to_mhdc(rp, col, val, 0.6, bl)
    m = H.to_mhdc(H.CsrMatrix(n, val, col, rp.astype(np.int32)), 0.6, bl)
    x0 = synth.x_vector(n, 5)
    nt = m.info.n_tiles
    bufs = [torch.from_numpy(x0).cuda(), torch.empty(n, dtype=torch.float64, device="cuda")]
    tiles = torch.empty(nt, dtype=torch.float64, device="cuda")
    red = torch.tensor([0.0, 1.0], dtype=torch.float64, device="cuda")
    x_prev, s_prev = x0, 1.0
    for k in range(steps):
        H.spmv_slab(m, bufs[0].data_ptr(), bufs[1].data_ptr(), 0, m.n_blocks, red.data_ptr() + 8, tiles.data_ptr())
        H.tree_sum(tiles.data_ptr(), nt, red.data_ptr())
        torch.cuda.synchronize()
        y = bufs[1].cpu().numpy()
        want = port.spmv_mhdc(ref, x_prev * s_prev)
        assert y.tobytes() == want.tobytes(), k
        s2, s = red.cpu().numpy()
        dot = float(np.dot(y, y))
        assert abs(s2 - dot) <= 1e-12 * dot, k
        assert s == 1.0 / np.sqrt(s2), k  # the kernel's own division
        x_prev, s_prev = y, s
        bufs.reverse()

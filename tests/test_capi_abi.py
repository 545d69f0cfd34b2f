"""The C-ABI library (no GPU needed): it loads, exports exactly what
include/hdcgpu.h declares, is built for sm_100a only, and refuses to compute
without a B200 (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2105_04937_b200 import hdcgpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hdcgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    decl = r"^(?:hdcg_status|int|const char\*)\s+(hdcg_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_header_lists_match_wrapper():
    assert declared_symbols() == sorted(hdcgpu.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = hdcgpu.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", hdcgpu.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hdcg_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert L.hdcg_version() >= 100


def test_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", hdcgpu.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is visible")
def test_no_cpu_fallback_without_device():
    """Every compute entry point fails loudly when no device is present."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rp, col, val = np.array([0, 1], np.int32), np.array([0], np.int32), np.array([2.0])
    m = hdcgpu.CsrMatrix(1, val, col, rp)
    with pytest.raises(hdcgpu.NoDeviceError):
        hdcgpu.to_mhdc(m, 0.6, 1)
    with pytest.raises(hdcgpu.NoDeviceError):
        hdcgpu.to_hdc(m, 0.6)
    with pytest.raises(hdcgpu.NoDeviceError):
        hdcgpu.init(0)


def test_host_side_validation():
    """Argument checks that mirror the reference before any device work."""
    with pytest.raises(ValueError):
        hdcgpu.CsrMatrix(-1, [], [], [0])
    with pytest.raises(ValueError):
        hdcgpu.CsrMatrix(2, [1.0], [0, 1], [0, 1, 2])
    with pytest.raises(ValueError):
        hdcgpu.BlockPlan.rows(4, 0)
    with pytest.raises(ValueError):
        hdcgpu.BlockPlan.rows(-1, 2)
    p = hdcgpu.BlockPlan.rows(10, 4)
    assert (p.n_blocks, p.begin(2), p.end(2), p.length(2)) == (3, 8, 10, 2)
    assert hdcgpu.BlockPlan.rows(0, 4).n_blocks == 0
    assert hdcgpu.BlockPlan.rows(3, 100).end(0) == 3


def test_host_spmv_rejects_unsafe_y():
    """The library writes 8*n bytes through y's pointer: float32, strided, read-only
    or wrong-length outputs are rejected before any device call (ValueError, like
    the reference's length check, kernels.cpp:21-24)."""
    class Fake:  # a matrix handle of 4 rows; never reaches the library
        n = 4
        handle = None

    x = np.ones(4)
    bad = [np.zeros(4, np.float32), np.zeros(8)[::2], np.zeros(5), np.zeros((2, 2)), [0.0] * 4]
    ro = np.zeros(4)
    ro.flags.writeable = False
    bad.append(ro)
    for y in bad:
        with pytest.raises(ValueError):
            hdcgpu._spmv_host(Fake(), x, y, "spmv_mhdc")
    with pytest.raises(ValueError):
        hdcgpu._spmv_host(Fake(), np.ones(3), None, "spmv_mhdc")

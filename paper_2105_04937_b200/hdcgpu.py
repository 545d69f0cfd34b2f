"""Python mirror of the reference's HDC / M-HDC interface over the C-ABI.

The reference is a C++ library (proj/include/hdc/*.hpp); its drop-in
replacement for C++ callers is the shim in shim/hdc_gpu_shim.cpp.  This module
is the same boundary for Python callers (tests, bench.py): names, argument
meaning and error behaviour follow the reference:

    reference (proj/include/hdc)            here
    ----------------------------------      --------------------------------
    CsrMatrix(n, values, col_ind, row_ptr)  CsrMatrix(n, values, col_ind, row_ptr)
    to_mhdc(m, theta, bl)  convert.hpp:39   to_mhdc(m, theta, bl)
    to_hdc(m, theta)       convert.hpp:34   to_hdc(m, theta)
    to_dia(m)              convert.hpp:31   to_dia(m)
    rates(h)               convert.hpp:45   rates(h)
    census_blocked/global  convert.hpp:26   census_blocked / census_global
    BlockPlan::rows        kernels.hpp:12   BlockPlan.rows
    spmv_{csr,dia,bdia,hdc,bhdc,mhdc}       same names, allocating form returns y
    std::invalid_argument / out_of_range /  ValueError / IndexError /
    overflow_error                          OverflowError

Every compute call goes through libhdcgpu.so (sm_100a).  There is no CPU
fallback: importing works anywhere, but any call without a B200 raises
NoDeviceError, and a missing library raises LibraryMissing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

# HDCG_LIBRARY: another in-tree build of the same library (same-box A/B of kernel versions)
_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhdcgpu.so")
LIB_PATH = os.environ.get("HDCG_LIBRARY") or _DEFAULT_LIB

HDCG_INPUT_DEVICE = 1
HDCG_VALIDATE = 2
HDCG_ROWPTR_I64 = 4

KIND_MHDC, KIND_HDC, KIND_CSR = 0, 1, 2

# every symbol include/hdcgpu.h declares (checked by tests/test_capi_abi.py)
EXPORTS = (
    "hdcg_last_error", "hdcg_version", "hdcg_init", "hdcg_build_mhdc", "hdcg_build_hdc",
    "hdcg_build_csr", "hdcg_upload_mhdc", "hdcg_upload_hdc", "hdcg_free", "hdcg_get_info",
    "hdcg_export", "hdcg_rates", "hdcg_census", "hdcg_spmv", "hdcg_spmv_host", "hdcg_spmv_slab",
    "hdcg_tree_sum", "hdcg_gen_uniform_pm1", "hdcg_gen_laplacian7", "hdcg_set_kernel_policy",
    "hdcg_membench", "hdcg_analyze", "hdcg_read_matrix_market", "hdcg_spmv_slab_halo",
    "hdcg_peer_alloc", "hdcg_peer_open", "hdcg_peer_close", "hdcg_peer_free", "hdcg_export_blocks",
)

POLICY_AUTO, POLICY_GENERAL, POLICY_TMA = 0, 1, 2
REST_DEFAULT, REST_GLOBAL, REST_SPLIT, REST_FUSED = 0, 1, 2, 3


class LibraryMissing(ImportError):
    pass


class NoDeviceError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class MatrixMarketError(RuntimeError):
    """std::runtime_error of hdc::io::read_matrix_market (proj/src/io.cpp)."""


_STATUS_EXC = {1: ValueError, 2: IndexError, 3: OverflowError, 4: CudaError, 5: NoDeviceError,
               6: MemoryError, 7: MatrixMarketError}


class Info(C.Structure):
    _fields_ = [("kind", C.c_int32), ("device", C.c_int32), ("n_rows", C.c_int64),
                ("n_cols", C.c_int64), ("row0", C.c_int64), ("bl", C.c_int64),
                ("n_blocks", C.c_int64), ("n_seg", C.c_int64), ("nnz_rest", C.c_int64),
                ("dia_slots", C.c_int64), ("nnz_input", C.c_int64), ("n_tiles", C.c_int64),
                ("tile_rows", C.c_int64), ("blocks_per_tile", C.c_int64),
                ("device_bytes", C.c_int64), ("max_seg_per_block", C.c_int64), ("packed_stages", C.c_int64),
                ("rest_rows_kernel", C.c_int64)]


_lib = None


def lib():
    """Load libhdcgpu.so (once).  Raises LibraryMissing when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(f"{LIB_PATH} not built: run `python -m paper_2105_04937_b200.build`")
    L = C.CDLL(LIB_PATH)
    i64, i32, f64, vp, u = C.c_int64, C.c_int32, C.c_double, C.c_void_p, C.c_uint
    L.hdcg_last_error.restype = C.c_char_p
    L.hdcg_version.restype = C.c_int
    sig = {
        "hdcg_init": [C.c_int],
        "hdcg_build_mhdc": [i64, i64, i64, i64, vp, vp, vp, f64, i64, u, vp, C.POINTER(vp)],
        "hdcg_build_hdc": [i64, i64, vp, vp, vp, f64, u, vp, C.POINTER(vp)],
        "hdcg_build_csr": [i64, i64, vp, vp, vp, u, vp, C.POINTER(vp)],
        "hdcg_upload_mhdc": [i64, i64, vp, i64, vp, vp, vp, i64, vp, vp, u, C.POINTER(vp)],
        "hdcg_upload_hdc": [i64, i64, vp, vp, vp, i64, vp, vp, u, C.POINTER(vp)],
        "hdcg_free": [vp],
        "hdcg_get_info": [vp, C.POINTER(Info)],
        "hdcg_export": [vp, vp, vp, vp, vp, vp, vp],
        "hdcg_export_blocks": [vp, i64, i64, vp, vp, vp, vp, vp, vp, vp],
        "hdcg_rates": [vp, C.POINTER(f64), C.POINTER(f64), C.POINTER(i64)],
        "hdcg_census": [i64, i64, vp, vp, i64, u, vp, vp, vp, C.POINTER(i64)],
        "hdcg_spmv": [vp, vp, vp, vp],
        "hdcg_spmv_host": [vp, vp, vp],
        "hdcg_spmv_slab": [vp, vp, vp, i64, i64, vp, vp, vp],
        "hdcg_spmv_slab_halo": [vp, vp, vp, i64, i64, vp, vp, vp, vp, i64, vp],
        "hdcg_peer_alloc": [i64, C.POINTER(vp), C.c_char_p],
        "hdcg_peer_open": [C.c_char_p, C.POINTER(vp)],
        "hdcg_peer_close": [vp],
        "hdcg_peer_free": [vp],
        "hdcg_tree_sum": [vp, i64, vp, vp],
        "hdcg_set_kernel_policy": [C.c_int],
        "hdcg_membench": [i64, C.c_int, C.c_int, C.c_int, C.POINTER(f64), C.POINTER(f64), vp],
        "hdcg_analyze": [i64, i64, vp, vp, vp, vp, C.c_int, vp, C.c_int, u, vp],
        "hdcg_read_matrix_market": [C.c_char_p, C.POINTER(vp)],
        "hdcg_gen_uniform_pm1": [C.c_uint64, C.c_uint64, i64, i64, vp, vp],
        "hdcg_gen_laplacian7": [i64, i64, i64, i64, i64, vp, vp, vp, C.POINTER(i64), vp],
    }
    for name, args in sig.items():
        if LIB_PATH != _DEFAULT_LIB and not hasattr(L, name):
            continue  # an older build loaded for an A/B (HDCG_LIBRARY): bind what it has
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def check(status: int):
    if status != 0:
        msg = lib().hdcg_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, RuntimeError)(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


# ---------------------------------------------------------------------------
# containers

class CsrMatrix:
    """Host CSR (formats.hpp:37-54).  Arrays are kept as given (int32 col_ind,
    int32 or int64 row_ptr); the reference constructor's checks are applied
    on the device when a format is built (HDCG_VALIDATE)."""

    def __init__(self, n, values, col_ind, row_ptr):
        self.n = int(n)
        if self.n < 0:
            raise ValueError("CsrMatrix: negative dimension")
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.col_ind = np.ascontiguousarray(col_ind, dtype=np.int32)
        rp = np.asarray(row_ptr)
        self.row_ptr = np.ascontiguousarray(rp, dtype=np.int64 if rp.dtype == np.int64 else np.int32)
        if self.values.size != self.col_ind.size:
            raise ValueError("CsrMatrix: values / col_ind length mismatch")
        if self.row_ptr.size != self.n + 1:
            raise ValueError("CsrMatrix: row_ptr must have n + 1 entries")

    @classmethod
    def from_arrays(cls, rp, col, val):
        return cls(len(rp) - 1, val, col, rp)

    @property
    def nnz(self):
        return int(self.values.size)

    def _flags(self):
        return HDCG_VALIDATE | (HDCG_ROWPTR_I64 if self.row_ptr.dtype == np.int64 else 0)


class HybridRates(NamedTuple):
    alpha: float
    beta: float
    dia_slots: int


class OffsetCount(NamedTuple):
    offset: int
    count: int


@dataclass
class DiagonalCensus:
    n: int
    bl: int
    n_blocks: int
    per_block: list

    def total(self):
        return sum(oc.count for b in self.per_block for oc in b)


class DeviceMatrix:
    """A device-resident, immutable format (hdcg_matrix handle)."""

    kind_name = "mhdc"

    def __init__(self, handle, theta=None):
        self._h = C.c_void_p(handle)
        self.theta = theta
        info = Info()
        check(lib().hdcg_get_info(self._h, C.byref(info)))
        self.info = info

    @property
    def handle(self):
        return self._h

    @property
    def n(self):
        return self.info.n_rows

    @property
    def bl(self):
        return self.info.bl

    @property
    def n_blocks(self):
        return self.info.n_blocks

    @property
    def n_segments(self):
        return self.info.n_seg

    def free(self):
        if self._h is not None and self._h.value:
            lib().hdcg_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def export(self):
        """Host copies: dict of dia_ptr, dia_offsets, segments, rest_row_ptr, rest_col_ind, rest_values."""
        i = self.info
        out = dict(
            dia_ptr=np.zeros(i.n_blocks + 1, np.int32),
            dia_offsets=np.zeros(i.n_seg, np.int32),
            segments=np.zeros(i.n_seg * i.bl, np.float64),
            rest_row_ptr=np.zeros(i.n_rows + 1, np.int32),
            rest_col_ind=np.zeros(i.nnz_rest, np.int32),
            rest_values=np.zeros(i.nnz_rest, np.float64),
        )
        check(lib().hdcg_export(self._h, *[_ptr(out[k]) for k in (
            "dia_ptr", "dia_offsets", "segments", "rest_row_ptr", "rest_col_ind", "rest_values")]))
        return out


    def export_blocks(self, b0, b1):
        """The format over row blocks [b0, b1) (hdcg_export_blocks): dia_ptr and the
        remainder row pointer rebased to 0, columns global."""
        i = self.info
        cnt = np.zeros(2, np.int64)
        check(lib().hdcg_export_blocks(self._h, b0, b1, None, None, None, None, None, None, _ptr(cnt)))
        rows = min(i.n_rows, b1 * i.bl) - min(i.n_rows, b0 * i.bl)
        out = dict(
            dia_ptr=np.zeros(b1 - b0 + 1, np.int32),
            dia_offsets=np.zeros(cnt[0], np.int32),
            segments=np.zeros(cnt[0] * i.bl, np.float64),
            rest_row_ptr=np.zeros(rows + 1, np.int32),
            rest_col_ind=np.zeros(cnt[1], np.int32),
            rest_values=np.zeros(cnt[1], np.float64),
        )
        check(lib().hdcg_export_blocks(self._h, b0, b1, *[_ptr(out[k]) for k in (
            "dia_ptr", "dia_offsets", "segments", "rest_row_ptr", "rest_col_ind", "rest_values")], None))
        return out


class MHdcMatrix(DeviceMatrix):
    kind_name = "mhdc"


class HdcMatrix(DeviceMatrix):
    kind_name = "hdc"

    @property
    def n_diags(self):
        return self.info.n_seg


class DeviceCsr(DeviceMatrix):
    kind_name = "csr"


class DiaMatrix(HdcMatrix):
    """to_dia result: HDC at theta = 0 (every populated diagonal is a lane, empty remainder)."""
    kind_name = "dia"


# ---------------------------------------------------------------------------
# converters (convert.hpp)

def _new_handle():
    return C.c_void_p()


def to_mhdc(m: CsrMatrix, theta: float, bl: int, validate=True) -> MHdcMatrix:
    h = _new_handle()
    flags = m._flags() if validate else (m._flags() & ~HDCG_VALIDATE)
    check(lib().hdcg_build_mhdc(m.n, m.n, 0, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), _ptr(m.values),
                                float(theta), int(bl), flags, None, C.byref(h)))
    return MHdcMatrix(h.value, theta)


def to_hdc(m: CsrMatrix, theta: float, validate=True) -> HdcMatrix:
    h = _new_handle()
    flags = m._flags() if validate else (m._flags() & ~HDCG_VALIDATE)
    check(lib().hdcg_build_hdc(m.n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), _ptr(m.values),
                               float(theta), flags, None, C.byref(h)))
    return HdcMatrix(h.value, theta)


def to_dia(m: CsrMatrix) -> DiaMatrix:
    h = _new_handle()
    check(lib().hdcg_build_hdc(m.n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), _ptr(m.values), 0.0,
                               m._flags(), None, C.byref(h)))
    return DiaMatrix(h.value, 0.0)


def device_csr(m: CsrMatrix) -> DeviceCsr:
    h = _new_handle()
    check(lib().hdcg_build_csr(m.n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), _ptr(m.values),
                               m._flags(), None, C.byref(h)))
    return DeviceCsr(h.value)


def read_matrix_market(path: str) -> DeviceCsr:
    """hdc::io::read_matrix_market + CsrMatrix::from_coo (io.cpp:69-121,
    formats.cpp:19-88): parsed on the host threads, normalised on the device;
    the result is a device-resident CSR (see csr_from_device for host arrays)."""
    h = _new_handle()
    check(lib().hdcg_read_matrix_market(os.fsencode(path), C.byref(h)))
    return DeviceCsr(h.value)


def csr_from_device(d: DeviceCsr) -> CsrMatrix:
    """Host copy of a device CSR (row_ptr int32, as index_t)."""
    e = d.export()
    return CsrMatrix(d.n, e["rest_values"], e["rest_col_ind"], e["rest_row_ptr"])


def rates(m: DeviceMatrix) -> HybridRates:
    a, b, s = C.c_double(), C.c_double(), C.c_int64()
    check(lib().hdcg_rates(m.handle, C.byref(a), C.byref(b), C.byref(s)))
    return HybridRates(a.value, b.value, s.value)


def _census(m: CsrMatrix, bl: int) -> DiagonalCensus:
    n = m.n
    tot = C.c_int64()
    nb = (1 if n > 0 else 0) if bl <= 0 else (0 if n == 0 else (n + bl - 1) // bl)
    bp = np.zeros(nb + 1, np.int64)
    flags = m._flags()
    check(lib().hdcg_census(n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), bl, flags, _ptr(bp), None,
                            None, C.byref(tot)))
    offs = np.zeros(tot.value, np.int32)
    cnt = np.zeros(tot.value, np.int64)
    check(lib().hdcg_census(n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), bl, flags, _ptr(bp), _ptr(offs),
                            _ptr(cnt), C.byref(tot)))
    per_block = [[OffsetCount(int(offs[k]), int(cnt[k])) for k in range(bp[b], bp[b + 1])]
                 for b in range(nb)]
    return DiagonalCensus(n, (n if bl <= 0 else bl), nb, per_block)


def census_blocked(m: CsrMatrix, bl: int) -> DiagonalCensus:
    if bl < 1:
        raise ValueError("census_blocked: block width must be >= 1")
    return _census(m, bl)


def census_global(m: CsrMatrix) -> DiagonalCensus:
    if m.n == 0:
        return DiagonalCensus(0, 0, 0, [])
    return _census(m, 0)


# ---------------------------------------------------------------------------
# kernels (kernels.hpp)

@dataclass
class BlockPlan:
    n: int
    bl: int
    n_blocks: int

    @staticmethod
    def rows(n: int, bl: int) -> "BlockPlan":
        """kernels.cpp:33-37"""
        if n < 0:
            raise ValueError("BlockPlan: negative row count")
        if bl < 1:
            raise ValueError("BlockPlan: block width must be >= 1")
        return BlockPlan(n, bl, 0 if n == 0 else (n + bl - 1) // bl)

    def begin(self, ib):
        return ib * self.bl

    def end(self, ib):
        return min((ib + 1) * self.bl, self.n)

    def length(self, ib):
        return self.end(ib) - self.begin(ib)


def _check_plan(plan: BlockPlan, n: int, what: str):
    """kernels.cpp:26-29"""
    if plan.n != n or plan.bl < 1 or plan.n_blocks != (0 if n == 0 else (n + plan.bl - 1) // plan.bl):
        raise ValueError(f"{what}: block plan does not match matrix")


def _spmv_host(m: DeviceMatrix, x, y, what):
    n = m.n
    x = np.ascontiguousarray(x, dtype=np.float64)
    if y is not None:
        # the library writes 8*n bytes through y's pointer: only a writeable,
        # C-contiguous float64 array of length n may be passed through
        if not isinstance(y, np.ndarray) or y.dtype != np.float64 or not y.flags.c_contiguous \
                or not y.flags.writeable or y.ndim != 1:
            raise ValueError(f"{what}: y must be a writeable, contiguous float64 vector of length n")
    if x.size != n or (y is not None and y.size != n):
        raise ValueError(f"{what}: x and y must have length n")
    out = np.empty(n, np.float64) if y is None else y
    if n:
        check(lib().hdcg_spmv_host(m.handle, _ptr(x), _ptr(out)))
    return out


def spmv_mhdc(m: MHdcMatrix, x, y=None, workers=0):
    return _spmv_host(m, x, y, "spmv_mhdc")


def spmv_hdc(m: HdcMatrix, x, y=None, workers=0):
    return _spmv_host(m, x, y, "spmv_hdc")


def spmv_bhdc(m: HdcMatrix, plan: BlockPlan, x, y=None, workers=0):
    _check_plan(plan, m.n, "spmv_bhdc")
    return _spmv_host(m, x, y, "spmv_bhdc")


def spmv_dia(m: DiaMatrix, x, y=None, workers=0):
    return _spmv_host(m, x, y, "spmv_dia")


def spmv_bdia(m: DiaMatrix, plan: BlockPlan, x, y=None, workers=0):
    _check_plan(plan, m.n, "spmv_bdia")
    return _spmv_host(m, x, y, "spmv_bdia")


def spmv_csr(m, x, y=None, workers=0):
    if isinstance(m, CsrMatrix):
        m = device_csr(m)
    return _spmv_host(m, x, y, "spmv_csr")


# ---------------------------------------------------------------------------
# device-pointer entry points (torch tensors / cupy-style integers)

def spmv_device(m: DeviceMatrix, x_ptr: int, y_ptr: int, stream: int = 0):
    check(lib().hdcg_spmv(m.handle, x_ptr, y_ptr, stream or None))


def spmv_slab(m: DeviceMatrix, x_local_ptr: int, y_ptr: int, block_begin: int, block_end: int,
              x_scale_ptr: int = 0, tile_sumsq_ptr: int = 0, stream: int = 0):
    check(lib().hdcg_spmv_slab(m.handle, x_local_ptr, y_ptr, block_begin, block_end,
                               x_scale_ptr or None, tile_sumsq_ptr or None, stream or None))


def spmv_slab_halo(m: DeviceMatrix, x_local_ptr: int, y_ptr: int, block_begin: int, block_end: int,
                   x_scale_ptr: int, tile_sumsq_ptr: int, peer_lo_ptr: int, peer_hi_ptr: int, halo: int,
                   stream: int = 0):
    """spmv_slab that also stores the slab's first/last `halo` rows into the
    neighbours' halo buffers (peer memory) from the kernel epilogue."""
    check(lib().hdcg_spmv_slab_halo(m.handle, x_local_ptr, y_ptr, block_begin, block_end, x_scale_ptr or None,
                                    tile_sumsq_ptr or None, peer_lo_ptr or None, peer_hi_ptr or None, halo,
                                    stream or None))


class PeerBuffer:
    """A float64 device buffer another process can map (CUDA IPC through
    hdcg_peer_alloc); exposes __cuda_array_interface__, so torch.as_tensor(buf,
    device="cuda") views it without a copy."""

    def __init__(self, count: int):
        self.count = count
        p = C.c_void_p()
        h = C.create_string_buffer(64)
        check(lib().hdcg_peer_alloc(8 * max(1, count), C.byref(p), h))
        self.ptr, self.handle = p.value, h.raw
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (self.ptr, False),
                                         "version": 3, "strides": None}

    def free(self):
        if self.ptr:
            check(lib().hdcg_peer_free(self.ptr))
            self.ptr = None


def peer_open(handle: bytes) -> int:
    """Map a PeerBuffer of another process; returns the device address."""
    p = C.c_void_p()
    check(lib().hdcg_peer_open(handle, C.byref(p)))
    return p.value


def peer_close(ptr: int):
    check(lib().hdcg_peer_close(ptr))


def tree_sum(vals_ptr: int, count: int, out_ptr: int, stream: int = 0):
    check(lib().hdcg_tree_sum(vals_ptr or None, count, out_ptr, stream or None))


def build_mhdc_device(n_rows, n_cols, row0, nnz, rp_ptr, col_ptr, val_ptr, theta, bl, rp64=True,
                      validate=False, stream=0) -> MHdcMatrix:
    h = _new_handle()
    flags = HDCG_INPUT_DEVICE | (HDCG_ROWPTR_I64 if rp64 else 0) | (HDCG_VALIDATE if validate else 0)
    check(lib().hdcg_build_mhdc(n_rows, n_cols, row0, nnz, rp_ptr, col_ptr, val_ptr, float(theta),
                                int(bl), flags, stream or None, C.byref(h)))
    return MHdcMatrix(h.value, theta)


def build_hdc_device(n, nnz, rp_ptr, col_ptr, val_ptr, theta, rp64=True, validate=False, stream=0) -> "HdcMatrix":
    """to_hdc from device-resident CSR arrays (the device twin of to_hdc)."""
    h = _new_handle()
    flags = HDCG_INPUT_DEVICE | (HDCG_ROWPTR_I64 if rp64 else 0) | (HDCG_VALIDATE if validate else 0)
    check(lib().hdcg_build_hdc(n, nnz, rp_ptr, col_ptr, val_ptr, float(theta), flags, stream or None, C.byref(h)))
    return HdcMatrix(h.value, theta)


def gen_uniform_pm1(seed: int, rng_stream: int, first: int, count: int, out_ptr: int, stream=0):
    check(lib().hdcg_gen_uniform_pm1(seed, rng_stream, first, count, out_ptr, stream or None))


def gen_laplacian7_nnz(nx, ny, nz, z0, z1) -> int:
    nnz = C.c_int64()
    check(lib().hdcg_gen_laplacian7(nx, ny, nz, z0, z1, None, None, None, C.byref(nnz), None))
    return nnz.value


def gen_laplacian7(nx, ny, nz, z0, z1, rp_ptr, col_ptr, val_ptr, stream=0):
    nnz = C.c_int64()
    check(lib().hdcg_gen_laplacian7(nx, ny, nz, z0, z1, rp_ptr, col_ptr, val_ptr, C.byref(nnz),
                                    stream or None))
    return nnz.value


def spmv_kernels(info: Info, scale: bool = False, norm: bool = False) -> list:
    """The kernels one SpMV call launches for a matrix under the default policy
    (mirrors spmv.cu::tiling_of and spmv_tma.cu::spmv_tma_launch)."""
    r = info.tile_rows // 256
    b = lambda v: str(v).lower()  # noqa: E731
    if info.packed_stages > 0:  # tile-packed small blocks (pack.cu)
        rest = 0 if info.nnz_rest == 0 else (3 if info.nnz_rest * 4 >= info.n_rows else 1)
        if rest == 3 and info.rest_rows_kernel:  # banded heavy remainder: summed first (spmv_rows.cu)
            return ["hdcg::rest_rows_kernel", f"hdcg::spmv_tma_kernel<4,{b(scale)},{b(norm)},2,5>"]
        return [f"hdcg::spmv_tma_kernel<4,{b(scale)},{b(norm)},{rest},5>"]
    inside = info.bl >= info.tile_rows  # tiles inside one block, else whole blocks per tile
    mb = not inside and r == 4 and info.bl % 128 == 0
    blk = not inside and r == 1 and 8 <= info.bl < 256 and info.max_seg_per_block <= 16
    if not ((info.bl >= 256 and inside) or mb or blk):
        return [f"hdcg::spmv_kernel<{r},{b(scale)},{b(norm)}>"]
    rest = 0 if info.nnz_rest == 0 else (2 if info.nnz_rest * 4 >= info.n_rows else 1)
    if rest == 2 and info.n_seg > 0 and not blk and info.kind == KIND_MHDC and not info.rest_rows_kernel:
        rest = 3  # gather warps inside the segment kernel (scattered columns)
    # remainder sums first: banded rows take the row-per-lane kernel with a TMA-staged
    # entry ring (spmv_rows.cu; info.rest_rows_kernel, decided from a sample of the
    # rows at build time), scattered columns the entry-major rest_pipe_kernel
    ks = [("hdcg::rest_rows_kernel" if info.rest_rows_kernel else "hdcg::rest_pipe_kernel")] if rest == 2 else []
    if rest == 2 and info.n_seg == 0 and not norm:
        return ks  # a CSR: the remainder kernel's sums are y
    if blk:
        return ks + [f"hdcg::spmv_blk_kernel<{b(scale)},{b(norm)},{rest}>"]
    # tile layout: inside one block (0) / multi-block (1; without a remainder 3 = bl 256, 4 = bl 128) / odd bl (2)
    lay = ({256: 3, 128: 4}.get(info.bl, 1) if info.nnz_rest == 0 else 1) if mb else (2 if info.bl % 2 else 0)
    ks.append(f"hdcg::spmv_tma_kernel<{r},{b(scale)},{b(norm)},{rest},{lay}>")
    return ks


def init(device: int = 0):
    check(lib().hdcg_init(device))


class AnalyzeRow(NamedTuple):
    """One line of `hdcmv analyze` (proj/tools/hdcmv.cpp:105-133)."""
    kernel: str      # "hdc" or "mhdc"
    theta: float
    bl: int          # 0 for hdc
    n_diag: int      # HdcMatrix::dia().n_diags() / MHdcMatrix::n_segments()
    alpha: float     # NaN where rates() throws (no nonzeros)
    beta: float
    dia_slots: int


def analyze(m: CsrMatrix, thetas, bls) -> list:
    """The (theta, bl) sweep of `hdcmv analyze` (hdcmv.cpp:93-140): for each theta
    the HDC split, then the M-HDC split for each bl -- rates computed from one
    device census per block width (no format is built)."""
    thetas = np.ascontiguousarray(thetas, dtype=np.float64)
    bls = np.ascontiguousarray(bls, dtype=np.int64)
    nt, nb = thetas.size, bls.size
    out = np.zeros(nt * (1 + nb) * 4, np.float64)
    check(lib().hdcg_analyze(m.n, m.nnz, _ptr(m.row_ptr), _ptr(m.col_ind), _ptr(m.values), _ptr(thetas), nt,
                             _ptr(bls), nb, m._flags(), _ptr(out)))
    out = out.reshape(nt, 1 + nb, 4)
    rows = []
    for t in range(nt):
        for j in range(1 + nb):
            a, b, slots, nd = out[t, j]
            rows.append(AnalyzeRow("hdc" if j == 0 else "mhdc", float(thetas[t]), 0 if j == 0 else int(bls[j - 1]),
                                   int(nd), float(a), float(b), int(slots)))
    return rows


class Measurement(NamedTuple):
    """hdc::bench::Measurement (proj/include/hdc/bench.hpp:18-23)."""
    best_time_s: float
    loop_times_s: list
    bytes_per_s: float


MEM_BYTES_DIRECT = 32.0    # bench.hpp:40
MEM_BYTES_INDIRECT = 36.0  # bench.hpp:41


def membench(n: int, mode: str = "direct", n_loops: int = 20, n_ites: int = 1000) -> Measurement:
    """hdc::bench::membench on the device (bench.cpp:68-110): c[i] += a[i]*b[i]
    (direct) or a[i]*b[idx[i]] (indirect); best per-call average of n_loops
    loops of n_ites calls after one warm-up loop."""
    modes = {"direct": 0, "indirect": 1}
    if mode not in modes:
        raise ValueError(f"unknown memory mode: {mode}")
    best, bps = C.c_double(), C.c_double()
    loops = np.zeros(max(n_loops, 1), np.float64)
    check(lib().hdcg_membench(n, modes[mode], n_loops, n_ites, C.byref(best), C.byref(bps), _ptr(loops)))
    return Measurement(best.value, loops.tolist(), bps.value)


def set_kernel_policy(policy: int, rest_mode: int = 0):
    """policy: 0 auto (TMA kernel where eligible), 1 general kernel only, 2 TMA kernel only.
    rest_mode (TMA kernel's CSR remainder): 0 default, 1 global loads, 2 summed first
    by a separate kernel, 3 summed by gather warps of the same kernel (shared memory)."""
    check(lib().hdcg_set_kernel_policy(policy + 16 * rest_mode))

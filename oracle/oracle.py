"""Python handle on the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module (see oracle/hdc_oracle.c).

* ``Port``: our C restatement (oracle/liboracle.so, built from hdc_oracle.c).
* ``Ref``:  the unmodified reference library (oracle/_ref/libhdcref.so, built
  by oracle/Makefile from /root/reference/proj/src in place).  Present in
  this container and, as a prebuilt file, on the GPU box.

Both expose the same numpy-level API; matrices are ``Mhdc`` tuples (HDC is
the bl = n special case: one block, lanes of length n).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import NamedTuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhdcref.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class Mhdc(NamedTuple):
    n: int
    bl: int
    dia_ptr: np.ndarray      # int64[n_blocks+1]
    offsets: np.ndarray      # int32[n_seg]
    segments: np.ndarray     # float64[n_seg*bl]
    rest_rp: np.ndarray      # int64[n+1]
    rest_col: np.ndarray     # int32[nnz_rest]
    rest_val: np.ndarray     # float64[nnz_rest]

    @property
    def n_blocks(self):
        return self.dia_ptr.size - 1

    @property
    def n_seg(self):
        return self.offsets.size


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _empty_i64(k):
    return np.zeros(max(k, 0), dtype=np.int64)


class OracleError(RuntimeError):
    pass


def dense_multiply(n, rp, col, val, x):
    """proj/tests/oracles.hpp:16-24: dense row sums in column order."""
    a = np.zeros((n, n))
    for i in range(n):
        a[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    y = np.zeros(n)
    for i in range(n):
        s = 0.0
        for j in range(n):
            s += a[i, j] * x[j]
        y[i] = s
    return y


def max_rel_err(a, b):
    """proj/tests/oracles.hpp:27-35."""
    a = np.asarray(a); b = np.asarray(b)
    scale = np.maximum(np.abs(a), np.abs(b))
    m = scale != 0
    if not m.any():
        return 0.0
    return float(np.max(np.abs(a[m] - b[m]) / scale[m]))


def row_abs_norm(rp, col, val, x):
    """sum_j |a_ij x_j| per row: the BASELINE.json tolerance denominator."""
    prod = np.abs(val * x[col])
    out = np.zeros(rp.size - 1)
    nz = np.diff(rp) > 0
    sums = np.add.reduceat(prod, rp[:-1][nz]) if prod.size else np.zeros(0)
    out[nz] = sums
    return out


class Port:
    """Our C restatement (hdc_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle liboracle.so`")
        L = self.lib = C.CDLL(path)
        L.orc_census_count.restype = C.c_int64
        L.orc_census_count.argtypes = [C.c_int64, _i64p, _i32p, C.c_int64, _i64p]
        L.orc_census_fill.argtypes = [C.c_int64, _i64p, _i32p, C.c_int64, _i64p, _i32p, _i64p]
        L.orc_mhdc_plan.restype = C.c_int64
        L.orc_mhdc_plan.argtypes = [C.c_int64, _i64p, _i32p, C.c_double, C.c_int64, _i64p,
                                    C.POINTER(C.c_int64)]
        L.orc_mhdc_fill.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.c_double, C.c_int64, _i64p,
                                    _i32p, _f64p, _i64p, _i32p, _f64p]
        L.orc_rates.restype = C.c_int
        L.orc_rates.argtypes = [C.c_int64, C.c_int64, _i64p, _f64p, C.c_int64,
                                C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.orc_spmv_mhdc.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p,
                                    _f64p, _f64p, C.c_int]
        L.orc_spmv_csr.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p, C.c_int]
        L.orc_max_threads.restype = C.c_int

    def max_threads(self):
        return self.lib.orc_max_threads()

    def census(self, rp, col, bl):
        rp, col = _c(rp, np.int64), _c(col, np.int32)
        n = rp.size - 1
        nb = 0 if n == 0 else (n + bl - 1) // bl
        bp = np.zeros(nb + 1, dtype=np.int64)
        tot = self.lib.orc_census_count(n, rp, col, bl, bp)
        offs = np.zeros(tot, dtype=np.int32)
        cnt = np.zeros(tot, dtype=np.int64)
        self.lib.orc_census_fill(n, rp, col, bl, bp, offs, cnt)
        return bp, offs, cnt

    def to_mhdc(self, rp, col, val, theta, bl) -> Mhdc:
        if not (0.0 <= theta <= 1.0):
            raise ValueError("to_mhdc: theta must be in [0, 1]")
        if bl < 1:
            raise ValueError("to_mhdc: block width must be >= 1")
        rp, col, val = _c(rp, np.int64), _c(col, np.int32), _c(val, np.float64)
        n = rp.size - 1
        nb = 0 if n == 0 else (n + bl - 1) // bl
        dp = np.zeros(nb + 1, dtype=np.int64)
        nr = C.c_int64(0)
        nseg = self.lib.orc_mhdc_plan(n, rp, col, theta, bl, dp, C.byref(nr))
        offs = np.zeros(nseg, dtype=np.int32)
        segs = np.zeros(nseg * bl, dtype=np.float64)
        rrp = np.zeros(n + 1, dtype=np.int64)
        rcol = np.zeros(nr.value, dtype=np.int32)
        rval = np.zeros(nr.value, dtype=np.float64)
        self.lib.orc_mhdc_fill(n, rp, col, val, theta, bl, dp, offs, segs, rrp, rcol, rval)
        return Mhdc(n, bl, dp, offs, segs, rrp, rcol, rval)

    def to_hdc(self, rp, col, val, theta) -> Mhdc:
        """convert.cpp:89-121 == to_mhdc with one block of width n."""
        n = len(rp) - 1
        if n == 0:
            if not (0.0 <= theta <= 1.0):
                raise ValueError("to_hdc: theta must be in [0, 1]")
            z = np.zeros(0)
            return Mhdc(0, 1, np.zeros(1, np.int64), np.zeros(0, np.int32), z,
                        np.zeros(1, np.int64), np.zeros(0, np.int32), z)
        return self.to_mhdc(rp, col, val, theta, n)

    def rates(self, m: Mhdc):
        a, b, s = C.c_double(), C.c_double(), C.c_int64()
        rc = self.lib.orc_rates(m.n, m.bl, _c(m.dia_ptr, np.int64), _c(m.segments, np.float64),
                                m.rest_col.size, C.byref(a), C.byref(b), C.byref(s))
        if rc != 0:
            raise ValueError("rates: matrix has no nonzeros")
        return a.value, b.value, s.value

    def spmv_mhdc(self, m: Mhdc, x, nthreads=1, out=None):
        y = np.empty(m.n, dtype=np.float64) if out is None else out
        self.lib.orc_spmv_mhdc(m.n, m.bl, _c(m.dia_ptr, np.int64), _c(m.offsets, np.int32),
                               _c(m.segments, np.float64), _c(m.rest_rp, np.int64),
                               _c(m.rest_col, np.int32), _c(m.rest_val, np.float64),
                               _c(x, np.float64), y, nthreads)
        return y

    def spmv_csr(self, rp, col, val, x, nthreads=1):
        n = len(rp) - 1
        y = np.empty(n, dtype=np.float64)
        self.lib.orc_spmv_csr(n, _c(rp, np.int64), _c(col, np.int32), _c(val, np.float64),
                              _c(x, np.float64), y, nthreads)
        return y


class Ref:
    """The unmodified reference library (oracle/_ref/libhdcref.so via ref_capi.cpp)."""

    KIND = {"csr": 0, "hdc": 1, "bhdc": 2, "mhdc": 3, "dia": 4, "bdia": 5}

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.refc_last_error.restype = C.c_char_p
        L.refc_max_threads.restype = C.c_int
        L.refc_csr_new.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.POINTER(vp)]
        L.refc_csr_free.argtypes = [vp]
        L.refc_example_matrix.argtypes = [C.POINTER(vp)]
        L.refc_csr_sizes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.refc_csr_export.argtypes = [vp, _i64p, _i32p, _f64p]
        L.refc_census.argtypes = [vp, C.c_int64, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                  vp, vp, vp]
        L.refc_to_mhdc.argtypes = [vp, C.c_double, C.c_int64, C.POINTER(vp)]
        L.refc_mhdc_free.argtypes = [vp]
        L.refc_mhdc_sizes.argtypes = [vp] + [C.POINTER(C.c_int64)] * 5
        L.refc_mhdc_export.argtypes = [vp, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p]
        L.refc_to_hdc.argtypes = [vp, C.c_double, C.POINTER(vp)]
        L.refc_hdc_free.argtypes = [vp]
        L.refc_hdc_sizes.argtypes = [vp] + [C.POINTER(C.c_int64)] * 3
        L.refc_hdc_export.argtypes = [vp, _i32p, _f64p, _i64p, _i32p, _f64p]
        L.refc_rates_mhdc.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64)]
        L.refc_rates_hdc.argtypes = L.refc_rates_mhdc.argtypes
        L.refc_spmv.argtypes = [C.c_int, vp, C.c_int64, _f64p, _f64p, C.c_int64, C.c_int]
        L.refc_time_spmv.argtypes = [C.c_int, vp, C.c_int64, _f64p, _f64p, C.c_int64, C.c_int,
                                     C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.refc_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.refc_membench.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.refc_last_error().decode()
            exc = {-1: ValueError, -2: IndexError, -3: OverflowError}.get(rc, RuntimeError)
            raise exc(msg)

    def max_threads(self):
        return self.lib.refc_max_threads()

    # -- handles ------------------------------------------------------------
    class _Handle:
        def __init__(self, ref, h, free, kind, n, bl=0):
            self.ref, self.h, self._free, self.kind, self.n, self.bl = ref, h, free, kind, n, bl

        def __del__(self):
            if self.h:
                self._free(self.h)
                self.h = None

    def csr(self, rp, col, val):
        h = C.c_void_p()
        self._check(self.lib.refc_csr_new(len(rp) - 1, _c(rp, np.int64), _c(col, np.int32),
                                          _c(val, np.float64), C.byref(h)))
        return Ref._Handle(self, h.value, self.lib.refc_csr_free, "csr", len(rp) - 1)

    def example_matrix(self):
        h = C.c_void_p()
        self._check(self.lib.refc_example_matrix(C.byref(h)))
        n, nnz = C.c_int64(), C.c_int64()
        self.lib.refc_csr_sizes(h, C.byref(n), C.byref(nnz))
        rp = np.zeros(n.value + 1, np.int64)
        col = np.zeros(nnz.value, np.int32)
        val = np.zeros(nnz.value)
        self.lib.refc_csr_export(h, rp, col, val)
        self.lib.refc_csr_free(h)
        return rp, col, val

    def read_matrix_market(self, path):
        """io.cpp:69-121 + CsrMatrix::from_coo -> (rp, col, val) host arrays."""
        h = C.c_void_p()
        self._check(self.lib.refc_read_matrix_market(os.fsencode(path), C.byref(h)))
        n, nnz = C.c_int64(), C.c_int64()
        self.lib.refc_csr_sizes(h, C.byref(n), C.byref(nnz))
        rp = np.zeros(n.value + 1, np.int64)
        col = np.zeros(nnz.value, np.int32)
        val = np.zeros(nnz.value)
        self.lib.refc_csr_export(h, rp, col, val)
        self.lib.refc_csr_free(h)
        return rp, col, val

    def census(self, rp, col, val, bl, global_=False):
        c = self.csr(rp, col, val)
        nb, tot = C.c_int64(), C.c_int64()
        self._check(self.lib.refc_census(c.h, bl, int(global_), C.byref(nb), C.byref(tot),
                                         None, None, None))
        bp = np.zeros(nb.value + 1, np.int64)
        offs = np.zeros(tot.value, np.int32)
        cnt = np.zeros(tot.value, np.int64)
        self._check(self.lib.refc_census(c.h, bl, int(global_), C.byref(nb), C.byref(tot),
                                         bp.ctypes.data, offs.ctypes.data, cnt.ctypes.data))
        return bp, offs, cnt

    def mhdc_handle(self, rp, col, val, theta, bl):
        c = self.csr(rp, col, val)
        h = C.c_void_p()
        self._check(self.lib.refc_to_mhdc(c.h, theta, bl, C.byref(h)))
        return Ref._Handle(self, h.value, self.lib.refc_mhdc_free, "mhdc", len(rp) - 1, bl)

    def hdc_handle(self, rp, col, val, theta):
        c = self.csr(rp, col, val)
        h = C.c_void_p()
        self._check(self.lib.refc_to_hdc(c.h, theta, C.byref(h)))
        return Ref._Handle(self, h.value, self.lib.refc_hdc_free, "hdc", len(rp) - 1)

    def export_mhdc(self, hd) -> Mhdc:
        s = [C.c_int64() for _ in range(5)]
        self.lib.refc_mhdc_sizes(hd.h, *[C.byref(v) for v in s])
        n, bl, nb, nseg, nr = (v.value for v in s)
        dp = np.zeros(nb + 1, np.int64)
        offs = np.zeros(nseg, np.int32)
        segs = np.zeros(nseg * bl)
        rrp = np.zeros(n + 1, np.int64)
        rcol = np.zeros(nr, np.int32)
        rval = np.zeros(nr)
        self.lib.refc_mhdc_export(hd.h, dp, offs, segs, rrp, rcol, rval)
        return Mhdc(n, bl, dp, offs, segs, rrp, rcol, rval)

    def export_hdc(self, hd) -> Mhdc:
        s = [C.c_int64() for _ in range(3)]
        self.lib.refc_hdc_sizes(hd.h, *[C.byref(v) for v in s])
        n, nd, nr = (v.value for v in s)
        offs = np.zeros(nd, np.int32)
        lanes = np.zeros(nd * n)
        rrp = np.zeros(n + 1, np.int64)
        rcol = np.zeros(nr, np.int32)
        rval = np.zeros(nr)
        self.lib.refc_hdc_export(hd.h, offs, lanes, rrp, rcol, rval)
        dp = np.array([0, nd] if n > 0 else [0], np.int64)
        return Mhdc(n, max(n, 1), dp, offs, lanes, rrp, rcol, rval)

    def to_mhdc(self, rp, col, val, theta, bl) -> Mhdc:
        return self.export_mhdc(self.mhdc_handle(rp, col, val, theta, bl))

    def to_hdc(self, rp, col, val, theta) -> Mhdc:
        return self.export_hdc(self.hdc_handle(rp, col, val, theta))

    def rates(self, hd):
        a, b, s = C.c_double(), C.c_double(), C.c_int64()
        f = self.lib.refc_rates_mhdc if hd.kind == "mhdc" else self.lib.refc_rates_hdc
        self._check(f(hd.h, C.byref(a), C.byref(b), C.byref(s)))
        return a.value, b.value, s.value

    def spmv(self, kernel, hd, x, bl=0, workers=0, out=None):
        y = np.empty(hd.n, dtype=np.float64) if out is None else out
        self._check(self.lib.refc_spmv(self.KIND[kernel], hd.h, bl, _c(x, np.float64), y, hd.n,
                                       workers))
        return y

    def membench(self, n, mode="direct", n_loops=3, n_ites=5, workers=0):
        """The reference's host membench (bench.cpp:68-110): (bytes_per_s, best_time_s)."""
        bps, best = C.c_double(), C.c_double()
        self._check(self.lib.refc_membench(n, 0 if mode == "direct" else 1, n_loops, n_ites, workers,
                                           C.byref(bps), C.byref(best)))
        return bps.value, best.value

    def time_spmv(self, kernel, hd, x, bl=0, workers=0, n_loops=5, n_ites=10):
        y = np.empty(hd.n, dtype=np.float64)
        best = C.c_double()
        self._check(self.lib.refc_time_spmv(self.KIND[kernel], hd.h, bl, _c(x, np.float64), y, hd.n,
                                            workers, n_loops, n_ites, C.byref(best)))
        return best.value, y

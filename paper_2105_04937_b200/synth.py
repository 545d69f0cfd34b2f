"""Seeded synthetic inputs for the BASELINE.json configurations (host, numpy).

No dataset is involved: BASELINE.json names only synthetic matrices, and the
reference's own stencil generator (proj/src/stencil.cpp:88-118) is *not* the
BASELINE Laplacian (it clips offsets without Dirichlet omission and uses the
values 1+((31i+17j) mod 7)), so the configurations are generated here.

Random numbers come from a counter-based generator so host (numpy) and device
(csrc/gen.cu) produce identical bits in any order:

    key(seed, stream) = splitmix64(seed*0x9E3779B97F4A7C15 + stream*0xD1B54A32D192ED03)
    u(seed, stream, i) = (splitmix64(key + i) >> 11) * 2**-53        in [0, 1)
    uniform[-1, 1]      = 2*u - 1          (exact in fp64)
    uniform[-1, 0)      = u - 1            (exact in fp64)

Every CSR returned here is (row_ptr int64[n+1], col_ind int32[nnz],
values float64[nnz]) with strictly ascending columns per row, i.e. it
satisfies the reference CsrMatrix invariants (proj/src/formats.cpp:45-67).
"""
from __future__ import annotations

import numpy as np

PHI = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = float(2.0 ** -53)


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + PHI
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.array([seed], dtype=np.uint64) * PHI + np.array([stream], dtype=np.uint64) * STREAM_MUL
    return splitmix64(z)[0]


def u01(seed: int, stream: int, idx) -> np.ndarray:
    """u(seed, stream, idx) in [0,1), vectorised over idx (int64/uint64 array)."""
    key = stream_key(seed, stream)
    with np.errstate(over="ignore"):
        z = np.asarray(idx).astype(np.uint64) + key
    return (splitmix64(z) >> np.uint64(11)).astype(np.float64) * _TWO_M53


def uniform_pm1(seed: int, stream: int, idx) -> np.ndarray:
    return 2.0 * u01(seed, stream, idx) - 1.0


def x_vector(n: int, seed: int) -> np.ndarray:
    """x_i = uniform[-1,1] from `seed`, stream 0 (BASELINE.json configs 'x ... from seed s')."""
    return uniform_pm1(seed, 0, np.arange(n, dtype=np.int64))


# ---------------------------------------------------------------------------
# helpers

def _csr_from_slots(cols: np.ndarray, vals: np.ndarray, present: np.ndarray):
    """cols/vals/present are [n, w] with slots already in ascending column order."""
    counts = present.sum(axis=1, dtype=np.int64)
    rp = np.zeros(cols.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return rp, cols[present].astype(np.int32), vals[present].astype(np.float64)


# ---------------------------------------------------------------------------
# configs 0, 1, 4: 7-point Laplacian with Dirichlet boundary

def laplacian7_offsets(nx: int, ny: int, nz: int):
    p = nx * ny
    return [-p, -nx, -1, 0, 1, nx, p]


def laplacian7(nx: int, ny: int, nz: int, z0: int = 0, z1: int | None = None):
    """7-point 3D Laplacian, rows of z-planes [z0, z1): diag 6.0, -1.0 at +-1, +-nx,
    +-nx*ny where the neighbour exists (couplings across the boundary omitted).
    Columns are global.  Row index i = x + nx*(y + ny*z)."""
    z1 = nz if z1 is None else z1
    p = nx * ny
    i = np.arange(z0 * p, z1 * p, dtype=np.int64)
    xx = i % nx
    yy = (i // nx) % ny
    zz = i // p
    dx = [(-p, zz > 0), (-nx, yy > 0), (-1, xx > 0), (0, None), (1, xx < nx - 1),
          (nx, yy < ny - 1), (p, zz < nz - 1)]
    n_loc = i.size
    cols = np.empty((n_loc, 7), dtype=np.int64)
    vals = np.empty((n_loc, 7), dtype=np.float64)
    present = np.empty((n_loc, 7), dtype=bool)
    for t, (off, mask) in enumerate(dx):
        cols[:, t] = i + off
        vals[:, t] = 6.0 if off == 0 else -1.0
        present[:, t] = True if mask is None else mask
    return _csr_from_slots(cols, vals, present)


def laplacian7_slab_square(nx: int, ny: int, nz: int, z0: int, z1: int):
    """The rows of z-planes [z0, z1) of the 7-point Laplacian with everything they
    read, as a SQUARE matrix over the planes [z0-1, z1+1): the halo planes' rows
    are empty, columns are shifted by g0 = (z0-1)*nx*ny.  Its middle rows are the
    slab's rows exactly (same entries, same order; M-HDC blocks of any bl dividing
    nx*ny are the global blocks), so a square-matrix library (the reference) can
    compute one rank's slab of config 4.  Returns (rp, col, val, g0)."""
    p = nx * ny
    rp_s, col_s, val_s = laplacian7(nx, ny, nz, z0, z1)
    g0 = (z0 - 1) * p
    n = (z1 - z0 + 2) * p
    rp = np.empty(n + 1, dtype=np.int64)
    rp[:p] = 0
    rp[p:p + rp_s.size] = rp_s
    rp[p + rp_s.size:] = rp_s[-1]
    col = (col_s.astype(np.int64) - g0).astype(np.int32)
    return rp, col, val_s, g0


# ---------------------------------------------------------------------------
# config 2: 27-point stencil, off-diagonals uniform[-1,0) (stream 1), diag 1 + sum|off|

def stencil27(g: int, seed: int = 2):
    """27-point stencil on a g^3 grid, offsets dx + g*dy + g^2*dz.  Off-diagonal
    value of neighbour t (t = 9*(dz+1) + 3*(dy+1) + (dx+1), ascending offset order)
    of row i is u(seed, 1, 27*i + t) - 1.  The diagonal is 1.0 + s where
    s = sum of |off-diagonals| accumulated in ascending column order from 0.0."""
    n = g ** 3
    i = np.arange(n, dtype=np.int64)
    xx = i % g
    yy = (i // g) % g
    zz = i // (g * g)
    cols = np.empty((n, 27), dtype=np.int64)
    vals = np.empty((n, 27), dtype=np.float64)
    present = np.empty((n, 27), dtype=bool)
    s = np.zeros(n, dtype=np.float64)
    t = 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                m = ((xx + dx >= 0) & (xx + dx < g) & (yy + dy >= 0) & (yy + dy < g)
                     & (zz + dz >= 0) & (zz + dz < g))
                cols[:, t] = i + dx + g * dy + g * g * dz
                present[:, t] = m
                if t != 13:
                    v = u01(seed, 1, 27 * i + t) - 1.0
                    vals[:, t] = v
                    s = np.where(m, s + np.abs(v), s)
                t += 1
    vals[:, 13] = 1.0 + s
    return _csr_from_slots(cols, vals, present)


# ---------------------------------------------------------------------------
# config 3: quasi-diagonal matrix with partial diagonals and scattered nonzeros

QD_CANDIDATES = (-1025, -1024, -2, -1, 1, 2, 1024, 1025)
QD_EXTRA_RADIUS = 1 << 16


def quasi_diag(n: int = 1 << 24, seed: int = 4, seg_min: int = 2048, seg_max: int = 65536,
               p_on: float = 0.6, n_extra: int = 6):
    """BASELINE config 3.  Interpretation (recorded in DESIGN.md):
    * main diagonal always present, value 10.0;
    * candidate offset d_t (QD_CANDIDATES[t]) covers consecutive row segments of
      length seg_min + floor(u(seed,10+t,2k)*(seg_max-seg_min+1)); segment k is on
      iff u(seed,10+t,2k+1) < p_on; value 2u(seed,1,16i+t)-1;
    * n_extra extra columns per row, attempt a draws
      j = lo + floor(u(seed,20,64i+a)*(hi-lo+1)), lo/hi = i -+ (2^16-1) clipped;
      rejected when j-i is 0 or a candidate offset, or already taken in the row
      ("non-colliding"); the e-th accepted extra has value 2u(seed,2,8i+e)-1.
    """
    i = np.arange(n, dtype=np.int64)
    w = 1 + len(QD_CANDIDATES) + n_extra
    cols = np.full((n, w), np.iinfo(np.int64).max, dtype=np.int64)
    vals = np.zeros((n, w), dtype=np.float64)
    cols[:, 0] = i
    vals[:, 0] = 10.0
    for t, d in enumerate(QD_CANDIDATES):
        on_rows = np.zeros(n, dtype=bool)
        start, k = 0, 0
        while start < n:
            ln = seg_min + int(np.floor(u01(seed, 10 + t, np.array([2 * k]))[0] * (seg_max - seg_min + 1)))
            if u01(seed, 10 + t, np.array([2 * k + 1]))[0] < p_on:
                on_rows[start:min(start + ln, n)] = True
            start += ln
            k += 1
        m = on_rows & (i + d >= 0) & (i + d < n)
        cols[m, 1 + t] = i[m] + d
        vals[m, 1 + t] = uniform_pm1(seed, 1, 16 * i[m] + t)
    # extras
    lo = np.maximum(0, i - (QD_EXTRA_RADIUS - 1))
    hi = np.minimum(n - 1, i + (QD_EXTRA_RADIUS - 1))
    span = hi - lo + 1
    forbidden = np.array((0,) + QD_CANDIDATES, dtype=np.int64)
    taken = np.zeros(n, dtype=np.int64)
    extra_cols = np.full((n, n_extra), -1, dtype=np.int64)
    for a in range(64):
        need = taken < n_extra
        if not need.any():
            break
        rows = np.nonzero(need)[0]
        j = lo[rows] + np.floor(u01(seed, 20, 64 * rows + a) * span[rows]).astype(np.int64)
        ok = ~np.isin(j - rows, forbidden)
        for e in range(n_extra):
            ok &= extra_cols[rows, e] != j
        rows, j = rows[ok], j[ok]
        e_idx = taken[rows]
        extra_cols[rows, e_idx] = j
        taken[rows] += 1
    for e in range(n_extra):
        m = extra_cols[:, e] >= 0
        cols[m, 1 + len(QD_CANDIDATES) + e] = extra_cols[m, e]
        vals[m, 1 + len(QD_CANDIDATES) + e] = uniform_pm1(seed, 2, 8 * i[m] + e)
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    present = cols < n
    return _csr_from_slots(cols, vals, present)


# ---------------------------------------------------------------------------
# small fixtures

def example_matrix():
    """The reference's 8x8 fixture (proj/src/stencil.cpp:120-126)."""
    rp = np.array([0, 3, 6, 9, 10, 13, 15, 17, 20], dtype=np.int64)
    col = np.array([0, 2, 5, 1, 3, 6, 2, 4, 7, 3, 0, 4, 6, 5, 7, 2, 6, 0, 3, 7], dtype=np.int32)
    val = np.arange(1, 21, dtype=np.float64)
    return rp, col, val


def coo_to_csr(n: int, rows, cols, vals):
    """CooMatrix normalisation (proj/src/formats.cpp:19-43: stable sort by (row,col),
    duplicates summed in order) followed by CsrMatrix::from_coo (:69-88)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        key = rows * n + cols
        first = np.ones(rows.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        starts = np.nonzero(first)[0]
        # sequential left-to-right sums of duplicate runs, like the reference's in-place loop
        out_vals = vals[starts].copy()
        run_id = np.cumsum(first) - 1
        dup = np.nonzero(~first)[0]
        for k in dup:  # duplicates are rare in test matrices; keep the exact order
            out_vals[run_id[k]] += vals[k]
        rows, cols, vals = rows[starts], cols[starts], out_vals
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    np.cumsum(rp, out=rp)
    return rp, cols.astype(np.int32), vals


def random_matrix(n: int, density: float, rng: np.random.Generator):
    """Uniform random coordinates at roughly `density`, values in [0.5, 1.5]
    (the shape of proj/tests/oracles.hpp:45-55; our own RNG)."""
    target = int(density * n * n)
    r = rng.integers(0, n, size=target)
    c = rng.integers(0, n, size=target)
    v = rng.uniform(0.5, 1.5, size=target)
    return coo_to_csr(n, r, c, v)


def single_diagonal_matrix(n: int, offset: int):
    """proj/tests/oracles.hpp:58-64 shape: one full diagonal, values 1 + 0.25*(i%4)."""
    i = np.arange(max(0, -offset), min(n, n - offset), dtype=np.int64)
    return coo_to_csr(n, i, i + offset, 1.0 + 0.25 * (i % 4))


def dense_row_matrix(n: int, dense_row: int, rng: np.random.Generator):
    """proj/tests/oracles.hpp:67-75 shape: unit-ish diagonal plus one dense row."""
    i = np.arange(n, dtype=np.int64)
    r = np.concatenate([i, np.full(n, dense_row, dtype=np.int64)])
    c = np.concatenate([i, i])
    v = rng.uniform(0.5, 1.5, size=2 * n)
    return coo_to_csr(n, r, c, v)


def reference_stencil(kind: str, n: int):
    """The reference's own gen_stencil (proj/src/stencil.cpp:60-118) restated: offsets
    p3_1d {0,+-1}, p5_2d {0,+-1,+-nx} (nx=floor(sqrt n)), p7_3d adds +-nx^2
    (nx=floor(cbrt n)), duplicates collapsed, |off|<n kept, every in-range slot
    populated with 1 + ((31 i + 17 j) mod 7)."""
    if kind == "p3_1d":
        offs = [0, 1, -1]
    elif kind == "p5_2d":
        nx = int(np.floor(np.sqrt(n)))
        while (nx + 1) * (nx + 1) <= n:
            nx += 1
        while nx * nx > n:
            nx -= 1
        offs = [0, 1, -1, nx, -nx]
    elif kind == "p7_3d":
        nx = int(round(n ** (1.0 / 3.0)))
        while nx ** 3 > n:
            nx -= 1
        while (nx + 1) ** 3 <= n:
            nx += 1
        offs = [0, 1, -1, nx, -nx, nx * nx, -nx * nx]
    else:
        raise ValueError(kind)
    offs = sorted(set(o for o in offs if -n < o < n))
    rows, cols = [], []
    for o in offs:
        i = np.arange(max(0, -o), min(n, n - o), dtype=np.int64)
        rows.append(i)
        cols.append(i + o)
    r = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    c = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    v = (1 + (r * 31 + c * 17) % 7).astype(np.float64)
    return coo_to_csr(n, r, c, v)

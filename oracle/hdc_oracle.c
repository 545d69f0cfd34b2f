/*
 * hdc_oracle.c -- CPU restatement of the reference's HDC / M-HDC path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2105_04937_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls it (there is no CPU fallback).
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below
 * against the reference's own fixtures (proj/tests/test_convert.cpp:14-188,
 * proj/tests/test_kernels.cpp:34-146, proj/tests/acceptance.cpp:62-218) and,
 * when oracle/_ref/libhdcref.so was built from /root/reference, bit-for-bit
 * against the reference library on random matrices.
 *
 * Everything is restated from the reference's algorithm, not copied:
 *   census        proj/src/convert.cpp:39-67   (per-block (offset,count), ascending)
 *   theta test    proj/src/convert.cpp:12-14   (double(count)/double(len) >= theta)
 *   to_mhdc       proj/src/convert.cpp:123-169 (dia_ptr, segments, remainder)
 *   to_hdc        proj/src/convert.cpp:89-121  (== to_mhdc with bl = n)
 *   rates         proj/src/convert.cpp:173-196
 *   spmv_mhdc     proj/src/kernels.cpp:173-206 (remainder first, then segments)
 *   spmv_hdc      proj/src/kernels.cpp:107-137 (same per-row order, lanes)
 *   spmv_csr      proj/src/kernels.cpp:39-54
 * The census here sorts each block's offsets instead of tallying them in a
 * hash map; counts are counts, so the output is identical.
 *
 * Index conventions: row pointers / dia_ptr are int64, column indices and
 * offsets int32, values fp64.  Compile with -ffp-contract=off: the reference
 * oracle (x86-64 -O3) has no FMA, and neither may we.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

static int64_t n_blocks_of(int64_t n, int64_t bl) { return n == 0 ? 0 : (n + bl - 1) / bl; }

/* Sorted distinct offsets (with counts) of block ib; returns the number of
 * distinct offsets.  scratch must hold the block's entry count. */
static int64_t block_census(int64_t n, const int64_t* rp, const int32_t* col, int64_t bl,
                            int64_t ib, int32_t* scratch, int32_t* offs, int64_t* counts) {
    const int64_t r0 = ib * bl, r1 = min64(r0 + bl, n);
    int64_t m = 0;
    for (int64_t i = r0; i < r1; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) scratch[m++] = (int32_t)(col[k] - i);
    qsort(scratch, (size_t)m, sizeof(int32_t), cmp_i32);
    int64_t d = 0;
    for (int64_t k = 0; k < m; ++k) {
        if (d > 0 && offs[d - 1] == scratch[k]) {
            ++counts[d - 1];
        } else {
            offs[d] = scratch[k];
            counts[d] = 1;
            ++d;
        }
    }
    return d;
}

static int64_t max_block_nnz(int64_t n, const int64_t* rp, int64_t bl) {
    int64_t best = 0;
    for (int64_t ib = 0; ib < n_blocks_of(n, bl); ++ib) {
        const int64_t r0 = ib * bl, r1 = min64(r0 + bl, n);
        best = max64(best, rp[r1] - rp[r0]);
    }
    return best;
}

/* convert.cpp:12-14 */
static int dense_enough(int64_t count, int64_t slots, double theta) {
    return (double)count / (double)slots >= theta;
}

/* ---- census (convert.cpp:39-67) ------------------------------------------
 * Pass 1 fills block_ptr[n_blocks+1] (prefix of distinct offsets per block)
 * and returns the total.  Pass 2 writes offsets/counts. */
int64_t orc_census_count(int64_t n, const int64_t* rp, const int32_t* col, int64_t bl,
                         int64_t* block_ptr) {
    const int64_t nb = n_blocks_of(n, bl);
    const int64_t cap = max_block_nnz(n, rp, bl) + 1;
    int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * cap);
    int32_t* offs = (int32_t*)malloc(sizeof(int32_t) * cap);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * cap);
    block_ptr[0] = 0;
    for (int64_t ib = 0; ib < nb; ++ib)
        block_ptr[ib + 1] = block_ptr[ib] + block_census(n, rp, col, bl, ib, scratch, offs, cnt);
    free(scratch); free(offs); free(cnt);
    return block_ptr[nb];
}

void orc_census_fill(int64_t n, const int64_t* rp, const int32_t* col, int64_t bl,
                     const int64_t* block_ptr, int32_t* offsets, int64_t* counts) {
    const int64_t nb = n_blocks_of(n, bl);
    const int64_t cap = max_block_nnz(n, rp, bl) + 1;
    int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * cap);
    for (int64_t ib = 0; ib < nb; ++ib)
        block_census(n, rp, col, bl, ib, scratch, offsets + block_ptr[ib], counts + block_ptr[ib]);
    free(scratch);
}

/* ---- to_mhdc (convert.cpp:123-169); to_hdc is the bl = n case ------------
 * Plan: dia_ptr[n_blocks+1] and the remainder size.  Fill: offsets,
 * segments (n_seg*bl, zero-initialised here), remainder CSR. */
int64_t orc_mhdc_plan(int64_t n, const int64_t* rp, const int32_t* col, double theta, int64_t bl,
                      int64_t* dia_ptr, int64_t* nnz_rest) {
    const int64_t nb = n_blocks_of(n, bl);
    const int64_t cap = max_block_nnz(n, rp, bl) + 1;
    int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * cap);
    int32_t* offs = (int32_t*)malloc(sizeof(int32_t) * cap);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * cap);
    int64_t captured = 0;
    dia_ptr[0] = 0;
    for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t len = min64(bl, n - ib * bl);
        const int64_t d = block_census(n, rp, col, bl, ib, scratch, offs, cnt);
        int64_t s = 0;
        for (int64_t k = 0; k < d; ++k)
            if (dense_enough(cnt[k], len, theta)) { ++s; captured += cnt[k]; }
        dia_ptr[ib + 1] = dia_ptr[ib] + s;
    }
    *nnz_rest = rp[n] - rp[0] - captured;
    free(scratch); free(offs); free(cnt);
    return dia_ptr[nb];
}

void orc_mhdc_fill(int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                   double theta, int64_t bl, const int64_t* dia_ptr, int32_t* dia_offsets,
                   double* segments, int64_t* rest_rp, int32_t* rest_col, double* rest_val) {
    const int64_t nb = n_blocks_of(n, bl);
    const int64_t cap = max_block_nnz(n, rp, bl) + 1;
    int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * cap);
    int32_t* offs = (int32_t*)malloc(sizeof(int32_t) * cap);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * cap);
    memset(segments, 0, sizeof(double) * (size_t)(dia_ptr[nb] * bl));
    int64_t w = 0;
    rest_rp[0] = 0;
    for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t r0 = ib * bl, r1 = min64(r0 + bl, n), len = r1 - r0;
        const int64_t d = block_census(n, rp, col, bl, ib, scratch, offs, cnt);
        int64_t s = dia_ptr[ib];
        for (int64_t k = 0; k < d; ++k)
            if (dense_enough(cnt[k], len, theta)) dia_offsets[s++] = offs[k];
        const int32_t* sel = dia_offsets + dia_ptr[ib];
        const int64_t ns = dia_ptr[ib + 1] - dia_ptr[ib];
        for (int64_t i = r0; i < r1; ++i) {
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int32_t off = (int32_t)(col[k] - i);
                /* lower_bound over the block's selected offsets */
                int64_t lo = 0, hi = ns;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) / 2;
                    if (sel[mid] < off) lo = mid + 1; else hi = mid;
                }
                if (lo < ns && sel[lo] == off) {
                    segments[(dia_ptr[ib] + lo) * bl + (i - r0)] = val[k];
                } else {
                    rest_col[w] = col[k];
                    rest_val[w] = val[k];
                    ++w;
                }
            }
            rest_rp[i + 1] = w;
        }
    }
    free(scratch); free(offs); free(cnt);
}

/* ---- rates (convert.cpp:173-196) -----------------------------------------
 * Returns 0, or -1 when the matrix holds no nonzeros (the reference throws
 * invalid_argument there).  dia_nnz counts nonzero segment values only. */
int orc_rates(int64_t n, int64_t bl, const int64_t* dia_ptr, const double* segments,
              int64_t rest_nnz, double* alpha, double* beta, int64_t* dia_slots) {
    const int64_t nb = n_blocks_of(n, bl);
    int64_t slots = 0, dia_nnz = 0;
    for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t len = min64(bl, n - ib * bl);
        slots += (dia_ptr[ib + 1] - dia_ptr[ib]) * len;
    }
    for (int64_t k = 0; k < dia_ptr[nb] * bl; ++k) dia_nnz += segments[k] != 0.0;
    const int64_t total = dia_nnz + rest_nnz;
    if (total == 0) return -1;
    *beta = (double)rest_nnz / (double)total;
    *alpha = slots == 0 ? 1.0 : (double)dia_nnz / (double)slots;
    *dia_slots = slots;
    return 0;
}

/* ---- SpMV ---------------------------------------------------------------
 * spmv_mhdc (kernels.cpp:173-206): per block, remainder rows summed from 0.0
 * in stored order, then each segment (ascending stored order) added over the
 * clamped row range.  With bl = n this is spmv_hdc / spmv_bhdc
 * (kernels.cpp:107-171), whose per-row order is the same. */
void orc_spmv_mhdc(int64_t n, int64_t bl, const int64_t* dia_ptr, const int32_t* offs,
                   const double* segs, const int64_t* rest_rp, const int32_t* rest_col,
                   const double* rest_val, const double* x, double* y, int nthreads) {
    const int64_t nb = n_blocks_of(n, bl);
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t r0 = ib * bl, r1 = min64(r0 + bl, n);
        for (int64_t i = r0; i < r1; ++i) {
            double s = 0.0;
            for (int64_t k = rest_rp[i]; k < rest_rp[i + 1]; ++k) s += rest_val[k] * x[rest_col[k]];
            y[i] = s;
        }
        for (int64_t k = dia_ptr[ib]; k < dia_ptr[ib + 1]; ++k) {
            const int64_t o = offs[k];
            const int64_t first = max64(r0, -o), last = min64(r1, n - o);
            const double* seg = segs + k * bl;
            for (int64_t i = first; i < last; ++i) y[i] += seg[i - r0] * x[i + o];
        }
    }
    (void)nthreads;
}

/* spmv_csr (kernels.cpp:39-54) */
void orc_spmv_csr(int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                  const double* x, double* y, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += val[k] * x[col[k]];
        y[i] = s;
    }
    (void)nthreads;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

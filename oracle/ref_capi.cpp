// ref_capi.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/hdc_oracle.c).  oracle/Makefile
// compiles this file together with /root/reference/proj/src/*.cpp, in place
// and out of tree, into oracle/_ref/libhdcref.so.  Nothing here re-implements
// the reference: every function forwards to the reference's public API
// (proj/include/hdc/{convert,kernels,bench}.hpp) so that Python tests and
// bench.py's reference arm can drive the real CPU implementation through
// ctypes.  Errors (the reference throws) come back as negative status codes
// with the message in refc_last_error().
#include "hdc/bench.hpp"
#include "hdc/convert.hpp"
#include "hdc/kernels.hpp"
#include "hdc/stencil.hpp"

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(_OPENMP)
#include <omp.h>
#endif

using namespace hdc;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// 1 invalid_argument, 2 out_of_range, 3 overflow_error, 4 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::out_of_range& e) {
        return fail(e, -2);
    } catch (const std::overflow_error& e) {
        return fail(e, -3);
    } catch (const std::exception& e) {
        return fail(e, -4);
    }
}

CsrMatrix make_csr(int64_t n, const int64_t* rp, const int32_t* col, const double* val) {
    const int64_t nnz = n > 0 ? rp[n] : 0;
    std::vector<index_t> row_ptr(static_cast<std::size_t>(n) + 1);
    for (int64_t i = 0; i <= n; ++i) row_ptr[i] = static_cast<index_t>(rp[i]);
    std::vector<index_t> c(col, col + nnz);
    std::vector<real_t> v(val, val + nnz);
    return CsrMatrix(static_cast<index_t>(n), std::move(v), std::move(c), std::move(row_ptr));
}

struct RefCsr {
    CsrMatrix m;
};
struct RefHdc {
    HdcMatrix m;
};
struct RefMhdc {
    MHdcMatrix m;
};

}  // namespace

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }

int refc_max_threads() {
#if defined(_OPENMP)
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int refc_csr_new(int64_t n, const int64_t* rp, const int32_t* col, const double* val, void** out) {
    return guarded([&] { *out = new RefCsr{make_csr(n, rp, col, val)}; });
}
void refc_csr_free(void* h) { delete static_cast<RefCsr*>(h); }

int refc_example_matrix(void** out) {
    return guarded([&] { *out = new RefCsr{example_matrix()}; });
}

int refc_csr_sizes(void* h, int64_t* n, int64_t* nnz) {
    const CsrMatrix& m = static_cast<RefCsr*>(h)->m;
    *n = m.n();
    *nnz = static_cast<int64_t>(m.values().size());
    return 0;
}

int refc_csr_export(void* h, int64_t* rp, int32_t* col, double* val) {
    const CsrMatrix& m = static_cast<RefCsr*>(h)->m;
    for (std::size_t i = 0; i < m.row_ptr().size(); ++i) rp[i] = m.row_ptr()[i];
    for (std::size_t k = 0; k < m.col_ind().size(); ++k) col[k] = m.col_ind()[k];
    std::memcpy(val, m.values().data(), m.values().size() * sizeof(double));
    return 0;
}

// ---- census (convert.hpp:26-32) -------------------------------------------
int refc_census(void* csr, int64_t bl, int global, int64_t* n_blocks, int64_t* total_entries,
                int64_t* block_ptr, int32_t* offsets, int64_t* counts) {
    return guarded([&] {
        const CsrMatrix& m = static_cast<RefCsr*>(csr)->m;
        const DiagonalCensus c = global ? census_global(m) : census_blocked(m, static_cast<index_t>(bl));
        *n_blocks = static_cast<int64_t>(c.per_block.size());
        int64_t tot = 0;
        for (const auto& b : c.per_block) tot += static_cast<int64_t>(b.size());
        *total_entries = tot;
        if (block_ptr) {
            int64_t w = 0;
            block_ptr[0] = 0;
            for (std::size_t ib = 0; ib < c.per_block.size(); ++ib) {
                for (const OffsetCount& oc : c.per_block[ib]) {
                    offsets[w] = oc.offset;
                    counts[w] = oc.count;
                    ++w;
                }
                block_ptr[ib + 1] = w;
            }
        }
    });
}

// ---- to_mhdc / to_hdc (convert.hpp:34-39) ----------------------------------
int refc_to_mhdc(void* csr, double theta, int64_t bl, void** out) {
    return guarded([&] {
        *out = new RefMhdc{to_mhdc(static_cast<RefCsr*>(csr)->m, theta, static_cast<index_t>(bl))};
    });
}
void refc_mhdc_free(void* h) { delete static_cast<RefMhdc*>(h); }

int refc_mhdc_sizes(void* h, int64_t* n, int64_t* bl, int64_t* n_blocks, int64_t* n_seg,
                    int64_t* nnz_rest) {
    const MHdcMatrix& m = static_cast<RefMhdc*>(h)->m;
    *n = m.n();
    *bl = m.bl();
    *n_blocks = m.n_blocks();
    *n_seg = m.n_segments();
    *nnz_rest = static_cast<int64_t>(m.csr().values().size());
    return 0;
}

int refc_mhdc_export(void* h, int64_t* dia_ptr, int32_t* offs, double* segs, int64_t* rest_rp,
                     int32_t* rest_col, double* rest_val) {
    const MHdcMatrix& m = static_cast<RefMhdc*>(h)->m;
    for (std::size_t i = 0; i < m.dia_ptr().size(); ++i) dia_ptr[i] = m.dia_ptr()[i];
    for (std::size_t k = 0; k < m.dia_offsets().size(); ++k) offs[k] = m.dia_offsets()[k];
    std::memcpy(segs, m.segments().data(), m.segments().size() * sizeof(double));
    for (std::size_t i = 0; i < m.csr().row_ptr().size(); ++i) rest_rp[i] = m.csr().row_ptr()[i];
    for (std::size_t k = 0; k < m.csr().col_ind().size(); ++k) rest_col[k] = m.csr().col_ind()[k];
    std::memcpy(rest_val, m.csr().values().data(), m.csr().values().size() * sizeof(double));
    return 0;
}

int refc_to_hdc(void* csr, double theta, void** out) {
    return guarded([&] { *out = new RefHdc{to_hdc(static_cast<RefCsr*>(csr)->m, theta)}; });
}
void refc_hdc_free(void* h) { delete static_cast<RefHdc*>(h); }

int refc_hdc_sizes(void* h, int64_t* n, int64_t* n_diag, int64_t* nnz_rest) {
    const HdcMatrix& m = static_cast<RefHdc*>(h)->m;
    *n = m.n();
    *n_diag = m.dia().n_diags();
    *nnz_rest = static_cast<int64_t>(m.csr().values().size());
    return 0;
}

int refc_hdc_export(void* h, int32_t* offs, double* lanes, int64_t* rest_rp, int32_t* rest_col,
                    double* rest_val) {
    const HdcMatrix& m = static_cast<RefHdc*>(h)->m;
    for (std::size_t k = 0; k < m.dia().offsets().size(); ++k) offs[k] = m.dia().offsets()[k];
    std::memcpy(lanes, m.dia().lanes().data(), m.dia().lanes().size() * sizeof(double));
    for (std::size_t i = 0; i < m.csr().row_ptr().size(); ++i) rest_rp[i] = m.csr().row_ptr()[i];
    for (std::size_t k = 0; k < m.csr().col_ind().size(); ++k) rest_col[k] = m.csr().col_ind()[k];
    std::memcpy(rest_val, m.csr().values().data(), m.csr().values().size() * sizeof(double));
    return 0;
}

// ---- rates (convert.hpp:45-52) ---------------------------------------------
int refc_rates_mhdc(void* h, double* alpha, double* beta, int64_t* slots) {
    return guarded([&] {
        const HybridRates r = rates(static_cast<RefMhdc*>(h)->m);
        *alpha = r.alpha;
        *beta = r.beta;
        *slots = r.dia_slots;
    });
}
int refc_rates_hdc(void* h, double* alpha, double* beta, int64_t* slots) {
    return guarded([&] {
        const HybridRates r = rates(static_cast<RefHdc*>(h)->m);
        *alpha = r.alpha;
        *beta = r.beta;
        *slots = r.dia_slots;
    });
}

// ---- kernels (kernels.hpp:31-49) -------------------------------------------
// kind: 0 csr, 1 hdc, 2 bhdc(bl), 3 mhdc, 4 dia (to_dia of the csr), 5 bdia(bl)
int refc_spmv(int kind, void* h, int64_t bl, const double* x, double* y, int64_t n, int workers) {
    return guarded([&] {
        std::span<const real_t> xs(x, static_cast<std::size_t>(n));
        std::span<real_t> ys(y, static_cast<std::size_t>(n));
        switch (kind) {
            case 0: spmv_csr(static_cast<RefCsr*>(h)->m, xs, ys, workers); break;
            case 1: spmv_hdc(static_cast<RefHdc*>(h)->m, xs, ys, workers); break;
            case 2: {
                const HdcMatrix& m = static_cast<RefHdc*>(h)->m;
                spmv_bhdc(m, BlockPlan::rows(m.n(), static_cast<index_t>(bl)), xs, ys, workers);
                break;
            }
            case 3: spmv_mhdc(static_cast<RefMhdc*>(h)->m, xs, ys, workers); break;
            case 4: spmv_dia(to_dia(static_cast<RefCsr*>(h)->m), xs, ys, workers); break;
            case 5: {
                const CsrMatrix& m = static_cast<RefCsr*>(h)->m;
                spmv_bdia(to_dia(m), BlockPlan::rows(m.n(), static_cast<index_t>(bl)), xs, ys,
                          workers);
                break;
            }
            default: throw std::invalid_argument("refc_spmv: unknown kernel kind");
        }
    });
}

// The reference's own timing protocol (bench.cpp:44-60): one warm-up loop of
// n_ites calls, n_loops timed loops, best per-call average.
int refc_time_spmv(int kind, void* h, int64_t bl, const double* x, double* y, int64_t n,
                   int workers, int n_loops, int n_ites, double* best_s) {
    return guarded([&] {
        bench::TimingConfig cfg;
        cfg.n_loops = n_loops;
        cfg.n_ites = n_ites;
        cfg.workers = workers;
        int rc = 0;
        const bench::Measurement m = bench::time_kernel(
            [&] { rc |= refc_spmv(kind, h, bl, x, y, n, workers); }, cfg, 0.0);
        if (rc != 0) throw std::runtime_error(g_err);
        *best_s = m.best_time_s;
    });
}

// The reference's streaming micro-benchmark (bench.hpp:33-46, bench.cpp:68-110):
// mode 0 direct (32 B/element), 1 indirect (36 B/element).
int refc_membench(int64_t n, int mode, int n_loops, int n_ites, int workers, double* bytes_per_s,
                  double* best_s) {
    return guarded([&] {
        bench::TimingConfig cfg;
        cfg.n_loops = n_loops;
        cfg.n_ites = n_ites;
        cfg.workers = workers;
        const bench::Measurement m = bench::membench(static_cast<index_t>(n),
                                                     mode ? bench::MemMode::indirect : bench::MemMode::direct, cfg);
        *bytes_per_s = m.bytes_per_s;
        *best_s = m.best_time_s;
    });
}

}  // extern "C"

// ---- io (io.hpp:14-20): Matrix Market -> CsrMatrix via CooMatrix ------------
#include "hdc/io.hpp"
extern "C" int refc_read_matrix_market(const char* path, void** out) {
    try {
        *out = new RefCsr{CsrMatrix::from_coo(hdc::io::read_matrix_market(std::string(path)))};
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::out_of_range& e) {
        return fail(e, -2);
    } catch (const std::overflow_error& e) {
        return fail(e, -3);
    } catch (const std::exception& e) {
        return fail(e, -4);
    }
}

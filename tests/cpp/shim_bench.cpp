// shim_bench.cpp -- what a C++ caller of the reference API sees with the GPU shim
// linked in (oracle/Makefile target `shim`): wall time of hdc::to_mhdc and of
// repeated hdc::spmv_mhdc calls on host containers (std::vector storage), for the
// BASELINE config-1 matrix (7-point Dirichlet Laplacian, 256^3 by default).
//   shim_bench [nx ny nz] [bl] [calls]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hdc/convert.hpp"
#include "hdc/formats.hpp"
#include "hdc/kernels.hpp"

using namespace hdc;
using clk = std::chrono::steady_clock;

static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main(int argc, char** argv) {
    const long nx = argc > 3 ? atol(argv[1]) : 256, ny = argc > 3 ? atol(argv[2]) : 256, nz = argc > 3 ? atol(argv[3]) : 256;
    const index_t bl = argc > 4 ? (index_t)atol(argv[4]) : 4096;
    const int calls = argc > 5 ? atoi(argv[5]) : 10;
    const long n = nx * ny * nz;
    std::vector<index_t> rp(n + 1, 0), ci;
    std::vector<real_t> cv;
    ci.reserve(7 * n);
    cv.reserve(7 * n);
    for (long z = 0; z < nz; ++z)
        for (long y = 0; y < ny; ++y)
            for (long x = 0; x < nx; ++x) {
                const long i = x + nx * (y + ny * z);
                auto put = [&](bool ok, long j, double v) {
                    if (ok) {
                        ci.push_back((index_t)j);
                        cv.push_back(v);
                    }
                };
                put(z > 0, i - nx * ny, -1.0);
                put(y > 0, i - nx, -1.0);
                put(x > 0, i - 1, -1.0);
                put(true, i, 6.0);
                put(x + 1 < nx, i + 1, -1.0);
                put(y + 1 < ny, i + nx, -1.0);
                put(z + 1 < nz, i + nx * ny, -1.0);
                rp[i + 1] = (index_t)ci.size();
            }
    const double nnz = (double)ci.size();
    CsrMatrix A((index_t)n, std::move(cv), std::move(ci), std::move(rp));
    std::vector<real_t> x(n), y(n);
    for (long i = 0; i < n; ++i) x[i] = 1.0 / (1.0 + (double)(i % 97));
    auto t0 = clk::now();
    MHdcMatrix M = to_mhdc(A, 0.6, bl);
    auto t1 = clk::now();
    std::printf("{\"n\": %ld, \"nnz\": %.0f, \"bl\": %ld, \"to_mhdc_ms\": %.2f, \"spmv_mhdc_ms\": [", n, nnz, (long)bl, ms(t0, t1));
    double best = 1e30;
    for (int k = 0; k < calls; ++k) {
        auto a = clk::now();
        spmv_mhdc(M, x, y);
        auto b = clk::now();
        std::printf("%s%.2f", k ? ", " : "", ms(a, b));
        if (k) best = std::min(best, ms(a, b));
    }
    double s = 0;
    for (long i = 0; i < n; ++i) s += y[i];
    std::printf("], \"best_ms\": %.2f, \"gflops\": %.1f, \"y_sum\": %.6e}\n", best, 2 * nnz / best / 1e6, s);
    return 0;
}

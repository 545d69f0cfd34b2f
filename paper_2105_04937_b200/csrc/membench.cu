// membench.cu -- the reference's streaming micro-benchmark on the device
// (hdc::bench::membench, proj/src/bench.cpp:68-110): it supplies
// the sustained memory bandwidth w_mem the §5 model divides byte volumes by
// (model.cpp:113-117), measured on the B200 instead of the host.
//
//   direct:   c[i] += a[i] * b[i]          32 bytes per element (bench.hpp:40)
//   indirect: c[i] += a[i] * b[idx[i]]     36 bytes per element, idx[i] = i
//
// Same protocol as bench::time_kernel (bench.cpp:44-60): one untimed loop of
// n_ites calls, n_loops timed loops (CUDA events), best per-call average; the
// result is checked (every slot must equal the number of calls, bench.cpp:99-104).
#include <vector>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

__global__ void fill_kernel_f64(double* p, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
__global__ void iota_kernel_i32(int32_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

template <bool INDIRECT>
__global__ void triad_kernel(const double* __restrict__ a, const double* __restrict__ b,
                             const int32_t* __restrict__ idx, double* __restrict__ c, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double bv = INDIRECT ? __ldg(b + __ldg(idx + i)) : __ldg(b + i);
        c[i] = __dadd_rn(c[i], __dmul_rn(__ldg(a + i), bv));
    }
}

__global__ void check_kernel(const double* c, int64_t n, double want, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (c[i] != want) atomicAdd(bad, 1ULL);
}

}  // namespace

void membench(int64_t n, int mode, int n_loops, int n_ites, double* best_s, double* bytes_per_s,
              double* loop_times) {
    if (n_loops < 1 || n_ites < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "timing: n_loops and n_ites must be >= 1");
    if (n < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "membench: n must be >= 1");
    if (mode != 0 && mode != 1) fail(HDCG_ERR_INVALID_ARGUMENT, "unknown memory mode");
    if (mode == 1 && n > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "membench: indirect index exceeds int32");
    cudaStream_t st = nullptr;
    double* a = dev_alloc<double>(n, st);
    double* b = dev_alloc<double>(n, st);
    double* c = dev_alloc<double>(n, st);
    int32_t* idx = mode == 1 ? dev_alloc<int32_t>(n, st) : nullptr;
    const int grid = grid_cap(ceil_div(n, 256));
    fill_kernel_f64<<<grid, 256, 0, st>>>(a, n, 1.0);
    fill_kernel_f64<<<grid, 256, 0, st>>>(b, n, 1.0);
    fill_kernel_f64<<<grid, 256, 0, st>>>(c, n, 0.0);
    if (idx) iota_kernel_i32<<<grid, 256, 0, st>>>(idx, n);
    HDCG_LAUNCH_CHECK("membench init");
    auto call = [&] {
        if (mode == 1) triad_kernel<true><<<grid, 256, 0, st>>>(a, b, idx, c, n);
        else triad_kernel<false><<<grid, 256, 0, st>>>(a, b, idx, c, n);
    };
    for (int it = 0; it < n_ites; ++it) call();  // untimed warm-up loop
    cudaEvent_t e0, e1;
    HDCG_CUDA(cudaEventCreate(&e0));
    HDCG_CUDA(cudaEventCreate(&e1));
    double best = 1e300;
    for (int loop = 0; loop < n_loops; ++loop) {
        HDCG_CUDA(cudaEventRecord(e0, st));
        for (int it = 0; it < n_ites; ++it) call();
        HDCG_CUDA(cudaEventRecord(e1, st));
        HDCG_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        HDCG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        const double per_call = (double)ms * 1e-3 / n_ites;
        if (loop_times) loop_times[loop] = per_call;
        best = per_call < best ? per_call : best;
    }
    HDCG_LAUNCH_CHECK("triad_kernel");
    unsigned long long* bad = dev_alloc<unsigned long long>(1, st);
    HDCG_CUDA(cudaMemsetAsync(bad, 0, sizeof(*bad), st));
    check_kernel<<<grid, 256, 0, st>>>(c, n, (double)n_ites * ((double)n_loops + 1.0), bad);
    unsigned long long nbad = 0;
    HDCG_CUDA(cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dev_free(bad, st);
    dev_free(a, st);
    dev_free(b, st);
    dev_free(c, st);
    dev_free(idx, st);
    HDCG_CUDA(cudaStreamSynchronize(st));
    if (nbad) fail(HDCG_ERR_CUDA, "membench: result check failed");
    *best_s = best;
    *bytes_per_s = (mode == 1 ? 36.0 : 32.0) * (double)n / best;
}

}  // namespace hdcg

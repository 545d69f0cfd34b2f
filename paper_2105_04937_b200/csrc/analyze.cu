// analyze.cu -- (theta, bl) parameter sweep with census reuse.
//
// The reference's `hdcmv analyze` (proj/tools/hdcmv.cpp:93-140) rebuilds the
// full HDC / M-HDC format for every grid point just to read rates() off it
// (convert.cpp:173-196).  The rates only depend on the per-(block, offset)
// census, so here each block width is censused ONCE on the device and every
// theta is evaluated from the census runs:
//
//   run (block b, offset o): count c (stored entries, convert.cpp:53-54) and
//                            nz (entries with a nonzero value)
//   selected(theta)       <=> double(c) / double(len_b) >= theta  (convert.cpp:12-14)
//   dia_slots             = sum over selected runs of len_b       (convert.cpp:190-194)
//   dia nnz               = sum over selected runs of nz          (nnz(MHdcMatrix) counts
//                                                                  nonzero slots, formats.cpp:185-190)
//   remainder nnz         = sum over unselected runs of c         (stored entries)
//   n_seg / n_diags       = number of selected runs
//
// which reproduces rates(to_mhdc(m, theta, bl)) and rates(to_hdc(m, theta))
// exactly (integer sums, then the same two divisions).  Census: the entries'
// offsets and nonzero flags are segment-sorted per block (CUB), runs found by
// comparing neighbours, nonzero counts from a prefix sum of the sorted flags.
#include <cub/cub.cuh>

#include <cmath>
#include <limits>
#include <vector>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

constexpr int MAX_THETA = 64;

template <class RP>
__global__ void census_keys_kernel(const RP* rp, const int32_t* col, const double* val, int64_t n, int32_t* keys,
                                   int32_t* nzflag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k1 = rp[i + 1];
        for (int64_t k = rp[i]; k < k1; ++k) {
            keys[k] = (int32_t)((int64_t)col[k] - i);
            nzflag[k] = val[k] != 0.0;
        }
    }
}

template <class RP>
__global__ void block_offsets_kernel(const RP* rp, int64_t n, int64_t bl, int64_t nb, int32_t* off) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x)
        off[b] = (int32_t)rp[b * bl < n ? b * bl : n];
}

// One CTA per block: runs of the sorted keys -> per-theta integer sums.
// sums layout: [theta][4] = {n_sel, dia_slots, dia_nnz, rest_nnz}.
__global__ void __launch_bounds__(256) runs_kernel(const int32_t* keys, const int32_t* nzpre, const int32_t* off,
                                                   int64_t n, int64_t bl, const double* thetas, int n_theta,
                                                   unsigned long long* sums) {
    __shared__ unsigned long long s[MAX_THETA * 4];
    for (int t = threadIdx.x; t < n_theta * 4; t += blockDim.x) s[t] = 0;
    __syncthreads();
    const int64_t b = blockIdx.x;
    const int64_t len = min(bl, n - b * bl);
    const int p0 = off[b], p1 = off[b + 1];
    for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const int32_t key = keys[p];
        if (p != p0 && keys[p - 1] == key) continue;  // not a run start
        int lo = p, hi = p1;                           // end of run: upper_bound in [p, p1)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (keys[mid] <= key) lo = mid + 1;
            else hi = mid;
        }
        const unsigned long long c = (unsigned long long)(lo - p);
        const unsigned long long nz = (unsigned long long)(nzpre[lo] - nzpre[p]);
        for (int t = 0; t < n_theta; ++t) {
            if ((double)c / (double)len >= thetas[t]) {
                atomicAdd(&s[4 * t + 0], 1ULL);
                atomicAdd(&s[4 * t + 1], (unsigned long long)len);
                atomicAdd(&s[4 * t + 2], nz);
            } else {
                atomicAdd(&s[4 * t + 3], c);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_theta * 4; t += blockDim.x)
        if (s[t]) atomicAdd(&sums[t], s[t]);
}

template <class RP>
void census_sums(const CsrInput& in, int64_t bl, const double* d_thetas, int n_theta,
                 std::vector<unsigned long long>& sums, cudaStream_t st) {
    const int64_t n = in.n_rows, nnz = in.nnz;
    const int64_t nb = n_blocks_of(n, bl);
    sums.assign((size_t)n_theta * 4, 0);
    if (nb == 0 || nnz == 0) return;
    int32_t* keys = dev_alloc<int32_t>(nnz, st);
    int32_t* flags = dev_alloc<int32_t>(nnz, st);
    int32_t* skeys = dev_alloc<int32_t>(nnz, st);
    int32_t* sflags = dev_alloc<int32_t>(nnz + 1, st);
    int32_t* pre = dev_alloc<int32_t>(nnz + 1, st);
    int32_t* off = dev_alloc<int32_t>(nb + 1, st);
    unsigned long long* d_sums = dev_alloc<unsigned long long>(n_theta * 4, st);
    HDCG_CUDA(cudaMemsetAsync(d_sums, 0, sizeof(unsigned long long) * n_theta * 4, st));
    census_keys_kernel<RP><<<grid_cap(ceil_div(n, 256)), 256, 0, st>>>((const RP*)in.row_ptr, in.col, in.val, n,
                                                                       keys, flags);
    block_offsets_kernel<RP><<<grid_cap(ceil_div(nb + 1, 256)), 256, 0, st>>>((const RP*)in.row_ptr, n, bl, nb, off);
    HDCG_LAUNCH_CHECK("census_keys_kernel");
    size_t bytes = 0;
    HDCG_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, keys, skeys, flags, sflags, (int)nnz, (int)nb, off,
                                                  off + 1, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp, bytes, keys, skeys, flags, sflags, (int)nnz, (int)nb, off,
                                                  off + 1, st));
    dev_free(tmp, st);
    HDCG_CUDA(cudaMemsetAsync(sflags + nnz, 0, sizeof(int32_t), st));
    size_t sbytes = 0;
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sbytes, sflags, pre, nnz + 1, st));
    tmp = dev_alloc<char>((int64_t)sbytes + 1, st);
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, sbytes, sflags, pre, nnz + 1, st));
    dev_free(tmp, st);
    if (nb > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "analyze: too many blocks");
    runs_kernel<<<(unsigned)nb, 256, 0, st>>>(skeys, pre, off, n, bl, d_thetas, n_theta, d_sums);
    HDCG_LAUNCH_CHECK("runs_kernel");
    HDCG_CUDA(cudaMemcpyAsync(sums.data(), d_sums, sizeof(unsigned long long) * n_theta * 4, cudaMemcpyDeviceToHost,
                              st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    dev_free(keys, st);
    dev_free(flags, st);
    dev_free(skeys, st);
    dev_free(sflags, st);
    dev_free(pre, st);
    dev_free(off, st);
    dev_free(d_sums, st);
}

}  // namespace

void analyze(const CsrInput& in, const double* thetas, int n_theta, const int64_t* bls, int n_bl, double* out,
             cudaStream_t st) {
    if (n_theta < 1 || n_theta > MAX_THETA) fail(HDCG_ERR_INVALID_ARGUMENT, "analyze: 1..64 theta values");
    if (n_bl < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "analyze: negative bl count");
    for (int t = 0; t < n_theta; ++t)
        if (!(thetas[t] >= 0.0 && thetas[t] <= 1.0)) fail(HDCG_ERR_INVALID_ARGUMENT, "to_hdc: theta must be in [0, 1]");
    for (int j = 0; j < n_bl; ++j)
        if (bls[j] < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "to_mhdc: block width must be >= 1");
    if (in.nnz > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "analyze: nnz exceeds the int32 index range");
    double* d_thetas = dev_alloc<double>(n_theta, st);
    HDCG_CUDA(cudaMemcpyAsync(d_thetas, thetas, sizeof(double) * n_theta, cudaMemcpyHostToDevice, st));
    const int64_t n = in.n_rows;
    const int n_cen = 1 + n_bl;
    for (int ci = 0; ci < n_cen; ++ci) {
        const int64_t bl = ci == 0 ? (n > 0 ? n : 1) : bls[ci - 1];  // census 0: global (HDC)
        std::vector<unsigned long long> sums;
        if (in.rp64) census_sums<int64_t>(in, bl, d_thetas, n_theta, sums, st);
        else census_sums<int32_t>(in, bl, d_thetas, n_theta, sums, st);
        for (int t = 0; t < n_theta; ++t) {
            const unsigned long long n_sel = sums[4 * t], slots = sums[4 * t + 1], dia = sums[4 * t + 2],
                                     rest = sums[4 * t + 3];
            double* o = out + ((size_t)t * n_cen + ci) * 4;
            const unsigned long long total = dia + rest;
            if (total == 0) {  // rates() throws invalid_argument (convert.cpp:175)
                o[0] = o[1] = std::numeric_limits<double>::quiet_NaN();
            } else {
                o[1] = (double)rest / (double)total;
                o[0] = slots == 0 ? 1.0 : (double)dia / (double)slots;
            }
            o[2] = (double)slots;
            o[3] = (double)n_sel;
        }
    }
    dev_free(d_thetas, st);
    HDCG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hdcg

// Microbenchmark behind the column-sorted remainder layout (config 3): how fast can
// one B200 gather 8-byte x values for CSR-remainder entries whose columns lie in a
// +-2^16 window around the row, (a) in row-major entry order and (b) with the
// entries of a T-row group sorted by column, the products scattered into shared
// memory at their row-major positions and summed per row in stored order.
// The order is data only: (col, dest) arrays; one kernel serves both.
// Also: random 8-byte loads from a 1 MB window held in the shared memory of a
// cluster of 8 CTAs (ld.shared::cluster).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
//        -o scripts/libgather_probe.so scripts/gather_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
namespace cg = cooperative_groups;

template <int NT, int U>
__global__ void __launch_bounds__(NT, 1)
probe_kernel(const int* __restrict__ col, const uint16_t* __restrict__ dest, const double* __restrict__ val,
             const double* __restrict__ x, double* __restrict__ y, int T, int per_row, int n_groups, int dmod, int n)
{
    extern __shared__ double prod[];
    const long long epg = (long long)T * per_row;
    for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
        const long long e0 = (g % dmod) * epg;   // dmod < n_groups: the entry streams stay in L2
        const int cbase = g * T - (1 << 16);
        for (int b = threadIdx.x; b < epg; b += NT * U) {
            int c[U];
            uint16_t d[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int i = b + u * NT;
                bool ok = i < epg;
                c[u] = ok ? __ldcs(col + e0 + i) : 0;
                d[u] = ok ? __ldcs(dest + e0 + i) : 0xffff;
                v[u] = ok ? __ldcs(val + e0 + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = __ldg(x + min(max(c[u] + cbase, 0), n - 1));
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (d[u] != 0xffff) prod[d[u]] = __dmul_rn(v[u], xv[u]);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < T; t += NT) {
            double a = 0.0;
            for (int k = 0; k < per_row; ++k) a = __dadd_rn(a, prod[t * per_row + k]);
            __stcs(y + (long long)g * T + t, a);
        }
        __syncthreads();
    }
}

// Cluster of 8: each CTA holds `per` doubles of a window in shared memory; every
// thread does `iters` rounds of U random 8-byte loads from the whole window.
template <int NT, int U>
__global__ void __launch_bounds__(NT, 1)
dsmem_kernel(const int* __restrict__ idx, double* __restrict__ out, int per, int iters)
{
    extern __shared__ double win[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < per; i += NT) win[i] = (double)(cl.block_rank() * per + i);
    cl.sync();
    const int nr = cl.num_blocks();
    double acc = 0.0;
    const int* p = idx + (size_t)blockIdx.x * NT * U * iters;
    for (int it = 0; it < iters; ++it) {
        int j[U];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = __ldcs(p + (it * U + u) * NT + threadIdx.x);
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int r = j[u] / per, o = j[u] - r * per;
            r = r < nr ? r : nr - 1;
            const double* q = cl.map_shared_rank(win, r);
            xv[u] = q[o];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += xv[u];
    }
    out[blockIdx.x * NT + threadIdx.x] = acc;
    cl.sync();
}

// Pure gather rate: no index streams.  Lane groups of K lanes share one 128-byte
// line (K = 1: every lane its own random line inside a +-2^16 window that moves
// with the CTA's position, like config 3's remainder).
__device__ __forceinline__ unsigned mix(unsigned a)
{
    a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
    return a;
}
// FLAVOR: 0 ld.global.nc (__ldg), 1 ld.global.cg (L2 only), 2 texture fetch (int2 texels
// of a linear texture over x), 3 ld.global.cv
template <int U, int FLAVOR = 0>
__global__ void __launch_bounds__(1024, 1)
pure_kernel(const double* __restrict__ x, double* __restrict__ out, int iters, int K, int n, int wbits,
            cudaTextureObject_t tex = 0)
{
    double acc = 0.0;
    const unsigned lane = threadIdx.x & 31, grp = lane / K;
    const unsigned wmask = (1u << wbits) - 1;
    for (int it = 0; it < iters; ++it) {
        // the window drifts through x as the iterations go on
        const long long base = ((long long)blockIdx.x * iters + it) * (n - (1 << wbits)) / ((long long)gridDim.x * iters);
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            unsigned h = mix(((blockIdx.x * 1024u + (threadIdx.x & ~31u) + grp) * 131u + it) * 16u + u);
            unsigned line = (h & wmask) >> 4;
            unsigned within = mix(h + lane) & 15;
            const long long idx = base + line * 16 + within;
            if (FLAVOR == 0) xv[u] = __ldg(x + idx);
            else if (FLAVOR == 1) xv[u] = __ldcg(x + idx);
            else if (FLAVOR == 3) xv[u] = __ldcv(x + idx);
            else {
                const int2 t = tex1Dfetch<int2>(tex, (int)idx);
                xv[u] = __hiloint2double(t.y, t.x);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += xv[u];
    }
    out[blockIdx.x * 1024 + threadIdx.x] = acc;
}
extern "C" int gp_pure(const double* x, double* out, int iters, int K, int n, int wbits, int u, int grid, void* stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (u == 4) pure_kernel<4><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else if (u == 8) pure_kernel<8><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else if (u == 16) pure_kernel<16><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else return -1;
    return (int)cudaGetLastError();
}

extern "C" int gp_pure_flavor(const double* x, double* out, int iters, int K, int n, int wbits, int flavor, int grid,
                              void* stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    static cudaTextureObject_t tex = 0;
    if (flavor == 2 && !tex) {
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = const_cast<double*>(x);
        rd.res.linear.desc = cudaCreateChannelDesc<int2>();
        rd.res.linear.sizeInBytes = (size_t)n * 8;
        cudaTextureDesc td = {};
        td.readMode = cudaReadModeElementType;
        cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
        if (e != cudaSuccess) return (int)e;
    }
    if (flavor == 0) pure_kernel<8, 0><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else if (flavor == 1) pure_kernel<8, 1><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else if (flavor == 2) pure_kernel<8, 2><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits, tex);
    else if (flavor == 3) pure_kernel<8, 3><<<grid, 1024, 0, s>>>(x, out, iters, K, n, wbits);
    else return -1;
    return (int)cudaGetLastError();
}

template <int NT, int U>
static int launch_probe(const int* col, const uint16_t* dest, const double* val, const double* x, double* y, int T,
                        int per_row, int n_groups, int dmod, int n, int grid, cudaStream_t s)
{
    size_t sm = (size_t)T * per_row * 8;
    cudaFuncSetAttribute(probe_kernel<NT, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    probe_kernel<NT, U><<<grid, NT, sm, s>>>(col, dest, val, x, y, T, per_row, n_groups, dmod, n);
    return (int)cudaGetLastError();
}

extern "C" int gp_probe(const int* col, const uint16_t* dest, const double* val, const double* x, double* y, int T,
                        int per_row, int n_groups, int dmod, int n, int grid, int nt, int u, void* stream)
{
    cudaStream_t s = (cudaStream_t)stream;
#define C(NT, U) \
    if (nt == NT && u == U) return launch_probe<NT, U>(col, dest, val, x, y, T, per_row, n_groups, dmod, n, grid, s);
    C(512, 4) C(512, 8) C(1024, 4) C(1024, 8) C(1024, 2) C(768, 8) C(768, 4)
#undef C
    return -1;
}

extern "C" int gp_dsmem(const int* idx, double* out, int per, int iters, int grid, int csize, int u, void* stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto kern) {
        size_t sm = (size_t)per * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (csize > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csize;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&cfg, kern, idx, out, per, iters);
    };
    if (u == 4) return go(dsmem_kernel<1024, 4>);
    if (u == 8) return go(dsmem_kernel<1024, 8>);
    return -1;
}

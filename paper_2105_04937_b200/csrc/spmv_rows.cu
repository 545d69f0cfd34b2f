// spmv_rows.cu -- remainder / CSR row sums with one row per lane and the entry
// streams staged through shared memory by TMA (sm_100a).
//
// The reference sums a row's remainder entries in stored order onto +0.0
// (kernels.cpp:39-60 spmv_csr, :192-197 the M-HDC remainder).  rest_pipe_kernel
// (spmv_tma.cu) keeps that order with entry-major lanes: 32 lanes load 32
// consecutive entries, gather x, and pass the products through shared memory to
// the lane that owns the row.  For structured rows (a stencil stored as CSR: 27
// consecutive entries are 27 different x lines) every warp gather touches ~32
// lines, and the kernel is bound by L1 wavefronts (config 2 as CSR: 68% of the
// HBM peak), not by bytes.
//
// Here a lane owns a row and walks its entries in order (the reference's loop,
// no product hand-off), so the k-th gathers of 32 adjacent rows are adjacent
// columns for banded matrices: 2-3 lines per warp gather.  Column indices and
// values never touch L1: a producer warp streams the CTA's contiguous entry range
// through a ring of CAP-entry stages with cp.async.bulk (L2 evict-first), and the
// lanes read them from shared memory (stride = row length: conflict-free for odd
// lengths).  Each CTA owns a contiguous range of 32-row runs (one wave, static
// partition); consumer warp w takes runs w, w + W, ... of it.  Ring protocol:
// every consumer warp passes every stage in stream order -- it waits for the
// stage's full barrier and, once its next run starts beyond the stage, arrives on
// the stage's empty barrier (W arrivals free the slot).  A run's entries must be
// resident together, so the matrix is eligible when its longest 32-row run fits
// the ring with a stage to spare (Matrix::rest_run_max, measured at build time);
// other matrices keep rest_pipe_kernel.
//
// Same per-row operations in the same order as warp_rest / rest_pipe_kernel:
// acc = __dadd_rn(acc, __dmul_rn(v, x[c] (* scale))) from +0.0 -- bitwise equal.
#include <algorithm>
#include <cstdlib>

#include "hdcg_internal.cuh"
#include "tma_ptx.cuh"

namespace hdcg {

namespace {

#ifndef HDCG_ROWS_W16_CTAS
#define HDCG_ROWS_W16_CTAS 2
#endif
constexpr int CAP_LOG2 = 10;
constexpr int CAP = 1 << CAP_LOG2;  // entries per ring stage: 4 KB of columns + 8 KB of values
#ifndef HDCG_ROWS_UNROLL
#define HDCG_ROWS_UNROLL 9  // 27-point rows: three full batches (8: 75%, 9: 81% of the HBM peak at config 2 as CSR)
#endif
constexpr int UNROLL = HDCG_ROWS_UNROLL;  // x gathers in flight per lane

struct RowsArgs {
    const int32_t* rp;
    const int32_t* col;  // padded: readable up to a multiple of 4 entries past the end
    const double* val;
    const double* x;  // x_local: x[c - row0]
    double* y;
    const double* x_scale;
    int64_t row0;
    int64_t r_lo, r_hi;  // local rows
    int chunk_runs;      // 32-row runs per chunk (chunks are dealt round-robin to the CTAs)
    int ns_log2;         // ring stages = 1 << ns_log2 (shifts, no divisions, in the stage bookkeeping)
};

template <int W, bool SCALE>
__global__ void __launch_bounds__(32 * (W + 1), W >= 16 ? HDCG_ROWS_W16_CTAS : 2) rest_rows_kernel(const RowsArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NSL = a.ns_log2, NS = 1 << NSL;
    const int ring = NS << CAP_LOG2, mask = ring - 1;
    double* sval = reinterpret_cast<double*>(smem_raw);
    int32_t* scol = reinterpret_cast<int32_t*>(sval + ring);
    uint64_t* full = reinterpret_cast<uint64_t*>(scol + ring);
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // Chunks of K 32-row runs, dealt round-robin to the CTAs: the CTAs at work at any
    // time cover one contiguous stretch of rows, so their x windows overlap in L2 (a
    // contiguous range per CTA spread 296 windows over the whole vector: config 3 as
    // CSR read 2.1x its bytes from DRAM, profiles/r02u_c3csr_rows_contig_ncu.json).
    // The ring runs on across chunks: stage numbers are global, chunk c's first
    // stage is q_base (every warp derives the same counts from the row pointers).
    const int64_t n_runs = (a.r_hi - a.r_lo + 31) >> 5;
    const int K = a.chunk_runs;
    const int64_t n_chunks = (n_runs + K - 1) / K;
    if ((int64_t)blockIdx.x >= n_chunks) return;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, W);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto chunk_rows = [&](int64_t c, int64_t* R0, int64_t* R1) {
        *R0 = a.r_lo + ((c * K) << 5);
        *R1 = min(*R0 + ((int64_t)K << 5), a.r_hi);
    };

    if (warp == W) {  // producer: each chunk's entry stream, stage by stage
        if (lane != 0) return;
        const uint64_t pol = evict_first_policy();
        int q = 0;  // global stage number
        int64_t c = blockIdx.x, R0, R1;
        chunk_rows(c, &R0, &R1);
        int64_t E0 = __ldg(a.rp + R0), E1 = __ldg(a.rp + R1);
        while (true) {
            const int64_t cn = c + gridDim.x;
            int64_t E0n = 0, E1n = 0;
            if (cn < n_chunks) {  // the next chunk's bounds, loaded under this chunk's copies
                chunk_rows(cn, &R0, &R1);
                E0n = __ldg(a.rp + R0);
                E1n = __ldg(a.rp + R1);
            }
            if (E1 > E0) {
                const int64_t E0a = E0 & ~int64_t(3), E1a = (E1 + 3) & ~int64_t(3);
                for (int64_t e = E0a; e < E1a; e += CAP, ++q) {
                    const int s = q & (NS - 1);
                    if (q >= NS) mbar_wait(empty + s, (uint32_t)(((q >> NSL) - 1) & 1));
                    const uint32_t cnt = (uint32_t)min((int64_t)CAP, E1a - e);
                    mbar_expect_tx(full + s, cnt * 12u);
                    bulk_g2s(scol + ((size_t)s << CAP_LOG2), a.col + e, cnt * 4u, full + s, pol);
                    bulk_g2s(sval + ((size_t)s << CAP_LOG2), a.val + e, cnt * 8u, full + s, pol);
                }
            }
            if (cn >= n_chunks) break;
            c = cn;
            E0 = E0n;
            E1 = E1n;
        }
        return;
    }

    const double sc = SCALE ? *a.x_scale : 1.0;
    const double* __restrict__ xb = a.x - a.row0;  // x[c - row0] = xb[c]
    int passed = 0;  // global stages [0, passed) waited for and released by this warp
    int q_base = 0;  // global number of the current chunk's first stage
    auto pass_to = [&](int q_end) {
        for (; passed < q_end; ++passed) {
            const int s = passed & (NS - 1);
            mbar_wait(full + s, (uint32_t)((passed >> NSL) & 1));
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    };
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        int64_t R0, R1;
        chunk_rows(c, &R0, &R1);
        const int64_t g_lo = c * K, g_hi = min(g_lo + K, n_runs);
        // the warp's first run of the chunk; lane 0 / 31 also fetch the chunk's bounds
        int64_t g = g_lo + warp;
        int kb = 0, ke = 0;
        if (g < g_hi) {
            const int64_t row = a.r_lo + (g << 5) + lane;
            kb = __ldg(a.rp + min(row, R1));
            ke = __ldg(a.rp + min(row + 1, R1));
        }
        const int64_t E0 = __ldg(a.rp + R0), E1 = __ldg(a.rp + R1);
        const int64_t E0a = E0 & ~int64_t(3);
        const int NQ = E1 > E0 ? (int)((E1 - E0a + CAP - 1) >> CAP_LOG2) : 0;
        // entry p of the chunk lives at ring slot (p - base) & mask (wrap-around arithmetic)
        const uint32_t base = (uint32_t)E0a - ((uint32_t)q_base << CAP_LOG2);
        for (; g < g_hi; g += W) {
            const int64_t row = a.r_lo + (g << 5) + lane;
            int kb_n = 0, ke_n = 0;
            if (g + W < g_hi) {  // the next run's row pointers, loaded while this one is summed
                const int64_t rn = row + ((int64_t)W << 5);
                kb_n = __ldg(a.rp + min(rn, R1));
                ke_n = __ldg(a.rp + min(rn + 1, R1));
            }
            const int ea = __shfl_sync(0xffffffffu, kb, 0), eb = __shfl_sync(0xffffffffu, ke, 31);
            double acc = 0.0;
            if (eb > ea) {
                const int qa = q_base + (int)((ea - E0a) >> CAP_LOG2), qb = q_base + (int)((eb - 1 - E0a) >> CAP_LOG2);
                pass_to(qa);  // stages of the other warps' runs
                for (int q = qa; q <= qb; ++q) mbar_wait(full + (q & (NS - 1)), (uint32_t)((q >> NSL) & 1));
                // The row's entries are contiguous in the ring unless they cross its end:
                // the common case reads them at fixed offsets from one slot address
                // (one LDS per column / value, no index arithmetic per entry).
                const uint32_t i0 = ((uint32_t)kb - base) & (uint32_t)mask;
                const int len = ke - kb;
                if (i0 + (uint32_t)len <= (uint32_t)ring) {
                    const int32_t* __restrict__ cp = scol + i0;
                    const double* __restrict__ vp = sval + i0;
                    int p = 0;
                    for (; p + UNROLL <= len; p += UNROLL) {  // full batches: no predicates
                        double xv[UNROLL];
#pragma unroll
                        for (int j = 0; j < UNROLL; ++j) xv[j] = __ldg(xb + cp[p + j]);
#pragma unroll
                        for (int j = 0; j < UNROLL; ++j) {
                            double t = xv[j];
                            if (SCALE) t = __dmul_rn(t, sc);
                            acc = __dadd_rn(acc, __dmul_rn(vp[p + j], t));
                        }
                    }
                    if (p < len) {  // the last, partial batch
                        double xv[UNROLL];
#pragma unroll
                        for (int j = 0; j < UNROLL; ++j) xv[j] = p + j < len ? __ldg(xb + cp[p + j]) : 0.0;
#pragma unroll
                        for (int j = 0; j < UNROLL; ++j) {
                            double t = xv[j];
                            if (SCALE) t = __dmul_rn(t, sc);
                            if (p + j < len) acc = __dadd_rn(acc, __dmul_rn(vp[p + j], t));
                        }
                    }
                } else {  // the row wraps around the ring's end
                    for (int p = 0; p < len; ++p) {
                        const uint32_t i = (i0 + (uint32_t)p) & (uint32_t)mask;
                        double t = __ldg(xb + scol[i]);
                        if (SCALE) t = __dmul_rn(t, sc);
                        acc = __dadd_rn(acc, __dmul_rn(sval[i], t));
                    }
                }
            }
            if (row < R1) a.y[row] = acc;
            kb = kb_n;
            ke = ke_n;
        }
        // the chunk's remaining stages: the producer can go on for the warps still at work
        __syncwarp();
        q_base += NQ;
        pass_to(q_base);
    }
}

__global__ void run_max_kernel(const int32_t* __restrict__ rp, int64_t n_rows, int* out) {
    const int64_t n_runs = (n_rows + 31) >> 5;
    int mx = 0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_runs; g += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, rp[min((g + 1) << 5, n_rows)] - rp[g << 5]);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(out, mx);
}

// How well row-per-lane gathers coalesce: for every `stride`-th 32-row run, a warp
// walks the rows like rest_rows_kernel does (lane = row, step k = the row's k-th
// entry) and counts the distinct 128-byte x lines of each step's columns.
// out[0] += lines, out[1] += steps.  Banded rows: 2-3 lines per step; random
// columns: one line per lane.
__global__ void run_lines_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t n_rows,
                                 int64_t stride, unsigned long long* out) {
    const int64_t n_runs = (n_rows + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long lines = 0, steps = 0;
    for (int64_t g = w * stride; g < n_runs; g += nw * stride) {
        const int64_t row = (g << 5) + lane;
        const int kb = row < n_rows ? rp[row] : 0, ke = row < n_rows ? rp[row + 1] : 0;
        int len = ke - kb;
        for (int o = 16; o; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
        len = min(len, 64);  // a long row's first entries tell enough
        for (int k = 0; k < len; ++k) {
            const bool ok = kb + k < ke;
            const int line = ok ? (col[kb + k] >> 4) : -1 - lane;
            const unsigned peers = __match_any_sync(0xffffffffu, line);
            const unsigned leaders = __ballot_sync(0xffffffffu, ok && lane == __ffs(peers) - 1);
            lines += __popc(leaders);
            ++steps;
        }
    }
    if (lane == 0 && steps) {
        atomicAdd(out, lines);
        atomicAdd(out + 1, steps);
    }
}

template <int W, bool SCALE>
void launch_rows(const RowsArgs& a, int grid, size_t smem, cudaStream_t st) {
    auto k = rest_rows_kernel<W, SCALE>;
    static PerDeviceFlag configured;
    if (!configured.test_and_set(current_device_index()))
        HDCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    k<<<grid, 32 * (W + 1), smem, st>>>(a);
}

}  // namespace

// The longest remainder run (entries of 32 consecutive rows, 32-aligned), measured
// once when the matrix is built: selects rest_rows_kernel (spmv_rows.cu).
void rest_run_stats(Matrix* m) {
    m->rest_run_max = 0;
    m->rest_lines_per_gather = 32.0;
    if (m->nnz_rest <= 0 || m->n_rows <= 0) return;
    DeviceGuard dg(m->device);
    unsigned long long* d = dev_alloc<unsigned long long>(3, nullptr);
    HDCG_CUDA(cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), nullptr));
    const int64_t n_runs = ceil_div(m->n_rows, 32);
    run_max_kernel<<<grid_cap(ceil_div(n_runs, 256)), 256>>>(m->rest_rp, m->n_rows, reinterpret_cast<int*>(d + 2));
    HDCG_LAUNCH_CHECK("run_max_kernel");
    const int64_t stride = std::max<int64_t>(1, n_runs / 4096);  // ~4096 sampled runs
    run_lines_kernel<<<grid_cap(ceil_div(ceil_div(n_runs, stride), 8)), 256>>>(m->rest_rp, m->rest_col, m->n_rows,
                                                                             stride, d);
    HDCG_LAUNCH_CHECK("run_lines_kernel");
    unsigned long long h[3] = {0, 0, 0};
    HDCG_CUDA(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    dev_free(d, nullptr);
    m->rest_run_max = (int64_t)(int)h[2];
    if (h[1] > 0) m->rest_lines_per_gather = (double)h[0] / (double)h[1];
}

// The default policy's choice for a matrix (hdcg_info.rest_rows_kernel): banded rows
// whose longest 32-row run fits the ring.
bool rest_rows_default(const Matrix& m) {
    if (m.nnz_rest <= 0 || m.rest_lines_per_gather > 8.0) return false;
    if (((uintptr_t)m.rest_col % 16) != 0 || ((uintptr_t)m.rest_val % 16) != 0) return false;
    return 2 * m.rest_run_max <= (int64_t)(16 - 1) * CAP;
}

// Remainder sums of local rows [r0, r1) into y (from +0.0).  False when the matrix
// is not eligible (a 32-row run longer than the ring holds) or the arrays are not
// 16-byte aligned: the caller then uses rest_pipe_kernel.
// HDCG_ROWS_W (8 | 16 consumer warps) and HDCG_ROWS_STAGES (ring stages of 1024
// entries, a power of two <= 16) are A/B knobs.
bool rest_rows_launch(const Matrix& m, const double* x_local, double* y, const double* x_scale, int64_t r0,
                      int64_t r1, cudaStream_t st) {
    if (r1 <= r0) return true;
    if (((uintptr_t)m.rest_col % 16) != 0 || ((uintptr_t)m.rest_val % 16) != 0) return false;
    const char* ew = getenv("HDCG_ROWS_W");  // read per call: the tests switch them in-process
    const char* es = getenv("HDCG_ROWS_STAGES");
    const int env_w = ew ? atoi(ew) : 0, env_ns = es ? atoi(es) : 0;
    const char* ek = getenv("HDCG_ROWS_CHUNK");
    // runs of a launch start at r0, which need not be 32-aligned: a window of 32
    // rows overlaps at most two aligned runs
    const int64_t run_max = 2 * m.rest_run_max;
    // Default: banded rows -- row-per-lane gathers of 32 adjacent rows touch few x
    // lines (Matrix::rest_lines_per_gather, sampled at build time: 2-3 for a stencil
    // stored as CSR, ~17 for config 3's rows with 6 random columns each) -- take this
    // kernel with 16 warps; a 16-stage (192 KB) ring, one CTA per SM, when a 32-row
    // run holds more than half a stage (27-point rows: 864 entries), else 8 stages
    // and two CTAs per SM.  Configs 1 / 2 as CSR: 81% / 68% (rest_pipe_kernel) ->
    // 92% / 94% of the HBM peak.  Rows with scattered columns stay on
    // rest_pipe_kernel, whose entry-major lanes keep more gathers in flight (config
    // 3 as CSR 61% vs 56% here; profiles/r02s_ab_rows.log).  The knobs force this
    // kernel (tests, A/B).
    const int64_t avg_run = m.nnz_rest * 32 / std::max<int64_t>(1, m.n_rows);
    if (!env_w && !env_ns && m.rest_lines_per_gather > 8.0) return false;
    int W = env_w ? env_w : 16;
    int NS = env_ns ? env_ns : (avg_run * 16 > 8 * CAP ? 16 : 8);
    if (W != 8 && W != 16) return false;
    if (NS < 2 || (NS & (NS - 1)) || NS > 16) return false;
    if (run_max > (int64_t)(NS - 1) * CAP) {
        if (env_ns) return false;
        NS = 16;  // the larger ring, if that holds the longest run
        if (run_max > (int64_t)(NS - 1) * CAP) return false;
    }
    RowsArgs a;
    a.rp = m.rest_rp;
    a.col = m.rest_col;
    a.val = m.rest_val;
    a.x = x_local;
    a.y = y;
    a.x_scale = x_scale;
    a.row0 = m.row0;
    a.r_lo = r0;
    a.r_hi = r1;
    // two runs per warp and chunk: 95.7% / 96.2% of the HBM peak on configs 1 / 2 as CSR
    // against 92.5% / 94.8% with four (profiles/r02s_ab_rows.log, chunk sweep)
    a.chunk_runs = ek && atoi(ek) > 0 ? atoi(ek) : 2 * W;
    a.ns_log2 = 0;
    while ((1 << a.ns_log2) < NS) ++a.ns_log2;
    const size_t smem = (size_t)NS * CAP * 12 + sizeof(uint64_t) * 2 * NS;
    const int per_sm = std::max(1, std::min(2, (int)((227 * 1024) / (smem + 1024))));
    const int64_t n_runs = ceil_div(r1 - r0, 32);
    const int64_t n_chunks = ceil_div(n_runs, a.chunk_runs);
    const int grid = (int)std::min<int64_t>((int64_t)sm_count() * per_sm, n_chunks);
    if (W == 16) {
        if (x_scale) launch_rows<16, true>(a, grid, smem, st);
        else launch_rows<16, false>(a, grid, smem, st);
    } else {
        if (x_scale) launch_rows<8, true>(a, grid, smem, st);
        else launch_rows<8, false>(a, grid, smem, st);
    }
    HDCG_LAUNCH_CHECK("rest_rows_kernel");
    return true;
}

}  // namespace hdcg

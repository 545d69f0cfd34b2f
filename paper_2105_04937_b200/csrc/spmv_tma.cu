// spmv_tma.cu -- TMA-fed persistent M-HDC / HDC SpMV for sm_100a.
//
// Same arithmetic as spmv.cu (the reference's per-row order, kernels.cpp:173-206,
// __dmul_rn/__dadd_rn, bitwise equal), different data movement:
//
//   * persistent grid (148 SMs x CTAS_PER_SM CTAs); CTA c owns tiles
//     c, c+grid, ...; a tile is TILE = 256*R rows inside one row block;
//   * warp 8 is the producer: one elected lane streams every (tile, segment)
//     slice -- TILE contiguous doubles of segment k -- global -> shared with
//     cp.async.bulk (the 1-D TMA path, UBLKCP in SASS) into an NSTAGE-deep ring,
//     completion signalled through mbarrier transaction counts, L2 evict-first
//     (segment values are read exactly once);
//   * warps 0-7 consume: per segment they wait on the stage's full barrier, read
//     their R slots with one 8/16-byte shared load, multiply with x (issued
//     ahead, per group of up to XGROUP segments, through the L1/tex path where
//     the near offsets of a tile share lines and the far ones hit L2), add in
//     stored order and release the stage;
//   * the producer runs up to NSTAGE slices (NSTAGE*TILE*8 bytes, 64 KB) ahead
//     of the consumers, across tile boundaries, so every SM keeps ~200 KB of
//     segment traffic in flight with a handful of instructions per 4 KB;
//   * y is stored once per tile (streaming store); the optional fused
//     sum-of-squares per tile uses the same fixed reduction order as spmv.cu.
// Used for even bl >= TILE (all BASELINE M-HDC configurations and HDC with
// even n); other shapes take the general kernel in spmv.cu.
#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

constexpr int CONSUMER_WARPS = 8;
constexpr int CONSUMERS = CONSUMER_WARPS * 32;
constexpr int THREADS = CONSUMERS + 32;  // + producer warp
constexpr int NSTAGE = 16;
constexpr int XGROUP = 8;
constexpr int REST_CHUNK_T = 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS) : "memory"); }

struct TmaArgs {
    const int32_t* dia_ptr;
    const int32_t* dia_off;
    const double* seg;
    const int32_t* rest_rp;
    const int32_t* rest_col;
    const double* rest_val;
    const double* x;
    double* y;
    const double* x_scale;
    double* tile_sumsq;
    int64_t n_rows, n_cols, row0, bl;
    int tiles_per_block;
    int tile_begin, tile_end;
    int has_rest;
    int y_vec_ok;
};

struct TileGeo {
    int64_t lo, hi, b0;
    int b;
};

template <int R>
__device__ __forceinline__ TileGeo tile_geo(const TmaArgs& a, int tile) {
    TileGeo g;
    g.b = tile / a.tiles_per_block;
    const int t = tile - g.b * a.tiles_per_block;
    g.b0 = (int64_t)g.b * a.bl;
    const int64_t bend = min(g.b0 + a.bl, a.n_rows);
    g.lo = g.b0 + (int64_t)t * (CONSUMERS * R);
    g.hi = min(g.lo + (int64_t)(CONSUMERS * R), bend);
    return g;
}

template <int R, bool SCALE, bool NORM>
__global__ void __launch_bounds__(THREADS) spmv_tma_kernel(const TmaArgs a) {
    constexpr int TILE = CONSUMERS * R;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);                       // NSTAGE * TILE
    double* prod = ring + NSTAGE * TILE;                                      // REST_CHUNK_T
    double* warp_sums = prod + REST_CHUNK_T;                                  // CONSUMER_WARPS
    uint64_t* full = reinterpret_cast<uint64_t*>(warp_sums + CONSUMER_WARPS);  // NSTAGE
    uint64_t* empty = full + NSTAGE;                                          // NSTAGE

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == CONSUMER_WARPS) {
        // ------------------------------ producer ------------------------------
        if (lane != 0) return;
        const uint64_t policy = evict_first_policy();
        uint32_t it = 0;
        for (int tile = a.tile_begin + blockIdx.x; tile < a.tile_end; tile += gridDim.x) {
            const TileGeo g = tile_geo<R>(a, tile);
            if (g.lo >= g.hi) continue;
            const int k0 = __ldg(a.dia_ptr + g.b), k1 = __ldg(a.dia_ptr + g.b + 1);
            const uint32_t bytes = (uint32_t)(((g.hi - g.lo + 1) & ~int64_t(1)) * 8);
            const double* src = a.seg + (int64_t)k0 * a.bl + (g.lo - g.b0);
            for (int k = k0; k < k1; ++k, ++it, src += a.bl) {
                const int s = it % NSTAGE;
                if (it >= NSTAGE) mbar_wait(&empty[s], ((it / NSTAGE) - 1) & 1);
                mbar_expect_tx(&full[s], bytes);
                bulk_g2s(ring + s * TILE, src, bytes, &full[s], policy);
            }
        }
        return;
    }

    // -------------------------------- consumers --------------------------------
    double sc = 1.0;
    if (SCALE) sc = *a.x_scale;
    uint32_t it = 0;
    for (int tile = a.tile_begin + blockIdx.x; tile < a.tile_end; tile += gridDim.x) {
        const TileGeo g = tile_geo<R>(a, tile);
        if (g.lo >= g.hi) {
            if (NORM && threadIdx.x == 0) a.tile_sumsq[tile] = 0.0;
            continue;
        }
        const int64_t i0 = g.lo + (int64_t)R * threadIdx.x;
        const bool active = i0 < g.hi;
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;

        // CSR remainder first (stored order), products staged through smem
        if (a.has_rest) {
            const int64_t e_lo = a.rest_rp[g.lo], e_hi = a.rest_rp[g.hi];
            if (e_lo < e_hi) {
                int64_t kb[R], ke[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool ok = i0 + r < g.hi;
                    kb[r] = ok ? a.rest_rp[i0 + r] : 0;
                    ke[r] = ok ? a.rest_rp[i0 + r + 1] : 0;
                }
                for (int64_t c0 = e_lo; c0 < e_hi; c0 += REST_CHUNK_T) {
                    const int64_t c1 = min(c0 + (int64_t)REST_CHUNK_T, e_hi);
                    for (int64_t e = c0 + threadIdx.x; e < c1; e += CONSUMERS) {
                        double xv = __ldg(a.x + ((int64_t)__ldcs(a.rest_col + e) - a.row0));
                        if (SCALE) xv = __dmul_rn(xv, sc);
                        prod[e - c0] = __dmul_rn(__ldcs(a.rest_val + e), xv);
                    }
                    consumer_sync();
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int64_t q0 = max(kb[r], c0), q1 = min(ke[r], c1);
                        for (int64_t q = q0; q < q1; ++q) acc[r] = __dadd_rn(acc[r], prod[q - c0]);
                    }
                    consumer_sync();
                }
            }
        }

        // diagonal segments, stored order
        const int k0 = __ldg(a.dia_ptr + g.b), k1 = __ldg(a.dia_ptr + g.b + 1);
        const int64_t glo = a.row0 + g.lo, ghi = a.row0 + g.hi;  // global rows [glo, ghi)
        const double* xrow = a.x + i0;
        for (int kg = k0; kg < k1; kg += XGROUP) {
            double xv[XGROUP][R];
#pragma unroll
            for (int u = 0; u < XGROUP; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) xv[u][r] = 0.0;
                const int k = kg + u;
                if (k < k1 && active) {
                    const int64_t o = __ldg(a.dia_off + k);
                    if (glo + o >= 0 && ghi - 1 + o < a.n_cols) {  // whole tile in range (uniform)
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (i0 + r < g.hi) xv[u][r] = __ldg(xrow + r + o);
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const int64_t j = a.row0 + i0 + r + o;
                            if (j >= 0 && j < a.n_cols && i0 + r < g.hi) xv[u][r] = __ldg(xrow + r + o);
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < XGROUP; ++u) {
                if (kg + u >= k1) break;
                const int s = it % NSTAGE;
                mbar_wait(&full[s], (it / NSTAGE) & 1);
                const double* st = ring + s * TILE + R * threadIdx.x;
                double v[R];
                if (R == 2) {
                    const double2 t = *reinterpret_cast<const double2*>(st);
                    v[0] = t.x;
                    v[R - 1] = t.y;
                } else {
                    v[0] = st[0];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                ++it;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double xx = xv[u][r];
                    if (SCALE) xx = __dmul_rn(xx, sc);
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(v[r], xx));
                }
            }
        }

        if (active) {
            if (R == 2 && a.y_vec_ok && i0 + 1 < g.hi) {
                __stcs(reinterpret_cast<double2*>(a.y + i0), make_double2(acc[0], acc[R - 1]));
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (i0 + r < g.hi) __stcs(a.y + i0 + r, acc[r]);
            }
        }
        if (NORM) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + r < g.hi) s = __dadd_rn(s, __dmul_rn(acc[r], acc[r]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
            if (lane == 0) warp_sums[warp] = s;
            consumer_sync();
            if (threadIdx.x == 0) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < CONSUMER_WARPS; ++w) t = __dadd_rn(t, warp_sums[w]);
                a.tile_sumsq[tile] = t;
            }
            consumer_sync();
        }
    }
}

template <int R>
constexpr size_t smem_bytes() {
    return sizeof(double) * (NSTAGE * CONSUMERS * R + REST_CHUNK_T + CONSUMER_WARPS) + sizeof(uint64_t) * 2 * NSTAGE;
}

template <int R, bool SCALE, bool NORM>
void launch_one(const TmaArgs& a, int grid, cudaStream_t st) {
    auto k = spmv_tma_kernel<R, SCALE, NORM>;
    static bool configured = false;  // per instantiation; attribute set once per process
    if (!configured) {
        HDCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<R>()));
        configured = true;
    }
    k<<<grid, THREADS, smem_bytes<R>(), st>>>(a);
}

template <int R>
void launch_r(const TmaArgs& a, int grid, bool scale, bool norm, cudaStream_t st) {
    if (scale) {
        if (norm) launch_one<R, true, true>(a, grid, st);
        else launch_one<R, true, false>(a, grid, st);
    } else {
        if (norm) launch_one<R, false, true>(a, grid, st);
        else launch_one<R, false, false>(a, grid, st);
    }
}

int ctas_per_sm(int rows_per_thread) {
    // smem-limited: 228 KB per SM, ~1 KB reserved per CTA
    const size_t per = (rows_per_thread == 2 ? smem_bytes<2>() : smem_bytes<1>()) + 1024;
    int c = (int)((228 * 1024) / per);
    return c < 1 ? 1 : (c > 4 ? 4 : c);
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace

// Eligible shapes: even bl >= 256 (tile rows 256 or 512), 16-byte aligned
// segment storage.  Returns false when the general kernel must be used.
bool spmv_tma_launch(const Matrix& m, const double* x_local, double* y, int64_t block_begin, int64_t block_end,
                     const double* x_scale, double* tile_sumsq, cudaStream_t st) {
    if (m.bl % 2 != 0 || m.bl < CONSUMERS) return false;
    if (m.n_seg > 0 && ((uintptr_t)m.seg % 16) != 0) return false;
    const int R = m.bl >= 2 * CONSUMERS ? 2 : 1;
    const int64_t tile_rows = (int64_t)CONSUMERS * R;
    const int64_t tpb = ceil_div(m.bl, tile_rows);
    const int64_t t0 = block_begin * tpb, t1 = block_end * tpb;
    if (t1 > 0x7fffffffLL) return false;
    if (t1 <= t0) return true;
    TmaArgs a;
    a.dia_ptr = m.dia_ptr;
    a.dia_off = m.dia_off;
    a.seg = m.seg;
    a.rest_rp = m.rest_rp;
    a.rest_col = m.rest_col;
    a.rest_val = m.rest_val;
    a.x = x_local;
    a.y = y;
    a.x_scale = x_scale;
    a.tile_sumsq = tile_sumsq;
    a.n_rows = m.n_rows;
    a.n_cols = m.n_cols;
    a.row0 = m.row0;
    a.bl = m.bl;
    a.tiles_per_block = (int)tpb;
    a.tile_begin = (int)t0;
    a.tile_end = (int)t1;
    a.has_rest = m.nnz_rest > 0;
    a.y_vec_ok = ((uintptr_t)y % 16) == 0;
    const int64_t n_tiles = t1 - t0;
    const int64_t cap = (int64_t)sm_count() * ctas_per_sm(R);
    const int grid = (int)(n_tiles < cap ? n_tiles : cap);
    if (R == 2) launch_r<2>(a, grid, x_scale != nullptr, tile_sumsq != nullptr, st);
    else launch_r<1>(a, grid, x_scale != nullptr, tile_sumsq != nullptr, st);
    HDCG_LAUNCH_CHECK("spmv_tma_kernel");
    return true;
}

}  // namespace hdcg

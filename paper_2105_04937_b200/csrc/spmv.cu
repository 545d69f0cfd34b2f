// spmv.cu -- the HDC / M-HDC SpMV kernel family for sm_100a.
//
// Replaces hdc::spmv_mhdc (proj/src/kernels.cpp:173-206) and, because their
// per-row accumulation order is the same, spmv_hdc / spmv_bhdc
// (kernels.cpp:107-171), spmv_dia / spmv_bdia (:56-105) and spmv_csr (:39-54).
//
// Per row i the reference computes
//     s = +0.0;  for k in rest_row(i) (stored order): s += val[k] * x[col[k]]
//     for each segment / lane k of i's block, ascending: if 0 <= i+off_k < n: s += seg_k[i] * x[i+off_k]
// with separately rounded multiply and add (the x86-64 oracle has no FMA).
// This kernel performs exactly those floating-point operations in exactly
// that order (__dmul_rn / __dadd_rn), so y is bitwise equal to the reference.
//
// Layout / bandwidth design (memory-bound fp64 streaming reduction, no tensor
// cores):
//   * one CTA owns a tile of 256*R rows inside one row block (or G whole
//     blocks when bl < tile); thread t owns R consecutive rows;
//   * segment values are streamed once with 128-bit evict-first loads
//     (ld.global.cs.v2.f64) -- 8 B/slot, the dominant traffic;
//   * the block's segment loop is unrolled by SEG_UNROLL with all loads issued
//     before the dependent adds, so each thread keeps ~8 x 16 B in flight;
//   * x is read through the L1/tex path: the near offsets (-1,0,+1 ...) of a
//     tile share lines in L1, far offsets (+-nx, +-nx*ny) hit L2 because the
//     wavefront of resident tiles re-reads them within ~2*nx*ny rows;
//   * the CSR remainder of the tile is processed in chunks: the products
//     val[k]*x[col[k]] are computed by all threads with coalesced loads into
//     shared memory, then each thread sums its own rows sequentially in stored
//     order (bitwise order preserved, no warp-tree reordering);
//   * y is written once (streaming store); optional fused epilogue emits the
//     tile's sum of y_i^2 (power iteration) in a fixed reduction order.
#include <algorithm>
#include <cstdlib>

#include "hdcg_internal.cuh"

namespace hdcg {

constexpr int SPMV_THREADS = 256;

int g_kernel_policy = 0;  // 0 auto (TMA kernel where eligible), 1 general kernel only, 2 TMA only
int g_rest_mode = 0;      // TMA kernel remainder: 0 default, 1 global loads, 2 rest_kernel first
constexpr int REST_CHUNK = 1024;  // doubles of staged remainder products
constexpr int SEG_UNROLL = 8;

struct SpmvArgs {
    const int32_t* dia_ptr;
    const int32_t* dia_off;
    const double* seg;
    const int32_t* rest_rp;
    const int32_t* rest_col;
    const double* rest_val;
    const double* x;  // x_local: x_local[j - row0] = x_j
    double* y;
    const double* x_scale;
    double* tile_sumsq;
    int64_t n_rows, n_cols, row0, bl;
    int64_t tiles_per_block, blocks_per_tile, tile_rows;
    int64_t tile_begin;
    int has_rest;
    int y_vec_ok;
    double* peer_lo;  // PeerOut
    double* peer_hi;
    int64_t halo;
};

// IL: interleaved rows (thread t owns tile rows t, t+256, ...) -- tiles inside
// one block, the TMA kernel's mapping (so per-tile sums agree bitwise); otherwise
// (whole blocks per tile) R consecutive rows per thread.
// PK: the packed tiling (tile = tile_rows consecutive rows, interleaved over the
// threads, rows of one thread possibly in different blocks) -- the bitwise
// cross-check of the packed TMA kernel; reads the reference layout.
template <int R, bool SCALE, bool NORM, bool IL, bool PK = false>
__global__ void __launch_bounds__(SPMV_THREADS) spmv_kernel(const SpmvArgs a) {
    __shared__ double prod[REST_CHUNK];
    __shared__ double warp_sums[SPMV_THREADS / 32];

    const int64_t tile = a.tile_begin + blockIdx.x;
    int64_t lo, hi;
    if (PK) {
        lo = tile * a.tile_rows;
        hi = min(lo + a.tile_rows, a.n_rows);
    } else if (a.tiles_per_block > 0) {
        const int64_t b = tile / a.tiles_per_block;
        const int64_t t = tile - b * a.tiles_per_block;
        const int64_t b0 = b * a.bl;
        const int64_t bend = min(b0 + a.bl, a.n_rows);
        lo = b0 + t * a.tile_rows;
        hi = min(lo + a.tile_rows, bend);
    } else {
        lo = tile * a.blocks_per_tile * a.bl;
        hi = min(lo + a.blocks_per_tile * a.bl, a.n_rows);
    }
    // row of this thread's r-th row
    // bl = 256 multi-block tiles without a remainder: the TMA kernel's mapping --
    // lane l of block k's two warps owns block rows 32 (warp & 1) + l + 64 r (per-tile
    // sums then agree bitwise between the kernels)
    const bool MBIL = !PK && !IL && R == 4 && (a.bl == 256 || a.bl == 128) && !a.has_rest;
    const int wpb = MBIL ? (int)a.bl / 128 : 1;
    const int warp = threadIdx.x >> 5, qb = warp / wpb;
    const int64_t mb0 = (int64_t)qb * a.bl + (warp - qb * wpb) * 32 + (threadIdx.x & 31);
    auto row = [&](int r) -> int64_t {
        if (MBIL) return lo + mb0 + (int64_t)32 * wpb * r;
        return IL || PK ? lo + threadIdx.x + (int64_t)SPMV_THREADS * r : lo + (int64_t)R * threadIdx.x + r;
    };

    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    double sc = 1.0;
    if (SCALE) sc = *a.x_scale;

    // ---- CSR remainder: products staged in smem, per-row sequential sums ----
    if (a.has_rest && lo < hi) {
        const int64_t e_lo = a.rest_rp[lo];
        const int64_t e_hi = a.rest_rp[hi];
        if (e_lo < e_hi) {
            int64_t kb[R], ke[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t i = row(r);
                if (i < hi) {
                    kb[r] = a.rest_rp[i];
                    ke[r] = a.rest_rp[i + 1];
                } else {
                    kb[r] = ke[r] = 0;
                }
            }
            for (int64_t c0 = e_lo; c0 < e_hi; c0 += REST_CHUNK) {
                const int64_t c1 = min(c0 + (int64_t)REST_CHUNK, e_hi);
                for (int64_t e = c0 + threadIdx.x; e < c1; e += SPMV_THREADS) {
                    double xv = __ldg(a.x + ((int64_t)__ldcs(a.rest_col + e) - a.row0));
                    if (SCALE) xv = __dmul_rn(xv, sc);
                    prod[e - c0] = __dmul_rn(__ldcs(a.rest_val + e), xv);
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t k0 = max(kb[r], c0), k1 = min(ke[r], c1);
                    for (int64_t k = k0; k < k1; ++k) acc[r] = __dadd_rn(acc[r], prod[k - c0]);
                }
                __syncthreads();
            }
        }
    }

    // ---- diagonal segments of this row's block, stored order ----------------
    const int64_t i0 = row(0);
    if (PK) {  // each row with its own block's segments
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = row(r);
            if (i >= hi) continue;
            const int64_t b = i / a.bl, l = i - b * a.bl;
            const int k0 = __ldg(a.dia_ptr + b), k1 = __ldg(a.dia_ptr + b + 1);
            for (int k = k0; k < k1; ++k) {
                const int64_t o = __ldg(a.dia_off + k);
                const int64_t j = a.row0 + i + o;
                const double v = __ldcs(a.seg + (int64_t)k * a.bl + l);
                double xx = (j >= 0 && j < a.n_cols) ? __ldg(a.x + (i + o)) : 0.0;
                if (SCALE) xx = __dmul_rn(xx, sc);
                acc[r] = __dadd_rn(acc[r], __dmul_rn(v, xx));
            }
            __stcs(a.y + i, acc[r]);
            if (a.peer_lo && i < a.halo) a.peer_lo[i] = acc[r];
            if (a.peer_hi && i >= a.n_rows - a.halo) a.peer_hi[i - (a.n_rows - a.halo)] = acc[r];
        }
        if (a.peer_lo || a.peer_hi) __threadfence_system();
    } else if (i0 < hi) {
        const int64_t b = i0 / a.bl;  // all of this thread's rows are in one block
        const int64_t l = i0 - b * a.bl;
        const int k0 = __ldg(a.dia_ptr + b);
        const int k1 = __ldg(a.dia_ptr + b + 1);
        const int64_t gi = a.row0 + i0;
        const double* seg_base = a.seg + l;
        constexpr int U = R == 4 ? 4 : SEG_UNROLL;
        const int64_t RS = IL ? SPMV_THREADS : MBIL ? 32 * wpb : 1;  // row stride between a thread's rows
        for (int k = k0; k < k1; k += U) {
            double v[U][R];
            double xv[U][R];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int kk = k + u;
#pragma unroll
                for (int r = 0; r < R; ++r) { v[u][r] = 0.0; xv[u][r] = 0.0; }
                if (kk < k1) {
                    const int64_t o = __ldg(a.dia_off + kk);
                    const double* sp = seg_base + (int64_t)kk * a.bl;
                    // 16-byte loads for consecutive rows unless the slice starts on an
                    // odd slot (odd bl, odd segment index: l is a multiple of R)
                    if (!IL && !MBIL && R >= 2 && !(kk & a.bl & 1)) {
#pragma unroll
                        for (int h = 0; h < R / 2; ++h) {
                            const double2 t = __ldcs(reinterpret_cast<const double2*>(sp) + h);
                            v[u][2 * h] = t.x;
                            v[u][2 * h + 1] = t.y;
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (i0 + RS * r < hi) v[u][r] = __ldcs(sp + RS * r);
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int64_t j = gi + RS * r + o;
                        const bool ok = (j >= 0) & (j < a.n_cols) & (i0 + RS * r < hi);
                        if (ok) xv[u][r] = __ldg(a.x + (i0 + RS * r + o));
                    }
                }
            }
            // zero slots contribute +-0.0, an identity on an accumulator that
            // can never be -0.0 (it starts at +0.0), so masked rows add nothing.
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double xx = xv[u][r];
                    if (SCALE) xx = __dmul_rn(xx, sc);
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(v[u][r], xx));
                }
            }
        }
        if (!IL && !MBIL && R >= 2 && a.y_vec_ok && i0 + R - 1 < hi) {
#pragma unroll
            for (int h = 0; h < R / 2; ++h)
                __stcs(reinterpret_cast<double2*>(a.y + i0) + h, make_double2(acc[2 * h], acc[2 * h + 1]));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + RS * r < hi) __stcs(a.y + i0 + RS * r, acc[r]);
        }
        if (a.peer_lo || a.peer_hi) {  // halo rows also to the neighbours (peer memory)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t i = i0 + RS * r;
                if (i >= hi) continue;
                if (a.peer_lo && i < a.halo) a.peer_lo[i] = acc[r];
                if (a.peer_hi && i >= a.n_rows - a.halo) a.peer_hi[i - (a.n_rows - a.halo)] = acc[r];
            }
            __threadfence_system();
        }
    }

    if (NORM) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (row(r) < hi) s = __dadd_rn(s, __dmul_rn(acc[r], acc[r]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
        if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < SPMV_THREADS / 32; ++w) t = __dadd_rn(t, warp_sums[w]);
            a.tile_sumsq[tile] = t;
        }
    }
}

// One tiling for both kernels (spmv_kernel and spmv_tma_kernel), so per-tile
// partial sums and block-range alignment do not depend on which one runs:
//   <= 32 segments per block (stencil-like) and bl >= 1024, or bl in {128, 256,
//   512}: 4 rows/thread, 1024-row tiles, ceil(bl/1024) tiles per block (or
//                         1024/bl whole blocks per tile)
//   other bl >= 512      : 2 rows/thread, 512-row tiles
//   bl in [256,512)      : 1 row/thread, 256-row tiles, 2 tiles per block
//   other bl < 256       : 1 row/thread, 256/bl whole blocks per tile
// (odd bl: a slice of segment k starts on an odd slot when k is odd, so both
// kernels fall back to 8-byte segment loads / y stores there)
Tiling tiling_of(const Matrix& m) {
    Tiling t;
    const int64_t t4 = 4 * SPMV_THREADS;
    if (m.packed) {  // tile-packed small blocks (pack.cu): 1024-row tiles, 4 rows per thread
        t.rows_per_thread = 4;
        t.tile_rows = PACK_TILE;
        t.tiles_per_block = t.blocks_per_tile = 0;
        t.n_tiles = ceil_div(m.n_rows, PACK_TILE);
        t.packed = true;
        int64_t a = PACK_TILE, b = m.bl;  // block ranges align to lcm(1024, bl) rows
        while (b) { const int64_t r = a % b; a = b; b = r; }
        t.align_blocks = PACK_TILE / a;
        return t;
    }
    // 4 rows/thread up to 32 segments per block: with the interleaved row mapping
    // config 2 (27 segments) went 90% -> 97% of peak (profiles/r01_v18_r4_c2_ab.log)
    static const int r4_max_seg = getenv("HDCG_R4_MAXSEG") ? atoi(getenv("HDCG_R4_MAXSEG")) : 32;  // A/B knob
    if (m.max_seg_per_block <= r4_max_seg && (m.bl >= t4 || (m.bl >= 128 && m.bl % 4 == 0 && t4 % m.bl == 0)))
        t.rows_per_thread = 4;
    else if (m.bl >= 2 * SPMV_THREADS) t.rows_per_thread = 2;
    else t.rows_per_thread = 1;  // incl. bl < 256: 256/bl whole blocks per tile (spmv_blk_kernel)
    t.tile_rows = (int64_t)SPMV_THREADS * t.rows_per_thread;
    if (m.bl >= t.tile_rows) {
        t.tiles_per_block = ceil_div(m.bl, t.tile_rows);
        t.blocks_per_tile = 0;
        t.n_tiles = m.n_blocks * t.tiles_per_block;
    } else {
        t.tiles_per_block = 0;
        t.blocks_per_tile = t.tile_rows / m.bl;
        t.n_tiles = ceil_div(m.n_blocks, t.blocks_per_tile);
    }
    t.align_blocks = t.blocks_per_tile > 0 ? t.blocks_per_tile : 1;
    return t;
}

template <int R, bool SCALE, bool NORM>
static void launch_t(const SpmvArgs& a, int64_t n_tiles, cudaStream_t st) {
    if constexpr (R == 4) {
        if (a.tiles_per_block == 0 && a.blocks_per_tile == 0) {
            spmv_kernel<4, SCALE, NORM, false, true><<<(unsigned)n_tiles, SPMV_THREADS, 0, st>>>(a);
            return;
        }
    }
    if (a.tiles_per_block > 0) spmv_kernel<R, SCALE, NORM, true><<<(unsigned)n_tiles, SPMV_THREADS, 0, st>>>(a);
    else spmv_kernel<R, SCALE, NORM, false><<<(unsigned)n_tiles, SPMV_THREADS, 0, st>>>(a);
}

template <int R>
static void launch_r(const SpmvArgs& a, int64_t n_tiles, bool scale, bool norm, cudaStream_t st) {
    if (scale) {
        if (norm) launch_t<R, true, true>(a, n_tiles, st);
        else launch_t<R, true, false>(a, n_tiles, st);
    } else {
        if (norm) launch_t<R, false, true>(a, n_tiles, st);
        else launch_t<R, false, false>(a, n_tiles, st);
    }
}

void spmv_launch(const Matrix& m, const double* x_local, double* y, int64_t block_begin,
                 int64_t block_end, const double* x_scale, double* tile_sumsq, cudaStream_t st,
                 const PeerOut& peer) {
    if (block_begin < 0 || block_end > m.n_blocks || block_begin > block_end)
        fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: block range outside the matrix");
    const Tiling t = tiling_of(m);
    int64_t tile_begin, tile_end;
    if (t.packed) {
        auto aligned = [&](int64_t b) { return b % t.align_blocks == 0 || b * m.bl >= m.n_rows; };
        if (!aligned(block_begin) || !aligned(block_end))
            fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: block range not aligned to the packed 1024-row tiles");
        tile_begin = std::min(block_begin * m.bl, m.n_rows) / PACK_TILE;
        tile_end = ceil_div(std::min(block_end * m.bl, m.n_rows), PACK_TILE);
        if (block_begin == block_end) tile_end = tile_begin;
    } else if (t.tiles_per_block > 0) {
        tile_begin = block_begin * t.tiles_per_block;
        tile_end = block_end * t.tiles_per_block;
    } else {
        if (block_begin % t.blocks_per_tile != 0 ||
            (block_end % t.blocks_per_tile != 0 && block_end != m.n_blocks))
            fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: block range not aligned to blocks_per_tile");
        tile_begin = block_begin / t.blocks_per_tile;
        tile_end = ceil_div(block_end, t.blocks_per_tile);
    }
    spmv_launch_tiles(m, x_local, y, tile_begin, tile_end, x_scale, tile_sumsq, st, peer);
}

void spmv_launch_tiles(const Matrix& m, const double* x_local, double* y, int64_t tile_begin, int64_t tile_end,
                       const double* x_scale, double* tile_sumsq, cudaStream_t st, const PeerOut& peer) {
    static const int env_policy = [] {  // HDCG_KERNEL_POLICY: profiling override of the default
        const char* e = getenv("HDCG_KERNEL_POLICY");
        if (e) g_kernel_policy = atoi(e);
        return 0;
    }();
    (void)env_policy;
    const Tiling t = tiling_of(m);
    if (tile_begin < 0 || tile_end > t.n_tiles || tile_begin > tile_end)
        fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: tile range outside the matrix");
    const int64_t n_tiles = tile_end - tile_begin;
    if (n_tiles <= 0) return;
    if (tile_end > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "spmv: too many tiles for one launch");
    if (g_kernel_policy != 1 && spmv_tma_launch(m, x_local, y, tile_begin, tile_end, x_scale, tile_sumsq, st, peer))
        return;
    if (g_kernel_policy == 2) fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: TMA kernel requested for an ineligible shape");
    SpmvArgs a;
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
    a.tiles_per_block = t.tiles_per_block;
    a.blocks_per_tile = t.blocks_per_tile;
    a.tile_rows = t.tile_rows;
    a.tile_begin = tile_begin;
    a.has_rest = m.nnz_rest > 0;
    a.y_vec_ok = ((uintptr_t)y % 16) == 0 && m.bl % 2 == 0;  // odd bl: tiles may start on odd rows
    a.peer_lo = peer.lo;
    a.peer_hi = peer.hi;
    a.halo = peer.halo;
    const bool scale = x_scale != nullptr, norm = tile_sumsq != nullptr;
    if (t.rows_per_thread == 4) launch_r<4>(a, n_tiles, scale, norm, st);
    else if (t.rows_per_thread == 2) launch_r<2>(a, n_tiles, scale, norm, st);
    else launch_r<1>(a, n_tiles, scale, norm, st);
    HDCG_LAUNCH_CHECK("spmv_kernel");
}

// ---- deterministic pairwise tree sum ------------------------------------------
constexpr int TREE_CHUNK = 2048;

__global__ void __launch_bounds__(1024) tree_chunk_kernel(const double* in, int64_t count,
                                                          int chunk, double* out, int last) {
    __shared__ double s[TREE_CHUNK];
    const int64_t base = (int64_t)blockIdx.x * chunk;
    for (int t = threadIdx.x; t < chunk; t += blockDim.x)
        s[t] = (base + t < count) ? in[base + t] : 0.0;
    __syncthreads();
    for (int stride = 1; stride < chunk; stride <<= 1) {
        for (int t = threadIdx.x * 2 * stride; t < chunk; t += blockDim.x * 2 * stride)
            s[t] = __dadd_rn(s[t], s[t + stride]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[blockIdx.x] = s[0];
        if (last) out[1] = 1.0 / sqrt(s[0]);
    }
}

void tree_sum_launch(const double* vals, int64_t count, double* out, cudaStream_t st) {
    int64_t p = 1;
    while (p < count) p <<= 1;
    const double* cur = vals;
    int64_t cur_count = count;
    double* tmp[2] = {nullptr, nullptr};
    int which = 0;
    while (true) {
        const int chunk = (int)(p < TREE_CHUNK ? p : TREE_CHUNK);
        const int64_t n_chunks = p / chunk;
        const bool last = n_chunks == 1;
        double* dst;
        if (last) {
            dst = out;
        } else {
            if (!tmp[which]) tmp[which] = dev_alloc<double>(n_chunks, st);
            dst = tmp[which];
        }
        tree_chunk_kernel<<<(unsigned)n_chunks, 1024, 0, st>>>(cur, cur_count, chunk, dst, last);
        HDCG_LAUNCH_CHECK("tree_chunk_kernel");
        if (last) break;
        cur = dst;
        cur_count = n_chunks;
        p = n_chunks;
        which ^= 1;
        if (tmp[which]) { dev_free(tmp[which], st); tmp[which] = nullptr; }
    }
    dev_free(tmp[0], st);
    dev_free(tmp[1], st);
}

}  // namespace hdcg

// spmv_tma.cu -- TMA-fed persistent M-HDC / HDC SpMV for sm_100a.
//
// Same arithmetic as spmv.cu (the reference's per-row order, kernels.cpp:173-206,
// __dmul_rn/__dadd_rn, bitwise equal), different data movement:
//
//   * persistent grid (SMs x CTAs/SM); CTA c owns tiles c, c+grid, ... of the
//     shared tiling (tiling_of: TILE = 256*R rows inside one row block);
//   * warp 8 is the producer.  One lane streams every segment slice of the tile
//     (TILE contiguous doubles of segment k) into an NSTAGE-deep ring with
//     cp.async.bulk (the 1-D TMA path, UBLKCP in SASS), completion through
//     mbarrier transaction counts, L2 evict-first (segments are read once).  The
//     ring holds only matrix data -- the bytes that come from DRAM -- so ~70 KB
//     per CTA (~210 KB per SM) of HBM traffic is in flight;
//   * warps 0-7 consume in the reference's order: first the CSR remainder
//     (each warp for its own rows: their entries are contiguous per 32-row run:
//     coalesced evict-first loads, 8 independent x gathers per lane in flight,
//     products in a per-warp scratch, per-row sequential sums; warp-synchronous),
//     then per segment: the block's offsets were loaded once per tile by each
//     warp (one coalesced load, broadcast with shuffles); x values are loaded for
//     a group of XGROUP segments ahead of the stage waits through the L1/tex
//     path, where the near offsets of a tile share lines and the far ones hit
//     L2; a warp-uniform whole-tile range test keeps per-row checks off the
//     common path; ring bookkeeping is a (stage, phase) pair, no divisions;
//   * rows are interleaved over the threads (thread t: tile rows t, t+256, ...),
//     so each x load, shared read and y store of a warp touches 32 consecutive
//     rows -- the L1 data pipe was 90% busy with 4 consecutive rows per thread
//     (8 wavefronts per x load, 2-way conflicted 16-byte shared reads);
//     multi-block tiles keep consecutive rows so a warp stays in one block;
//   * y is stored once per tile (streaming store); the optional fused per-tile
//     sum of squares has the same fixed reduction order as spmv.cu, with one
//     consumer barrier per tile (double-buffered warp partials).
// Used for bl >= 256 (all BASELINE M-HDC configurations, HDC; odd bl: slices
// that start on an odd slot are copied from one slot early) and for small
// blocks that tile evenly (bl in {128, 256, 512} with R = 4: a tile = G =
// 1024/bl whole blocks; ring stage j then carries segment j of each of the G
// blocks, each warp's rows lie in one block); other shapes take the general
// kernel in spmv.cu.
#include <algorithm>
#include <cstdlib>

#include "hdcg_internal.cuh"
#include "tma_ptx.cuh"

namespace hdcg {

namespace {

constexpr int CONSUMER_WARPS = 8;
constexpr int CONSUMERS = CONSUMER_WARPS * 32;
constexpr int THREADS = CONSUMERS + 32;  // + producer warp
constexpr int XGROUP_ROWS = 16;          // x values loaded ahead per thread (segments x rows)
constexpr int WPASS = 256;               // remainder scratch per warp (entries per pass <= this)
// fused remainder mode (REST == 3): gather warps sum the CSR remainder of the
// tiles ahead into y while the consumers stream segments
#ifndef HDCG_GATHER_WARPS
#define HDCG_GATHER_WARPS 15
#endif
constexpr int GATHER_WARPS = HDCG_GATHER_WARPS;  // + 8 consumers + the producer = 24 warps: one CTA per SM, 80 registers
constexpr int GPER = 8;                  // x gathers per lane per pass
constexpr int GPASS = 32 * GPER;         // entries per gather-warp pass
constexpr int RS_SLOTS = 2 * 32;         // tile hand-off barriers (>= 2 * GATHER_WARPS, power of 2)

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS) : "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// The lines the consumers read at the start of a tile (the block's offsets, the
// remainder row pointers at warp boundaries), pulled into L2 by the producer when
// it starts the tile's copies -- one or more tiles before the consumers get there.
__device__ __forceinline__ void prefetch_range_l2(const int32_t* base, int64_t first, int64_t last) {
    const uintptr_t a = (uintptr_t)(base + first) & ~uintptr_t(127), e = (uintptr_t)(base + last);
    for (uintptr_t q = a; q < e; q += 128) prefetch_l2((const void*)q);
}

struct TmaArgs {
    const int32_t* dia_ptr;
    const int32_t* dia_off;
    const double* seg;
    const int32_t* rest_rp;
    const int32_t* rest_col;  // padded: readable up to a multiple of 4 entries past nnz_rest
    const double* rest_val;
    const double* x;  // x_local
    double* y;
    const double* x_scale;
    double* tile_sumsq;
    int64_t n_rows, n_cols, row0, bl;
    int tiles_per_block;  // > 0: a tile is a part of one block
    int blocks_per_tile;  // > 0: a tile is G whole blocks (bl < TILE, bl % (32 R) == 0)
    int64_t n_blocks;
    int tile_begin, tile_end;
    int nstage;
    int has_rest;
    int init_y;       // remainder sums already in y (rest_kernel ran first)
    int y_vec_ok;
    double* peer_lo;  // PeerOut: halo rows also stored to the neighbours
    double* peer_hi;
    int64_t halo;
    int prefetch;  // producer prefetches the consumers' tile-start lines into L2
    int fused;     // REST == 3: remainder sums by the gather warps (shared memory)
    const double* pk_val;  // LAY 5: the tile-packed segment copy (pack.cu)
    const int4* pk_meta;
    const int32_t* pk_tab;
};

struct Geo {
    int64_t lo, hi, b0;
    int b;
};

template <int R, bool MB, bool PK = false>
__device__ __forceinline__ Geo geo(const TmaArgs& a, int tile) {
    Geo g;
    if constexpr (PK) {  // packed: 1024 consecutive rows, b = the tile's first block
        g.lo = (int64_t)tile * (CONSUMERS * R);
        g.hi = min(g.lo + (int64_t)(CONSUMERS * R), a.n_rows);
        g.b = (int)(g.lo / a.bl);
        g.b0 = (int64_t)g.b * a.bl;
        return g;
    }
    if constexpr (MB) {  // G whole blocks: b = the first one
        g.b = tile * a.blocks_per_tile;
        g.b0 = g.lo = (int64_t)g.b * a.bl;
        g.hi = min(g.lo + (int64_t)a.blocks_per_tile * a.bl, a.n_rows);
        return g;
    }
    g.b = tile / a.tiles_per_block;
    const int t = tile - g.b * a.tiles_per_block;
    g.b0 = (int64_t)g.b * a.bl;
    const int64_t bend = min(g.b0 + a.bl, a.n_rows);
    g.lo = g.b0 + (int64_t)t * (CONSUMERS * R);
    g.hi = min(g.lo + (int64_t)(CONSUMERS * R), bend);
    return g;
}

// Doubles per ring stage: a tile's slice + 2 -- with odd bl a slice can start on
// an odd slot; the 16-byte aligned copy then starts one slot early.
__host__ __device__ constexpr int ring_stride(int R) { return CONSUMERS * R + 2; }

// has_rest: the consumers' per-warp remainder scratch (CONSUMER_WARPS * WPASS doubles)
// fused: the gather warps' product scratch and staged row pointers (a gather
// warp sums its tiles in chunks of GCHUNK rows), the tile hand-off barriers
constexpr int GCHUNK = 256;
__host__ __device__ inline size_t fused_int_bytes(int) {
    return ((size_t)GATHER_WARPS * (GCHUNK + 1) * sizeof(int32_t) + 15) & ~size_t(15);
}
__host__ __device__ inline size_t smem_bytes(int R, int nstage, int has_rest, int fused = 0) {
    size_t b = sizeof(double) * ((size_t)nstage * ring_stride(R) + (has_rest ? CONSUMER_WARPS * WPASS : 0) +
                                 2 * CONSUMER_WARPS) +
               sizeof(uint64_t) * (2 * nstage);
    if (fused)
        b += sizeof(double) * ((size_t)GATHER_WARPS * GPASS) + fused_int_bytes(R) + sizeof(uint64_t) * 2 * RS_SLOTS;
    return b;
}

struct Smem {
    double* ring;     // nstage * ring_stride(R)
    double* scratch;  // CONSUMER_WARPS * WPASS (remainder products) when has_rest
    double* wsum;     // 2 * CONSUMER_WARPS (fused norm: double-buffered warp partials)
    double* gscratch; // fused: GATHER_WARPS * GPASS products
    int32_t* grp;     // fused: GATHER_WARPS * (GCHUNK + 1) row pointers
    uint64_t* full;
    uint64_t* empty;
    uint64_t* rs_full;   // fused: a tile's sums are in y (its gather warp's arrival)
    uint64_t* rs_empty;  // fused: the consumers have read them (CONSUMER_WARPS arrivals)
};

__device__ __forceinline__ Smem carve(unsigned char* base, int R, int nstage, int has_rest, int fused = 0) {
    Smem s;
    s.ring = reinterpret_cast<double*>(base);
    s.scratch = s.ring + (size_t)nstage * ring_stride(R);
    s.wsum = s.scratch + (has_rest ? CONSUMER_WARPS * WPASS : 0);
    double* d = s.wsum + 2 * CONSUMER_WARPS;
    s.gscratch = d;
    d = s.gscratch + (fused ? GATHER_WARPS * GPASS : 0);
    s.grp = reinterpret_cast<int32_t*>(d);
    unsigned char* u = reinterpret_cast<unsigned char*>(d) + (fused ? fused_int_bytes(R) : 0);
    s.full = reinterpret_cast<uint64_t*>(u);
    s.empty = s.full + nstage;
    s.rs_full = s.empty + nstage;
    s.rs_empty = s.rs_full + RS_SLOTS;
    return s;
}

// Remainder sums (stored order, onto +0.0 accumulators) of one warp's 32*R rows
// of the tile [lo, hi): the rows' entries are contiguous, so lanes stream them
// coalesced (evict-first), gather x for PER entries each (independent loads in
// flight), leave the products in the warp's scratch, and each lane then adds its
// rows' products sequentially.  Warp-synchronous.
template <int R, bool SCALE, int PER = (R == 4 ? 4 : 8)>
__device__ __forceinline__ void warp_rest(const int32_t* __restrict__ rest_rp, const int32_t* __restrict__ rest_col,
                                          const double* __restrict__ rest_val, const double* __restrict__ x,
                                          int64_t row0, double sc, int64_t lo, int64_t hi, int warp, int lane,
                                          double* scratch, double (&acc)[R]) {
    const int t0 = R * (warp * 32 + lane);
    const int rows = (int)(hi - lo);
    const int64_t i0 = lo + t0;
    const int64_t w_lo = min(lo + (int64_t)warp * 32 * R, hi);
    const int64_t w_hi = min(w_lo + 32 * R, hi);
    const int e_lo = __ldg(rest_rp + w_lo), e_hi = __ldg(rest_rp + w_hi);  // int32: nnz_rest < 2^31
    if (e_lo >= e_hi) return;
    int kb[R], ke[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const bool ok = t0 + r < rows;
        kb[r] = ok ? __ldg(rest_rp + i0 + r) : 0;
        ke[r] = ok ? __ldg(rest_rp + i0 + r + 1) : 0;
    }
    constexpr int PASS = 32 * PER;  // PER entries per lane per pass (x gathers in flight); scratch >= PASS
    for (int c = e_lo; c < e_hi; c += PASS) {
        int32_t cl[PER];
        double vl[PER], xl[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int q = c + lane + 32 * j;
            cl[j] = q < e_hi ? __ldcs(rest_col + q) : 0;
            vl[j] = q < e_hi ? __ldcs(rest_val + q) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int q = c + lane + 32 * j;
            xl[j] = q < e_hi ? __ldg(x + ((int64_t)cl[j] - row0)) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            double xv = xl[j];
            if (SCALE) xv = __dmul_rn(xv, sc);
            scratch[lane + 32 * j] = __dmul_rn(vl[j], xv);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p0 = max(kb[r], c), p1 = min(ke[r], c + PASS);
            for (int p = p0; p < p1; ++p) acc[r] = __dadd_rn(acc[r], scratch[p - c]);
        }
        __syncwarp();
    }
}

// Remainder-heavy matrices: the remainder sums of every tile, written to y, by a
// non-persistent high-occupancy kernel (one CTA of 8 warps per tile, no ring), so
// far more x gathers are in flight than beside the segment ring.  spmv_tma_kernel
// then starts each row from y -- the same operations in the same order.
// It only writes y, so its row mapping is free: one row per lane (a warp's 32 rows
// usually fit one pass of 8 gathers per lane), 256 rows per CTA, many CTAs per SM.
template <bool SCALE, int MINB, int RR, int PER>
__global__ void __launch_bounds__(CONSUMERS, MINB) rest_kernel(const TmaArgs a, int64_t row_lo, int64_t row_hi) {
    __shared__ double scratch[CONSUMER_WARPS * 32 * PER];
    const int64_t lo = row_lo + (int64_t)blockIdx.x * (CONSUMERS * RR);
    const int64_t hi = min(lo + CONSUMERS * RR, row_hi);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double sc = 1.0;
    if (SCALE) sc = *a.x_scale;
    double acc[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) acc[r] = 0.0;
    warp_rest<RR, SCALE, PER>(a.rest_rp, a.rest_col, a.rest_val, a.x, a.row0, sc, lo, hi, warp, lane,
                              scratch + warp * 32 * PER, acc);
    const int64_t i0 = lo + RR * threadIdx.x;
#pragma unroll
    for (int r = 0; r < RR; ++r)
        if (i0 + r < hi) a.y[i0 + r] = acc[r];
}

// Software-pipelined remainder sums (the default for remainder-heavy matrices and
// CSR).  rest_kernel pays three dependent round trips per 32 rows (row pointers ->
// columns/values -> x gathers); here a warp owns G runs of 32 rows (one contiguous
// entry range), stages their row pointers in shared memory once, and walks the range
// in passes of 32*PER entries with the next pass's columns loaded while this pass's
// gathers and values are in flight -- one round trip per pass.  Lanes own the rows
// of the current 32-row run; a pass's products go to the warp's scratch and each
// lane adds those of its row in stored order (runs finished inside the pass are
// stored and the lanes move to the next run).  Same operations in the same order as
// warp_rest: bitwise equal.
template <bool SCALE, int MINB, int G, int PER>
__global__ void __launch_bounds__(CONSUMERS, MINB) rest_pipe_kernel(const TmaArgs a, int64_t row_lo, int64_t row_hi) {
    constexpr int PASS = 32 * PER;
    constexpr int WROWS = 32 * G;
    __shared__ double scratch_all[CONSUMER_WARPS][PASS];
    __shared__ int32_t rp_all[CONSUMER_WARPS][WROWS + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* scratch = scratch_all[warp];
    int32_t* rps = rp_all[warp];
    const int64_t w0 = row_lo + ((int64_t)blockIdx.x * CONSUMER_WARPS + warp) * WROWS;
    if (w0 >= row_hi) return;
    const int nrows = (int)min((int64_t)WROWS, row_hi - w0);
    for (int i = lane; i <= WROWS; i += 32) rps[i] = __ldg(a.rest_rp + w0 + min(i, nrows));
    __syncwarp();
    const double sc = SCALE ? *a.x_scale : 1.0;
    const int e0 = rps[0], e1 = rps[WROWS];
    int g = 0;  // current 32-row run
    int kb = rps[lane], ke = rps[lane + 1];
    int gend = rps[32];  // first entry past the run (warp-uniform)
    double acc = 0.0;
    int32_t cn[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int q = e0 + lane + 32 * j;
        cn[j] = q < e1 ? __ldcs(a.rest_col + q) : 0;
    }
    int c = e0;
    do {
        int32_t cl[PER];
        double xl[PER], vl[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) cl[j] = cn[j];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int q = c + lane + 32 * j;
            xl[j] = q < e1 ? __ldg(a.x + ((int64_t)cl[j] - a.row0)) : 0.0;
            vl[j] = q < e1 ? __ldcs(a.rest_val + q) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {  // the next pass's columns
            const int q = c + PASS + lane + 32 * j;
            cn[j] = q < e1 ? __ldcs(a.rest_col + q) : 0;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            double xv = xl[j];
            if (SCALE) xv = __dmul_rn(xv, sc);
            scratch[lane + 32 * j] = __dmul_rn(vl[j], xv);
        }
        __syncwarp();
        const int cend = c + PASS;
        while (true) {
            const int p0 = max(kb, c), p1 = min(ke, cend);
            for (int p = p0; p < p1; ++p) acc = __dadd_rn(acc, scratch[p - c]);
            if (gend > cend || g >= G) break;  // the run continues in the next pass
            const int r = 32 * g + lane;
            if (r < nrows) a.y[w0 + r] = acc;
            acc = 0.0;
            if (++g >= G || 32 * g >= nrows) {
                g = G;
                break;
            }
            kb = rps[32 * g + lane];
            ke = rps[32 * g + lane + 1];
            gend = rps[min(32 * g + 32, WROWS)];
        }
        __syncwarp();
        c = cend;
    } while (c < e1);
}

// One gather warp's rows [w0, w0 + nrows) of a tile (nrows <= 32 * G): the
// remainder sums in stored order onto +0.0 (kernels.cpp:192-197), written to
// out[0 .. nrows) in shared memory.  rest_pipe_kernel's pipeline: the warp's row
// pointers staged once, the entry range walked in passes of GPASS entries with
// the next pass's columns loaded while this pass's x gathers and values are in
// flight, products through the warp's scratch, each lane adding its row's
// products in order.  Bitwise equal to warp_rest / rest_pipe_kernel.
template <bool SCALE, int G>
__device__ __forceinline__ void gather_rest_rows(const TmaArgs& a, int64_t w0, int nrows, double sc, double* scratch,
                                                 int32_t* rps, double* out, int lane) {
    constexpr int WROWS = 32 * G;
    for (int i = lane; i <= WROWS; i += 32) rps[i] = __ldg(a.rest_rp + w0 + min(i, nrows));
    __syncwarp();
    const int e0 = rps[0], e1 = rps[WROWS];
    int g = 0;
    int kb = rps[lane], ke = rps[lane + 1];
    int gend = rps[32];
    double acc = 0.0;
    int32_t cn[GPER];
#pragma unroll
    for (int j = 0; j < GPER; ++j) {
        const int q = e0 + lane + 32 * j;
        cn[j] = q < e1 ? __ldcs(a.rest_col + q) : 0;
    }
    int c = e0;
    do {
        int32_t cl[GPER];
        double xl[GPER], vl[GPER];
#pragma unroll
        for (int j = 0; j < GPER; ++j) cl[j] = cn[j];
#pragma unroll
        for (int j = 0; j < GPER; ++j) {
            const int q = c + lane + 32 * j;
            xl[j] = q < e1 ? __ldg(a.x + ((int64_t)cl[j] - a.row0)) : 0.0;
            vl[j] = q < e1 ? __ldcs(a.rest_val + q) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < GPER; ++j) {
            const int q = c + GPASS + lane + 32 * j;
            cn[j] = q < e1 ? __ldcs(a.rest_col + q) : 0;
        }
#pragma unroll
        for (int j = 0; j < GPER; ++j) {
            double xv = xl[j];
            if (SCALE) xv = __dmul_rn(xv, sc);
            scratch[lane + 32 * j] = __dmul_rn(vl[j], xv);
        }
        __syncwarp();
        const int cend = c + GPASS;
        while (true) {
            const int p0 = max(kb, c), p1 = min(ke, cend);
            for (int p = p0; p < p1; ++p) acc = __dadd_rn(acc, scratch[p - c]);
            if (gend > cend || g >= G) break;  // the run continues in the next pass
            const int r = 32 * g + lane;
            if (r < nrows) out[r] = acc;
            acc = 0.0;
            if (++g >= G || 32 * g >= nrows) {
                g = G;
                break;
            }
            kb = rps[32 * g + lane];
            ke = rps[32 * g + lane + 1];
            gend = rps[min(32 * g + 32, WROWS)];
        }
        __syncwarp();
        c = cend;
    } while (c < e1);
    // rows of runs the pass loop never reached (no entries left): +0.0
    for (int r = 32 * g + lane; r < nrows; r += 32) out[r] = 0.0;
}

// REST: 0 no remainder, 1 remainder summed here from global memory (fused),
// 2 remainder sums already in y (rest_kernel ran first)
// LAY: tile layout.  0 tiles inside one block, even bl; 1 multi-block tiles
// (a.blocks_per_tile > 0, R = 4 only); 2 tiles inside one block, odd bl
// (slices of odd segments start on an odd slot); 3 / 4 multi-block tiles of
// bl = 256 / 128 without a remainder, rows interleaved inside each block.
// REST == 3 (fused): warps 9 .. 9+GATHER_WARPS-1 are gather warps (remainder
// sums of whole tiles ahead into y, up to RS_SLOTS tiles in flight); the
// consumers start each row from its sum.  One CTA per SM: the x gathers need
// about as many warps in flight as rest_pipe_kernel has (24 per SM).
// Tile order of a persistent CTA.  HDCG_TILE_GROUP = 1 (default): tiles c, c + grid,
// ...; G > 1 (A/B builds): G adjacent tiles in a row, then the next group -- the x
// lines one tile loads for its +tile_rows offsets are the next tile's own rows.
// Measured slower: config 4 1292 -> 1244 (G = 2) / 1242 (G = 4) GFLOP/s, configs 1-2
// unchanged (profiles/r03o_ab_tile_group.log); the interleaved order stays.
#ifndef HDCG_TILE_GROUP
#define HDCG_TILE_GROUP 1
#endif
__device__ __forceinline__ int first_tile(const TmaArgs& a) { return a.tile_begin + HDCG_TILE_GROUP * (int)blockIdx.x; }
__device__ __forceinline__ int next_tile(const TmaArgs& a, int tile) {
    if (HDCG_TILE_GROUP == 1) return tile + (int)gridDim.x;
    return (tile - a.tile_begin) % HDCG_TILE_GROUP != HDCG_TILE_GROUP - 1
               ? tile + 1
               : tile + HDCG_TILE_GROUP * (int)gridDim.x - (HDCG_TILE_GROUP - 1);
}

template <int R, bool SCALE, bool NORM, int REST, int LAY>
__global__ void __launch_bounds__(REST == 3 ? THREADS + 32 * GATHER_WARPS : THREADS, REST == 3 ? 1 : 3)
    spmv_tma_kernel(const TmaArgs a) {
    constexpr bool MB = LAY == 1 || LAY == 3 || LAY == 4;
    constexpr bool ODD = LAY == 2;
    constexpr bool PK = LAY == 5;  // tile-packed small blocks (pack.cu), R = 4
    constexpr int TILE = CONSUMERS * R;
    constexpr int STRIDE = ring_stride(R);
    // x registers per thread stay at XGROUP_ROWS doubles (8 for the multi-block layout
    // with consecutive rows per thread, whose wider address math otherwise spills)
    constexpr int XG = (LAY == 1 || (SCALE && NORM && (LAY == 4 || REST == 3)) ? XGROUP_ROWS / 2 : XGROUP_ROWS) / R;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NS = a.nstage;
    const Smem S = carve(smem_raw, R, NS, a.has_rest, REST == 3);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], CONSUMER_WARPS);
        }
        if (REST == 3) {
            for (int s = 0; s < RS_SLOTS; ++s) {
                mbar_init(&S.rs_full[s], 1);
                mbar_init(&S.rs_empty[s], CONSUMER_WARPS);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if constexpr (REST == 3) {
        if (warp > CONSUMER_WARPS) {
            // -------------------------- gather warps --------------------------
            // Gather warp gw sums the remainder of every GATHER_WARPS-th tile of this
            // CTA's sequence (in 256-row chunks, rest_pipe_kernel's pipeline) into y
            // (the rows' starting values; the consumers add the segments and store
            // y again, normally while the line is still in L2), then arrives on the
            // tile's hand-off barrier.  Up to RS_SLOTS tiles ahead of the consumers.
            const int gw = warp - CONSUMER_WARPS - 1;
            double* scratch = S.gscratch + gw * GPASS;
            int32_t* rps = S.grp + gw * (GCHUNK + 1);
            const double sc = SCALE ? *a.x_scale : 1.0;
            int k = 0;  // index among this CTA's non-empty tiles (the consumers count the same)
            for (int tile = first_tile(a); tile < a.tile_end; tile = next_tile(a, tile)) {
                const Geo g = geo<R, MB, PK>(a, tile);
                if (g.lo >= g.hi) continue;  // the consumers skip it too
                const int kk = k++;
                if (kk % GATHER_WARPS != gw) continue;
                const int slot = kk & (RS_SLOTS - 1);
                if (kk >= RS_SLOTS) mbar_wait(&S.rs_empty[slot], ((kk / RS_SLOTS) - 1) & 1);
                for (int64_t c0 = g.lo; c0 < g.hi; c0 += GCHUNK)  // rest_pipe_kernel's 256-row runs
                    gather_rest_rows<SCALE, GCHUNK / 32>(a, c0, (int)min((int64_t)GCHUNK, g.hi - c0), sc, scratch, rps,
                                                         a.y + c0, lane);
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.rs_full[slot]);
            }
            return;
        }
    }

    if (warp == CONSUMER_WARPS) {
        // ------------------------------ producer ------------------------------
        // one lane streams tiles inside a block; multi-block tiles use the whole
        // warp (lane q issues block q's copies: no per-block register arrays)
        if (!MB && lane != 0) return;
        const uint64_t policy = evict_first_policy();
        int ps = 0;              // ring stage the next slice goes to
        uint32_t pphase = 0;     // parity of that stage's current use
        bool p_wrapped = false;  // every stage has been used once
        for (int tile = first_tile(a); tile < a.tile_end; tile = next_tile(a, tile)) {
            const Geo g = geo<R, MB, PK>(a, tile);
            if (g.lo >= g.hi) continue;
            if (a.prefetch && lane == 0) {
                if constexpr (REST == 1) {
#pragma unroll
                    for (int w = 0; w <= CONSUMER_WARPS; ++w)
                        prefetch_l2(a.rest_rp + min(g.lo + (int64_t)w * 32 * R, g.hi));
                }
                const int64_t bl_last = MB ? min((int64_t)g.b + a.blocks_per_tile, a.n_blocks) : (int64_t)g.b + 1;
                prefetch_range_l2(a.dia_off, __ldg(a.dia_ptr + g.b), __ldg(a.dia_ptr + bl_last));
            }
            if constexpr (MB) {
                // stage j = segment j of each of the tile's blocks, block q's slots at
                // q*bl (the tile-local row); blocks with fewer segments leave theirs
                // unused.  Lane q < G (<= 8) owns block q.
                const int nbt = (int)min((int64_t)a.blocks_per_tile, a.n_blocks - g.b);
                const int64_t last_len = min((int64_t)a.bl, a.n_rows - (int64_t)(g.b + nbt - 1) * a.bl);
                const int kst = lane < nbt ? __ldg(a.dia_ptr + g.b + lane) : 0;
                const int cnt = lane < nbt ? __ldg(a.dia_ptr + g.b + lane + 1) - kst : 0;
                const uint32_t pb = (uint32_t)(((lane == nbt - 1 ? last_len : a.bl) + 1) & ~int64_t(1)) * 8u;
                const int J = __reduce_max_sync(0xffffffffu, cnt);
                const double* src = a.seg + (int64_t)kst * a.bl;
                for (int j = 0; j < J; ++j, src += a.bl) {
                    const uint32_t bytes = __reduce_add_sync(0xffffffffu, j < cnt ? pb : 0u);
                    if (lane == 0) {
                        if (p_wrapped) mbar_wait(&S.empty[ps], pphase ^ 1u);
                        mbar_expect_tx(&S.full[ps], bytes);
                    }
                    __syncwarp();
                    if (j < cnt) bulk_g2s(S.ring + ps * STRIDE + lane * a.bl, src, pb, &S.full[ps], policy);
                    if (++ps == NS) {
                        ps = 0;
                        pphase ^= 1u;
                        p_wrapped = true;
                    }
                }
                continue;
            }
            if constexpr (PK) {  // K_t whole 8 KB stages, contiguous
                const int4 md = __ldg(a.pk_meta + tile);
                const int K = md.y & 0xffff;
                const double* src = a.pk_val + (int64_t)md.x * TILE;
                for (int k = 0; k < K; ++k, src += TILE) {
                    if (p_wrapped) mbar_wait(&S.empty[ps], pphase ^ 1u);
                    mbar_expect_tx(&S.full[ps], TILE * 8u);
                    bulk_g2s(S.ring + ps * STRIDE, src, TILE * 8u, &S.full[ps], policy);
                    if (++ps == NS) {
                        ps = 0;
                        pphase ^= 1u;
                        p_wrapped = true;
                    }
                }
                continue;
            }
            const int k0 = __ldg(a.dia_ptr + g.b), k1 = __ldg(a.dia_ptr + g.b + 1);
            const int64_t off0 = g.lo - g.b0;
            uint32_t bytes = (uint32_t)(((g.hi - g.lo + 1) & ~int64_t(1)) * 8);
            const double* src = a.seg + (int64_t)k0 * a.bl + off0;
            for (int k = k0; k < k1; ++k, src += a.bl) {
                // odd bl: the slice starts on an odd slot (k odd, or an odd tile start
                // for R = 1); copy from one slot earlier (16-byte aligned), consumers
                // read at +1
                const int sh = ODD ? ((k & (int)a.bl) ^ (int)off0) & 1 : 0;
                if (ODD) bytes = (uint32_t)(((g.hi - g.lo + sh + 1) & ~int64_t(1)) * 8);
                if (p_wrapped) mbar_wait(&S.empty[ps], pphase ^ 1u);  // previous use released
                mbar_expect_tx(&S.full[ps], bytes);
                bulk_g2s(S.ring + ps * STRIDE, src - sh, bytes, &S.full[ps], policy);
                if (++ps == NS) {
                    ps = 0;
                    pphase ^= 1u;
                    p_wrapped = true;
                }
            }
        }
        return;
    }

    // -------------------------------- consumers --------------------------------
    // Row mapping: tiles inside one block (LAY 0, 2) are interleaved -- thread t
    // owns tile rows t, t+256, ..., so every x load, shared-memory read and y store
    // of a warp covers 32 consecutive rows (2 L1 wavefronts per 8-byte access
    // instead of 8 with 4 consecutive rows per thread).  Multi-block tiles (LAY 1)
    // keep 4 consecutive rows per thread (a warp's rows stay in one block), except
    // without a remainder for bl = 256 (layout 3: lane l of the block's k-th warp
    // owns block rows 32 k + l + 64 r; 87% -> 95-97%) and bl = 128 (layout 4: one
    // warp per block, rows l + 32 r; 83% -> 91%).  Compile-time layouts: with a
    // runtime warps-per-block, or per-run remainder sums (bl = 512), it was slower
    // (profiles/r01_v19_*rejected*).
    constexpr bool mbil = LAY == 3 || LAY == 4;
    constexpr bool IL = !MB || mbil;
    double sc = 1.0;
    if (SCALE) sc = *a.x_scale;
    int cs = 0;             // ring stage of the next slice to consume
    uint32_t cphase = 0;    // parity of that stage's current use
    uint32_t par = 0;
    // this warp's block in the tile: two warps per block for bl = 256, one for 128
    const int qb = LAY == 3 ? warp / 2 : LAY == 4 ? warp : 0;
    // local row of this thread's first row, and the stride between its rows
    const int t0 = LAY == 3   ? qb * 256 + (warp & 1) * 32 + lane
                   : LAY == 4 ? qb * 128 + lane
                   : MB       ? R * (int)threadIdx.x
                              : (int)threadIdx.x;
    const int rstride = LAY == 3 ? 64 : LAY == 4 ? 32 : MB ? 1 : CONSUMERS;
    auto lr = [&](int r) { return t0 + rstride * r; };  // local row of its r-th row
    const int64_t xlo_valid = -a.row0, xhi_valid = a.n_cols - a.row0;  // x_local index range
    int kt = 0;          // REST == 3: index among this CTA's non-empty tiles
    int pe0 = 0, pe1 = 0;  // REST == 1: the next tile's remainder entry range
    auto probe = [&](int tl) {
        pe0 = pe1 = 0;
        if (REST != 1 || tl >= a.tile_end) return;
        const Geo q = geo<R, MB, PK>(a, tl);
        if (q.lo >= q.hi) return;
        pe0 = __ldg(a.rest_rp + q.lo);
        pe1 = __ldg(a.rest_rp + q.hi);
    };
    probe(first_tile(a));
    for (int tile = first_tile(a); tile < a.tile_end; tile = next_tile(a, tile)) {
        const Geo g = geo<R, MB, PK>(a, tile);
        if (g.lo >= g.hi) {
            if (NORM && threadIdx.x == 0) a.tile_sumsq[tile] = 0.0;
            probe(next_tile(a, tile));
            continue;
        }
        const int rows = (int)(g.hi - g.lo);
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;

        // CSR remainder first (stored order).  Fused here (few remainder entries),
        // already summed into y by rest_kernel (REST 2), or summed by this CTA's
        // gather warps into shared memory (REST 3, remainder-heavy matrices).
        if constexpr (REST == 3) {
            const int slot = kt & (RS_SLOTS - 1);
            mbar_wait(&S.rs_full[slot], (kt / RS_SLOTS) & 1);
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = lr(r) < rows ? a.y[g.lo + lr(r)] : 0.0;
            // release the slot once the sums are in registers
#pragma unroll
            for (int r = 0; r < R; ++r) asm volatile("" ::"d"(acc[r]));
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.rs_empty[slot]);
            ++kt;
        } else if constexpr (REST == 2) {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = lr(r) < rows ? a.y[g.lo + lr(r)] : 0.0;
        } else if constexpr (REST == 1) {
            // a light remainder: most tiles have no entries.  The tile's entry range
            // was loaded one tile ahead, so those tiles issue no dependent load here.
            const bool any = pe0 < pe1;
            probe(next_tile(a, tile));
            if (any) {
                if constexpr (!MB) {  // the warp's rows are R runs of 32
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int64_t lo = g.lo + (int64_t)CONSUMERS * r;
                        if (lo >= g.hi) break;
                        double a1[1] = {0.0};
                        warp_rest<1, SCALE>(a.rest_rp, a.rest_col, a.rest_val, a.x, a.row0, sc, lo,
                                            min(lo + CONSUMERS, g.hi), warp, lane, S.scratch + warp * WPASS, a1);
                        acc[r] = a1[0];
                    }
                } else {  // R consecutive rows per lane (mbil needs REST == 0)
                    warp_rest<R, SCALE>(a.rest_rp, a.rest_col, a.rest_val, a.x, a.row0, sc, g.lo, g.hi, warp, lane,
                                        S.scratch + warp * WPASS, acc);
                }
            }
        }

        // diagonal segments, stored order.  [k0, k1): the ring stages of the tile;
        // [k0, kw): this warp's block's segments (MB: k1 - k0 is the largest
        // segment count over the tile's blocks; otherwise kw = k1, the one block's).
        int k0, k1, kw;
        const int32_t* offs = a.dia_off;  // the offsets [k0, k1) index
        bool uniform = true;              // PK: every block of the tile has the same offsets
        int4 md = make_int4(0, 0, 0, 0);
        if constexpr (PK) {
            md = __ldg(a.pk_meta + tile);
            k0 = 0;
            k1 = kw = md.y & 0xffff;
            uniform = (md.y >> 16) & 1;
            offs = a.pk_tab + md.z;
        } else if constexpr (MB) {  // warp-uniform: bl % (32 R) == 0
            const int64_t bw = (int64_t)g.b + (mbil ? qb : t0 / (int)a.bl);
            const int nbt = (int)min((int64_t)a.blocks_per_tile, a.n_blocks - g.b);
            k0 = bw < a.n_blocks ? __ldg(a.dia_ptr + bw) : 0;
            kw = bw < a.n_blocks ? __ldg(a.dia_ptr + bw + 1) : 0;
            const int c = lane < nbt ? __ldg(a.dia_ptr + g.b + lane + 1) - __ldg(a.dia_ptr + g.b + lane) : 0;
            k1 = k0 + __reduce_max_sync(0xffffffffu, c);
        } else {
            k0 = __ldg(a.dia_ptr + g.b);
            k1 = kw = __ldg(a.dia_ptr + g.b + 1);
        }
        const double* xrow = a.x + g.lo;
        const bool full = rows == TILE;  // warp-uniform: no per-row predicates needed
        if (PK && !uniform) {
            // packed tile whose blocks differ: each row looks its k-th offset up in
            // its block's list (INT32_MIN: that block has no k-th segment -- skip)
            int q[R];
            const int rel = (int)(g.lo - (int64_t)md.w * a.bl);  // < bl
#pragma unroll
            for (int r = 0; r < R; ++r) q[r] = (rel + lr(r)) / (int)a.bl * k1;
            constexpr int XGN = XG / 2 > 0 ? XG / 2 : 1;  // per-row offsets: fewer x registers
            for (int kg = 0; kg < k1; kg += XGN) {
                const int ng = min(XGN, k1 - kg);
                double xv[XGN][R];
                uint32_t okm = 0;  // bit u*R + r: row r has a k-th segment
#pragma unroll
                for (int u = 0; u < XGN; ++u)
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        xv[u][r] = 0.0;
                        if (u < ng && lr(r) < rows) {
                            const int o = __ldg(offs + q[r] + kg + u);
                            const int64_t j = g.lo + lr(r) + (int64_t)o;
                            if (o != INT32_MIN) {
                                okm |= 1u << (u * R + r);
                                if (j >= xlo_valid && j < xhi_valid) xv[u][r] = __ldg(xrow + lr(r) + o);
                            }
                        }
                    }
#pragma unroll
                for (int u = 0; u < XGN; ++u) {
                    if (u < ng) {
                        mbar_wait(&S.full[cs], cphase);
                        const double* st = S.ring + cs * STRIDE;
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const double v = st[lr(r)];
                            double xx = xv[u][r];
                            if (SCALE) xx = __dmul_rn(xx, sc);
                            if ((okm >> (u * R + r)) & 1u) acc[r] = __dadd_rn(acc[r], __dmul_rn(v, xx));
                            else asm volatile("" ::"d"(v));
                        }
#pragma unroll
                        for (int r = 0; r < R; ++r) asm volatile("" ::"d"(acc[r]));
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&S.empty[cs]);
                        if (++cs == NS) {
                            cs = 0;
                            cphase ^= 1u;
                        }
                    }
                }
            }
            k1 = k0;  // done: skip the uniform loop below
        }
        for (int kb0 = k0; kb0 < k1; kb0 += 32) {
            // the next <= 32 offsets of the block: one coalesced load, then shuffles
            const int nk = min(32, k1 - kb0);
            const int nko = MB ? min(32, kw - kb0) : nk;  // of which this warp's block has
            const int my_off = lane < nko ? __ldg(offs + kb0 + lane) : 0;
            for (int kg = 0; kg < nk; kg += XG) {
                const int ng = min(XG, nk - kg);  // warp-uniform
                const int nv = MB ? min(ng, kw - kb0 - kg) : ng;  // of which this warp's block has
                double xv[XG][R];
#pragma unroll
                for (int u = 0; u < XG; ++u) {
                    const int64_t o = __shfl_sync(0xffffffffu, my_off, (kg + u) & 31);
#pragma unroll
                    for (int r = 0; r < R; ++r) xv[u][r] = 0.0;
                    if (u < nv) {
                        if (full && g.lo + o >= xlo_valid && g.hi + o <= xhi_valid) {  // common case
#pragma unroll
                            for (int r = 0; r < R; ++r) xv[u][r] = __ldg(xrow + lr(r) + o);
                        } else {
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const int64_t j = g.lo + lr(r) + o;
                                if (lr(r) < rows && j >= xlo_valid && j < xhi_valid) xv[u][r] = __ldg(xrow + lr(r) + o);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < XG; ++u) {
                    if (u < ng) {
                        mbar_wait(&S.full[cs], cphase);
                        const double* st = S.ring + cs * STRIDE;
                        double v[R];
                        if constexpr (IL) {
                            // odd bl: the slice may sit one slot in (see the producer;
                            // k*bl has k's parity, tile starts are even for R >= 2)
                            const int sh = !ODD ? 0
                                                : R >= 2 ? (kb0 + kg + u) & 1
                                                         : ((kb0 + kg + u) ^ (int)(g.lo - g.b0)) & 1;
#pragma unroll
                            for (int r = 0; r < R; ++r) v[r] = st[lr(r) + sh];
                        } else {
#pragma unroll
                            for (int h = 0; h < R / 2; ++h) {
                                const double2 t = reinterpret_cast<const double2*>(st + t0)[h];
                                v[2 * h] = t.x;
                                v[2 * h + 1] = t.y;
                            }
                        }
                        if (u < nv) {
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                double xx = xv[u][r];
                                if (SCALE) xx = __dmul_rn(xx, sc);
                                acc[r] = __dadd_rn(acc[r], __dmul_rn(v[r], xx));
                            }
                        }
                        // Release the stage only once this thread's shared loads have
                        // delivered (acc depends on them), then order the warp's reads
                        // before lane 0's arrive.
#pragma unroll
                        for (int r = 0; r < R; ++r) asm volatile("" ::"d"(acc[r]));
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&S.empty[cs]);
                        if (++cs == NS) {
                            cs = 0;
                            cphase ^= 1u;
                        }
                    }
                }
            }
        }

        if constexpr (IL) {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (lr(r) < rows) __stcs(a.y + g.lo + lr(r), acc[r]);
        } else if (t0 < rows) {
            if (a.y_vec_ok && t0 + R - 1 < rows) {
#pragma unroll
                for (int h = 0; h < R / 2; ++h)
                    __stcs(reinterpret_cast<double2*>(a.y + g.lo + t0) + h, make_double2(acc[2 * h], acc[2 * h + 1]));
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (t0 + r < rows) __stcs(a.y + g.lo + t0 + r, acc[r]);
            }
        }
        if (a.peer_lo || a.peer_hi) {  // halo rows also to the neighbours (peer memory)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t i = g.lo + lr(r);
                if (lr(r) >= rows) continue;
                if (a.peer_lo && i < a.halo) a.peer_lo[i] = acc[r];
                if (a.peer_hi && i >= a.n_rows - a.halo) a.peer_hi[i - (a.n_rows - a.halo)] = acc[r];
            }
        }
        if (NORM) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (lr(r) < rows) s = __dadd_rn(s, __dmul_rn(acc[r], acc[r]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
            // the tile's 8 warp partials in warp order, one consumer barrier per tile
            // (double-buffered partials).  A barrier-free variant (partials to a global
            // scratch, summed by a second kernel) measured 8% more DRAM reads at config 4
            // -- the x lines' L2 reuse across the +-nx*ny offsets suffered -- and was
            // dropped (profiles/r01_v14_norm_variants.log).
            double* ws = S.wsum + par * CONSUMER_WARPS;
            if (lane == 0) ws[warp] = s;
            consumer_sync();
            if (threadIdx.x == 0) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < CONSUMER_WARPS; ++w) t = __dadd_rn(t, ws[w]);
                a.tile_sumsq[tile] = t;
            }
            par ^= 1;  // the next tile writes the other buffer; its barrier orders this read
        }
    }
    // remote halo stores are visible system-wide before the kernel completes
    if (a.peer_lo || a.peer_hi) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Small blocks (8 <= bl < 256 outside the multi-block layout -- the paper's
// recommended bl = 50 / 100, and hdcmv's default bl = 100,
// hdcmv.cpp:148): a tile is G = 256/bl whole blocks, and its segments are ONE
// contiguous run of the segment array, seg[dia_ptr[b0]*bl, dia_ptr[b0+G]*bl).
// A ring stage holds a whole tile: the producer warp stages the tile's block
// starts (relative) and offsets in the stage header with plain loads/stores, and
// one cp.async.bulk brings the values (16-byte aligned: an odd start is copied
// from one slot earlier, the shift is in the header).  Consumer thread t owns
// tile row t (block q = t / bl, slot t % bl -- fixed for the whole kernel) and
// reads everything but x from shared memory: no dependent global loads before
// its x gathers.  Same per-row operations in the same order as spmv_kernel.
constexpr int BLK_MAX_SEG = 16;  // eligibility: max segments per block (27 segments measured slower)
constexpr int BLK_MAX_G = 32;    // bl >= 8
constexpr int BLK_XG = 8;        // x gathers in flight per thread

__host__ __device__ inline int blk_vals_stride(int max_seg, int G, int bl) {  // doubles, even
    return ((max_seg * G * bl + 2) + 1) & ~1;
}
__host__ __device__ inline int blk_hdr_ints(int max_seg, int G) {  // 4-int aligned
    return ((4 + G + 1 + max_seg * G) + 3) & ~3;
}

template <bool SCALE, bool NORM, int REST>
__global__ void __launch_bounds__(THREADS, 3) spmv_blk_kernel(const TmaArgs a, int max_seg) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NS = a.nstage;
    const int G = a.blocks_per_tile;
    const int bl = (int)a.bl;
    const int VST = blk_vals_stride(max_seg, G, bl);
    const int HST = blk_hdr_ints(max_seg, G);
    const size_t stage_bytes = sizeof(double) * VST + sizeof(int32_t) * HST;  // multiple of 16
    double* scratch = reinterpret_cast<double*>(smem_raw + stage_bytes * NS);  // CONSUMER_WARPS * WPASS
    double* wsum = scratch + (a.has_rest ? CONSUMER_WARPS * WPASS : 0);          // 2 * CONSUMER_WARPS
    uint64_t* full = reinterpret_cast<uint64_t*>(wsum + 2 * CONSUMER_WARPS);
    uint64_t* empty = full + NS;
    auto vals = [&](int s) { return reinterpret_cast<double*>(smem_raw + stage_bytes * s); };
    // header: [0] value shift, [1] segment count, [2] / [3] least / greatest offset,
    // [4 .. 4+G] block starts (relative), then the offsets
    auto hdr = [&](int s) { return reinterpret_cast<int32_t*>(smem_raw + stage_bytes * s + sizeof(double) * VST); };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == CONSUMER_WARPS) {
        // ------------------------------ producer warp ------------------------------
        const uint64_t policy = evict_first_policy();
        constexpr int OFR = 4;  // offsets per lane held in registers (nk <= 128; more: a loop)
        int ps = 0;
        uint32_t pphase = 0;
        bool p_wrapped = false;
        // the next tile's block starts are loaded while this tile's offsets are, and
        // both before the wait for a free stage (a deeper look-ahead measured no faster)
        int tile = a.tile_begin + blockIdx.x;
        auto starts = [&](int tl, int& dp, int& k1) {
            if (tl >= a.tile_end) return;
            const int64_t b0 = (int64_t)tl * G;
            const int nb = (int)min((int64_t)G, a.n_blocks - b0);
            dp = lane < nb ? __ldg(a.dia_ptr + b0 + lane) : 0;
            k1 = __ldg(a.dia_ptr + b0 + nb);
        };
        int dp_n = 0, k1_n = 0;
        starts(tile, dp_n, k1_n);
        for (; tile < a.tile_end; tile += gridDim.x) {
            const int64_t b0 = (int64_t)tile * G;
            const int nb = (int)min((int64_t)G, a.n_blocks - b0);
            const int dp = dp_n, k1 = k1_n;
            const int k0 = __shfl_sync(0xffffffffu, dp, 0);
            const int nk = k1 - k0;
            int ofr[OFR];
#pragma unroll
            for (int u = 0; u < OFR; ++u) {
                const int j = lane + 32 * u;
                ofr[u] = j < nk ? __ldg(a.dia_off + k0 + j) : 0;
            }
            starts(tile + gridDim.x, dp_n, k1_n);
            if (p_wrapped) mbar_wait(&empty[ps], pphase ^ 1u);
            int32_t* h = hdr(ps);
            const int sh = (int)(((int64_t)k0 * bl) & 1);
            if (lane < nb) h[4 + lane] = dp - k0;
            int32_t* ho = h + 4 + G + 1;
            int omin = 0x7fffffff, omax = -0x7fffffff;
#pragma unroll
            for (int u = 0; u < OFR; ++u) {
                const int j = lane + 32 * u;
                if (j < nk) {
                    ho[j] = ofr[u];
                    omin = min(omin, ofr[u]);
                    omax = max(omax, ofr[u]);
                }
            }
            for (int j = lane + 32 * OFR; j < nk; j += 32) {
                const int o = __ldg(a.dia_off + k0 + j);
                ho[j] = o;
                omin = min(omin, o);
                omax = max(omax, o);
            }
            omin = __reduce_min_sync(0xffffffffu, omin);
            omax = __reduce_max_sync(0xffffffffu, omax);
            if (lane == 0) {
                h[0] = sh;
                h[1] = nk;
                h[2] = omin;
                h[3] = omax;
                h[4 + nb] = nk;
            }
            __syncwarp();
            if (lane == 0) {
                if (nk > 0) {
                    const uint32_t bytes = (uint32_t)((((int64_t)nk * bl + sh + 1) & ~int64_t(1)) * 8);
                    mbar_expect_tx(&full[ps], bytes);
                    bulk_g2s(vals(ps), a.seg + (int64_t)k0 * bl - sh, bytes, &full[ps], policy);
                } else {
                    mbar_arrive(&full[ps]);
                }
            }
            if (++ps == NS) {
                ps = 0;
                pphase ^= 1u;
                p_wrapped = true;
            }
        }
        return;
    }

    // -------------------------------- consumers --------------------------------
    const int t = threadIdx.x;
    const int q = t / bl, l = t - q * bl;  // this thread's block in the tile and slot in it
    double sc = 1.0;
    if (SCALE) sc = *a.x_scale;
    const int64_t xlo_valid = -a.row0, xhi_valid = a.n_cols - a.row0;
    int cs = 0;
    uint32_t cphase = 0, par = 0;
    // REST == 1: the remainder entry range of this warp's rows, loaded one tile ahead
    // (most tiles of a light remainder have none: no dependent load on their path)
    auto probe = [&](int tl, int& e0, int& e1) {
        e0 = e1 = 0;
        if (REST != 1 || tl >= a.tile_end) return;
        const int64_t lo_t = (int64_t)tl * G * bl;
        const int64_t hi_t = min(lo_t + (int64_t)G * bl, a.n_rows);
        const int64_t w_lo = min(lo_t + 32 * warp, hi_t), w_hi = min(w_lo + 32, hi_t);
        e0 = __ldg(a.rest_rp + w_lo);
        e1 = __ldg(a.rest_rp + w_hi);
    };
    int pe0, pe1;
    probe(a.tile_begin + blockIdx.x, pe0, pe1);
    for (int tile = a.tile_begin + blockIdx.x; tile < a.tile_end; tile += gridDim.x) {
        const int64_t b0 = (int64_t)tile * G;
        const int nb = (int)min((int64_t)G, a.n_blocks - b0);
        const int64_t lo = b0 * bl;
        const int64_t hi = min(lo + (int64_t)nb * bl, a.n_rows);
        const int64_t i = lo + t;
        const bool active = q < nb && i < hi;
        double acc = 0.0;
        if constexpr (REST == 2) {
            if (active) acc = a.y[i];
        } else if constexpr (REST == 1) {
            const bool any = pe0 < pe1;
            probe(tile + gridDim.x, pe0, pe1);
            if (any) {
                double a1[1] = {0.0};
                warp_rest<1, SCALE>(a.rest_rp, a.rest_col, a.rest_val, a.x, a.row0, sc, lo, hi, warp, lane,
                                    scratch + warp * WPASS, a1);
                acc = a1[0];
            }
        }
        mbar_wait(&full[cs], cphase);
        const int32_t* h = hdr(cs);
        const int kst = active ? h[4 + q] : 0, kend = active ? h[4 + q + 1] : 0;
        const int cnt = kend - kst;
        const int cmax = __reduce_max_sync(0xffffffffu, cnt);
        const int32_t* op = h + 4 + G + 1 + kst;             // this row's offsets
        const double* vp = vals(cs) + h[0] + l + kst * bl;  // this row's first value
        // tile-uniform: every x index of the tile in range (the common case)
        const bool inr = lo + h[2] >= xlo_valid && hi + h[3] <= xhi_valid;
        const double* xr = a.x + i;
        for (int j0 = 0; j0 < cmax; j0 += BLK_XG) {
            double xv[BLK_XG];
#pragma unroll
            for (int u = 0; u < BLK_XG; ++u) {
                xv[u] = 0.0;
                if (j0 + u < cnt) {
                    const int o = op[j0 + u];
                    if (inr || (i + o >= xlo_valid && i + o < xhi_valid)) xv[u] = __ldg(xr + o);
                }
            }
            const double* vq = vp + j0 * bl;
#pragma unroll
            for (int u = 0; u < BLK_XG; ++u) {
                if (j0 + u < cnt) {
                    double xx = xv[u];
                    if (SCALE) xx = __dmul_rn(xx, sc);
                    acc = __dadd_rn(acc, __dmul_rn(*vq, xx));
                }
                vq += bl;
            }
        }
        asm volatile("" ::"d"(acc));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cs]);
        if (++cs == NS) {
            cs = 0;
            cphase ^= 1u;
        }
        if (active) {
            __stcs(a.y + i, acc);
            if (a.peer_lo && i < a.halo) a.peer_lo[i] = acc;
            if (a.peer_hi && i >= a.n_rows - a.halo) a.peer_hi[i - (a.n_rows - a.halo)] = acc;
        }
        if (NORM) {  // spmv_kernel's order: warp shuffle tree, then the warps in order
            double s = active ? __dmul_rn(acc, acc) : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
            double* ws = wsum + par * CONSUMER_WARPS;
            if (lane == 0) ws[warp] = s;
            consumer_sync();
            if (threadIdx.x == 0) {
                double tot = 0.0;
#pragma unroll
                for (int w = 0; w < CONSUMER_WARPS; ++w) tot = __dadd_rn(tot, ws[w]);
                a.tile_sumsq[tile] = tot;
            }
            par ^= 1;
        }
    }
    if (a.peer_lo || a.peer_hi) __threadfence_system();
}

template <bool SCALE, bool NORM, int REST>
void launch_blk(const TmaArgs& a, int max_seg, int grid, size_t smem, cudaStream_t st) {
    auto k = spmv_blk_kernel<SCALE, NORM, REST>;
    static PerDeviceFlag configured;  // the attribute is per device
    if (!configured.test_and_set(current_device_index()))
        HDCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    k<<<grid, THREADS, smem, st>>>(a, max_seg);
}

template <int REST>
void launch_blk_r(const TmaArgs& a, int max_seg, int grid, size_t smem, bool scale, bool norm, cudaStream_t st) {
    if (scale) {
        if (norm) launch_blk<true, true, REST>(a, max_seg, grid, smem, st);
        else launch_blk<true, false, REST>(a, max_seg, grid, smem, st);
    } else {
        if (norm) launch_blk<false, true, REST>(a, max_seg, grid, smem, st);
        else launch_blk<false, false, REST>(a, max_seg, grid, smem, st);
    }
}

template <int R, bool SCALE, bool NORM, int REST, int LAY>
void launch_one(const TmaArgs& a, int grid, size_t smem, cudaStream_t st) {
    auto k = spmv_tma_kernel<R, SCALE, NORM, REST, LAY>;
    static PerDeviceFlag configured;  // per instantiation and device
    if (!configured.test_and_set(current_device_index())) {
        HDCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        // fused: ~100 KB of the unified 228 KB as shared memory, the rest L1
        if (REST == 3)
            HDCG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           std::min(100, (int)((smem + 1023) / 1024 * 100 + 227) / 228)));
    }
    constexpr int threads = REST == 3 ? THREADS + 32 * GATHER_WARPS : THREADS;
    k<<<grid, threads, smem, st>>>(a);
}

template <int R, int REST, int LAY>
void launch_rr(const TmaArgs& a, int grid, size_t smem, bool scale, bool norm, cudaStream_t st) {
    if (scale) {
        if (norm) launch_one<R, true, true, REST, LAY>(a, grid, smem, st);
        else launch_one<R, true, false, REST, LAY>(a, grid, smem, st);
    } else {
        if (norm) launch_one<R, false, true, REST, LAY>(a, grid, smem, st);
        else launch_one<R, false, false, REST, LAY>(a, grid, smem, st);
    }
}

template <int R, int LAY>
void launch_m(const TmaArgs& a, int grid, size_t smem, bool scale, bool norm, cudaStream_t st) {
    if (a.fused) launch_rr<R, 3, LAY>(a, grid, smem, scale, norm, st);
    else if (a.init_y) launch_rr<R, 2, LAY>(a, grid, smem, scale, norm, st);
    else if (a.has_rest) launch_rr<R, 1, LAY>(a, grid, smem, scale, norm, st);
    else launch_rr<R, 0, LAY>(a, grid, smem, scale, norm, st);
}

template <int R>
void launch_r(const TmaArgs& a, int grid, size_t smem, bool scale, bool norm, cudaStream_t st) {
    if constexpr (R == 4) {
        if (a.pk_meta) return launch_m<4, 5>(a, grid, smem, scale, norm, st);
        if (a.blocks_per_tile > 0) {
            // bl = 256 without a remainder: block-local interleaved rows (tile layout 3)
            const bool plain = !a.has_rest && !a.init_y && !a.fused;
            if (a.bl == 256 && plain) return launch_rr<4, 0, 3>(a, grid, smem, scale, norm, st);
            if (a.bl == 128 && plain) return launch_rr<4, 0, 4>(a, grid, smem, scale, norm, st);
            return launch_m<4, 1>(a, grid, smem, scale, norm, st);
        }
    }
    if (a.bl % 2) launch_m<R, 2>(a, grid, smem, scale, norm, st);
    else launch_m<R, 0>(a, grid, smem, scale, norm, st);
}

}  // namespace

int sm_count() {
    static int n[64] = {0};
    const int dev = current_device_index() & 63;
    if (!n[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
}

bool spmv_tma_launch(const Matrix& m, const double* x_local, double* y, int64_t tile_begin, int64_t tile_end,
                     const double* x_scale, double* tile_sumsq, cudaStream_t st, const PeerOut& peer) {
    if (m.n_seg > 0 && ((uintptr_t)m.seg % 16) != 0) return false;
    if (m.nnz_rest > 0 && (((uintptr_t)m.rest_col % 16) != 0 || ((uintptr_t)m.rest_val % 16) != 0)) return false;
    const Tiling t = tiling_of(m);
    const int R = t.rows_per_thread;
    if (t.tile_rows != (int64_t)CONSUMERS * R) return false;
    // multi-block tiles: R = 4 (bl in {128, 256, 512}, tiling_of) only
    // small blocks, 8 <= bl < 256: whole-tile stages (spmv_blk_kernel); HDCG_BLK=0 disables (A/B)
    const char* eb = getenv("HDCG_BLK");
    const bool blk = (!eb || atoi(eb) != 0) && t.blocks_per_tile > 0 && R == 1 && m.bl >= CONSUMERS / BLK_MAX_G &&
                     m.bl < CONSUMERS && m.max_seg_per_block <= BLK_MAX_SEG;
    if (!blk && !t.packed && t.tiles_per_block <= 0 && (R != 4 || t.blocks_per_tile <= 0 || m.bl % (32 * R) != 0))
        return false;
    if (tile_end <= tile_begin) return true;
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
    a.tiles_per_block = (int)t.tiles_per_block;
    a.blocks_per_tile = (int)t.blocks_per_tile;
    a.n_blocks = m.n_blocks;
    a.tile_begin = (int)tile_begin;
    a.tile_end = (int)tile_end;
    a.has_rest = m.nnz_rest > 0;
    a.init_y = 0;
    a.pk_val = t.packed ? m.pk_val : nullptr;
    a.pk_meta = t.packed ? m.pk_meta : nullptr;
    a.pk_tab = t.packed ? m.pk_tab : nullptr;
    a.y_vec_ok = ((uintptr_t)y % 16) == 0;  // (odd bl: tiles may start on odd rows, tested per thread)
    a.peer_lo = peer.lo;
    a.peer_hi = peer.hi;
    a.halo = peer.halo;
    {  // HDCG_TMA_PREFETCH: A/B knob (read per call).  Default: on for multi-block
       // tiles only -- there every tile starts on fresh block pointers and offsets
       // (+0.5-1.5 points at bl = 256/512), while for tiles inside large blocks it
       // cost 4-8 points at config 4 (profiles/r01_v11_prefetch_ab.log)
        const char* e = getenv("HDCG_TMA_PREFETCH");
        a.prefetch = e ? atoi(e) : (t.blocks_per_tile > 0 ? 1 : 0);
    }
    // Remainder mode (hdcg_set_kernel_policy / HDCG_REST_MODE override the default):
    // 3 summed into y by the CTA's gather warps, tiles ahead of the consumers --
    // remainder-heavy (>= 1 entry per 4 rows) M-HDC; 2 summed first into y by
    // rest_pipe_kernel -- remainder-heavy HDC and CSR; 1 loaded from global
    // memory by the consumers -- every other matrix.  (A producer staging the remainder through the ring
    // measured 33% at config 3 and was removed: profiles/README.md.)
    static const int env_mode = getenv("HDCG_REST_MODE") ? atoi(getenv("HDCG_REST_MODE")) : 0;
    const int req = g_rest_mode ? g_rest_mode : env_mode;
    const bool heavy = m.nnz_rest * 4 >= m.n_rows;
    const bool fusable = !blk && m.n_seg > 0;
    // Mode 3 is the default for remainder-heavy M-HDC (config 3: 0.62-0.65 ms
    // against 0.68 ms for mode 2, profiles/r02i_ab_fused_smem_sweep.log); HDC
    // (one block of n rows) measured 3% slower fused than split, so it keeps mode 2.
    // A banded heavy remainder (a stencil converted with a high theta: rows of
    // adjacent columns) is summed first by rest_rows_kernel, which runs near the HBM
    // peak there (27-point 192^3 at theta = 1: 0.39 ms split vs 0.57 ms fused,
    // profiles/r03k_ab_theta1.log); the gather warps are for scattered columns.
    const bool banded = rest_rows_default(m);
    int mode = req >= 1 && req <= 3 ? req
                                    : (heavy ? (fusable && m.kind == HDCG_KIND_MHDC && !banded ? 3 : 2) : 1);
    if (mode == 3 && !fusable) mode = 2;
    const bool split = a.has_rest && mode == 2;
    a.fused = a.has_rest && mode == 3;
    if (a.fused) a.has_rest = 0;  // no consumer scratch: the gather warps own the remainder
    auto rest_rows = [&](int64_t tb, int64_t te, cudaStream_t s) {
        // rows covered by the tile range (tiles are contiguous in rows)
        int64_t r0, r1, dummy;
        tile_rows(tb, t.tiles_per_block, t.blocks_per_tile, t.tile_rows, m.bl, m.n_rows, &r0, &dummy);
        tile_rows(te - 1, t.tiles_per_block, t.blocks_per_tile, t.tile_rows, m.bl, m.n_rows, &dummy, &r1);
        r0 = std::min(r0, m.n_rows);
        if (r1 <= r0) return;
        // HDCG_REST_VARIANT: A/B knob, read per call (tests switch it in-process):
        // 0 rest_kernel, 1-4 rest_pipe_kernel shapes, 5 (default) rest_rows_kernel
        const char* ev = getenv("HDCG_REST_VARIANT");
        const int variant = ev ? atoi(ev) : 5;
        auto pipe = [&](auto kern, int g) {
            kern<<<(unsigned)ceil_div(r1 - r0, (int64_t)CONSUMERS * g), CONSUMERS, 0, s>>>(a, r0, r1);
        };
        switch (variant) {
            case 0: {  // rest_kernel: 5 CTAs/SM, one row per lane, 8 gathers per lane in flight
                const unsigned nb = (unsigned)ceil_div(r1 - r0, CONSUMERS);
                if (x_scale) rest_kernel<true, 5, 1, 8><<<nb, CONSUMERS, 0, s>>>(a, r0, r1);
                else rest_kernel<false, 5, 1, 8><<<nb, CONSUMERS, 0, s>>>(a, r0, r1);
                break;
            }
            case 2:
                if (x_scale) pipe(rest_pipe_kernel<true, 3, 4, 8>, 4);
                else pipe(rest_pipe_kernel<false, 3, 4, 8>, 4);
                break;
            case 3:
                if (x_scale) pipe(rest_pipe_kernel<true, 4, 8, 4>, 8);
                else pipe(rest_pipe_kernel<false, 4, 8, 4>, 8);
                break;
            case 4:
                if (x_scale) pipe(rest_pipe_kernel<true, 3, 16, 8>, 16);
                else pipe(rest_pipe_kernel<false, 3, 16, 8>, 16);
                break;
            case 5:  // one row per lane, entry streams staged by TMA (spmv_rows.cu), when eligible
                if (rest_rows_launch(m, x_local, y, x_scale, r0, r1, s)) break;
                [[fallthrough]];
            default:
                if (x_scale) pipe(rest_pipe_kernel<true, 3, 8, 8>, 8);
                else pipe(rest_pipe_kernel<false, 3, 8, 8>, 8);
        }
        HDCG_LAUNCH_CHECK("rest_kernel");
    };
    // ring of segment slices: ~64 KB per CTA, 3 CTAs per SM (tunable for profiling)
    static const int env_kb = getenv("HDCG_TMA_STAGE_KB") ? atoi(getenv("HDCG_TMA_STAGE_KB")) : 0;
    static const int env_ctas = getenv("HDCG_TMA_CTAS") ? atoi(getenv("HDCG_TMA_CTAS")) : 0;
    auto tma = [&](const TmaArgs& base, int64_t tb, int64_t te, int want_ctas, cudaStream_t s) {
        // (REST 3 needs one CTA's gather warps and consumers on the same tiles: any grid works)
        TmaArgs b = base;
        b.tile_begin = (int)tb;
        b.tile_end = (int)te;
        if (blk) {
            const int G = (int)t.blocks_per_tile, ms = (int)std::max<int64_t>(1, m.max_seg_per_block);
            const size_t stage = sizeof(double) * blk_vals_stride(ms, G, (int)m.bl) + sizeof(int32_t) * blk_hdr_ints(ms, G);
            const size_t fixed = sizeof(double) * ((b.has_rest ? CONSUMER_WARPS * WPASS : 0) + 2 * CONSUMER_WARPS) +
                                 sizeof(uint64_t) * 2 * 32;
            // >= 3 stages per CTA: fewer CTAs per SM when the stages are large
            int want = want_ctas;
            auto stages_for = [&](int w) {
                const size_t budget = env_kb > 0 ? (size_t)env_kb * 1024 + fixed : (227 * 1024) / w - 1024;
                return std::max(2, std::min(32, (int)((budget > fixed ? budget - fixed : 0) / stage)));
            };
            while (want > 1 && stages_for(want) < 3) --want;
            b.nstage = stages_for(want);
            const size_t smem = stage * b.nstage + fixed;
            const int fit = (int)((227 * 1024) / (smem + 1024));
            const int per_sm = std::max(1, std::min(want, fit));
            const int64_t cap = (int64_t)sm_count() * per_sm;
            const int grid = (int)(te - tb < cap ? te - tb : cap);
            const bool sc = x_scale != nullptr, nm = tile_sumsq != nullptr;
            if (b.init_y) launch_blk_r<2>(b, ms, grid, smem, sc, nm, s);
            else if (b.has_rest) launch_blk_r<1>(b, ms, grid, smem, sc, nm, s);
            else launch_blk_r<0>(b, ms, grid, smem, sc, nm, s);
            HDCG_LAUNCH_CHECK("spmv_blk_kernel");
            return;
        }
        // fused: 24 warps per CTA, one CTA per SM, and at most ~98 KB of shared
        // memory -- the rest of the unified 228 KB stays L1, which holds the
        // gather warps' outstanding x misses (with the whole array as shared
        // memory the gathers crawled: profiles/r02g_ab_fused_v2.log)
        if (b.fused) want_ctas = 1;
        const size_t stage = smem_bytes(R, 1, 0) - smem_bytes(R, 0, 0);
        const size_t fixed = smem_bytes(R, 0, b.has_rest, b.fused);
        static const int fused_kb = getenv("HDCG_FUSED_KB") ? atoi(getenv("HDCG_FUSED_KB")) : 98;  // A/B knob
        // Ring of ~48 KB per CTA (3 CTAs per SM: ~150 KB of shared memory): the
        // rest of the unified 228 KB stays L1, where the x lines of a tile's
        // offsets are reused.  With the whole array as ring (3 x 73 KB) the x loads
        // missed L1 (18% hits) and config 4 ran at 92% of the copy peak; with 48 KB
        // it runs at 104%, configs 1-2 at 96-99% (profiles/r02n_ab_ring_sweep.log).
        const size_t budget = env_kb > 0 ? (size_t)env_kb * 1024 + fixed
                              : b.fused ? (size_t)fused_kb * 1024
                                        : std::min<size_t>((227 * 1024) / want_ctas - 1024, 48 * 1024 + fixed);
        b.nstage = std::max(2, std::min(32, (int)((budget > fixed ? budget - fixed : 0) / stage)));
        const size_t smem = smem_bytes(R, b.nstage, b.has_rest, b.fused);
        const int fit = (int)((227 * 1024) / (smem + 1024));
        const int per_sm = std::max(1, std::min(want_ctas, fit));
        const int64_t cap = (int64_t)sm_count() * per_sm;
        const int grid = (int)(te - tb < cap ? te - tb : cap);
        if (R == 4) launch_r<4>(b, grid, smem, x_scale != nullptr, tile_sumsq != nullptr, s);
        else if (R == 2) launch_r<2>(b, grid, smem, x_scale != nullptr, tile_sumsq != nullptr, s);
        else launch_r<1>(b, grid, smem, x_scale != nullptr, tile_sumsq != nullptr, s);
        HDCG_LAUNCH_CHECK("spmv_tma_kernel");
    };
    if (split) {
        rest_rows(tile_begin, tile_end, st);
        // no segments (a CSR, spmv_csr): rest_kernel's sums are y -- unless the
        // TMA kernel's epilogue is needed (fused norm, peer halo stores)
        if (m.n_seg == 0 && !tile_sumsq && !peer.lo && !peer.hi) return true;
        a.has_rest = 0;
        a.init_y = 1;
    }
    tma(a, tile_begin, tile_end, env_ctas > 0 ? env_ctas : 3, st);
    return true;
}

}  // namespace hdcg

/*
 * hdcgpu.h -- C-ABI of the B200 (sm_100a) HDC / M-HDC SpMV library
 *             (paper_2105_04937_b200/libhdcgpu.so).
 *
 * This is the drop-in boundary for the reference's format-build and SpMV
 * path (arXiv 2105.04937; reference at proj/include/hdc/*.hpp).  Every entry
 * point below names the reference interface it replaces.  The reference's
 * C++ signatures (hdc::to_mhdc, hdc::spmv_mhdc, ...) are re-declared on top
 * of this ABI by the shim in paper_2105_04937_b200/shim/hdc_gpu_shim.cpp;
 * see INTEGRATION.md for the binding a maintainer links in.
 *
 * Conventions
 *   - plain pointers and sizes only; sizes are int64_t.
 *   - index arrays follow the reference's default index_t = int32
 *     (proj/include/hdc/types.hpp:8-12); an input row pointer may be int64
 *     (HDCG_ROWPTR_I64) so inputs with nnz > 2^31-1 can be converted.
 *   - a matrix is an opaque, immutable, device-resident handle (the
 *     reference's matrices are immutable after construction).
 *   - every function returns an hdcg_status; on failure hdcg_last_error()
 *     returns the message (thread-local).  Status codes map one-to-one onto
 *     the exception types the reference throws (convert.cpp:16-19,125,175;
 *     kernels.cpp:21-29; formats.cpp:45-163).
 *   - there is no CPU fallback: without a usable sm_100 device every call
 *     fails with HDCG_ERR_NO_DEVICE.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Functions
 *     taking device pointers and a stream are asynchronous; the *_host
 *     variants are synchronous like the reference (y valid on return).
 */
#ifndef HDCGPU_H
#define HDCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HDCG_OK = 0,
    HDCG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    HDCG_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    HDCG_ERR_OVERFLOW = 3,         /* std::overflow_error (index range exceeded) */
    HDCG_ERR_CUDA = 4,             /* CUDA runtime failure */
    HDCG_ERR_NO_DEVICE = 5,        /* no usable sm_100 device */
    HDCG_ERR_OUT_OF_MEMORY = 6,    /* std::bad_alloc */
    HDCG_ERR_IO = 7                /* std::runtime_error from Matrix Market reading (io.cpp) */
} hdcg_status;

/* flags */
#define HDCG_INPUT_DEVICE 1u /* input arrays are device pointers (default: host) */
#define HDCG_VALIDATE 2u     /* apply the CsrMatrix invariants (formats.cpp:45-67) to the input */
#define HDCG_ROWPTR_I64 4u   /* the input row pointer is int64_t[] (default int32_t[]) */

typedef enum { HDCG_KIND_MHDC = 0, HDCG_KIND_HDC = 1, HDCG_KIND_CSR = 2 } hdcg_kind;

typedef struct hdcg_matrix_s* hdcg_matrix;

typedef struct {
    int32_t kind;       /* hdcg_kind */
    int32_t device;     /* CUDA ordinal the matrix lives on */
    int64_t n_rows;     /* rows held (a row slab for sharded matrices) */
    int64_t n_cols;     /* global dimension n */
    int64_t row0;       /* global index of local row 0 (multiple of bl) */
    int64_t bl;         /* block width; HDC: n, CSR: max(n_rows, 1) */
    int64_t n_blocks;   /* ceil(n_rows / bl) */
    int64_t n_seg;      /* stored diagonal segments (HDC: lanes) */
    int64_t nnz_rest;   /* CSR remainder entries */
    int64_t dia_slots;  /* rates().dia_slots: segments x true block lengths */
    int64_t nnz_input;  /* stored entries of the original CSR (2*nnz flops / SpMV) */
    int64_t n_tiles;    /* SpMV tiles (one sum-of-squares partial each) */
    int64_t tile_rows;  /* rows per tile (tiles never straddle a block, except packed tiles) */
    int64_t blocks_per_tile; /* block-range granularity of hdcg_spmv_slab: ranges start and end
                                at multiples of it (or at n_blocks); >1 when tiles hold several
                                blocks, lcm(1024, bl) / bl for packed small blocks */
    int64_t device_bytes;
    int64_t max_seg_per_block; /* most segments in one block (selects the SpMV kernel) */
    int64_t packed_stages; /* >0: small blocks also stored tile-packed (1024-value stages) */
    int64_t rest_rows_kernel; /* 1: remainder-first / CSR row sums take the row-per-lane kernel
                                 (banded rows, sampled at build time), 0: the entry-major one */
} hdcg_info;

/* ---- runtime ------------------------------------------------------------ */
const char* hdcg_last_error(void);
int hdcg_version(void);
/* Selects / initialises the device (creates the context).  Optional. */
hdcg_status hdcg_init(int device);

/* ---- format build on the device ----------------------------------------- *
 * hdcg_build_mhdc replaces  hdc::to_mhdc(const CsrMatrix&, real_t theta, index_t bl)
 *                           (proj/include/hdc/convert.hpp:39; convert.cpp:123-169).
 * The input is a CSR row slab: rows [row0, row0+n_rows) of an n_cols x n_cols
 * matrix with global column indices.  row0 must be a multiple of bl and the
 * slab must end at n_cols or at a multiple of bl, so the slab's blocks are
 * exactly the global blocks and the result is bit-identical to the
 * corresponding rows of the global conversion.  Single-GPU use: row0 = 0,
 * n_rows = n_cols = n.  Errors: theta outside [0,1] or bl < 1 ->
 * INVALID_ARGUMENT (convert.cpp:16-19,125); with HDCG_VALIDATE, the CsrMatrix
 * constructor's checks (formats.cpp:45-67). */
hdcg_status hdcg_build_mhdc(int64_t n_rows, int64_t n_cols, int64_t row0, int64_t nnz,
                            const void* row_ptr, const int32_t* col_ind, const double* values,
                            double theta, int64_t bl, unsigned flags, void* stream,
                            hdcg_matrix* out);

/* Replaces hdc::to_hdc(const CsrMatrix&, real_t theta) (convert.hpp:34; convert.cpp:89-121).
 * With theta = 0 every populated diagonal becomes a lane: hdc::to_dia
 * (convert.cpp:69-87) is the DIA part of that result. */
hdcg_status hdcg_build_hdc(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                           const double* values, double theta, unsigned flags, void* stream,
                           hdcg_matrix* out);

/* A plain CSR held for hdcg_spmv (replaces the operand of hdc::spmv_csr,
 * kernels.hpp:31). */
hdcg_status hdcg_build_csr(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                           const double* values, unsigned flags, void* stream, hdcg_matrix* out);

/* Upload an already-built host M-HDC / HDC (the arrays of hdc::MHdcMatrix,
 * formats.hpp:107-132, or hdc::HdcMatrix, formats.hpp:86-100) so that the
 * shim's spmv_mhdc(const MHdcMatrix&, ...) can run on the device.  The
 * MHdcMatrix constructor's structural checks (formats.cpp:131-163) are
 * applied with HDCG_VALIDATE. */
hdcg_status hdcg_upload_mhdc(int64_t n, int64_t bl, const int32_t* dia_ptr, int64_t n_seg,
                             const int32_t* dia_offsets, const double* segments,
                             const int32_t* rest_row_ptr, int64_t nnz_rest,
                             const int32_t* rest_col_ind, const double* rest_values,
                             unsigned flags, hdcg_matrix* out);
hdcg_status hdcg_upload_hdc(int64_t n, int64_t n_diag, const int32_t* offsets, const double* lanes,
                            const int32_t* rest_row_ptr, int64_t nnz_rest,
                            const int32_t* rest_col_ind, const double* rest_values,
                            unsigned flags, hdcg_matrix* out);

/* Matrix Market file -> device-resident CSR handle (kind HDCG_KIND_CSR; the CSR
 * arrays are what hdcg_export returns as the remainder).  Replaces
 * hdc::io::read_matrix_market (proj/include/hdc/io.hpp:14-20, io.cpp:69-121) +
 * CooMatrix normalisation (formats.cpp:19-43) + CsrMatrix::from_coo
 * (formats.cpp:69-88): same accepted formats (coordinate real / integer /
 * pattern; general / symmetric / skew-symmetric), same checks and messages
 * (HDCG_ERR_IO), duplicates summed in file order, bit-identical arrays. */
hdcg_status hdcg_read_matrix_market(const char* path, hdcg_matrix* out);

hdcg_status hdcg_free(hdcg_matrix m);

/* ---- inspection ---------------------------------------------------------- */
hdcg_status hdcg_get_info(hdcg_matrix m, hdcg_info* info);

/* Copy the format out to HOST buffers sized from hdcg_info (any may be NULL):
 * dia_ptr[n_blocks+1], dia_offsets[n_seg], segments[n_seg*bl],
 * rest_row_ptr[n_rows+1], rest_col_ind[nnz_rest], rest_values[nnz_rest].
 * For HDC, segments are the lanes (n_diag*n) and dia_ptr is {0, n_diag}. */
hdcg_status hdcg_export(hdcg_matrix m, int32_t* dia_ptr, int32_t* dia_offsets, double* segments,
                        int32_t* rest_row_ptr, int32_t* rest_col_ind, double* rest_values);

/* The format restricted to the row blocks [block_begin, block_end) -- one slab
 * of a large matrix, for bit-exact checks of matrices too large to export whole
 * (config 4: 30 GB of segments).  Same layout as hdcg_export with the block
 * pointer and the remainder row pointer rebased to 0 at the first block / row:
 * dia_ptr int32[nb+1], dia_offsets int32[n_seg_range], segments
 * double[n_seg_range*bl], rest_row_ptr int32[rows+1], rest_col_ind /
 * rest_values [nnz_rest_range] (columns stay global).  counts (int64[2], may be
 * NULL) receives {n_seg_range, nnz_rest_range}; any array may be NULL (call
 * once with NULLs to size them).  No reference counterpart (the reference's
 * containers expose their vectors directly, formats.hpp:107-132). */
hdcg_status hdcg_export_blocks(hdcg_matrix m, int64_t block_begin, int64_t block_end, int32_t* dia_ptr,
                               int32_t* dia_offsets, double* segments, int32_t* rest_row_ptr,
                               int32_t* rest_col_ind, double* rest_values, int64_t* counts);

/* Replaces hdc::rates(const HdcMatrix&) / rates(const MHdcMatrix&)
 * (convert.hpp:45-52; convert.cpp:173-196), computed on the device from the
 * stored format.  INVALID_ARGUMENT when the matrix holds no nonzeros. */
hdcg_status hdcg_rates(hdcg_matrix m, double* alpha, double* beta, int64_t* dia_slots);

/* Replaces hdc::census_blocked / census_global (convert.hpp:26-32;
 * convert.cpp:39-67).  Two calls: with offsets == NULL only *n_entries and
 * block_ptr (host int64[n_blocks+1], may be NULL) are produced; then
 * offsets / counts (host, n_entries each) are filled.  bl <= 0 means the
 * global census (one block of width n). */
hdcg_status hdcg_census(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                        int64_t bl, unsigned flags, int64_t* block_ptr, int32_t* offsets,
                        int64_t* counts, int64_t* n_entries);

/* (theta, bl) parameter sweep, the loop of `hdcmv analyze` (proj/tools/hdcmv.cpp:93-140):
 * for every theta, rates(to_hdc(m, theta)) and, for every bl, rates(to_mhdc(m, theta, bl))
 * (convert.cpp:173-196), computed from ONE device census per block width instead of
 * building each format.  out (host) holds n_theta x (1 + n_bl) records of 4 doubles
 * {alpha, beta, dia_slots, n_diags or n_segments}, record (t, 0) for HDC and
 * (t, 1 + j) for M-HDC with bls[j]; alpha = beta = NaN where rates() would throw
 * (no nonzeros).  Requires nnz < 2^31 and 1 <= n_theta <= 64. */
hdcg_status hdcg_analyze(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                         const double* values, const double* thetas, int n_theta, const int64_t* bls,
                         int n_bl, unsigned flags, double* out);

/* ---- SpMV ------------------------------------------------------------------
 * hdcg_spmv replaces hdc::spmv_mhdc / spmv_hdc / spmv_bhdc / spmv_csr /
 * spmv_dia / spmv_bdia (proj/include/hdc/kernels.hpp:31-49).  One kernel
 * family serves all: per row, the CSR remainder is summed from +0.0 in stored
 * order, then each diagonal segment is added in stored (ascending-offset)
 * order over its valid rows, multiply and add separately rounded (no FMA) --
 * the reference's per-row order (kernels.cpp:123-135,158-169,192-204), so y
 * is bitwise equal to the reference for every kernel.
 * x and y are DEVICE pointers of n elements; asynchronous on `stream`. */
hdcg_status hdcg_spmv(hdcg_matrix m, const double* x, double* y, void* stream);

/* Same with HOST x / y (pageable or pinned); the host<->device copies are
 * part of the call, which returns when y is complete.  This is the call the
 * reference-facing shim makes. */
hdcg_status hdcg_spmv_host(hdcg_matrix m, const double* x, double* y);

/* Row-slab form used by the multi-GPU driver and the power iteration.
 *   x_local : device pointer such that x_local[j - row0] is x_j for every
 *             global column j the computed rows reference (a slab's x buffer
 *             with its halos, offset to the first owned row);
 *   y       : device pointer to the slab's n_rows outputs;
 *   [block_begin, block_end) : blocks to compute (aligned to
 *             blocks_per_tile, or ending at n_blocks);
 *   x_scale : NULL, or a device scalar s: x_j is used as x_j * s
 *             (power iteration x <- y * (1/||y||), fused into the load);
 *   tile_sumsq : NULL, or device double[n_tiles]: per-tile sum of y_i^2,
 *             summed in a fixed order (deterministic). */
hdcg_status hdcg_spmv_slab(hdcg_matrix m, const double* x_local, double* y, int64_t block_begin,
                           int64_t block_end, const double* x_scale, double* tile_sumsq,
                           void* stream);

/* Row-slab SpMV that also delivers the slab's halo rows to its neighbours
 * through peer memory (NVLink P2P stores from the SpMV epilogue -- the
 * exchange overlaps the computation tile by tile, no separate collective):
 * as hdcg_spmv_slab, and additionally rows i < halo are stored to
 * peer_lo[i] (the lower neighbour's upper halo) and rows i >= n_rows - halo to
 * peer_hi[i - (n_rows - halo)] (the upper neighbour's lower halo), followed by
 * a system-scope fence.  peer_lo / peer_hi may be NULL (no such neighbour) and
 * are device pointers valid on this device (hdcg_peer_open).  The caller orders
 * the neighbour's reads after this kernel (the power iteration's per-step norm
 * all-gather does).  There is no reference counterpart: the reference has no
 * distributed path. */
hdcg_status hdcg_spmv_slab_halo(hdcg_matrix m, const double* x_local, double* y, int64_t block_begin,
                                int64_t block_end, const double* x_scale, double* tile_sumsq, double* peer_lo,
                                double* peer_hi, int64_t halo, void* stream);

/* Peer memory for the halo exchange: hdcg_peer_alloc returns a device buffer
 * on the current device and its 64-byte inter-process handle; another process
 * (another GPU of the node, or the same GPU) maps it with hdcg_peer_open
 * (peer access enabled lazily) and unmaps it with hdcg_peer_close;
 * hdcg_peer_free releases the owner's buffer. */
hdcg_status hdcg_peer_alloc(int64_t bytes, void** ptr, unsigned char handle[64]);
hdcg_status hdcg_peer_open(const unsigned char handle[64], void** ptr);
hdcg_status hdcg_peer_close(void* ptr);
hdcg_status hdcg_peer_free(void* ptr);

/* Kernel selection (process-wide): policy & 3 = 0 automatic (the TMA-fed
 * persistent kernel for even bl >= 256, the general kernel otherwise), 1 general
 * kernel only, 2 TMA kernel only (ineligible shapes then fail with
 * INVALID_ARGUMENT); policy >> 4 = how the TMA kernel reads the CSR remainder:
 * 0 default, 1 consumers load it from global memory, 2 a separate kernel sums
 * it into y first, 3 gather warps of the same kernel sum it into shared memory
 * for the tiles ahead of the consumers (matrices with segments).  All produce
 * bitwise identical y and tile sums; this exists for testing. */
hdcg_status hdcg_set_kernel_policy(int policy);

/* Deterministic pairwise-tree sum of vals[0..count) (padded with +0.0 to a
 * power of two): out[0] = sum, out[1] = 1/sqrt(sum).  The tree over a
 * power-of-two aligned sub-range is a subtree of the tree over the whole
 * range, so per-rank partials combined by a second call give the same bits
 * as one call over all tiles. */
hdcg_status hdcg_tree_sum(const double* vals, int64_t count, double* out, void* stream);

/* ---- device memory benchmark -----------------------------------------------
 * Replaces hdc::bench::membench(n, mode, cfg) (proj/include/hdc/bench.hpp:33-45,
 * bench.cpp:68-110) on the device: c[i] += a[i]*b[i] (mode 0, direct, 32 B per
 * element) or c[i] += a[i]*b[idx[i]] (mode 1, indirect, 36 B per element),
 * one untimed loop then n_loops timed loops of n_ites calls, best per-call
 * average; loop_times (host, n_loops entries) may be NULL.  Errors as the
 * reference: INVALID_ARGUMENT for n < 1, n_loops < 1 or n_ites < 1. */
hdcg_status hdcg_membench(int64_t n, int mode, int n_loops, int n_ites, double* best_time_s,
                          double* bytes_per_s, double* loop_times);

/* ---- synthetic inputs (bench / test support, device side) ----------------
 * The same counter-based generator as paper_2105_04937_b200/synth.py:
 *   u(seed, stream, i) = (splitmix64(key(seed, stream) + i) >> 11) * 2^-53
 * out[k] = 2*u(seed, stream, first + k) - 1. */
hdcg_status hdcg_gen_uniform_pm1(uint64_t seed, uint64_t rng_stream, int64_t first, int64_t count,
                                 double* out, void* stream);

/* 7-point Dirichlet Laplacian (BASELINE configs 0, 1, 4), rows of z-planes
 * [z0, z1) of an nx*ny*nz grid, global columns.  Two calls: with row_ptr ==
 * NULL only *nnz is returned; then device row_ptr (int64[n_rows+1]),
 * col_ind, values are filled. */
hdcg_status hdcg_gen_laplacian7(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1,
                                int64_t* row_ptr, int32_t* col_ind, double* values, int64_t* nnz,
                                void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HDCGPU_H */

// Internal declarations shared by the CUDA translation units of libhdcgpu.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "hdcgpu.h"

namespace hdcg {

// ---- errors ---------------------------------------------------------------
// Internal code throws Error; the C-ABI layer (capi.cu) converts it into an
// hdcg_status + message.  Nothing ever falls back to the CPU.
struct Error : std::runtime_error {
    hdcg_status status;
    Error(hdcg_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(hdcg_status s, const std::string& msg) { throw Error(s, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation)
        fail(HDCG_ERR_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
        e == cudaErrorNoKernelImageForDevice)
        fail(HDCG_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    fail(HDCG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define HDCG_CUDA(call) ::hdcg::cuda_check((call), #call)
#define HDCG_LAUNCH_CHECK(name) ::hdcg::cuda_check(cudaGetLastError(), name)

// Makes `dev` current for the lifetime of the guard and restores the caller's
// device afterwards: every entry point that takes a matrix handle runs on the
// matrix's device, whatever the calling thread had selected.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        HDCG_CUDA(cudaGetDevice(&prev));
        if (prev != dev) HDCG_CUDA(cudaSetDevice(dev));
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Per-device one-time state: kernel attributes (max dynamic shared memory) apply
// to the current device only, so a process that uses matrices on several GPUs
// configures each kernel once per device.
inline int current_device_index() {
    int dev = 0;
    HDCG_CUDA(cudaGetDevice(&dev));
    return dev;
}
struct PerDeviceFlag {
    uint64_t bits = 0;  // devices 0..63
    bool test_and_set(int dev) {
        const uint64_t b = 1ull << (dev & 63);
        const bool was = (__atomic_fetch_or(&bits, b, __ATOMIC_ACQ_REL) & b) != 0;
        return was;
    }
};
int sm_count();  // of the current device (cached per device)

// ---- the device-resident matrix -------------------------------------------
// One storage layout serves M-HDC, HDC (bl = n, one block, lanes) and CSR
// (no diagonal part):
//   dia_ptr  int32[n_blocks+1]  exclusive prefix of per-block segment counts
//   dia_off  int32[n_seg]       ascending within a block
//   seg      f64[n_seg*bl]      segment k at [k*bl, (k+1)*bl), slot = i - ib*bl
//   rest_rp  int32[n_rows+1]    remainder CSR (rows local, columns global)
//   rest_col int32[nnz_rest]
//   rest_val f64[nnz_rest]
struct Matrix {
    hdcg_kind kind = HDCG_KIND_MHDC;
    int device = 0;
    int64_t n_rows = 0, n_cols = 0, row0 = 0, bl = 1, n_blocks = 0;
    int64_t n_seg = 0, nnz_rest = 0, nnz_input = 0, dia_slots = 0;
    int64_t max_seg_per_block = 0;  // selects rows per thread (tiling_of)
    int64_t rest_run_max = 0;       // most remainder entries in 32 aligned consecutive rows (rest_run_stats)
    double rest_lines_per_gather = 32.0;  // distinct x lines per row-per-lane warp gather (sampled; rest_run_stats)
    int32_t* dia_ptr = nullptr;
    int32_t* dia_off = nullptr;
    double* seg = nullptr;
    int32_t* rest_rp = nullptr;
    int32_t* rest_col = nullptr;
    double* rest_val = nullptr;
    // Tile-packed copy of the segments for small blocks (pack.cu; bl < 1024 where
    // 1024-row tiles do not hold whole blocks): tile t = rows [1024 t, 1024 t +
    // 1024) is K_t stages of 1024 values, stage k holding the k-th segment of each
    // row's block (0.0 where that block has fewer), so the SpMV streams whole
    // 8 KB stages with 4 rows per thread whatever bl is.  The reference layout
    // above stays the source of truth (export, rates, the general kernel).
    bool packed = false;
    double* pk_val = nullptr;     // stages * 1024 doubles
    int4* pk_meta = nullptr;      // per tile {first stage, K_t | uniform << 16, table start, first block}
    int32_t* pk_tab = nullptr;    // per tile: [blocks of the tile][K_t] offsets (one list when uniform)
    int64_t pk_stages = 0;
    // lazily built state of the host-buffer SpMV pipeline (host_spmv.cu): the
    // chunk plan is shared; each concurrent caller borrows its own context
    // (device x/y buffers, streams, events), so calls on disjoint outputs run
    // concurrently -- there is no process-wide lock
    std::mutex pipe_mu;
    bool pipe_planned = false;
    std::vector<int64_t> chunk_blocks;  // chunk c = tiles [chunk_blocks[c], chunk_blocks[c+1])
    std::vector<int64_t> chunk_x_hi;    // x entries [0, chunk_x_hi[c]) chunk c reads (global)
    std::vector<int64_t> x_pieces;      // H2D pieces of x: [x_pieces[p], x_pieces[p+1])
    std::vector<struct PipeCtx*> pipe_free;  // idle contexts
    std::vector<struct PipeCtx*> pipe_all;   // every context (released with the matrix)
    int64_t device_bytes = 0;
};

struct PipeCtx {
    double* dx = nullptr;
    double* dy = nullptr;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};  // H2D, compute, D2H
    std::vector<cudaEvent_t> events;
    // pageable host vectors (what the reference's std::vector-based API hands over):
    // pinned staging rings, allocated on the first such call (host_spmv.cu)
    double* hx = nullptr;      // STAGE_SLOTS slots of slot_elems doubles each
    double* hy = nullptr;
    int64_t slot_elems = 0;
    std::vector<cudaEvent_t> slot_ev;  // [0, S): x slot free again; [S, 2S): y slot filled
};
void pipe_ctx_release(PipeCtx* c);

void matrix_release(Matrix* m);

// ---- SpMV tiling -----------------------------------------------------------
// A tile is the row range one CTA owns.  Tiles never straddle a block: when
// bl >= tile_rows a block holds ceil(len/tile_rows) tiles; otherwise a tile
// holds G = tile_rows / bl whole blocks.
struct Tiling {
    int rows_per_thread;   // 2 (double2 segment loads) or 1 (odd bl)
    int64_t tile_rows;     // threads * rows_per_thread
    int64_t tiles_per_block;  // > 0 when bl >= tile_rows
    int64_t blocks_per_tile;  // > 0 when bl <  tile_rows and tiles hold whole blocks
    int64_t n_tiles;
    bool packed = false;      // tile-packed small blocks: tile t = rows [t*tile_rows, ...)
    int64_t align_blocks = 1; // block ranges must start/end at multiples of this (or at n)
};
Tiling tiling_of(const Matrix& m);
constexpr int64_t PACK_TILE = 1024;  // rows per tile of the packed layout
bool pack_eligible(int64_t bl, int64_t n_rows);

// Rows [lo, hi) of tile t (lo >= hi for the empty tail tiles of a short last block).
// tiles_per_block == blocks_per_tile == 0: packed tiles of tile_rows_n rows.
__host__ __device__ inline void tile_rows(int64_t t, int64_t tiles_per_block, int64_t blocks_per_tile,
                                          int64_t tile_rows_n, int64_t bl, int64_t n_rows, int64_t* lo,
                                          int64_t* hi) {
    if (tiles_per_block == 0 && blocks_per_tile == 0) {
        *lo = t * tile_rows_n;
        *hi = *lo + tile_rows_n < n_rows ? *lo + tile_rows_n : n_rows;
    } else if (tiles_per_block > 0) {
        const int64_t b = t / tiles_per_block;
        const int64_t b0 = b * bl;
        const int64_t bend = b0 + bl < n_rows ? b0 + bl : n_rows;
        *lo = b0 + (t - b * tiles_per_block) * tile_rows_n;
        *hi = *lo + tile_rows_n < bend ? *lo + tile_rows_n : bend;
    } else {
        *lo = t * blocks_per_tile * bl;
        const int64_t e = *lo + blocks_per_tile * bl;
        *hi = e < n_rows ? e : n_rows;
    }
}

// Peer-memory halo: rows i < halo of the slab are also stored to lo[i] (the lower
// neighbour's upper halo), rows i >= n_rows - halo to hi[i - (n_rows - halo)]
// (the upper neighbour's lower halo), from the kernel's epilogue, then fenced at
// system scope.  Either pointer may be null.
struct PeerOut {
    double* lo = nullptr;
    double* hi = nullptr;
    int64_t halo = 0;
};

// Launch over a tile range (both kernels); spmv_launch maps block ranges onto it.
void spmv_launch_tiles(const Matrix& m, const double* x_local, double* y, int64_t tile_begin, int64_t tile_end,
                       const double* x_scale, double* tile_sumsq, cudaStream_t st, const PeerOut& peer = PeerOut());

void spmv_launch(const Matrix& m, const double* x_local, double* y, int64_t block_begin,
                 int64_t block_end, const double* x_scale, double* tile_sumsq, cudaStream_t st,
                 const PeerOut& peer = PeerOut());
// the TMA-fed persistent kernel (spmv_tma.cu); false when the shape is not eligible
bool spmv_tma_launch(const Matrix& m, const double* x_local, double* y, int64_t tile_begin, int64_t tile_end,
                     const double* x_scale, double* tile_sumsq, cudaStream_t st, const PeerOut& peer);
// remainder / CSR row sums, one row per lane, entry streams staged by TMA (spmv_rows.cu);
// false when the matrix is not eligible
bool rest_rows_launch(const Matrix& m, const double* x_local, double* y, const double* x_scale, int64_t r0,
                      int64_t r1, cudaStream_t st);
bool rest_rows_default(const Matrix& m);  // the default policy picks rest_rows_kernel for this matrix
void rest_run_stats(Matrix* m);  // fills Matrix::rest_run_max / rest_lines_per_gather (synchronous; after the build)
extern int g_kernel_policy;  // 0 auto, 1 general kernel only, 2 TMA kernel only
extern int g_rest_mode;      // TMA kernel remainder mode (hdcg_set_kernel_policy), 0 default
// Matrix Market ingestion (mmio.cu)
void read_matrix_market(const char* path, Matrix* m);
int64_t coo_dedup_to_csr(const int64_t* skeys, const double* svals, int64_t total, int64_t n, Matrix* m,
                         cudaStream_t st);
// device membench (membench.cu)
void membench(int64_t n, int mode, int n_loops, int n_ites, double* best_s, double* bytes_per_s,
              double* loop_times);
// synchronous SpMV on host buffers, H2D / kernel / D2H overlapped chunk by chunk
void spmv_host_pipelined(Matrix* m, const double* x_host, double* y_host);
void tree_sum_launch(const double* vals, int64_t count, double* out, cudaStream_t st);
// bulk host <-> device copies, fast for pageable host memory too (host_spmv.cu): large
// pageable transfers are staged through a pinned ring and have completed on return;
// anything else is a cudaMemcpyAsync on st
void copy_h2d(void* dev, const void* host, size_t bytes, cudaStream_t st);
void copy_d2h(void* host, const void* dev, size_t bytes, cudaStream_t st);

// ---- converters (convert.cu) ------------------------------------------------
struct CsrInput {
    int64_t n_rows, n_cols, row0, nnz;
    const void* row_ptr;  // device
    bool rp64;
    const int32_t* col;   // device
    const double* val;    // device (may be null for census-only)
};
void validate_csr(const CsrInput& in, cudaStream_t st);
void build_mhdc(const CsrInput& in, double theta, int64_t bl, Matrix* out, cudaStream_t st);
void build_hdc(const CsrInput& in, double theta, Matrix* out, cudaStream_t st);
void build_csr(const CsrInput& in, Matrix* out, cudaStream_t st);
// census: returns the number of (block, offset) entries; fills host arrays when non-null
int64_t census(const CsrInput& in, int64_t bl, int64_t* block_ptr_host, int32_t* offsets_host,
               int64_t* counts_host, cudaStream_t st);
void rates(const Matrix& m, double* alpha, double* beta, int64_t* slots, cudaStream_t st);
// the tile-packed copy of a finished M-HDC (pack.cu); no-op unless pack_eligible
void build_packed(Matrix* m, cudaStream_t st);
// (theta, bl) sweep from one census per block width (analyze.cu)
void analyze(const CsrInput& in, const double* thetas, int n_theta, const int64_t* bls, int n_bl, double* out,
             cudaStream_t st);
// CUB exclusive scan of int64 (defined in convert.cu so only one TU includes CUB)
cudaError_t cub_exclusive_sum_i64(void* tmp, size_t& bytes, const int64_t* in, int64_t* out,
                                  int64_t count, cudaStream_t st);

// ---- small device helpers ----------------------------------------------------
// Small arrays come from the stream-ordered pool; arrays of HDCG_BIG_ALLOC_MB (default
// 16) or more from cudaMalloc: the pool maps fresh memory far more slowly than
// cudaMalloc does (30 GB of config-4 segments: 174 ms against 1 ms; the whole
// conversion 197 ms -> 36 ms, profiles/r03t_convert_alloc.log).  Either kind may be
// released with cudaFreeAsync (dev_free) or cudaFree (matrix_release).
inline size_t big_alloc_bytes() {
    static const long long mb = getenv("HDCG_BIG_ALLOC_MB") ? atoll(getenv("HDCG_BIG_ALLOC_MB")) : 16;
    return mb > 0 ? (size_t)mb << 20 : ~size_t(0);
}
template <class T>
T* dev_alloc(int64_t count, cudaStream_t st) {
    if (count <= 0) return nullptr;
    void* p = nullptr;
    const size_t bytes = sizeof(T) * (size_t)count;
    if (bytes >= big_alloc_bytes()) HDCG_CUDA(cudaMalloc(&p, bytes));
    else HDCG_CUDA(cudaMallocAsync(&p, bytes, st));
    return static_cast<T*>(p);
}
template <class T>
void dev_free(T* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// Remainder arrays carry REST_PAD zeroed entries past the end so the TMA kernel
// can move 16-byte aligned windows that run over the last entry.
constexpr int64_t REST_PAD = 8;
inline void alloc_rest(Matrix* m, int64_t nnz, cudaStream_t st) {
    m->rest_col = dev_alloc<int32_t>(nnz + REST_PAD, st);
    m->rest_val = dev_alloc<double>(nnz + REST_PAD, st);
    HDCG_CUDA(cudaMemsetAsync(m->rest_col + nnz, 0, sizeof(int32_t) * REST_PAD, st));
    HDCG_CUDA(cudaMemsetAsync(m->rest_val + nnz, 0, sizeof(double) * REST_PAD, st));
}

// Segment arrays carry SEG_PAD zeroed doubles past the end: for odd bl the TMA
// kernel moves 16-byte aligned windows that can start one slot early and end one
// slot late.
constexpr int64_t SEG_PAD = 2;
inline double* alloc_seg(int64_t count, cudaStream_t st) {
    double* p = dev_alloc<double>(count + SEG_PAD, st);
    HDCG_CUDA(cudaMemsetAsync(p + count, 0, sizeof(double) * SEG_PAD, st));
    return p;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t n_blocks_of(int64_t n, int64_t bl) { return n == 0 ? 0 : ceil_div(n, bl); }

inline int grid_cap(int64_t want) {
    const int64_t cap = 148LL * 64;  // enough CTAs for any grid-stride kernel
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

// splitmix64 counter RNG (synth.py)
__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return splitmix64(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL);
}

}  // namespace hdcg

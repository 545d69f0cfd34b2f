// capi.cu -- the extern "C" boundary of libhdcgpu.so (include/hdcgpu.h).
//
// Converts internal hdcg::Error exceptions into hdcg_status codes, owns the
// device-resident matrix handles, stages host inputs, and implements the
// synchronous host-buffer SpMV the reference-facing shim calls.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cstdlib>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

thread_local std::string g_last_error;

template <class F>
hdcg_status guard(F&& f) {
    try {
        f();
        return HDCG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return HDCG_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return HDCG_ERR_CUDA;
    }
}

int current_device() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        fail(HDCG_ERR_NO_DEVICE, std::string("no CUDA device available (libhdcgpu has no CPU fallback): ") +
                                     cudaGetErrorString(e));
    int dev = 0;
    HDCG_CUDA(cudaGetDevice(&dev));
    return dev;
}

void check_arch(int dev) {
    static std::once_flag once[64];
    static int ok[64];
    std::call_once(once[dev & 63], [&] {
        cudaDeviceProp p;
        ok[dev & 63] = cudaGetDeviceProperties(&p, dev) == cudaSuccess && p.major == 10 ? 1 : 0;
    });
    if (!ok[dev & 63]) fail(HDCG_ERR_NO_DEVICE, "libhdcgpu is built for sm_100a (B200) only");
}

int use_device() {
    const int dev = current_device();
    check_arch(dev);
    return dev;
}

// Input arrays staged on the device (copied when the caller passed host pointers).
struct Staged {
    CsrInput in{};
    std::vector<void*> owned;
    cudaStream_t st;
    explicit Staged(cudaStream_t s) : st(s) {}
    ~Staged() {
        for (void* p : owned) cudaFreeAsync(p, st);
    }
    template <class T>
    const T* stage(const T* p, int64_t count, bool on_device) {
        if (on_device || count <= 0 || p == nullptr) return p;
        T* d = dev_alloc<T>(count, st);
        owned.push_back(d);
        copy_h2d(d, p, sizeof(T) * count, st);
        return d;
    }
};

void stage_csr(Staged& s, int64_t n_rows, int64_t n_cols, int64_t row0, int64_t nnz,
               const void* row_ptr, const int32_t* col, const double* val, unsigned flags) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: negative dimension");
    if (row_ptr == nullptr) fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: row_ptr is null");
    if (nnz > 0 && col == nullptr) fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: col_ind is null");
    const bool dev = flags & HDCG_INPUT_DEVICE;
    const bool rp64 = flags & HDCG_ROWPTR_I64;
    s.in.n_rows = n_rows;
    s.in.n_cols = n_cols;
    s.in.row0 = row0;
    s.in.nnz = nnz;
    s.in.rp64 = rp64;
    s.in.row_ptr = rp64 ? (const void*)s.stage((const int64_t*)row_ptr, n_rows + 1, dev)
                        : (const void*)s.stage((const int32_t*)row_ptr, n_rows + 1, dev);
    s.in.col = s.stage(col, nnz, dev);
    s.in.val = s.stage(val, nnz, dev);
    if (flags & HDCG_VALIDATE) validate_csr(s.in, s.st);
}

void account(Matrix* m) {
    rest_run_stats(m);
    m->device_bytes = sizeof(int32_t) * (m->n_blocks + 1 + m->n_seg + m->n_rows + 1 + m->nnz_rest) +
                      sizeof(double) * (m->n_seg * m->bl + m->nnz_rest);
    if (m->packed) m->device_bytes += sizeof(double) * m->pk_stages * PACK_TILE;  // + small tables
}

template <class T>
T* upload(const T* host, int64_t count, cudaStream_t st) {
    T* d = dev_alloc<T>(count, st);
    if (count > 0) copy_h2d(d, host, sizeof(T) * count, st);
    return d;
}

double* upload_seg(const double* host, int64_t count, cudaStream_t st) {
    double* d = alloc_seg(count, st);
    if (count > 0) copy_h2d(d, host, sizeof(double) * count, st);
    return d;
}

void validate_mhdc_host(int64_t n, int64_t bl, const int32_t* dia_ptr, int64_t n_seg,
                        const int32_t* offs, const int32_t* rest_rp, int64_t nnz_rest,
                        const int32_t* rest_col) {
    // MHdcMatrix constructor (formats.cpp:131-163) and the remainder CsrMatrix (:45-67)
    if (n < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: negative dimension");
    if (bl < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: block width must be >= 1");
    const int64_t nb = n_blocks_of(n, bl);
    if (dia_ptr[0] != 0 || dia_ptr[nb] != n_seg)
        fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: dia_ptr endpoints do not match segment count");
    for (int64_t b = 0; b < nb; ++b) {
        if (dia_ptr[b] > dia_ptr[b + 1]) fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: dia_ptr not monotone");
        for (int64_t k = dia_ptr[b] + 1; k < dia_ptr[b + 1]; ++k)
            if (offs[k - 1] >= offs[k])
                fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: offsets must ascend within a block");
    }
    for (int64_t k = 0; k < n_seg; ++k)
        if (offs[k] <= -n || offs[k] >= n) fail(HDCG_ERR_OUT_OF_RANGE, "MHdcMatrix: offset outside matrix");
    if (rest_rp[0] != 0 || rest_rp[n] != nnz_rest)
        fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: row_ptr endpoints do not match value count");
    for (int64_t i = 0; i < n; ++i) {
        if (rest_rp[i] > rest_rp[i + 1])
            fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: row_ptr not monotone at row " + std::to_string(i));
        for (int64_t k = rest_rp[i]; k < rest_rp[i + 1]; ++k) {
            if (rest_col[k] < 0 || rest_col[k] >= n)
                fail(HDCG_ERR_OUT_OF_RANGE, "CsrMatrix: column index out of range in row " + std::to_string(i));
            if (k > rest_rp[i] && rest_col[k - 1] >= rest_col[k])
                fail(HDCG_ERR_INVALID_ARGUMENT,
                     "CsrMatrix: columns not strictly ascending in row " + std::to_string(i));
        }
    }
}

Matrix* new_matrix(int dev) {
    Matrix* m = new Matrix();
    m->device = dev;
    return m;
}

hdcg_matrix wrap(Matrix* m) { return reinterpret_cast<hdcg_matrix>(m); }
Matrix* unwrap(hdcg_matrix h) {
    if (!h) fail(HDCG_ERR_INVALID_ARGUMENT, "null matrix handle");
    return reinterpret_cast<Matrix*>(h);
}

}  // namespace

void matrix_release(Matrix* m) {
    if (!m) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    cudaFree(m->dia_ptr);
    cudaFree(m->dia_off);
    cudaFree(m->seg);
    cudaFree(m->rest_rp);
    cudaFree(m->rest_col);
    cudaFree(m->rest_val);
    cudaFree(m->pk_val);
    cudaFree(m->pk_meta);
    cudaFree(m->pk_tab);
    for (PipeCtx* c : m->pipe_all) pipe_ctx_release(c);
    cudaSetDevice(prev);
    delete m;
}

// ---- device generators (synth.py restated for the device) ----------------------

__global__ void gen_uniform_kernel(uint64_t key, int64_t first, int64_t count, double* out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = splitmix64(key + (uint64_t)(first + k));
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[k] = 2.0 * u - 1.0;
    }
}

__device__ __forceinline__ void lap7_row(int64_t g, int64_t nx, int64_t ny, int64_t nz, int64_t* cols,
                                         int* cnt) {
    const int64_t p = nx * ny;
    const int64_t x = g % nx, y = (g / nx) % ny, z = g / p;
    int c = 0;
    if (z > 0) cols[c++] = g - p;
    if (y > 0) cols[c++] = g - nx;
    if (x > 0) cols[c++] = g - 1;
    cols[c++] = g;
    if (x < nx - 1) cols[c++] = g + 1;
    if (y < ny - 1) cols[c++] = g + nx;
    if (z < nz - 1) cols[c++] = g + p;
    *cnt = c;
}

__global__ void lap7_count_kernel(int64_t nx, int64_t ny, int64_t nz, int64_t g0, int64_t n_rows,
                                  int64_t* counts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t cols[7];
        int c;
        lap7_row(g0 + i, nx, ny, nz, cols, &c);
        counts[i] = c;
    }
}

__global__ void lap7_fill_kernel(int64_t nx, int64_t ny, int64_t nz, int64_t g0, int64_t n_rows,
                                 const int64_t* rp, int32_t* col, double* val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = g0 + i;
        int64_t cols[7];
        int c;
        lap7_row(g, nx, ny, nz, cols, &c);
        const int64_t base = rp[i];
        for (int t = 0; t < c; ++t) {
            col[base + t] = (int32_t)cols[t];
            val[base + t] = cols[t] == g ? 6.0 : -1.0;
        }
    }
}

}  // namespace hdcg

using namespace hdcg;

extern "C" {

const char* hdcg_last_error(void) { return g_last_error.c_str(); }

int hdcg_version(void) { return 100; }

hdcg_status hdcg_init(int device) {
    return guard([&] {
        int count = 0;
        const cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            fail(HDCG_ERR_NO_DEVICE, std::string("no CUDA device available: ") + cudaGetErrorString(e));
        if (device < 0 || device >= count) fail(HDCG_ERR_INVALID_ARGUMENT, "hdcg_init: bad device ordinal");
        HDCG_CUDA(cudaSetDevice(device));
        check_arch(device);
        HDCG_CUDA(cudaFree(nullptr));
        // HDCG_POOL_RETAIN_MB: freed device memory up to this size stays in the
        // stream-ordered pool instead of going back to the driver at the next
        // synchronisation (default: released) -- repeated conversions then skip
        // the driver's page mapping, most of a large conversion's wall time
        // (scripts/convert_bench.py measures both)
        if (const char* e = getenv("HDCG_POOL_RETAIN_MB")) {
            cudaMemPool_t pool;
            HDCG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t keep = (uint64_t)atoll(e) << 20;
            HDCG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
    });
}

hdcg_status hdcg_build_mhdc(int64_t n_rows, int64_t n_cols, int64_t row0, int64_t nnz,
                            const void* row_ptr, const int32_t* col_ind, const double* values,
                            double theta, int64_t bl, unsigned flags, void* stream, hdcg_matrix* out) {
    return guard([&] {
        if (!out) fail(HDCG_ERR_INVALID_ARGUMENT, "null output handle");
        const int dev = use_device();
        cudaStream_t st = (cudaStream_t)stream;
        // parameter checks first, like convert.cpp:124-125
        if (!(theta >= 0.0 && theta <= 1.0)) fail(HDCG_ERR_INVALID_ARGUMENT, "to_mhdc: theta must be in [0, 1]");
        if (bl < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "to_mhdc: block width must be >= 1");
        Staged s(st);
        stage_csr(s, n_rows, n_cols, row0, nnz, row_ptr, col_ind, values, flags);
        Matrix* m = new_matrix(dev);
        try {
            build_mhdc(s.in, theta, bl, m, st);
            HDCG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_build_hdc(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                           const double* values, double theta, unsigned flags, void* stream,
                           hdcg_matrix* out) {
    return guard([&] {
        if (!out) fail(HDCG_ERR_INVALID_ARGUMENT, "null output handle");
        const int dev = use_device();
        cudaStream_t st = (cudaStream_t)stream;
        if (!(theta >= 0.0 && theta <= 1.0)) fail(HDCG_ERR_INVALID_ARGUMENT, "to_hdc: theta must be in [0, 1]");
        Staged s(st);
        stage_csr(s, n, n, 0, nnz, row_ptr, col_ind, values, flags);
        Matrix* m = new_matrix(dev);
        try {
            build_hdc(s.in, theta, m, st);
            HDCG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_build_csr(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                           const double* values, unsigned flags, void* stream, hdcg_matrix* out) {
    return guard([&] {
        if (!out) fail(HDCG_ERR_INVALID_ARGUMENT, "null output handle");
        const int dev = use_device();
        cudaStream_t st = (cudaStream_t)stream;
        Staged s(st);
        stage_csr(s, n, n, 0, nnz, row_ptr, col_ind, values, flags);
        Matrix* m = new_matrix(dev);
        try {
            build_csr(s.in, m, st);
            HDCG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_upload_mhdc(int64_t n, int64_t bl, const int32_t* dia_ptr, int64_t n_seg,
                             const int32_t* dia_offsets, const double* segments,
                             const int32_t* rest_row_ptr, int64_t nnz_rest,
                             const int32_t* rest_col_ind, const double* rest_values, unsigned flags,
                             hdcg_matrix* out) {
    return guard([&] {
        if (!out) fail(HDCG_ERR_INVALID_ARGUMENT, "null output handle");
        if (flags & HDCG_INPUT_DEVICE) fail(HDCG_ERR_INVALID_ARGUMENT, "hdcg_upload_mhdc takes host arrays");
        if (n < 0 || n_seg < 0 || nnz_rest < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "negative size");
        if (bl < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "MHdcMatrix: block width must be >= 1");
        if (flags & HDCG_VALIDATE)
            validate_mhdc_host(n, bl, dia_ptr, n_seg, dia_offsets, rest_row_ptr, nnz_rest, rest_col_ind);
        const int dev = use_device();
        cudaStream_t st = nullptr;
        Matrix* m = new_matrix(dev);
        try {
            m->kind = HDCG_KIND_MHDC;
            m->n_rows = m->n_cols = n;
            m->bl = bl;
            m->n_blocks = n_blocks_of(n, bl);
            m->n_seg = n_seg;
            m->nnz_rest = nnz_rest;
            m->dia_ptr = upload(dia_ptr, m->n_blocks + 1, st);
            m->dia_off = upload(dia_offsets, n_seg, st);
            m->seg = upload_seg(segments, n_seg * bl, st);
            m->rest_rp = upload(rest_row_ptr, n + 1, st);
            alloc_rest(m, nnz_rest, st);
            if (nnz_rest > 0) {
                copy_h2d(m->rest_col, rest_col_ind, sizeof(int32_t) * nnz_rest, st);
                copy_h2d(m->rest_val, rest_values, sizeof(double) * nnz_rest, st);
            }
            int64_t slots = 0, dia_nnz = 0;
            for (int64_t b = 0; b < m->n_blocks; ++b) {
                slots += (int64_t)(dia_ptr[b + 1] - dia_ptr[b]) * std::min(bl, n - b * bl);
                m->max_seg_per_block = std::max<int64_t>(m->max_seg_per_block, dia_ptr[b + 1] - dia_ptr[b]);
            }
            for (int64_t k = 0; k < n_seg * bl; ++k) dia_nnz += segments[k] != 0.0;
            m->dia_slots = slots;
            m->nnz_input = dia_nnz + nnz_rest;
            HDCG_CUDA(cudaStreamSynchronize(st));
            build_packed(m, st);
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_upload_hdc(int64_t n, int64_t n_diag, const int32_t* offsets, const double* lanes,
                            const int32_t* rest_row_ptr, int64_t nnz_rest,
                            const int32_t* rest_col_ind, const double* rest_values, unsigned flags,
                            hdcg_matrix* out) {
    return guard([&] {
        if (!out) fail(HDCG_ERR_INVALID_ARGUMENT, "null output handle");
        if (flags & HDCG_INPUT_DEVICE) fail(HDCG_ERR_INVALID_ARGUMENT, "hdcg_upload_hdc takes host arrays");
        if (n < 0 || n_diag < 0 || nnz_rest < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "negative size");
        if (flags & HDCG_VALIDATE) {
            // DiaMatrix constructor (formats.cpp:94-115)
            for (int64_t k = 0; k < n_diag; ++k) {
                if (offsets[k] <= -n || offsets[k] >= n)
                    fail(HDCG_ERR_OUT_OF_RANGE, "DiaMatrix: offset outside matrix");
                if (k > 0 && offsets[k - 1] >= offsets[k])
                    fail(HDCG_ERR_INVALID_ARGUMENT, "DiaMatrix: offsets must be strictly ascending");
                const int64_t first = std::max<int64_t>(0, -offsets[k]);
                const int64_t last = std::min<int64_t>(n, n - offsets[k]);
                for (int64_t i = 0; i < n; ++i)
                    if ((i < first || i >= last) && lanes[k * n + i] != 0.0)
                        fail(HDCG_ERR_INVALID_ARGUMENT, "DiaMatrix: lane value outside valid rows");
            }
            std::vector<int32_t> dp = {0, (int32_t)n_diag};
            if (n > 0) validate_mhdc_host(n, n, dp.data(), n_diag, offsets, rest_row_ptr, nnz_rest, rest_col_ind);
        }
        const int dev = use_device();
        cudaStream_t st = nullptr;
        Matrix* m = new_matrix(dev);
        try {
            m->kind = HDCG_KIND_HDC;
            m->n_rows = m->n_cols = n;
            m->bl = n > 0 ? n : 1;
            m->n_blocks = n_blocks_of(n, m->bl);
            m->n_seg = n > 0 ? n_diag : 0;
            m->nnz_rest = nnz_rest;
            std::vector<int32_t> dp = {0, (int32_t)m->n_seg};
            m->dia_ptr = upload(dp.data(), m->n_blocks + 1, st);
            m->dia_off = upload(offsets, m->n_seg, st);
            m->seg = upload_seg(lanes, m->n_seg * m->bl, st);
            m->rest_rp = upload(rest_row_ptr, n + 1, st);
            alloc_rest(m, nnz_rest, st);
            if (nnz_rest > 0) {
                copy_h2d(m->rest_col, rest_col_ind, sizeof(int32_t) * nnz_rest, st);
                copy_h2d(m->rest_val, rest_values, sizeof(double) * nnz_rest, st);
            }
            int64_t dia_nnz = 0;
            for (int64_t k = 0; k < m->n_seg * m->bl; ++k) dia_nnz += lanes[k] != 0.0;
            m->dia_slots = m->n_seg * n;
            m->max_seg_per_block = m->n_seg;
            m->nnz_input = dia_nnz + nnz_rest;
            HDCG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_read_matrix_market(const char* path, hdcg_matrix* out) {
    return guard([&] {
        if (!path || !out) fail(HDCG_ERR_INVALID_ARGUMENT, "null argument");
        const int dev = use_device();
        Matrix* m = new_matrix(dev);
        try {
            read_matrix_market(path, m);
        } catch (...) {
            matrix_release(m);
            throw;
        }
        account(m);
        *out = wrap(m);
    });
}

hdcg_status hdcg_free(hdcg_matrix h) {
    return guard([&] { matrix_release(reinterpret_cast<Matrix*>(h)); });
}

hdcg_status hdcg_get_info(hdcg_matrix h, hdcg_info* info) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        if (!info) fail(HDCG_ERR_INVALID_ARGUMENT, "null info");
        const Tiling t = tiling_of(*m);
        info->kind = m->kind;
        info->device = m->device;
        info->n_rows = m->n_rows;
        info->n_cols = m->n_cols;
        info->row0 = m->row0;
        info->bl = m->bl;
        info->n_blocks = m->n_blocks;
        info->n_seg = m->n_seg;
        info->nnz_rest = m->nnz_rest;
        info->dia_slots = m->dia_slots;
        info->nnz_input = m->nnz_input;
        info->n_tiles = t.n_tiles;
        info->tile_rows = t.tile_rows;
        // the block-range granularity of hdcg_spmv_slab (whole tiles)
        info->blocks_per_tile = t.align_blocks;
        info->device_bytes = m->device_bytes;
        info->max_seg_per_block = m->max_seg_per_block;
        info->packed_stages = m->packed ? m->pk_stages : 0;
        info->rest_rows_kernel = rest_rows_default(*m) ? 1 : 0;
    });
}

hdcg_status hdcg_export(hdcg_matrix h, int32_t* dia_ptr, int32_t* dia_offsets, double* segments,
                        int32_t* rest_row_ptr, int32_t* rest_col_ind, double* rest_values) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        const DeviceGuard dg(m->device);
        auto cp = [](void* dst, const void* src, size_t bytes) {
            if (dst && src && bytes) {
                copy_d2h(dst, src, bytes, nullptr);  // staged through pinned memory when dst is pageable
                HDCG_CUDA(cudaStreamSynchronize(nullptr));
            }
        };
        cp(dia_ptr, m->dia_ptr, sizeof(int32_t) * (m->n_blocks + 1));
        if (dia_ptr && m->n_blocks == 0) dia_ptr[0] = 0;
        cp(dia_offsets, m->dia_off, sizeof(int32_t) * m->n_seg);
        cp(segments, m->seg, sizeof(double) * m->n_seg * m->bl);
        cp(rest_row_ptr, m->rest_rp, sizeof(int32_t) * (m->n_rows + 1));
        cp(rest_col_ind, m->rest_col, sizeof(int32_t) * m->nnz_rest);
        cp(rest_values, m->rest_val, sizeof(double) * m->nnz_rest);
    });
}

hdcg_status hdcg_export_blocks(hdcg_matrix h, int64_t block_begin, int64_t block_end, int32_t* dia_ptr,
                               int32_t* dia_offsets, double* segments, int32_t* rest_row_ptr,
                               int32_t* rest_col_ind, double* rest_values, int64_t* counts) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        if (block_begin < 0 || block_end > m->n_blocks || block_begin > block_end)
            fail(HDCG_ERR_INVALID_ARGUMENT, "export_blocks: block range outside the matrix");
        const DeviceGuard dg(m->device);
        const int64_t nb = block_end - block_begin;
        const int64_t r0 = std::min(m->n_rows, block_begin * m->bl), r1 = std::min(m->n_rows, block_end * m->bl);
        int32_t k[2] = {0, 0}, e[2] = {0, 0};
        if (m->n_blocks > 0) {
            HDCG_CUDA(cudaMemcpy(&k[0], m->dia_ptr + block_begin, sizeof(int32_t), cudaMemcpyDeviceToHost));
            HDCG_CUDA(cudaMemcpy(&k[1], m->dia_ptr + block_end, sizeof(int32_t), cudaMemcpyDeviceToHost));
        }
        if (m->rest_rp) {
            HDCG_CUDA(cudaMemcpy(&e[0], m->rest_rp + r0, sizeof(int32_t), cudaMemcpyDeviceToHost));
            HDCG_CUDA(cudaMemcpy(&e[1], m->rest_rp + r1, sizeof(int32_t), cudaMemcpyDeviceToHost));
        }
        if (counts) {
            counts[0] = k[1] - k[0];
            counts[1] = e[1] - e[0];
        }
        auto cp = [](void* dst, const void* src, size_t bytes) {
            if (dst && src && bytes) {
                copy_d2h(dst, src, bytes, nullptr);  // staged through pinned memory when dst is pageable
                HDCG_CUDA(cudaStreamSynchronize(nullptr));
            }
        };
        if (dia_ptr) {
            if (m->n_blocks > 0) cp(dia_ptr, m->dia_ptr + block_begin, sizeof(int32_t) * (nb + 1));
            else dia_ptr[0] = 0;
            for (int64_t b = 0; b <= nb && m->n_blocks > 0; ++b) dia_ptr[b] -= k[0];
        }
        cp(dia_offsets, m->dia_off + k[0], sizeof(int32_t) * (k[1] - k[0]));
        cp(segments, m->seg + (int64_t)k[0] * m->bl, sizeof(double) * (int64_t)(k[1] - k[0]) * m->bl);
        if (rest_row_ptr) {
            if (m->rest_rp) {
                cp(rest_row_ptr, m->rest_rp + r0, sizeof(int32_t) * (r1 - r0 + 1));
                for (int64_t i = 0; i <= r1 - r0; ++i) rest_row_ptr[i] -= e[0];
            } else {
                for (int64_t i = 0; i <= r1 - r0; ++i) rest_row_ptr[i] = 0;
            }
        }
        cp(rest_col_ind, m->rest_col + e[0], sizeof(int32_t) * (e[1] - e[0]));
        cp(rest_values, m->rest_val + e[0], sizeof(double) * (e[1] - e[0]));
    });
}

hdcg_status hdcg_rates(hdcg_matrix h, double* alpha, double* beta, int64_t* dia_slots) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        const DeviceGuard dg(m->device);
        double a = 0, b = 0;
        int64_t s = 0;
        rates(*m, &a, &b, &s, nullptr);
        if (alpha) *alpha = a;
        if (beta) *beta = b;
        if (dia_slots) *dia_slots = s;
    });
}

hdcg_status hdcg_census(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind, int64_t bl,
                        unsigned flags, int64_t* block_ptr, int32_t* offsets, int64_t* counts,
                        int64_t* n_entries) {
    return guard([&] {
        use_device();
        cudaStream_t st = nullptr;
        Staged s(st);
        stage_csr(s, n, n, 0, nnz, row_ptr, col_ind, nullptr, flags);
        const int64_t total = census(s.in, bl, block_ptr, offsets, counts, st);
        if (n_entries) *n_entries = total;
        HDCG_CUDA(cudaStreamSynchronize(st));
    });
}

hdcg_status hdcg_spmv(hdcg_matrix h, const double* x, double* y, void* stream) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        if (m->n_rows > 0 && (!x || !y)) fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: x and y must have length n");
        const DeviceGuard dg(m->device);
        spmv_launch(*m, x ? x + m->row0 : nullptr, y, 0, m->n_blocks, nullptr, nullptr, (cudaStream_t)stream);
    });
}

hdcg_status hdcg_spmv_slab(hdcg_matrix h, const double* x_local, double* y, int64_t block_begin,
                           int64_t block_end, const double* x_scale, double* tile_sumsq, void* stream) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        const DeviceGuard dg(m->device);
        spmv_launch(*m, x_local, y, block_begin, block_end, x_scale, tile_sumsq, (cudaStream_t)stream);
    });
}

hdcg_status hdcg_spmv_slab_halo(hdcg_matrix h, const double* x_local, double* y, int64_t block_begin,
                                int64_t block_end, const double* x_scale, double* tile_sumsq, double* peer_lo,
                                double* peer_hi, int64_t halo, void* stream) {
    return guard([&] {
        const Matrix* m = unwrap(h);
        if (halo < 0 || halo > m->n_rows) fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: halo outside the slab");
        const DeviceGuard dg(m->device);
        PeerOut p;
        p.lo = peer_lo;
        p.hi = peer_hi;
        p.halo = halo;
        spmv_launch(*m, x_local, y, block_begin, block_end, x_scale, tile_sumsq, (cudaStream_t)stream, p);
    });
}

hdcg_status hdcg_peer_alloc(int64_t bytes, void** ptr, unsigned char handle[64]) {
    return guard([&] {
        if (!ptr || !handle || bytes < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "peer_alloc: bad arguments");
        use_device();
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        void* p = nullptr;
        HDCG_CUDA(cudaMalloc(&p, (size_t)bytes));
        cudaIpcMemHandle_t hd;
        const cudaError_t e = cudaIpcGetMemHandle(&hd, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            HDCG_CUDA(e);
        }
        std::memcpy(handle, &hd, 64);
        *ptr = p;
    });
}

hdcg_status hdcg_peer_open(const unsigned char handle[64], void** ptr) {
    return guard([&] {
        if (!ptr || !handle) fail(HDCG_ERR_INVALID_ARGUMENT, "peer_open: bad arguments");
        use_device();
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle, 64);
        HDCG_CUDA(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    });
}

hdcg_status hdcg_peer_close(void* ptr) {
    return guard([&] { HDCG_CUDA(cudaIpcCloseMemHandle(ptr)); });
}

hdcg_status hdcg_peer_free(void* ptr) {
    return guard([&] { HDCG_CUDA(cudaFree(ptr)); });
}

hdcg_status hdcg_spmv_host(hdcg_matrix h, const double* x, double* y) {
    return guard([&] {
        Matrix* m = unwrap(h);
        if (m->n_rows == 0) return;
        if (!x || !y) fail(HDCG_ERR_INVALID_ARGUMENT, "spmv: x and y must have length n");
        spmv_host_pipelined(m, x, y);  // per-matrix context pool: concurrent calls allowed
    });
}

hdcg_status hdcg_analyze(int64_t n, int64_t nnz, const void* row_ptr, const int32_t* col_ind,
                         const double* values, const double* thetas, int n_theta, const int64_t* bls,
                         int n_bl, unsigned flags, double* out) {
    return guard([&] {
        if (!thetas || !out || (n_bl > 0 && !bls)) fail(HDCG_ERR_INVALID_ARGUMENT, "analyze: null argument");
        use_device();
        cudaStream_t st = nullptr;
        Staged s(st);
        stage_csr(s, n, n, 0, nnz, row_ptr, col_ind, values, flags);
        if (nnz > 0 && !values) fail(HDCG_ERR_INVALID_ARGUMENT, "analyze: values are required");
        analyze(s.in, thetas, n_theta, bls, n_bl, out, st);
    });
}

hdcg_status hdcg_membench(int64_t n, int mode, int n_loops, int n_ites, double* best_time_s,
                          double* bytes_per_s, double* loop_times) {
    return guard([&] {
        if (!best_time_s || !bytes_per_s) fail(HDCG_ERR_INVALID_ARGUMENT, "membench: null output");
        if (n_loops < 1 || n_ites < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "timing: n_loops and n_ites must be >= 1");
        if (n < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "membench: n must be >= 1");
        use_device();
        membench(n, mode, n_loops, n_ites, best_time_s, bytes_per_s, loop_times);
    });
}

hdcg_status hdcg_set_kernel_policy(int policy) {
    return guard([&] {
        if (policy < 0 || (policy & 3) > 2 || (policy & 0xC) != 0 || (policy >> 4) > 3)
            fail(HDCG_ERR_INVALID_ARGUMENT, "kernel policy must be (0, 1 or 2) + 16 * (0, 1, 2 or 3)");
        g_kernel_policy = policy & 3;
        g_rest_mode = policy >> 4;
    });
}

hdcg_status hdcg_tree_sum(const double* vals, int64_t count, double* out, void* stream) {
    return guard([&] {
        if (count < 0 || !out) fail(HDCG_ERR_INVALID_ARGUMENT, "tree_sum: bad arguments");
        tree_sum_launch(vals, count, out, (cudaStream_t)stream);
    });
}

hdcg_status hdcg_gen_uniform_pm1(uint64_t seed, uint64_t rng_stream, int64_t first, int64_t count,
                                 double* out, void* stream) {
    return guard([&] {
        if (count <= 0) return;
        gen_uniform_kernel<<<grid_cap(ceil_div(count, 256)), 256, 0, (cudaStream_t)stream>>>(
            stream_key(seed, rng_stream), first, count, out);
        HDCG_LAUNCH_CHECK("gen_uniform_kernel");
    });
}

hdcg_status hdcg_gen_laplacian7(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1,
                                int64_t* row_ptr, int32_t* col_ind, double* values, int64_t* nnz,
                                void* stream) {
    return guard([&] {
        if (nx < 1 || ny < 1 || nz < 1 || z0 < 0 || z1 > nz || z0 > z1)
            fail(HDCG_ERR_INVALID_ARGUMENT, "gen_laplacian7: bad grid");
        // closed-form nnz of the slab: 7 per row minus the missing neighbours
        const int64_t p = nx * ny, rows = (z1 - z0) * p;
        int64_t count = 7 * rows;
        count -= 2 * (nx > 0 ? ny * (z1 - z0) : 0);          // x = 0 and x = nx-1 faces
        count -= 2 * (nx * (z1 - z0));                      // y = 0 and y = ny-1 faces
        count -= (z0 == 0 ? p : 0) + (z1 == nz ? p : 0);    // z faces inside the slab
        if (nnz) *nnz = count;
        if (!row_ptr) return;
        cudaStream_t st = (cudaStream_t)stream;
        int64_t* counts = dev_alloc<int64_t>(rows + 1, st);
        HDCG_CUDA(cudaMemsetAsync(counts + rows, 0, sizeof(int64_t), st));
        lap7_count_kernel<<<grid_cap(ceil_div(rows, 256)), 256, 0, st>>>(nx, ny, nz, z0 * p, rows, counts);
        HDCG_LAUNCH_CHECK("lap7_count_kernel");
        size_t bytes = 0;
        HDCG_CUDA(cub_exclusive_sum_i64(nullptr, bytes, counts, row_ptr, rows + 1, st));
        void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
        HDCG_CUDA(cub_exclusive_sum_i64(tmp, bytes, counts, row_ptr, rows + 1, st));
        dev_free(tmp, st);
        dev_free(counts, st);
        lap7_fill_kernel<<<grid_cap(ceil_div(rows, 256)), 256, 0, st>>>(nx, ny, nz, z0 * p, rows, row_ptr,
                                                                       col_ind, values);
        HDCG_LAUNCH_CHECK("lap7_fill_kernel");
    });
}

}  // extern "C"

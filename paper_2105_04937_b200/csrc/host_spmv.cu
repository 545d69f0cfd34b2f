// host_spmv.cu -- y = A x on HOST buffers (the call the reference-facing shim
// makes: hdc::spmv_mhdc(const MHdcMatrix&, span x, span y) is synchronous and
// works on host vectors, kernels.hpp:31-49).
//
// The matrix stays resident in HBM; per call only x goes down and y comes
// back.  PCIe (not HBM) bounds this path, so the three phases are overlapped:
//   stream 0: x copied host->device in pieces, an event after each piece;
//   stream 1: the rows are split into chunks of whole blocks; chunk c's kernel
//             waits only for the x pieces covering the highest column its
//             blocks reference (computed once per matrix from dia_offsets and
//             the remainder's columns), then runs;
//   stream 2: chunk c's y rows are copied device->host as soon as its kernel ends.
// With pinned host buffers H2D and D2H run concurrently (PCIe is full duplex),
// so a call costs about max(8 n_cols, 8 n_rows) / PCIe bandwidth instead of the sum.
//
// Pageable vectors -- what the reference API hands over: std::vector storage behind
// std::span (kernels.hpp:31-49) -- would make every cudaMemcpyAsync a synchronous,
// single-threaded staged copy inside the driver (7 GB/s each way, no overlap: 19 ms
// per call on config 1 against 3.4 ms pinned, slower than the reference on the
// CPU).  For those the pipeline stages the pieces itself: a small pool of host
// threads copies x piece p into a pinned ring slot while piece p-1 is on the wire,
// and copies finished y chunks out of their pinned slots into the caller's vector.
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

// Pipeline granularity: pieces of ~32 MB of x (at least 16, at most 256 chunks),
// so the fill (the first chunk's x) and the drain (the last chunk's y) stay a
// small part of the PCIe time.  Each chunk costs ~20 us of launches and event
// waits: 16 chunks beat 32 on the 134 MB vectors of configs 1 and 3 (3.40 vs
// 3.65 ms per call) and on config 2 (1.75 vs 1.94 ms).  HDCG_PIPE_CHUNKS overrides (A/B).
int pipe_chunks(int64_t n_cols) {
    static const int env = getenv("HDCG_PIPE_CHUNKS") ? atoi(getenv("HDCG_PIPE_CHUNKS")) : 0;
    if (env > 0) return env;
    const int64_t want = ceil_div(8 * n_cols, (int64_t)32 << 20);
    return (int)std::min<int64_t>(256, std::max<int64_t>(16, want));
}

// per tile: highest global column any of its rows reads (-1: none)
__global__ void tile_xhi_kernel(int64_t n_tiles, int64_t tpb, int64_t bpt, int64_t tile_rows_n, int64_t bl,
                                int64_t n_rows, int64_t row0, int64_t n_cols, const int32_t* dia_ptr,
                                const int32_t* dia_off, const int32_t* rest_rp, const int32_t* rest_col,
                                int64_t* hi_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < n_tiles; t += n_warps) {
        int64_t lo, hi_row;
        tile_rows(t, tpb, bpt, tile_rows_n, bl, n_rows, &lo, &hi_row);
        int64_t hi = -1;
        if (lo < hi_row) {
            // segments: the last block of the tile has the largest rows; offsets ascend per block
            for (int64_t b = lo / bl + lane; b <= (hi_row - 1) / bl; b += 32) {
                const int k0 = dia_ptr[b], k1 = dia_ptr[b + 1];
                const int64_t last_row = min(hi_row, (b + 1) * bl) - 1;
                if (k1 > k0) hi = max(hi, min(n_cols - 1, row0 + last_row + (int64_t)dia_off[k1 - 1]));
            }
            if (rest_rp) {
                const int64_t e0 = rest_rp[lo], e1 = rest_rp[hi_row];
                for (int64_t e = e0 + lane; e < e1; e += 32) hi = max(hi, (int64_t)rest_col[e]);
            }
        }
        for (int o = 16; o > 0; o >>= 1) hi = max(hi, (int64_t)__shfl_down_sync(0xffffffffu, hi, o));
        if (lane == 0) hi_out[t] = hi;
    }
}

void plan_pipeline(Matrix* m, cudaStream_t st) {
    const Tiling t = tiling_of(*m);
    const int64_t nt = t.n_tiles;
    const int chunks = pipe_chunks(m->n_cols);
    const int64_t per = std::max<int64_t>(1, ceil_div(nt, chunks));
    m->chunk_blocks.clear();  // holds TILE boundaries of the chunks
    for (int64_t q = 0; q < nt; q += per) m->chunk_blocks.push_back(q);
    m->chunk_blocks.push_back(nt);
    const int64_t n_chunks = (int64_t)m->chunk_blocks.size() - 1;

    std::vector<int64_t> hi((size_t)nt);
    int64_t* d_hi = dev_alloc<int64_t>(nt, st);
    tile_xhi_kernel<<<grid_cap(ceil_div(nt * 32, 256)), 256, 0, st>>>(
        nt, t.tiles_per_block, t.blocks_per_tile, t.tile_rows, m->bl, m->n_rows, m->row0, m->n_cols, m->dia_ptr,
        m->dia_off, m->nnz_rest > 0 ? m->rest_rp : nullptr, m->rest_col, d_hi);
    HDCG_LAUNCH_CHECK("tile_xhi_kernel");
    HDCG_CUDA(cudaMemcpyAsync(hi.data(), d_hi, sizeof(int64_t) * nt, cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    dev_free(d_hi, st);
    m->chunk_x_hi.assign((size_t)n_chunks, 0);
    int64_t run = 0;  // chunks run in order, so the requirement is cumulative
    for (int64_t c = 0; c < n_chunks; ++c) {
        for (int64_t q = m->chunk_blocks[c]; q < m->chunk_blocks[c + 1]; ++q) run = std::max(run, hi[q] + 1);
        m->chunk_x_hi[c] = run;
    }
    // x pieces: equal slices of [0, n_cols), 16-byte aligned boundaries
    m->x_pieces.clear();
    const int64_t np = std::max<int64_t>(1, std::min<int64_t>(chunks, m->n_cols));
    for (int64_t p = 0; p < np; ++p) m->x_pieces.push_back((m->n_cols * p / np) & ~int64_t(1));
    m->x_pieces.push_back(m->n_cols);
    m->pipe_planned = true;
}

PipeCtx* new_ctx(const Matrix* m) {
    PipeCtx* c = new PipeCtx();
    try {
        for (int s = 0; s < 3; ++s) HDCG_CUDA(cudaStreamCreateWithFlags(&c->s[s], cudaStreamNonBlocking));
        const size_t ne = m->x_pieces.size() - 1 + m->chunk_blocks.size() - 1;
        c->events.assign(ne, nullptr);
        for (auto& e : c->events) HDCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        HDCG_CUDA(cudaMalloc(&c->dx, sizeof(double) * std::max<int64_t>(1, m->n_cols)));
        HDCG_CUDA(cudaMalloc(&c->dy, sizeof(double) * std::max<int64_t>(1, m->n_rows)));
    } catch (...) {
        pipe_ctx_release(c);
        throw;
    }
    return c;
}

// Blocking memcpy spread over a few host threads (the caller takes a share): one
// core copies ~10 GB/s, a B200 host needs ~50 GB/s each way to keep PCIe busy.
// Threads start on the first pageable call; HDCG_COPY_THREADS sets their number.
class CopyPool {
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_work_, cv_done_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;

    static void slice(size_t n, int part, int parts, size_t* a, size_t* b) {
        *a = (n * (size_t)part / (size_t)parts) & ~size_t(63);
        *b = part + 1 == parts ? n : (n * (size_t)(part + 1) / (size_t)parts) & ~size_t(63);
    }
    void run(int id) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_work_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            char* d = dst_;
            const char* s = src_;
            const size_t n = bytes_;
            lk.unlock();
            size_t a, b;
            slice(n, id + 1, (int)workers_.size() + 1, &a, &b);
            if (b > a) std::memcpy(d + a, s + a, b - a);
            lk.lock();
            if (--pending_ == 0) cv_done_.notify_one();
        }
    }

public:
    CopyPool() {
        const char* e = getenv("HDCG_COPY_THREADS");
        const int hc = (int)std::thread::hardware_concurrency();
        int n = e ? atoi(e) : std::min(12, std::max(2, hc - 2));
        n = std::max(1, n) - 1;  // + the calling thread
        for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_work_.notify_all();
        for (auto& t : workers_) t.join();
    }
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    void copy(void* dst, const void* src, size_t n) {
        if (n < (size_t)1 << 20 || workers_.empty()) {
            std::memcpy(dst, src, n);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu_);  // one spread copy at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = (char*)dst;
            src_ = (const char*)src;
            bytes_ = n;
            pending_ = (int)workers_.size();
            ++gen_;
        }
        cv_work_.notify_all();
        size_t a, b;
        slice(n, 0, (int)workers_.size() + 1, &a, &b);
        if (b > a) std::memcpy((char*)dst + a, (const char*)src + a, b - a);
        std::unique_lock<std::mutex> lk(mu_);
        cv_done_.wait(lk, [&] { return pending_ == 0; });
    }
};

constexpr int STAGE_SLOTS = 4;

bool is_pageable(const void* p) {
    cudaPointerAttributes at;
    const cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();  // older drivers report unregistered host memory as an error
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// Borrow an idle pipeline context of m (creating one when every context is busy);
// returned to the pool when the call ends, also on error.
struct Borrow {
    Matrix* m;
    PipeCtx* c = nullptr;
    explicit Borrow(Matrix* mm) : m(mm) {
        std::lock_guard<std::mutex> lock(m->pipe_mu);
        if (!m->pipe_planned) plan_pipeline(m, nullptr);
        if (!m->pipe_free.empty()) {
            c = m->pipe_free.back();
            m->pipe_free.pop_back();
        } else {
            c = new_ctx(m);
            m->pipe_all.push_back(c);
        }
    }
    ~Borrow() {
        std::lock_guard<std::mutex> lock(m->pipe_mu);
        m->pipe_free.push_back(c);
    }
};

}  // namespace

// ---- bulk host <-> device copies for the upload / export entry points -------------
// The reference's containers are std::vectors (pageable): a plain cudaMemcpy of them
// runs at ~7 GB/s through the driver's own staging.  Large pageable transfers go
// through a process-wide pinned ring instead, filled / drained by the copy pool while
// the previous slot is on the wire.  Pinned or registered host memory, and small
// transfers, take cudaMemcpyAsync directly.
namespace {
constexpr size_t BULK_SLOT = (size_t)16 << 20;
constexpr int BULK_SLOTS = 4;
struct BulkRing {
    std::mutex mu;  // one staged transfer at a time
    char* ring = nullptr;
    cudaEvent_t ev[BULK_SLOTS] = {};
    void ensure() {
        if (ring) return;
        HDCG_CUDA(cudaHostAlloc(&ring, BULK_SLOT * BULK_SLOTS, cudaHostAllocPortable));
        for (auto& e : ev) HDCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
};
BulkRing& bulk_ring() {
    static BulkRing r;  // lives until process exit (pinned memory is released with the context)
    return r;
}
bool stage_bulk(const void* host, size_t bytes) {
    static const bool off = getenv("HDCG_STAGE_PAGEABLE") && atoi(getenv("HDCG_STAGE_PAGEABLE")) == 0;
    return !off && bytes >= ((size_t)8 << 20) && is_pageable(host);
}
}  // namespace

void copy_h2d(void* dev, const void* host, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (!stage_bulk(host, bytes)) {
        HDCG_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    BulkRing& r = bulk_ring();
    std::lock_guard<std::mutex> lock(r.mu);
    r.ensure();
    CopyPool& pool = CopyPool::get();
    int i = 0;
    for (size_t off = 0; off < bytes; off += BULK_SLOT, ++i) {
        const size_t n = std::min(BULK_SLOT, bytes - off);
        const int s = i % BULK_SLOTS;
        if (i >= BULK_SLOTS) HDCG_CUDA(cudaEventSynchronize(r.ev[s]));
        pool.copy(r.ring + s * BULK_SLOT, (const char*)host + off, n);
        HDCG_CUDA(cudaMemcpyAsync((char*)dev + off, r.ring + s * BULK_SLOT, n, cudaMemcpyHostToDevice, st));
        HDCG_CUDA(cudaEventRecord(r.ev[s], st));
    }
    HDCG_CUDA(cudaStreamSynchronize(st));  // the ring is free again when this returns
}

void copy_d2h(void* host, const void* dev, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (!stage_bulk(host, bytes)) {
        HDCG_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
        return;
    }
    BulkRing& r = bulk_ring();
    std::lock_guard<std::mutex> lock(r.mu);
    r.ensure();
    CopyPool& pool = CopyPool::get();
    const int total = (int)((bytes + BULK_SLOT - 1) / BULK_SLOT);
    auto finish = [&](int j) {  // slot of piece j -> the caller's memory
        const size_t off = (size_t)j * BULK_SLOT, n = std::min(BULK_SLOT, bytes - off);
        HDCG_CUDA(cudaEventSynchronize(r.ev[j % BULK_SLOTS]));
        pool.copy((char*)host + off, r.ring + (j % BULK_SLOTS) * BULK_SLOT, n);
    };
    for (int i = 0; i < total; ++i) {
        const size_t off = (size_t)i * BULK_SLOT, n = std::min(BULK_SLOT, bytes - off);
        if (i >= BULK_SLOTS) finish(i - BULK_SLOTS);
        HDCG_CUDA(cudaMemcpyAsync(r.ring + (i % BULK_SLOTS) * BULK_SLOT, (const char*)dev + off, n,
                                  cudaMemcpyDeviceToHost, st));
        HDCG_CUDA(cudaEventRecord(r.ev[i % BULK_SLOTS], st));
    }
    for (int j = std::max(0, total - BULK_SLOTS); j < total; ++j) finish(j);
}

void pipe_ctx_release(PipeCtx* c) {
    if (!c) return;
    cudaFree(c->dx);
    cudaFree(c->dy);
    cudaFreeHost(c->hx);
    cudaFreeHost(c->hy);
    for (cudaEvent_t e : c->slot_ev)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : c->s)
        if (s) cudaStreamDestroy(s);
    for (cudaEvent_t e : c->events)
        if (e) cudaEventDestroy(e);
    delete c;
}

void spmv_host_pipelined(Matrix* m, const double* x, double* y) {
    const DeviceGuard dg(m->device);
    const Borrow b(m);
    PipeCtx* ctx = b.c;
    cudaStream_t s_in = ctx->s[0], s_k = ctx->s[1], s_out = ctx->s[2];
    const int64_t np = (int64_t)m->x_pieces.size() - 1;
    const int64_t nc = (int64_t)m->chunk_blocks.size() - 1;
    cudaEvent_t* ev_in = ctx->events.data();
    cudaEvent_t* ev_k = ctx->events.data() + np;
    const Tiling t = tiling_of(*m);
    auto chunk_rows = [&](int64_t c, int64_t* r0, int64_t* r1) {
        const int64_t q0 = m->chunk_blocks[c], q1 = m->chunk_blocks[c + 1];
        int64_t dummy;
        tile_rows(q0, t.tiles_per_block, t.blocks_per_tile, t.tile_rows, m->bl, m->n_rows, r0, &dummy);
        tile_rows(q1 - 1, t.tiles_per_block, t.blocks_per_tile, t.tile_rows, m->bl, m->n_rows, &dummy, r1);
        *r0 = std::min(*r0, m->n_rows);
    };
    static const bool stage_off = getenv("HDCG_STAGE_PAGEABLE") && atoi(getenv("HDCG_STAGE_PAGEABLE")) == 0;
    const bool stage_x = !stage_off && is_pageable(x), stage_y = !stage_off && is_pageable(y);
    if (stage_x || stage_y) {
        if (!ctx->hx) {  // pinned rings, sized for the largest x piece / y chunk of this matrix
            int64_t mx = 1;
            for (int64_t p = 0; p < np; ++p) mx = std::max(mx, m->x_pieces[p + 1] - m->x_pieces[p]);
            for (int64_t c = 0; c < nc; ++c) {
                int64_t r0, r1;
                chunk_rows(c, &r0, &r1);
                mx = std::max(mx, r1 - r0);
            }
            ctx->slot_elems = mx;
            HDCG_CUDA(cudaHostAlloc(&ctx->hx, sizeof(double) * mx * STAGE_SLOTS, cudaHostAllocDefault));
            HDCG_CUDA(cudaHostAlloc(&ctx->hy, sizeof(double) * mx * STAGE_SLOTS, cudaHostAllocDefault));
            ctx->slot_ev.assign(2 * STAGE_SLOTS, nullptr);
            for (auto& e : ctx->slot_ev) HDCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    CopyPool* pool = (stage_x || stage_y) ? &CopyPool::get() : nullptr;
    cudaEvent_t* ev_xfree = ctx->slot_ev.data();
    cudaEvent_t* ev_yfull = ctx->slot_ev.data() + STAGE_SLOTS;

    int64_t c_next = 0;     // next chunk to launch
    int64_t c_drained = 0;  // staged y chunks [0, c_drained) are in the caller's vector
    int64_t p_done = -1;
    auto drain = [&](int64_t c) {  // y chunk c: pinned slot -> caller's vector
        int64_t r0, r1;
        chunk_rows(c, &r0, &r1);
        HDCG_CUDA(cudaEventSynchronize(ev_yfull[c % STAGE_SLOTS]));
        if (r1 > r0) pool->copy(y + r0, ctx->hy + (c % STAGE_SLOTS) * ctx->slot_elems, sizeof(double) * (r1 - r0));
    };
    auto launch_ready = [&](int64_t pieces_sent) {
        // every chunk whose x is on its way (pieces [0, pieces_sent) are enqueued)
        const int64_t have = m->x_pieces[pieces_sent];
        while (c_next < nc && (m->chunk_x_hi[c_next] <= have || pieces_sent == np)) {
            const int64_t c = c_next++;
            const int64_t need = m->chunk_x_hi[c];
            int64_t p = p_done;
            while (p + 1 < np && m->x_pieces[p + 1] < need) ++p;
            if (need > 0 && p < 0) p = 0;
            if (p > p_done) {
                HDCG_CUDA(cudaStreamWaitEvent(s_k, ev_in[p], 0));
                p_done = p;
            }
            spmv_launch_tiles(*m, ctx->dx + m->row0, ctx->dy, m->chunk_blocks[c], m->chunk_blocks[c + 1], nullptr,
                              nullptr, s_k);
            HDCG_CUDA(cudaEventRecord(ev_k[c], s_k));
            HDCG_CUDA(cudaStreamWaitEvent(s_out, ev_k[c], 0));
            int64_t r0, r1;
            chunk_rows(c, &r0, &r1);
            if (stage_y) {
                if (c >= STAGE_SLOTS) {  // the slot's previous chunk must be out first
                    for (; c_drained <= c - STAGE_SLOTS; ++c_drained) drain(c_drained);
                }
                if (r1 > r0)
                    HDCG_CUDA(cudaMemcpyAsync(ctx->hy + (c % STAGE_SLOTS) * ctx->slot_elems, ctx->dy + r0,
                                              sizeof(double) * (r1 - r0), cudaMemcpyDeviceToHost, s_out));
                HDCG_CUDA(cudaEventRecord(ev_yfull[c % STAGE_SLOTS], s_out));
            } else if (r1 > r0) {
                HDCG_CUDA(cudaMemcpyAsync(y + r0, ctx->dy + r0, sizeof(double) * (r1 - r0), cudaMemcpyDeviceToHost,
                                          s_out));
            }
        }
    };
    for (int64_t p = 0; p < np; ++p) {
        const int64_t a = m->x_pieces[p], e = m->x_pieces[p + 1];
        if (e > a) {
            if (stage_x) {
                double* slot = ctx->hx + (p % STAGE_SLOTS) * ctx->slot_elems;
                if (p >= STAGE_SLOTS) HDCG_CUDA(cudaEventSynchronize(ev_xfree[p % STAGE_SLOTS]));
                pool->copy(slot, x + a, sizeof(double) * (e - a));
                HDCG_CUDA(cudaMemcpyAsync(ctx->dx + a, slot, sizeof(double) * (e - a), cudaMemcpyHostToDevice, s_in));
                HDCG_CUDA(cudaEventRecord(ev_xfree[p % STAGE_SLOTS], s_in));
            } else {
                HDCG_CUDA(cudaMemcpyAsync(ctx->dx + a, x + a, sizeof(double) * (e - a), cudaMemcpyHostToDevice, s_in));
            }
        }
        HDCG_CUDA(cudaEventRecord(ev_in[p], s_in));
        // staging is host work: launch what can already run, so kernels and y copies overlap it
        if (stage_x || stage_y) launch_ready(p + 1);
    }
    launch_ready(np);
    if (stage_y)
        for (; c_drained < nc; ++c_drained) drain(c_drained);
    HDCG_CUDA(cudaStreamSynchronize(s_out));
    HDCG_CUDA(cudaStreamSynchronize(s_in));
}

}  // namespace hdcg

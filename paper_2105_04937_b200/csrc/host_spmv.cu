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
#include <algorithm>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

constexpr int PIPE_CHUNKS = 8;

// per block: highest global column any of its rows reads (-1: none)
__global__ void block_xhi_kernel(int64_t n_blocks, int64_t bl, int64_t n_rows, int64_t row0, int64_t n_cols,
                                 const int32_t* dia_ptr, const int32_t* dia_off, const int32_t* rest_rp,
                                 const int32_t* rest_col, int64_t* hi_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < n_blocks; b += n_warps) {
        const int64_t r0 = b * bl, r1 = min(r0 + bl, n_rows);
        int64_t hi = -1;
        if (lane == 0) {
            const int k0 = dia_ptr[b], k1 = dia_ptr[b + 1];
            if (k1 > k0) hi = min(n_cols - 1, row0 + r1 - 1 + (int64_t)dia_off[k1 - 1]);
        }
        if (rest_rp) {
            const int64_t e0 = rest_rp[r0], e1 = rest_rp[r1];
            for (int64_t e = e0 + lane; e < e1; e += 32) hi = max(hi, (int64_t)rest_col[e]);
        }
        for (int o = 16; o > 0; o >>= 1) hi = max(hi, (int64_t)__shfl_down_sync(0xffffffffu, hi, o));
        if (lane == 0) hi_out[b] = hi;
    }
}

void plan_pipeline(Matrix* m, cudaStream_t st) {
    const Tiling t = tiling_of(*m);
    const int64_t align = t.blocks_per_tile > 0 ? t.blocks_per_tile : 1;
    const int64_t nb = m->n_blocks;
    int64_t per = std::max<int64_t>(align, ceil_div(ceil_div(nb, PIPE_CHUNKS), align) * align);
    m->chunk_blocks.clear();
    for (int64_t b = 0; b < nb; b += per) m->chunk_blocks.push_back(b);
    m->chunk_blocks.push_back(nb);
    const int64_t n_chunks = (int64_t)m->chunk_blocks.size() - 1;

    std::vector<int64_t> hi((size_t)nb);
    int64_t* d_hi = dev_alloc<int64_t>(nb, st);
    block_xhi_kernel<<<grid_cap(ceil_div(nb * 32, 256)), 256, 0, st>>>(
        nb, m->bl, m->n_rows, m->row0, m->n_cols, m->dia_ptr, m->dia_off, m->nnz_rest > 0 ? m->rest_rp : nullptr,
        m->rest_col, d_hi);
    HDCG_LAUNCH_CHECK("block_xhi_kernel");
    HDCG_CUDA(cudaMemcpyAsync(hi.data(), d_hi, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    dev_free(d_hi, st);
    m->chunk_x_hi.assign((size_t)n_chunks, 0);
    int64_t run = 0;  // chunks run in order, so the requirement is cumulative
    for (int64_t c = 0; c < n_chunks; ++c) {
        for (int64_t b = m->chunk_blocks[c]; b < m->chunk_blocks[c + 1]; ++b) run = std::max(run, hi[b] + 1);
        m->chunk_x_hi[c] = run;
    }
    // x pieces: equal slices of [0, n_cols), 16-byte aligned boundaries
    m->x_pieces.clear();
    const int64_t np = std::max<int64_t>(1, std::min<int64_t>(PIPE_CHUNKS, m->n_cols));
    for (int64_t p = 0; p < np; ++p) m->x_pieces.push_back((m->n_cols * p / np) & ~int64_t(1));
    m->x_pieces.push_back(m->n_cols);

    for (int s = 0; s < 3; ++s) HDCG_CUDA(cudaStreamCreateWithFlags(&m->pipe[s], cudaStreamNonBlocking));
    m->pipe_events.resize((size_t)(np + n_chunks));
    for (auto& e : m->pipe_events) HDCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HDCG_CUDA(cudaMalloc(&m->dx, sizeof(double) * std::max<int64_t>(1, m->n_cols)));
    HDCG_CUDA(cudaMalloc(&m->dy, sizeof(double) * std::max<int64_t>(1, m->n_rows)));
}

}  // namespace

void spmv_host_pipelined(Matrix* m, const double* x, double* y) {
    HDCG_CUDA(cudaSetDevice(m->device));
    if (!m->pipe[0]) plan_pipeline(m, nullptr);
    cudaStream_t s_in = m->pipe[0], s_k = m->pipe[1], s_out = m->pipe[2];
    const int64_t np = (int64_t)m->x_pieces.size() - 1;
    const int64_t nc = (int64_t)m->chunk_blocks.size() - 1;
    cudaEvent_t* ev_in = m->pipe_events.data();
    cudaEvent_t* ev_k = m->pipe_events.data() + np;
    for (int64_t p = 0; p < np; ++p) {
        const int64_t a = m->x_pieces[p], b = m->x_pieces[p + 1];
        if (b > a) HDCG_CUDA(cudaMemcpyAsync(m->dx + a, x + a, sizeof(double) * (b - a), cudaMemcpyHostToDevice, s_in));
        HDCG_CUDA(cudaEventRecord(ev_in[p], s_in));
    }
    int64_t p_done = -1;
    for (int64_t c = 0; c < nc; ++c) {
        // wait for the x pieces up to the one holding column chunk_x_hi[c]-1
        const int64_t need = m->chunk_x_hi[c];
        int64_t p = p_done;
        while (p + 1 < np && m->x_pieces[p + 1] < need) ++p;
        if (need > 0 && p < 0) p = 0;
        if (p > p_done) {
            HDCG_CUDA(cudaStreamWaitEvent(s_k, ev_in[p], 0));
            p_done = p;
        }
        const int64_t b0 = m->chunk_blocks[c], b1 = m->chunk_blocks[c + 1];
        spmv_launch(*m, m->dx + m->row0, m->dy, b0, b1, nullptr, nullptr, s_k);
        HDCG_CUDA(cudaEventRecord(ev_k[c], s_k));
        HDCG_CUDA(cudaStreamWaitEvent(s_out, ev_k[c], 0));
        const int64_t r0 = b0 * m->bl, r1 = std::min(b1 * m->bl, m->n_rows);
        if (r1 > r0)
            HDCG_CUDA(cudaMemcpyAsync(y + r0, m->dy + r0, sizeof(double) * (r1 - r0), cudaMemcpyDeviceToHost, s_out));
    }
    HDCG_CUDA(cudaStreamSynchronize(s_out));
    HDCG_CUDA(cudaStreamSynchronize(s_in));
}

}  // namespace hdcg

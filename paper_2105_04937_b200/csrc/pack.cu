// pack.cu -- the tile-packed copy of a small-block M-HDC (bl < 1024).
//
// The reference layout (convert.cpp:141-156, formats.hpp:107-132) stores segment
// k of block ib as bl consecutive values.  For small blocks (the paper's
// recommended 50 <= bl <= 500; hdcmv's default bl = 100,
// hdcmv.cpp:148) a 1024-row tile of the SpMV then spans many blocks whose
// segments are 0.8 KB runs, and the kernel either idles threads or pays
// per-block bookkeeping for every few slots.  The packed copy re-lays the same
// values out per 1024-row tile t = rows [1024 t, 1024 t + 1024):
//
//   stage k of tile t (k < K_t = the most segments any block of the tile has) is
//   1024 consecutive values: row r's is the k-th segment of r's block at slot
//   r - ib*bl, or 0.0 where that block has fewer than k+1 segments.
//   pk_meta[t] = {first stage of t, K_t | uniform << 16, start of t's offset
//   table, first block of t}; the table is [blocks of t][K_t] offsets
//   (INT32_MIN where a block has no k-th segment), or ONE list of K_t offsets
//   when every block of the tile has the same list (uniform: stencils).
//
// So the SpMV moves whole 8 KB stages by TMA and runs the 4-rows-per-thread
// interleaved consumer loop of large blocks, whatever bl is.  Each row still
// adds its own block's segments in stored order (padding slots are skipped),
// so y is bitwise the reference's (kernels.cpp:192-204).  Costs one extra copy
// of the segment values in HBM; the reference layout remains for export, rates
// and the general kernel.
#include <cstdlib>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

// per tile: K_t, uniform flag, table entries
__global__ void pack_plan_kernel(int64_t n_tiles, int64_t n_rows, int64_t bl, const int32_t* dia_ptr,
                                 const int32_t* dia_off, int64_t* k_out, int64_t* tab_out, int32_t* uni_out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = t * PACK_TILE, hi = min(lo + PACK_TILE, n_rows);
        const int64_t b0 = lo / bl, b1 = (hi - 1) / bl;
        const int c0 = dia_ptr[b0 + 1] - dia_ptr[b0];
        int K = c0;
        bool uni = true;
        for (int64_t b = b0 + 1; b <= b1; ++b) {
            const int c = dia_ptr[b + 1] - dia_ptr[b];
            K = max(K, c);
            if (uni && c == c0) {
                for (int k = 0; k < c; ++k)
                    if (dia_off[dia_ptr[b] + k] != dia_off[dia_ptr[b0] + k]) {
                        uni = false;
                        break;
                    }
            } else {
                uni = false;
            }
        }
        k_out[t] = K;
        tab_out[t] = uni ? K : (b1 - b0 + 1) * K;
        uni_out[t] = uni;
    }
}

__global__ void pack_meta_kernel(int64_t n_tiles, int64_t bl, const int64_t* k, const int64_t* stage0,
                                 const int64_t* tab0, const int32_t* uni, int4* meta) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x)
        meta[t] = make_int4((int)stage0[t], (int)k[t] | (uni[t] << 16), (int)tab0[t], (int)(t * PACK_TILE / bl));
}

// one CTA per tile: the offset table and the K_t stages of values
__global__ void __launch_bounds__(256) pack_fill_kernel(int64_t n_rows, int64_t bl, const int32_t* dia_ptr,
                                                        const int32_t* dia_off, const double* seg,
                                                        const int4* meta, int32_t* tab, double* val) {
    const int64_t t = blockIdx.x;
    const int4 md = meta[t];
    const int K = md.y & 0xffff;
    const bool uni = (md.y >> 16) & 1;
    const int64_t lo = t * PACK_TILE, hi = min(lo + PACK_TILE, n_rows);
    const int64_t b0 = md.w, b1 = (hi - 1) / bl;
    if (uni) {
        for (int k = threadIdx.x; k < K; k += blockDim.x) tab[md.z + k] = dia_off[dia_ptr[b0] + k];
    } else {
        for (int64_t e = threadIdx.x; e < (b1 - b0 + 1) * K; e += blockDim.x) {
            const int64_t b = b0 + e / K;
            const int k = (int)(e % K);
            const int c = dia_ptr[b + 1] - dia_ptr[b];
            tab[md.z + e] = k < c ? dia_off[dia_ptr[b] + k] : INT32_MIN;
        }
    }
    double* out = val + (int64_t)md.x * PACK_TILE;
    for (int k = 0; k < K; ++k)
        for (int r = threadIdx.x; r < PACK_TILE; r += blockDim.x) {
            const int64_t i = lo + r;
            double v = 0.0;
            if (i < hi) {
                const int64_t b = i / bl;
                const int ks = dia_ptr[b];
                if (k < dia_ptr[b + 1] - ks) v = seg[(int64_t)(ks + k) * bl + (i - b * bl)];
            }
            out[(int64_t)k * PACK_TILE + r] = v;
        }
}

}  // namespace

// HDCG_PACKED (read per build): 0 never, 1 the default shapes, 2 every bl < 1024
bool pack_eligible(int64_t bl, int64_t n_rows) {
    const char* e = getenv("HDCG_PACKED");
    const int mode = e ? atoi(e) : 1;
    if (mode == 0 || bl >= PACK_TILE || n_rows <= 0) return false;
    if (mode == 2) return true;
    // 128 / 256 tile 1024 rows with whole blocks and run faster on the
    // multi-block layouts (97.5% vs 95% packed); 512 runs faster packed (98.9%
    // vs 92.4%, whose light remainder the multi-block layout sums per warp):
    // profiles/r02f_ab_small_bl.log
    return PACK_TILE % bl != 0 || bl < 128 || bl == 512;
}

void build_packed(Matrix* m, cudaStream_t st) {
    if (m->kind != HDCG_KIND_MHDC || m->n_seg == 0 || !pack_eligible(m->bl, m->n_rows)) return;
    const int64_t nt = ceil_div(m->n_rows, PACK_TILE);
    if (m->max_seg_per_block > 0xffff) return;
    int64_t* k = dev_alloc<int64_t>(nt + 1, st);
    int64_t* tabn = dev_alloc<int64_t>(nt + 1, st);
    int64_t* stage0 = dev_alloc<int64_t>(nt + 1, st);
    int64_t* tab0 = dev_alloc<int64_t>(nt + 1, st);
    int32_t* uni = dev_alloc<int32_t>(nt, st);
    HDCG_CUDA(cudaMemsetAsync(k + nt, 0, sizeof(int64_t), st));
    HDCG_CUDA(cudaMemsetAsync(tabn + nt, 0, sizeof(int64_t), st));
    pack_plan_kernel<<<grid_cap(ceil_div(nt, 256)), 256, 0, st>>>(nt, m->n_rows, m->bl, m->dia_ptr, m->dia_off, k,
                                                                  tabn, uni);
    HDCG_LAUNCH_CHECK("pack_plan_kernel");
    size_t bytes = 0;
    HDCG_CUDA(cub_exclusive_sum_i64(nullptr, bytes, k, stage0, nt + 1, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub_exclusive_sum_i64(tmp, bytes, k, stage0, nt + 1, st));
    HDCG_CUDA(cub_exclusive_sum_i64(tmp, bytes, tabn, tab0, nt + 1, st));
    dev_free(tmp, st);
    int64_t tot[2];
    HDCG_CUDA(cudaMemcpyAsync(&tot[0], stage0 + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaMemcpyAsync(&tot[1], tab0 + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    if (tot[0] > 0x7fffffffLL || tot[1] > 0x7fffffffLL) {  // beyond the int32 tile metadata
        dev_free(k, st);
        dev_free(tabn, st);
        dev_free(stage0, st);
        dev_free(tab0, st);
        dev_free(uni, st);
        return;
    }
    m->pk_stages = tot[0];
    m->pk_meta = dev_alloc<int4>(nt, st);
    m->pk_tab = dev_alloc<int32_t>(std::max<int64_t>(1, tot[1]), st);
    m->pk_val = alloc_seg(tot[0] * PACK_TILE, st);
    pack_meta_kernel<<<grid_cap(ceil_div(nt, 256)), 256, 0, st>>>(nt, m->bl, k, stage0, tab0, uni, m->pk_meta);
    HDCG_LAUNCH_CHECK("pack_meta_kernel");
    pack_fill_kernel<<<(unsigned)nt, 256, 0, st>>>(m->n_rows, m->bl, m->dia_ptr, m->dia_off, m->seg, m->pk_meta,
                                                   m->pk_tab, m->pk_val);
    HDCG_LAUNCH_CHECK("pack_fill_kernel");
    dev_free(k, st);
    dev_free(tabn, st);
    dev_free(stage0, st);
    dev_free(tab0, st);
    dev_free(uni, st);
    HDCG_CUDA(cudaStreamSynchronize(st));
    m->packed = true;
}

}  // namespace hdcg

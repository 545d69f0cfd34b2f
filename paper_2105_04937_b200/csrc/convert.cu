// convert.cu -- CSR -> M-HDC / HDC converters on the device, bit-exact with
// hdc::to_mhdc / hdc::to_hdc (proj/src/convert.cpp:89-169).
//
// Reference algorithm (per row block ib of width bl, last block shorter):
//   census     counts of stored entries per offset off = col - row (explicit
//              zeros count, convert.cpp:39-58);
//   select     off kept iff double(count)/double(len) >= theta (convert.cpp:12-14,
//              len = min(bl, n - ib*bl); HDC: len = n);
//   dia_ptr    exclusive prefix of per-block selected counts, offsets ascending;
//   segments   segment k zero-filled, slot i - ib*bl = value (convert.cpp:141,156);
//   remainder  unselected entries in original per-row order (convert.cpp:158-162).
//
// Device pipeline (each step a kernel; only the scalar sizes come back to the host):
//   1. census+select per block in shared memory: open-addressing hash with
//      warp-aggregated inserts (__match_any_sync); a block whose census does not
//      fit (too many distinct offsets) or that selects > SEL_MAX offsets goes to
//   1b. the general path: the block's offsets are gathered, segment-sorted (CUB),
//      run-length encoded and selected in order (exact for any offset count);
//      HDC uses a dense histogram over [-(n-1), n-1] instead of a hash;
//   2. scan of per-block counts -> dia_ptr; the sorted selections -> dia_offsets;
//   3. per row: remainder count by binary search in the block's offsets; scan -> row_ptr;
//   4. per row: a merge of the row's ascending offsets with the block's ascending
//      selected offsets writes every segment slot exactly once (value or 0.0,
//      coalesced across the rows of a block) and appends unselected entries to
//      the remainder in stored order.  Tail slots of a short last block get 0.0.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hdcg_internal.cuh"

namespace hdcg {

constexpr int CENSUS_THREADS = 512;
constexpr int HASH_LOG2 = 11;
constexpr int HASH_CAP = 1 << HASH_LOG2;
constexpr int HASH_MAX_PROBE = 64;
constexpr int SEL_MAX = 32;
constexpr int32_t EMPTY_KEY = INT32_MIN;

// HDCG_TRACE_BUILD=1: wall time of each conversion stage on stderr (each mark
// synchronises the stream: a diagnostic, not for timed runs)
struct BuildTrace {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t0;
    explicit BuildTrace(cudaStream_t s) : on(getenv("HDCG_TRACE_BUILD") != nullptr), st(s) {
        if (on) {
            cudaStreamSynchronize(st);
            t0 = std::chrono::steady_clock::now();
        }
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[hdcg build] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

template <class RP>
struct RowPtr {
    const RP* p;
    __device__ __forceinline__ int64_t operator[](int64_t i) const { return (int64_t)p[i]; }
};

// ---------------------------------------------------------------------------
// validation: the CsrMatrix constructor's per-row checks (formats.cpp:55-66).
// The first failing (row, position, check) in the reference's order wins, so
// the reported exception type is the one the reference would throw.
template <class RP>
__global__ void validate_kernel(RowPtr<RP> rp, const int32_t* col, int64_t n_rows, int64_t n_cols,
                                unsigned long long* first_err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = rp[i], b = rp[i + 1];
        unsigned long long key = ~0ULL;
        if (a > b) {
            key = (unsigned long long)i << 33;  // monotonicity, checked before the columns
        } else {
            for (int64_t k = a; k < b; ++k) {
                const int32_t c = col[k];
                const unsigned long long pos = (unsigned long long)(k - a + 1) << 1;
                if (c < 0 || c >= n_cols) { key = ((unsigned long long)i << 33) | pos; break; }
                if (k > a && col[k - 1] >= c) { key = ((unsigned long long)i << 33) | pos | 1ULL; break; }
            }
        }
        if (key != ~0ULL) atomicMin(first_err, key);
    }
}

template <class RP>
static void validate_t(const CsrInput& in, cudaStream_t st) {
    int64_t ends[2] = {0, 0};
    if (in.n_rows >= 0) {
        if (in.rp64) {
            HDCG_CUDA(cudaMemcpyAsync(&ends[0], (const int64_t*)in.row_ptr, 8, cudaMemcpyDeviceToHost, st));
            HDCG_CUDA(cudaMemcpyAsync(&ends[1], (const int64_t*)in.row_ptr + in.n_rows, 8,
                                      cudaMemcpyDeviceToHost, st));
        } else {
            int32_t e[2];
            HDCG_CUDA(cudaMemcpyAsync(&e[0], (const int32_t*)in.row_ptr, 4, cudaMemcpyDeviceToHost, st));
            HDCG_CUDA(cudaMemcpyAsync(&e[1], (const int32_t*)in.row_ptr + in.n_rows, 4,
                                      cudaMemcpyDeviceToHost, st));
            HDCG_CUDA(cudaStreamSynchronize(st));
            ends[0] = e[0];
            ends[1] = e[1];
        }
        HDCG_CUDA(cudaStreamSynchronize(st));
    }
    if (ends[0] != 0 || ends[1] != in.nnz)
        fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: row_ptr endpoints do not match value count");
    if (in.n_rows == 0) return;
    unsigned long long* d_err = dev_alloc<unsigned long long>(1, st);
    HDCG_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), st));
    validate_kernel<RP><<<grid_cap(ceil_div(in.n_rows, 256)), 256, 0, st>>>(
        RowPtr<RP>{(const RP*)in.row_ptr}, in.col, in.n_rows, in.n_cols, d_err);
    HDCG_LAUNCH_CHECK("validate_kernel");
    unsigned long long key = 0;
    HDCG_CUDA(cudaMemcpyAsync(&key, d_err, sizeof(key), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    dev_free(d_err, st);
    if (key == ~0ULL) return;
    const int64_t row = (int64_t)(key >> 33);
    const uint64_t pos = (key >> 1) & 0xffffffffULL;
    if (pos == 0)
        fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: row_ptr not monotone at row " + std::to_string(row));
    if (key & 1ULL)
        fail(HDCG_ERR_INVALID_ARGUMENT,
             "CsrMatrix: columns not strictly ascending in row " + std::to_string(row));
    fail(HDCG_ERR_OUT_OF_RANGE, "CsrMatrix: column index out of range in row " + std::to_string(row));
}

void validate_csr(const CsrInput& in, cudaStream_t st) {
    if (in.n_rows < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "CsrMatrix: negative dimension");
    if (in.rp64) validate_t<int64_t>(in, st);
    else validate_t<int32_t>(in, st);
}

// ---------------------------------------------------------------------------
// 1. shared-memory census + selection per block

// used / n_used: the slots that hold a key, in insertion order, while there are at
// most USED_MAX of them -- a block with few distinct offsets (any stencil) is then
// selected from and cleared through this list instead of the whole table, which
// matters for small blocks (256 rows x 7 entries against 2048 slots).
constexpr int USED_MAX = 128;
__device__ __forceinline__ bool hash_add(int32_t* keys, int32_t* cnts, int32_t off, int c, int32_t* used,
                                         int* n_used) {
    volatile int32_t* vkeys = keys;
    uint32_t h = ((uint32_t)off * 0x9E3779B1u) >> (32 - HASH_LOG2);
    for (int p = 0; p < HASH_MAX_PROBE; ++p) {
        const int32_t k = vkeys[h];
        if (k == off) { atomicAdd(&cnts[h], c); return true; }
        if (k == EMPTY_KEY) {
            const int32_t prev = atomicCAS(&keys[h], EMPTY_KEY, off);
            if (prev == EMPTY_KEY) {  // this thread claimed the slot
                const int u = atomicAdd(n_used, 1);
                if (u < USED_MAX) used[u] = (int32_t)h;
            }
            if (prev == EMPTY_KEY || prev == off) { atomicAdd(&cnts[h], c); return true; }
        }
        h = (h + 1) & (HASH_CAP - 1);
    }
    return false;
}

#ifndef HDCG_CENSUS_MINB
#define HDCG_CENSUS_MINB 3
#endif
template <class RP>
__global__ void __launch_bounds__(CENSUS_THREADS, HDCG_CENSUS_MINB)
census_select_kernel(RowPtr<RP> rp, const int32_t* col, int64_t n_rows, int64_t row0, int64_t bl,
                     int64_t n_blocks, double theta, int32_t* sel_count, int32_t* stash,
                     int32_t* blk_status, int32_t* ovf_list, int32_t* ovf_count, int32_t* blk_rest,
                     int bucket_filter) {
    __shared__ int32_t keys[HASH_CAP];
    __shared__ int32_t cnts[HASH_CAP];
    __shared__ int32_t sel[SEL_MAX];
    __shared__ int s_nsel;
    __shared__ int s_overflow;
    __shared__ unsigned long long s_selected;  // entries on the selected offsets
    __shared__ int32_t used[USED_MAX];
    __shared__ int s_nused;
    const int lane = threadIdx.x & 31;
    bool first = true;
    for (int64_t b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        // clear the table: only the slots the previous block used, when those are listed
        const int prev_used = first ? USED_MAX + 1 : s_nused;
        first = false;
        if (prev_used <= USED_MAX) {
            for (int s = threadIdx.x; s < prev_used; s += blockDim.x) {
                keys[used[s]] = EMPTY_KEY;
                cnts[used[s]] = 0;
            }
        } else {
            for (int s = threadIdx.x; s < HASH_CAP; s += blockDim.x) {
                keys[s] = EMPTY_KEY;
                cnts[s] = 0;
            }
        }
        __syncthreads();  // prev_used was read by every thread before it is reset
        if (threadIdx.x == 0) { s_nsel = 0; s_overflow = 0; s_selected = 0; s_nused = 0; }
        __syncthreads();
        const int64_t r0 = b * bl, r1 = min(r0 + bl, n_rows), len = r1 - r0;
        volatile int* vovf = &s_overflow;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            if (*vovf) break;
            const int64_t gi = row0 + i;
            const int64_t ke = rp[i + 1];
            for (int64_t k = rp[i]; k < ke; ++k) {
                const int32_t off = (int32_t)((int64_t)col[k] - gi);
                const unsigned peers = __match_any_sync(__activemask(), off);
                if (lane == __ffs(peers) - 1) {
                    if (!hash_add(keys, cnts, off, __popc(peers), used, &s_nused)) *vovf = 1;
                }
            }
        }
        __syncthreads();
        // The table overflowed: more distinct offsets than slots (rows with scattered
        // columns).  Only offsets with count >= theta * len matter, so count the
        // entries per hash bucket first (no keys, no probing): an offset can pass the
        // threshold only if its bucket's total does.  A second pass tallies exactly
        // the offsets of those candidate buckets -- a handful of keys -- and the
        // selection below proceeds as usual.  Exact: nothing that could be selected is
        // left out.  (If every present offset qualifies -- theta * len <= 1 -- or the
        // second pass overflows too, the block takes the sort path.)
        if (s_overflow && bucket_filter && !((double)1 / (double)len >= theta)) {
            __shared__ uint32_t cand[HASH_CAP / 32];
            for (int s = threadIdx.x; s < HASH_CAP; s += blockDim.x) cnts[s] = 0;
            for (int s = threadIdx.x; s < HASH_CAP / 32; s += blockDim.x) cand[s] = 0;
            __syncthreads();
            for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                const int64_t gi = row0 + i, ke = rp[i + 1];
                for (int64_t k = rp[i]; k < ke; ++k) {
                    const int32_t off = (int32_t)((int64_t)col[k] - gi);
                    const unsigned peers = __match_any_sync(__activemask(), off);
                    if (lane == __ffs(peers) - 1)
                        atomicAdd(&cnts[((uint32_t)off * 0x9E3779B1u) >> (32 - HASH_LOG2)], __popc(peers));
                }
            }
            __syncthreads();
            for (int s = threadIdx.x; s < HASH_CAP; s += blockDim.x)
                if ((double)cnts[s] / (double)len >= theta) atomicOr(&cand[s >> 5], 1u << (s & 31));
            __syncthreads();
            for (int s = threadIdx.x; s < HASH_CAP; s += blockDim.x) {
                keys[s] = EMPTY_KEY;
                cnts[s] = 0;
            }
            if (threadIdx.x == 0) { s_overflow = 0; s_nused = 0; }
            __syncthreads();
            for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                if (*vovf) break;
                const int64_t gi = row0 + i, ke = rp[i + 1];
                for (int64_t k = rp[i]; k < ke; ++k) {
                    const int32_t off = (int32_t)((int64_t)col[k] - gi);
                    const uint32_t h = ((uint32_t)off * 0x9E3779B1u) >> (32 - HASH_LOG2);
                    if ((cand[h >> 5] >> (h & 31)) & 1u) {
                        const unsigned peers = __match_any_sync(__activemask(), off);
                        if (lane == __ffs(peers) - 1) {
                            if (!hash_add(keys, cnts, off, __popc(peers), used, &s_nused)) *vovf = 1;
                        }
                    }
                }
            }
            __syncthreads();
        }
        if (!s_overflow) {
            const int nu = s_nused;
            const int n_scan = nu <= USED_MAX ? nu : HASH_CAP;
            for (int q = threadIdx.x; q < n_scan; q += blockDim.x) {
                const int s = nu <= USED_MAX ? used[q] : q;
                const int32_t k = keys[s];
                if (k != EMPTY_KEY && (double)cnts[s] / (double)len >= theta) {
                    const int p = atomicAdd(&s_nsel, 1);
                    if (p < SEL_MAX) sel[p] = k;
                    atomicAdd(&s_selected, (unsigned long long)cnts[s]);
                }
            }
        }
        __syncthreads();
        const bool fast = !s_overflow && s_nsel <= SEL_MAX;
        if (fast) {
            if (threadIdx.x < 32) {
                const int S = s_nsel;
                const int32_t v = lane < S ? sel[lane] : INT32_MAX;
                int rank = 0;
                for (int j = 0; j < 32; ++j) {
                    const int32_t w = __shfl_sync(0xffffffffu, v, j);
                    rank += (j < S) && (w < v);
                }
                if (lane < S) stash[b * SEL_MAX + rank] = v;
            }
            if (threadIdx.x == 0) {
                sel_count[b] = s_nsel;
                blk_status[b] = 0;
                // entries left for the remainder: 0 lets rest_count_kernel skip the block
                const int64_t left = (rp[r1] - rp[r0]) - (int64_t)s_selected;
                blk_rest[b] = (int32_t)min(left, (int64_t)INT32_MAX);
                if (left != 0) ovf_count[1] = 1;  // the matrix has a remainder (benign race: every writer stores 1)
            }
        } else if (threadIdx.x == 0) {
            sel_count[b] = 0;
            ovf_count[1] = 1;
            blk_rest[b] = -1;  // unknown: counted row by row
            blk_status[b] = -1;
            ovf_list[atomicAdd(ovf_count, 1)] = (int32_t)b;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// 1b. general path: gather -> segmented sort -> run-length encode + select

template <class RP>
__global__ void ovf_sizes_kernel(RowPtr<RP> rp, int64_t n_rows, int64_t bl, const int32_t* ovf_list,
                                 int n_ovf, int64_t* sizes) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_ovf; j += gridDim.x * blockDim.x) {
        const int64_t b = ovf_list[j];
        const int64_t r0 = b * bl, r1 = min(r0 + bl, n_rows);
        sizes[j] = rp[r1] - rp[r0];
    }
}

template <class RP>
__global__ void ovf_gather_kernel(RowPtr<RP> rp, const int32_t* col, int64_t n_rows, int64_t row0,
                                  int64_t bl, const int32_t* ovf_list, const int64_t* start,
                                  int32_t* keys) {
    const int j = blockIdx.x;
    const int64_t b = ovf_list[j];
    const int64_t r0 = b * bl, r1 = min(r0 + bl, n_rows);
    const int64_t e0 = rp[r0];
    int32_t* out = keys + start[j];
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const int64_t gi = row0 + i, ke = rp[i + 1];
        for (int64_t k = rp[i]; k < ke; ++k) out[k - e0] = (int32_t)((int64_t)col[k] - gi);
    }
}

// mode 0: select (sel_out = selected offsets ascending, sel_count[b] = #)
// mode 1: census export (sel_out = every distinct offset, cnt_out = counts)
template <int MODE>
__global__ void __launch_bounds__(256)
ovf_rle_kernel(const int32_t* keys, const int64_t* start, const int32_t* ovf_list, int64_t n_rows,
               int64_t bl, double theta, int32_t* sel_out, int64_t* cnt_out, int32_t* sel_count) {
    typedef cub::BlockScan<int, 256> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int carry;
    const int j = blockIdx.x;
    const int64_t b = ovf_list[j];
    const int64_t len = min(bl, n_rows - b * bl);
    const int64_t s = start[j], e = start[j + 1];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c = s; c < e; c += 256) {
        const int64_t p = c + threadIdx.x;
        int flag = 0;
        int32_t key = 0;
        int64_t count = 0;
        if (p < e) {
            key = keys[p];
            if (p == s || keys[p - 1] != key) {
                // end of run: upper_bound of key in [p, e)
                int64_t lo = p, hi = e;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (keys[mid] <= key) lo = mid + 1; else hi = mid;
                }
                count = lo - p;
                flag = MODE == 1 ? 1 : ((double)count / (double)len >= theta);
            }
        }
        int pos, total;
        Scan(scan_tmp).ExclusiveSum(flag, pos, total);
        if (flag) {
            sel_out[s + carry + pos] = key;
            if (MODE == 1) cnt_out[s + carry + pos] = count;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) sel_count[b] = carry;
}

__global__ void ovf_index_kernel(const int32_t* ovf_list, int n_ovf, int32_t* blk_status) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_ovf; j += gridDim.x * blockDim.x)
        blk_status[ovf_list[j]] = j + 1;
}

// ---------------------------------------------------------------------------
// 2. selected offsets into dia_offsets

__global__ void write_offsets_kernel(int64_t n_blocks, const int32_t* dia_ptr, const int32_t* blk_status,
                                     const int32_t* stash, const int32_t* sel_out,
                                     const int64_t* ovf_start, int32_t* dia_off) {
    for (int64_t b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        const int32_t base = dia_ptr[b], S = dia_ptr[b + 1] - base;
        const int32_t st = blk_status[b];
        const int32_t* src = st == 0 ? stash + b * SEL_MAX : sel_out + ovf_start[st - 1];
        for (int r = threadIdx.x; r < S; r += blockDim.x) dia_off[base + r] = src[r];
    }
}

// ---------------------------------------------------------------------------
// 3./4. per-row remainder count and fill (generic over M-HDC / HDC)

template <class RP>
__global__ void rest_count_kernel(RowPtr<RP> rp, const int32_t* col, int64_t n_rows, int64_t row0,
                                  int64_t bl, const int32_t* dia_ptr, const int32_t* dia_off,
                                  const int32_t* blk_rest, int32_t* rest_cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / bl;
        // every entry of the block lies on a selected offset (known from the census):
        // no column is read
        if (blk_rest && blk_rest[b] == 0) {
            rest_cnt[i] = 0;
            continue;
        }
        const int32_t base = dia_ptr[b];
        const int32_t S = dia_ptr[b + 1] - base;
        const int32_t* sel = dia_off + base;
        const int64_t gi = row0 + i, ke = rp[i + 1];
        int32_t cnt = 0;
        for (int64_t k = rp[i]; k < ke; ++k) {
            const int32_t off = (int32_t)((int64_t)col[k] - gi);
            int lo = 0, hi = S;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sel[mid] < off) lo = mid + 1; else hi = mid;
            }
            cnt += !(lo < S && sel[lo] == off);
        }
        rest_cnt[i] = cnt;
    }
}

template <class RP>
__global__ void fill_kernel(RowPtr<RP> rp, const int32_t* col, const double* val, int64_t n_rows,
                            int64_t row0, int64_t bl, int64_t n_blocks, const int32_t* dia_ptr,
                            const int32_t* dia_off, const int32_t* rest_rp, double* seg,
                            int32_t* rest_col, double* rest_val) {
    const int64_t total = n_blocks * bl;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = v / bl, l = v - b * bl;
        const int32_t base = dia_ptr[b];
        const int32_t S = dia_ptr[b + 1] - base;
        const int32_t* sel = dia_off + base;
        double* sp = seg + (int64_t)base * bl + l;
        if (v >= n_rows) {
            for (int r = 0; r < S; ++r) sp[(int64_t)r * bl] = 0.0;
            continue;
        }
        const int64_t gi = row0 + v;
        int64_t k = rp[v];
        const int64_t ke = rp[v + 1];
        int64_t w = rest_rp[v];
        int32_t off = k < ke ? (int32_t)((int64_t)col[k] - gi) : INT32_MAX;
        for (int r = 0; r < S; ++r) {
            const int32_t s = sel[r];
            while (k < ke && off < s) {
                rest_col[w] = col[k];
                rest_val[w] = val[k];
                ++w;
                ++k;
                off = k < ke ? (int32_t)((int64_t)col[k] - gi) : INT32_MAX;
            }
            double out = 0.0;
            if (k < ke && off == s) {
                out = val[k];
                ++k;
                off = k < ke ? (int32_t)((int64_t)col[k] - gi) : INT32_MAX;
            }
            sp[(int64_t)r * bl] = out;
        }
        for (; k < ke; ++k, ++w) {
            rest_col[w] = col[k];
            rest_val[w] = val[k];
        }
    }
}

// ---------------------------------------------------------------------------
// HDC census: dense histogram over offsets [-(n-1), n-1]

template <class RP>
__global__ void hist_kernel(RowPtr<RP> rp, const int32_t* col, int64_t n, int32_t* hist) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ke = rp[i + 1];
        for (int64_t k = rp[i]; k < ke; ++k) {
            const int64_t idx = (int64_t)col[k] - i + (n - 1);
            const unsigned peers = __match_any_sync(__activemask(), (unsigned long long)idx);
            if (lane == __ffs(peers) - 1) atomicAdd(&hist[idx], __popc(peers));
        }
    }
}

struct SelectPred {
    const int32_t* hist;
    int64_t n;
    double theta;
    int census;  // 1: every populated offset
    __device__ __forceinline__ bool operator()(const int64_t& j) const {
        const int32_t c = hist[j];
        if (c <= 0) return false;
        return census ? true : ((double)c / (double)n >= theta);
    }
};

__global__ void hist_emit_kernel(const int64_t* idx, const int32_t* n_sel, const int32_t* hist,
                                 int64_t n, int32_t* offs, int64_t* counts) {
    const int S = *n_sel;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < S; r += gridDim.x * blockDim.x) {
        const int64_t j = idx[r];
        offs[r] = (int32_t)(j - (n - 1));
        if (counts) counts[r] = hist[j];
    }
}

// ---------------------------------------------------------------------------
// scans (CUB, stream-ordered temporaries)

template <class In, class Out>
static void exclusive_scan(In in, Out out, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    size_t bytes = 0;
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, count, st));
    dev_free(tmp, st);
}

template <class T>
static T read_scalar(const T* p, cudaStream_t st) {
    T v;
    HDCG_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    return v;
}

struct I64Widen {
    __host__ __device__ __forceinline__ int64_t operator()(const int32_t& v) const { return v; }
};

static int64_t sum_i32_as_i64(const int32_t* d, int64_t count, cudaStream_t st) {
    if (count <= 0) return 0;
    int64_t* out = dev_alloc<int64_t>(1, st);
    auto it = thrust::make_transform_iterator(d, I64Widen());
    size_t bytes = 0;
    HDCG_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, it, out, count, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceReduce::Sum(tmp, bytes, it, out, count, st));
    const int64_t v = read_scalar(out, st);
    dev_free(tmp, st);
    dev_free(out, st);
    return v;
}

// Offsets selected per block, for either the blocked (M-HDC) or global path.
struct Selection {
    int32_t* dia_ptr = nullptr;  // [n_blocks+1]
    int32_t* dia_off = nullptr;  // [n_seg]
    int64_t n_seg = 0;
    int32_t* blk_rest = nullptr;  // [n_blocks] unselected entries per block (-1 unknown), or null
    bool no_rest = false;         // the census found every entry on a selected offset
};

// General-path machinery shared by to_mhdc (overflow blocks) and census export.
template <class RP>
struct OvfRun {
    int n_ovf = 0;
    int64_t* start = nullptr;   // [n_ovf+1]
    int32_t* sorted = nullptr;  // [E]
    int32_t* out = nullptr;     // [E]
    int64_t* cnt = nullptr;     // [E] (census mode)
    int64_t total = 0;

    void run(const CsrInput& in, int64_t bl, const int32_t* ovf_list, int n, double theta,
             int mode, int32_t* sel_count, cudaStream_t st) {
        n_ovf = n;
        RowPtr<RP> rp{(const RP*)in.row_ptr};
        start = dev_alloc<int64_t>(n_ovf + 1, st);
        int64_t* sizes = dev_alloc<int64_t>(n_ovf + 1, st);
        HDCG_CUDA(cudaMemsetAsync(sizes, 0, sizeof(int64_t) * (n_ovf + 1), st));
        ovf_sizes_kernel<RP><<<grid_cap(ceil_div(n_ovf, 256)), 256, 0, st>>>(rp, in.n_rows, bl,
                                                                             ovf_list, n_ovf, sizes);
        HDCG_LAUNCH_CHECK("ovf_sizes_kernel");
        exclusive_scan(sizes, start, n_ovf + 1, st);
        dev_free(sizes, st);
        total = read_scalar(start + n_ovf, st);
        if (total > 0x7fffffffLL)
            fail(HDCG_ERR_OVERFLOW, "census: more than 2^31-1 entries in irregular blocks");
        int32_t* keys = dev_alloc<int32_t>(total, st);
        sorted = dev_alloc<int32_t>(total, st);
        out = dev_alloc<int32_t>(total, st);
        if (mode == 1) cnt = dev_alloc<int64_t>(total, st);
        ovf_gather_kernel<RP><<<n_ovf, 256, 0, st>>>(rp, in.col, in.n_rows, in.row0, bl, ovf_list,
                                                     start, keys);
        HDCG_LAUNCH_CHECK("ovf_gather_kernel");
        if (total > 0) {
            size_t bytes = 0;
            HDCG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, keys, sorted, (int)total,
                                                         n_ovf, start, start + 1, st));
            void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
            HDCG_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, keys, sorted, (int)total, n_ovf,
                                                         start, start + 1, st));
            dev_free(tmp, st);
        }
        dev_free(keys, st);
        if (mode == 0)
            ovf_rle_kernel<0><<<n_ovf, 256, 0, st>>>(sorted, start, ovf_list, in.n_rows, bl, theta,
                                                     out, nullptr, sel_count);
        else
            ovf_rle_kernel<1><<<n_ovf, 256, 0, st>>>(sorted, start, ovf_list, in.n_rows, bl, theta,
                                                     out, cnt, sel_count);
        HDCG_LAUNCH_CHECK("ovf_rle_kernel");
    }
    void release(cudaStream_t st) {
        dev_free(start, st);
        dev_free(sorted, st);
        dev_free(out, st);
        dev_free(cnt, st);
        start = nullptr;
        sorted = out = nullptr;
        cnt = nullptr;
    }
};

template <class RP>
static Selection select_blocked(const CsrInput& in, double theta, int64_t bl, int64_t n_blocks,
                                cudaStream_t st) {
    Selection s;
    BuildTrace tr(st);
    RowPtr<RP> rp{(const RP*)in.row_ptr};
    int32_t* sel_count = dev_alloc<int32_t>(n_blocks + 1, st);
    int32_t* stash = dev_alloc<int32_t>(n_blocks * SEL_MAX, st);
    int32_t* blk_status = dev_alloc<int32_t>(n_blocks, st);
    int32_t* ovf_list = dev_alloc<int32_t>(n_blocks, st);
    int32_t* ovf_count = dev_alloc<int32_t>(2, st);  // [overflowed blocks, any block with a remainder]
    HDCG_CUDA(cudaMemsetAsync(ovf_count, 0, 2 * sizeof(int32_t), st));
    HDCG_CUDA(cudaMemsetAsync(sel_count + n_blocks, 0, sizeof(int32_t), st));
    s.blk_rest = dev_alloc<int32_t>(n_blocks, st);
    // one thread per row for blocks narrower than the CTA
    const int threads = (int)std::min<int64_t>(CENSUS_THREADS, std::max<int64_t>(64, (bl + 31) / 32 * 32));
    // HDCG_CENSUS_FILTER=0: overflowing blocks go straight to the sort path (A/B knob)
    const char* ef = getenv("HDCG_CENSUS_FILTER");
    const int bucket_filter = !ef || atoi(ef) != 0;
    census_select_kernel<RP><<<grid_cap(n_blocks), threads, 0, st>>>(
        rp, in.col, in.n_rows, in.row0, bl, n_blocks, theta, sel_count, stash, blk_status, ovf_list,
        ovf_count, s.blk_rest, bucket_filter);
    HDCG_LAUNCH_CHECK("census_select_kernel");
    int32_t flags[2] = {0, 0};
    HDCG_CUDA(cudaMemcpyAsync(flags, ovf_count, sizeof(flags), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    const int n_ovf = flags[0];
    s.no_rest = flags[1] == 0;
    tr.mark("census + select");
    OvfRun<RP> ovf;
    if (n_ovf > 0) {
        // deterministic order of the irregular blocks
        int32_t* sorted_list = dev_alloc<int32_t>(n_ovf, st);
        size_t bytes = 0;
        HDCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, ovf_list, sorted_list, n_ovf, 0, 32, st));
        void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
        HDCG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, ovf_list, sorted_list, n_ovf, 0, 32, st));
        dev_free(tmp, st);
        HDCG_CUDA(cudaMemcpyAsync(ovf_list, sorted_list, sizeof(int32_t) * n_ovf,
                                  cudaMemcpyDeviceToDevice, st));
        dev_free(sorted_list, st);
        ovf.run(in, bl, ovf_list, n_ovf, theta, 0, sel_count, st);
        ovf_index_kernel<<<grid_cap(ceil_div(n_ovf, 256)), 256, 0, st>>>(ovf_list, n_ovf, blk_status);
        HDCG_LAUNCH_CHECK("ovf_index_kernel");
    }
    s.dia_ptr = dev_alloc<int32_t>(n_blocks + 1, st);
    // n_seg must fit index_t: widen before scanning
    const int64_t n_seg = sum_i32_as_i64(sel_count, n_blocks, st);
    if (n_seg > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "to_mhdc: segment count exceeds index range");
    exclusive_scan(sel_count, s.dia_ptr, n_blocks + 1, st);
    s.n_seg = n_seg;
    s.dia_off = dev_alloc<int32_t>(n_seg, st);
    if (n_seg > 0) {
        write_offsets_kernel<<<grid_cap(n_blocks), 32, 0, st>>>(n_blocks, s.dia_ptr, blk_status, stash,
                                                                ovf.out, ovf.start, s.dia_off);
        HDCG_LAUNCH_CHECK("write_offsets_kernel");
    }
    tr.mark("overflow blocks, offsets");
    ovf.release(st);
    dev_free(sel_count, st);
    dev_free(stash, st);
    dev_free(blk_status, st);
    dev_free(ovf_list, st);
    dev_free(ovf_count, st);
    return s;
}

template <class RP>
static Selection select_global(const CsrInput& in, double theta, bool census_mode, int64_t** counts_out,
                               cudaStream_t st) {
    Selection s;
    const int64_t n = in.n_rows;
    RowPtr<RP> rp{(const RP*)in.row_ptr};
    const int64_t H = 2 * n - 1;
    int32_t* hist = dev_alloc<int32_t>(H, st);
    HDCG_CUDA(cudaMemsetAsync(hist, 0, sizeof(int32_t) * H, st));
    hist_kernel<RP><<<grid_cap(ceil_div(n, 256)), 256, 0, st>>>(rp, in.col, n, hist);
    HDCG_LAUNCH_CHECK("hist_kernel");
    int64_t* idx = dev_alloc<int64_t>(H, st);
    int32_t* n_sel = dev_alloc<int32_t>(1, st);
    SelectPred pred{hist, n, theta, census_mode ? 1 : 0};
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    HDCG_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, idx, n_sel, H, pred, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceSelect::If(tmp, bytes, it, idx, n_sel, H, pred, st));
    dev_free(tmp, st);
    const int32_t S = read_scalar(n_sel, st);
    s.n_seg = S;
    s.dia_off = dev_alloc<int32_t>(S, st);
    int64_t* counts = nullptr;
    if (census_mode && S > 0) counts = dev_alloc<int64_t>(S, st);
    if (S > 0) {
        hist_emit_kernel<<<grid_cap(ceil_div(S, 256)), 256, 0, st>>>(idx, n_sel, hist, n, s.dia_off,
                                                                     counts);
        HDCG_LAUNCH_CHECK("hist_emit_kernel");
    }
    if (counts_out) *counts_out = counts;
    s.dia_ptr = dev_alloc<int32_t>(2, st);
    const int32_t dp[2] = {0, S};
    HDCG_CUDA(cudaMemcpyAsync(s.dia_ptr, dp, sizeof(dp), cudaMemcpyHostToDevice, st));
    HDCG_CUDA(cudaStreamSynchronize(st));  // dp is a stack array
    dev_free(idx, st);
    dev_free(n_sel, st);
    dev_free(hist, st);
    return s;
}

// Remainder + segments from a finished selection (steps 3 and 4).
template <class RP>
static void finish_build(const CsrInput& in, int64_t bl, int64_t n_blocks, Selection sel, Matrix* m,
                         cudaStream_t st) {
    RowPtr<RP> rp{(const RP*)in.row_ptr};
    BuildTrace tr(st);
    m->n_rows = in.n_rows;
    m->n_cols = in.n_cols;
    m->row0 = in.row0;
    m->bl = bl;
    m->n_blocks = n_blocks;
    m->n_seg = sel.n_seg;
    m->nnz_input = in.nnz;
    m->dia_ptr = sel.dia_ptr;
    m->dia_off = sel.dia_off;
    // remainder row pointers: per-row counts written into rest_rp and scanned in place
    // (no second n-row array); a matrix whose census left nothing for the remainder
    // (every stencil configuration) just gets zeros
    m->rest_rp = dev_alloc<int32_t>(in.n_rows + 1, st);
    // HDCG_CONVERT_SKIP=0: count every row's remainder from its columns (A/B knob)
    const char* es = getenv("HDCG_CONVERT_SKIP");
    const bool skip = !es || atoi(es) != 0;
    if (skip && sel.no_rest) {
        HDCG_CUDA(cudaMemsetAsync(m->rest_rp, 0, sizeof(int32_t) * (in.n_rows + 1), st));
    } else {
        int32_t* rest_cnt = m->rest_rp;
        HDCG_CUDA(cudaMemsetAsync(rest_cnt + in.n_rows, 0, sizeof(int32_t), st));
        if (in.n_rows > 0) {
            rest_count_kernel<RP><<<grid_cap(ceil_div(in.n_rows, 256)), 256, 0, st>>>(
                rp, in.col, in.n_rows, in.row0, bl, m->dia_ptr, m->dia_off, skip ? sel.blk_rest : nullptr, rest_cnt);
            HDCG_LAUNCH_CHECK("rest_count_kernel");
        }
        const int64_t nnz_rest = in.nnz <= 0x7fffffffLL ? -1 : sum_i32_as_i64(rest_cnt, in.n_rows, st);
        if (nnz_rest > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "remainder nnz exceeds index range");
        exclusive_scan(rest_cnt, m->rest_rp, in.n_rows + 1, st);  // in place
    }
    dev_free(sel.blk_rest, st);
    m->nnz_rest = read_scalar(m->rest_rp + in.n_rows, st);
    tr.mark("remainder counts + scan");
    alloc_rest(m, m->nnz_rest, st);
    if (sel.n_seg > 0 && (int64_t)sel.n_seg * bl > (int64_t)1 << 40)
        fail(HDCG_ERR_OUT_OF_MEMORY, "segments too large");
    m->seg = alloc_seg(sel.n_seg * bl, st);
    tr.mark("allocate segments");
    const int64_t total = n_blocks * bl;
    if (total > 0) {
        fill_kernel<RP><<<grid_cap(ceil_div(total, 256)), 256, 0, st>>>(
            rp, in.col, in.val, in.n_rows, in.row0, bl, n_blocks, m->dia_ptr, m->dia_off, m->rest_rp,
            m->seg, m->rest_col, m->rest_val);
        HDCG_LAUNCH_CHECK("fill_kernel");
    }
    // dia_slots with the true (last-block) lengths, convert.cpp:190-194
    std::vector<int32_t> dp((size_t)n_blocks + 1);
    HDCG_CUDA(cudaMemcpyAsync(dp.data(), m->dia_ptr, sizeof(int32_t) * (n_blocks + 1),
                              cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    int64_t slots = 0, mx = 0;
    for (int64_t b = 0; b < n_blocks; ++b) {
        slots += (int64_t)(dp[b + 1] - dp[b]) * std::min(bl, in.n_rows - b * bl);
        mx = std::max<int64_t>(mx, dp[b + 1] - dp[b]);
    }
    m->dia_slots = slots;
    m->max_seg_per_block = mx;
    tr.mark("fill + slot count");
}

static void check_slab(const CsrInput& in, int64_t bl) {
    if (in.n_rows < 0 || in.n_cols < 0) fail(HDCG_ERR_INVALID_ARGUMENT, "negative dimension");
    if (in.row0 < 0 || in.row0 + in.n_rows > in.n_cols)
        fail(HDCG_ERR_INVALID_ARGUMENT, "row slab outside the matrix");
    if (in.row0 % bl != 0) fail(HDCG_ERR_INVALID_ARGUMENT, "row slab must start at a multiple of bl");
    if (in.row0 + in.n_rows != in.n_cols && in.n_rows % bl != 0)
        fail(HDCG_ERR_INVALID_ARGUMENT, "row slab must end at n or at a multiple of bl");
    if (in.n_cols > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "n exceeds the int32 index range");
}

void build_mhdc(const CsrInput& in, double theta, int64_t bl, Matrix* m, cudaStream_t st) {
    if (!(theta >= 0.0 && theta <= 1.0)) fail(HDCG_ERR_INVALID_ARGUMENT, "to_mhdc: theta must be in [0, 1]");
    if (bl < 1) fail(HDCG_ERR_INVALID_ARGUMENT, "to_mhdc: block width must be >= 1");
    check_slab(in, bl);
    const int64_t nb = n_blocks_of(in.n_rows, bl);
    m->kind = HDCG_KIND_MHDC;
    if (in.rp64) {
        Selection s = select_blocked<int64_t>(in, theta, bl, nb, st);
        finish_build<int64_t>(in, bl, nb, s, m, st);
    } else {
        Selection s = select_blocked<int32_t>(in, theta, bl, nb, st);
        finish_build<int32_t>(in, bl, nb, s, m, st);
    }
    build_packed(m, st);  // small blocks: the tile-packed copy the SpMV streams
}

void build_hdc(const CsrInput& in, double theta, Matrix* m, cudaStream_t st) {
    if (!(theta >= 0.0 && theta <= 1.0)) fail(HDCG_ERR_INVALID_ARGUMENT, "to_hdc: theta must be in [0, 1]");
    if (in.row0 != 0 || in.n_rows != in.n_cols)
        fail(HDCG_ERR_INVALID_ARGUMENT, "to_hdc: HDC is built from the whole matrix");
    if (in.n_cols > 0x3fffffffLL) fail(HDCG_ERR_OVERFLOW, "to_hdc: n exceeds the histogram index range");
    m->kind = HDCG_KIND_HDC;
    const int64_t n = in.n_rows;
    const int64_t bl = n > 0 ? n : 1;
    const int64_t nb = n_blocks_of(n, bl);
    Selection s;
    if (n == 0) {
        s.dia_ptr = dev_alloc<int32_t>(1, st);
        HDCG_CUDA(cudaMemsetAsync(s.dia_ptr, 0, sizeof(int32_t), st));
    } else if (in.rp64) {
        s = select_global<int64_t>(in, theta, false, nullptr, st);
    } else {
        s = select_global<int32_t>(in, theta, false, nullptr, st);
    }
    if (in.rp64) finish_build<int64_t>(in, bl, nb, s, m, st);
    else finish_build<int32_t>(in, bl, nb, s, m, st);
}

template <class RP>
__global__ void copy_rowptr_kernel(RowPtr<RP> rp, int64_t count, int32_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)rp[i];
}

void build_csr(const CsrInput& in, Matrix* m, cudaStream_t st) {
    if (in.nnz > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "CSR nnz exceeds the int32 index range");
    m->kind = HDCG_KIND_CSR;
    m->n_rows = in.n_rows;
    m->n_cols = in.n_cols;
    m->row0 = in.row0;
    m->bl = in.n_rows > 0 ? in.n_rows : 1;
    m->n_blocks = n_blocks_of(in.n_rows, m->bl);
    m->n_seg = 0;
    m->nnz_input = in.nnz;
    m->nnz_rest = in.nnz;
    m->dia_slots = 0;
    m->dia_ptr = dev_alloc<int32_t>(m->n_blocks + 1, st);
    HDCG_CUDA(cudaMemsetAsync(m->dia_ptr, 0, sizeof(int32_t) * (m->n_blocks + 1), st));
    m->rest_rp = dev_alloc<int32_t>(in.n_rows + 1, st);
    if (in.rp64)
        copy_rowptr_kernel<int64_t><<<grid_cap(ceil_div(in.n_rows + 1, 256)), 256, 0, st>>>(
            RowPtr<int64_t>{(const int64_t*)in.row_ptr}, in.n_rows + 1, m->rest_rp);
    else
        HDCG_CUDA(cudaMemcpyAsync(m->rest_rp, in.row_ptr, sizeof(int32_t) * (in.n_rows + 1),
                                  cudaMemcpyDeviceToDevice, st));
    alloc_rest(m, in.nnz, st);
    if (in.nnz > 0) {
        HDCG_CUDA(cudaMemcpyAsync(m->rest_col, in.col, sizeof(int32_t) * in.nnz, cudaMemcpyDeviceToDevice, st));
        HDCG_CUDA(cudaMemcpyAsync(m->rest_val, in.val, sizeof(double) * in.nnz, cudaMemcpyDeviceToDevice, st));
    }
}

// ---------------------------------------------------------------------------
// census export (convert.cpp:39-67): global = histogram, blocked = general path for all blocks

__global__ void iota_kernel(int32_t* out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

template <class RP>
static int64_t census_t(const CsrInput& in, int64_t bl, int64_t* bp_host, int32_t* off_host,
                        int64_t* cnt_host, cudaStream_t st) {
    const int64_t n = in.n_rows;
    if (bl <= 0) {  // global census: one block of width n (empty matrix: no blocks)
        if (n == 0) { if (bp_host) bp_host[0] = 0; return 0; }
        int64_t* counts = nullptr;
        Selection s = select_global<RP>(in, 0.0, true, &counts, st);
        if (bp_host) { bp_host[0] = 0; bp_host[1] = s.n_seg; }
        if (off_host && s.n_seg > 0) {
            HDCG_CUDA(cudaMemcpyAsync(off_host, s.dia_off, sizeof(int32_t) * s.n_seg, cudaMemcpyDeviceToHost, st));
            HDCG_CUDA(cudaMemcpyAsync(cnt_host, counts, sizeof(int64_t) * s.n_seg, cudaMemcpyDeviceToHost, st));
        }
        HDCG_CUDA(cudaStreamSynchronize(st));
        dev_free(counts, st);
        dev_free(s.dia_off, st);
        dev_free(s.dia_ptr, st);
        return s.n_seg;
    }
    const int64_t nb = n_blocks_of(n, bl);
    if (nb == 0) { if (bp_host) bp_host[0] = 0; return 0; }
    if (nb > 0x7fffffffLL) fail(HDCG_ERR_OVERFLOW, "census: too many blocks");
    int32_t* list = dev_alloc<int32_t>(nb, st);
    iota_kernel<<<grid_cap(ceil_div(nb, 256)), 256, 0, st>>>(list, nb);
    int32_t* per_block = dev_alloc<int32_t>(nb + 1, st);
    HDCG_CUDA(cudaMemsetAsync(per_block, 0, sizeof(int32_t) * (nb + 1), st));
    OvfRun<RP> ovf;
    ovf.run(in, bl, list, (int)nb, 0.0, 1, per_block, st);
    int64_t* bp = dev_alloc<int64_t>(nb + 1, st);
    auto it = thrust::make_transform_iterator((const int32_t*)per_block, I64Widen());
    exclusive_scan(it, bp, nb + 1, st);
    const int64_t total = read_scalar(bp + nb, st);
    if (bp_host)
        HDCG_CUDA(cudaMemcpyAsync(bp_host, bp, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost, st));
    if (off_host && total > 0) {
        // compact: block j's entries sit at ovf.start[j] .. + per_block[j]
        std::vector<int64_t> start((size_t)nb + 1), bph((size_t)nb + 1);
        HDCG_CUDA(cudaMemcpyAsync(start.data(), ovf.start, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost, st));
        HDCG_CUDA(cudaMemcpyAsync(bph.data(), bp, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost, st));
        HDCG_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> o((size_t)ovf.total);
        std::vector<int64_t> c((size_t)ovf.total);
        if (ovf.total > 0) {
            HDCG_CUDA(cudaMemcpyAsync(o.data(), ovf.out, sizeof(int32_t) * ovf.total, cudaMemcpyDeviceToHost, st));
            HDCG_CUDA(cudaMemcpyAsync(c.data(), ovf.cnt, sizeof(int64_t) * ovf.total, cudaMemcpyDeviceToHost, st));
        }
        HDCG_CUDA(cudaStreamSynchronize(st));
        for (int64_t b = 0; b < nb; ++b)
            for (int64_t r = 0; r < bph[b + 1] - bph[b]; ++r) {
                off_host[bph[b] + r] = o[start[b] + r];
                cnt_host[bph[b] + r] = c[start[b] + r];
            }
    }
    HDCG_CUDA(cudaStreamSynchronize(st));
    ovf.release(st);
    dev_free(bp, st);
    dev_free(per_block, st);
    dev_free(list, st);
    return total;
}

int64_t census(const CsrInput& in, int64_t bl, int64_t* bp, int32_t* off, int64_t* cnt, cudaStream_t st) {
    if (in.rp64) return census_t<int64_t>(in, bl, bp, off, cnt, st);
    return census_t<int32_t>(in, bl, bp, off, cnt, st);
}

// ---------------------------------------------------------------------------
// rates (convert.cpp:173-196): alpha = nonzero segment values / dia_slots

__global__ void count_nonzero_kernel(const double* v, int64_t count, unsigned long long* out) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        c += v[i] != 0.0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

void rates(const Matrix& m, double* alpha, double* beta, int64_t* slots, cudaStream_t st) {
    int64_t dia_nnz = 0;
    const int64_t n_vals = m.n_seg * m.bl;
    if (n_vals > 0) {
        unsigned long long* d = dev_alloc<unsigned long long>(1, st);
        HDCG_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), st));
        count_nonzero_kernel<<<grid_cap(ceil_div(n_vals, 256)), 256, 0, st>>>(m.seg, n_vals, d);
        HDCG_LAUNCH_CHECK("count_nonzero_kernel");
        dia_nnz = (int64_t)read_scalar(d, st);
        dev_free(d, st);
    }
    const int64_t total = dia_nnz + m.nnz_rest;
    if (total == 0) fail(HDCG_ERR_INVALID_ARGUMENT, "rates: matrix has no nonzeros");
    *beta = (double)m.nnz_rest / (double)total;
    *alpha = m.dia_slots == 0 ? 1.0 : (double)dia_nnz / (double)m.dia_slots;
    *slots = m.dia_slots;
}

cudaError_t cub_exclusive_sum_i64(void* tmp, size_t& bytes, const int64_t* in, int64_t* out,
                                  int64_t count, cudaStream_t st) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, count, st);
}

}  // namespace hdcg

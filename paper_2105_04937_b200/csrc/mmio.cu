// mmio.cu -- Matrix Market ingestion for the device path.
//
// Replaces hdc::io::read_matrix_market (proj/src/io.cpp:69-121) followed by
// CooMatrix normalisation (formats.cpp:19-43) and CsrMatrix::from_coo
// (formats.cpp:69-88), the step in front of the converters for real inputs:
//
//   host   : the file is read once (fread) and cut at line boundaries into one
//            piece per host thread, each piece's lines parsed into (row*n+col)
//            keys and values by its thread (std::from_chars: correctly rounded
//            like the reference's `iss >> v`), pieces copied to the device in
//            file order; the banner,
//            size line, entry count, bounds, trailing tokens / content and the
//            symmetric / skew-symmetric mirroring follow io.cpp exactly, with
//            the same messages (runtime_error -> HDCG_ERR_IO);
//   device : stable radix sort of (row*n + col) keys carrying the values (the
//            reference's stable_sort), duplicate runs summed left to right in
//            stored order by one thread each (bitwise the reference's in-place
//            loop), compaction, and row_ptr by counting + scan.
#include <cub/cub.cuh>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "hdcg_internal.cuh"

namespace hdcg {

namespace {

[[noreturn]] void bad_file(const std::string& what) { fail(HDCG_ERR_IO, "matrix market: " + what); }

std::string lower(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return (char)std::tolower(c); });
    return s;
}

bool is_blank(const char* b, const char* e) {
    for (; b < e; ++b)
        if (!std::isspace((unsigned char)*b)) return false;
    return true;
}

struct Line {
    const char* b;
    const char* e;
};

// whitespace-separated tokens of [b, e)
int tokens(const char* b, const char* e, Line* out, int max) {
    int n = 0;
    while (b < e) {
        while (b < e && std::isspace((unsigned char)*b)) ++b;
        if (b >= e) break;
        const char* s = b;
        while (b < e && !std::isspace((unsigned char)*b)) ++b;
        if (n < max) out[n] = Line{s, b};
        ++n;
    }
    return n;
}

std::string str(Line l) { return std::string(l.b, l.e); }

template <class T>
bool parse_num(Line t, T* v) {
    // std::from_chars does not accept a leading '+', istream extraction does
    const char* b = t.b;
    if (b < t.e && *b == '+') ++b;
    auto r = std::from_chars(b, t.e, *v);
    return r.ec == std::errc() && r.ptr == t.e;
}

enum Field { REAL, INTEGER, PATTERN };
enum Symmetry { GENERAL, SYMMETRIC, SKEW };

}  // namespace

// Parse + normalise; fills a device CSR (int32 row_ptr / col, f64 values).
void read_matrix_market(const char* path, Matrix* m) {
    std::string buf;
    {
        FILE* fp = std::fopen(path, "rb");
        if (!fp) fail(HDCG_ERR_IO, std::string("cannot open '") + path + "' for reading");
        std::fseek(fp, 0, SEEK_END);
        const long size = std::ftell(fp);
        std::fseek(fp, 0, SEEK_SET);
        buf.resize(size > 0 ? (size_t)size : 0);
        const size_t got = buf.empty() ? 0 : std::fread(&buf[0], 1, buf.size(), fp);
        std::fclose(fp);
        if (got != buf.size()) fail(HDCG_ERR_IO, std::string("cannot read '") + path + "'");
    }
    const char* p = buf.data();
    const char* end = p + buf.size();
    auto next_nonblank = [&](const char*& q, Line* line) {
        while (q < end) {
            const char* e = (const char*)memchr(q, '\n', end - q);
            if (!e) e = end;
            Line l{q, e};
            q = e < end ? e + 1 : end;
            if (!is_blank(l.b, l.e)) {
                *line = l;
                return true;
            }
        }
        return false;
    };
    Line line;
    if (!next_nonblank(p, &line)) bad_file("empty input");
    Line tk[8];
    const int nt = tokens(line.b, line.e, tk, 8);
    auto tok = [&](int i) { return i < nt ? str(tk[i]) : std::string(); };
    if (lower(tok(0)) != "%%matrixmarket") bad_file("missing %%MatrixMarket banner");
    if (lower(tok(1)) != "matrix") bad_file("unsupported object '" + tok(1) + "'");
    if (lower(tok(2)) != "coordinate") bad_file("unsupported format '" + tok(2) + "'");
    Field field;
    const std::string fs = lower(tok(3));
    if (fs == "real") field = REAL;
    else if (fs == "integer") field = INTEGER;
    else if (fs == "pattern") field = PATTERN;
    else bad_file("unsupported field '" + tok(3) + "'");
    Symmetry sym;
    const std::string ss = lower(tok(4));
    if (ss == "general") sym = GENERAL;
    else if (ss == "symmetric") sym = SYMMETRIC;
    else if (ss == "skew-symmetric") sym = SKEW;
    else bad_file("unsupported symmetry '" + tok(4) + "'");
    (void)field;

    // size line (comment lines start with '%' after leading blanks)
    do {
        if (!next_nonblank(p, &line)) bad_file("missing size line");
    } while (*std::find_if(line.b, line.e, [](char c) { return c != ' ' && c != '\t' && c != '\r'; }) == '%');
    long long rows = 0, cols = 0, declared = 0;
    {
        const int k = tokens(line.b, line.e, tk, 8);
        if (k < 3 || !parse_num(tk[0], &rows) || !parse_num(tk[1], &cols) || !parse_num(tk[2], &declared))
            bad_file("malformed size line '" + str(line) + "'");
        if (k > 3) bad_file("trailing tokens on size line");
        if (rows < 0 || cols < 0 || declared < 0) bad_file("negative size");
        if (rows != cols)
            bad_file("matrix is " + std::to_string(rows) + " x " + std::to_string(cols) +
                     ", only square matrices are supported");
        if (rows > std::numeric_limits<int32_t>::max()) bad_file("dimension exceeds index range");
    }
    const int64_t n = rows;

    // Entry lines: the rest of the file is cut at line boundaries into one piece
    // per host thread; each thread counts its non-blank lines and parses them into
    // (row*n + col) keys and values (mirrored entries right after their source, as
    // io.cpp pushes them), keeping its first error and that line's local index.
    // Afterwards the pieces are ordered by file position: the first error on a
    // line the reference would read (global index < declared) is reported, then
    // the entry-count checks -- the reference's messages and precedence.
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const int64_t body = end - p;
    const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(hw, body / (1 << 20) + 1));
    std::vector<const char*> cut((size_t)chunks + 1);
    cut[0] = p;
    cut[(size_t)chunks] = end;
    for (int64_t ci = 1; ci < chunks; ++ci) {
        const char* q = p + body * ci / chunks;
        const char* e = (const char*)memchr(q, '\n', end - q);
        cut[(size_t)ci] = std::max(cut[(size_t)ci - 1], e ? e + 1 : end);
    }
    struct Piece {
        std::vector<int64_t> key;
        std::vector<double> val;
        std::string err;
        int64_t err_line = -1;  // local index of the line with err
        int64_t lines = 0;      // non-blank lines in the piece
    };
    std::vector<Piece> parts((size_t)chunks);
    auto work = [&](int64_t ci) {
        Piece& P = parts[(size_t)ci];
        const char* q = cut[(size_t)ci];
        const char* qe = cut[(size_t)ci + 1];
        P.key.reserve((size_t)((qe - q) / 12 + 16) * (sym == GENERAL ? 1 : 2));
        P.val.reserve(P.key.capacity());
        Line t[4];
        while (q < qe) {
            const char* e = (const char*)memchr(q, '\n', qe - q);
            if (!e) e = qe;
            const Line L{q, e};
            q = e < qe ? e + 1 : qe;
            if (is_blank(L.b, L.e)) continue;
            const int64_t idx = P.lines++;
            if (P.err_line >= 0) continue;  // keep counting lines only
            const int nt = tokens(L.b, L.e, t, 4);
            long long i = 0, j = 0;
            double v = 1.0;
            std::string err;
            if (nt < 2 || !parse_num(t[0], &i) || !parse_num(t[1], &j))
                err = "malformed entry line '" + str(L) + "'";
            else if (field != PATTERN && (nt < 3 || !parse_num(t[2], &v)))
                err = "missing value on entry line '" + str(L) + "'";
            else if (nt > (field == PATTERN ? 2 : 3))
                err = "trailing tokens on entry line '" + str(L) + "'";
            else if (i < 1 || i > rows || j < 1 || j > cols)
                err = "entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside declared size";
            if (!err.empty()) {
                P.err = err;
                P.err_line = idx;
                continue;
            }
            P.key.push_back((int64_t)(i - 1) * n + (j - 1));
            P.val.push_back(v);
            if (i != j && sym != GENERAL) {
                P.key.push_back((int64_t)(j - 1) * n + (i - 1));
                P.val.push_back(sym == SKEW ? -v : v);
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int64_t ci = 1; ci < chunks; ++ci) th.emplace_back(work, ci);
        work(0);
        for (auto& t : th) t.join();
    }
    int64_t n_lines = 0;
    for (const Piece& P : parts) {
        if (P.err_line >= 0 && n_lines + P.err_line < declared) bad_file(P.err);
        n_lines += P.lines;
    }
    if (n_lines < declared)
        bad_file("expected " + std::to_string(declared) + " entries, got " + std::to_string(n_lines));
    if (n_lines > declared) bad_file("trailing content after " + std::to_string(declared) + " entries");

    int64_t total = 0;
    for (const Piece& P : parts) total += (int64_t)P.key.size();
    if (total > std::numeric_limits<int32_t>::max())
        fail(HDCG_ERR_OVERFLOW, "CsrMatrix::from_coo: entry count exceeds index range");

    // ---- device: stable sort by (row, col), in-order duplicate sums, CSR ----
    cudaStream_t st = nullptr;
    int64_t* keys = dev_alloc<int64_t>(total, st);
    int64_t* skeys = dev_alloc<int64_t>(total, st);
    double* vals = dev_alloc<double>(total, st);
    double* svals = dev_alloc<double>(total, st);
    {
        int64_t w = 0;
        for (const Piece& P : parts) {
            const int64_t k = (int64_t)P.key.size();
            if (k > 0) {
                HDCG_CUDA(cudaMemcpyAsync(keys + w, P.key.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, st));
                HDCG_CUDA(cudaMemcpyAsync(vals + w, P.val.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
            }
            w += k;
        }
        HDCG_CUDA(cudaStreamSynchronize(st));
    }
    m->kind = HDCG_KIND_CSR;
    m->n_rows = m->n_cols = n;
    m->bl = n > 0 ? n : 1;
    m->n_blocks = n_blocks_of(n, m->bl);
    m->dia_ptr = dev_alloc<int32_t>(m->n_blocks + 1, st);
    HDCG_CUDA(cudaMemsetAsync(m->dia_ptr, 0, sizeof(int32_t) * (m->n_blocks + 1), st));
    m->rest_rp = dev_alloc<int32_t>(n + 1, st);
    int64_t nnz = 0;
    if (total > 0) {
        int end_bit = 1;
        while (end_bit < 63 && ((int64_t)1 << end_bit) < n * n) ++end_bit;
        size_t bytes = 0;
        HDCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, skeys, vals, svals, total, 0, end_bit, st));
        void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
        HDCG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, skeys, vals, svals, total, 0, end_bit, st));
        dev_free(tmp, st);
        nnz = coo_dedup_to_csr(skeys, svals, total, n, m, st);
    }
    if (total == 0) {
        HDCG_CUDA(cudaMemsetAsync(m->rest_rp, 0, sizeof(int32_t) * (n + 1), st));
        alloc_rest(m, 0, st);
    }
    m->nnz_rest = nnz;
    m->nnz_input = nnz;
    dev_free(keys, st);
    dev_free(skeys, st);
    dev_free(vals, st);
    dev_free(svals, st);
    HDCG_CUDA(cudaStreamSynchronize(st));
}

namespace {

__global__ void run_start_kernel(const int64_t* k, int64_t total, int32_t* start) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        start[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// one thread per run: sum the duplicates left to right (CooMatrix ctor, formats.cpp:32-41)
__global__ void run_sum_kernel(const int64_t* k, const double* v, const int32_t* start, const int32_t* pos,
                               int64_t total, int64_t n, int32_t* row_count, int32_t* col, double* val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        if (!start[i]) continue;
        double s = v[i];
        for (int64_t j = i + 1; j < total && !start[j]; ++j) s = __dadd_rn(s, v[j]);
        const int32_t w = pos[i];
        const int64_t row = k[i] / n;
        col[w] = (int32_t)(k[i] - row * n);
        val[w] = s;
        atomicAdd(&row_count[row], 1);
    }
}

}  // namespace

int64_t coo_dedup_to_csr(const int64_t* skeys, const double* svals, int64_t total, int64_t n, Matrix* m,
                         cudaStream_t st) {
    int32_t* start = dev_alloc<int32_t>(total + 1, st);
    int32_t* pos = dev_alloc<int32_t>(total + 1, st);
    HDCG_CUDA(cudaMemsetAsync(start + total, 0, sizeof(int32_t), st));
    run_start_kernel<<<grid_cap(ceil_div(total, 256)), 256, 0, st>>>(skeys, total, start);
    size_t bytes = 0;
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, start, pos, total + 1, st));
    void* tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, start, pos, total + 1, st));
    dev_free(tmp, st);
    int32_t nnz32 = 0;
    HDCG_CUDA(cudaMemcpyAsync(&nnz32, pos + total, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HDCG_CUDA(cudaStreamSynchronize(st));
    const int64_t nnz = nnz32;
    alloc_rest(m, nnz, st);
    int32_t* cnt = dev_alloc<int32_t>(n + 1, st);
    HDCG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 1), st));
    run_sum_kernel<<<grid_cap(ceil_div(total, 256)), 256, 0, st>>>(skeys, svals, start, pos, total, n, cnt,
                                                                   m->rest_col, m->rest_val);
    HDCG_LAUNCH_CHECK("run_sum_kernel");
    bytes = 0;
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, m->rest_rp, n + 1, st));
    tmp = dev_alloc<char>((int64_t)bytes + 1, st);
    HDCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, m->rest_rp, n + 1, st));
    dev_free(tmp, st);
    dev_free(cnt, st);
    dev_free(start, st);
    dev_free(pos, st);
    return nnz;
}

}  // namespace hdcg

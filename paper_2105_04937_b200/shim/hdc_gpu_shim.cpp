// hdc_gpu_shim.cpp -- drop-in GPU implementation of the reference's format-build
// and SpMV entry points, on top of the C-ABI in include/hdcgpu.h.
//
// A C++ program written against the reference (proj/include/hdc/convert.hpp
// and kernels.hpp) links this file INSTEAD OF proj/src/convert.cpp and
// proj/src/kernels.cpp, keeps the reference's formats.cpp (the containers),
// and links libhdcgpu.so.  Nothing else changes: same declarations, same
// value semantics, same exception types (std::invalid_argument /
// std::out_of_range / std::overflow_error), same synchronous behaviour
// (y is complete when the call returns).  `workers` is accepted and ignored:
// the GPU result is bitwise identical for every worker count, as the
// reference guarantees for its own (kernels.hpp:24-27).
//
// Entry points replaced (reference file:line):
//   DiagonalCensus::total, census_global, census_blocked   convert.cpp:32-67
//   to_dia, to_hdc, to_mhdc                                 convert.cpp:69-169
//   rates(HdcMatrix), rates(MHdcMatrix)                     convert.cpp:185-196
//   BlockPlan::rows                                         kernels.cpp:33-37
//   spmv_csr / dia / bdia / hdc / bhdc / mhdc (+ allocating) kernels.cpp:39-244
//
// Matrices are immutable after construction, so each one is
// uploaded at most once: a small LRU cache maps a host matrix (its array
// addresses and sizes, verified on every lookup by a hash of every byte of
// its arrays) to its device handle.  Formats
// produced by to_hdc / to_mhdc / to_dia are built on the device and
// registered under the returned object, so their SpMVs never re-upload.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <list>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hdc/convert.hpp"
#include "hdc/kernels.hpp"
#include "hdcgpu.h"

namespace hdc {

namespace {

[[noreturn]] void rethrow(hdcg_status s) {
    const std::string msg = hdcg_last_error();
    switch (s) {
        case HDCG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case HDCG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case HDCG_ERR_OVERFLOW: throw std::overflow_error(msg);
        case HDCG_ERR_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error("hdcgpu: " + msg);
    }
}

void call(hdcg_status s) {
    if (s != HDCG_OK) rethrow(s);
}

// index_t is int32 in the default build.  An HDC_INDEX64 build (types.hpp:8-12)
// passes input row pointers through as int64 (RowPtrArg) and narrows the other
// index arrays here: the device formats index rows, columns, segments and
// remainder entries with int32 (n, n_seg, nnz_rest < 2^31; the segment values
// themselves are addressed with 64-bit arithmetic), and a value beyond that range
// raises std::overflow_error like the reference's own range checks.
struct I32View {
    std::vector<int32_t> tmp;
    const int32_t* ptr = nullptr;
    explicit I32View(std::span<const index_t> s) {
        if constexpr (sizeof(index_t) == sizeof(int32_t)) {
            ptr = reinterpret_cast<const int32_t*>(s.data());
        } else {
            tmp.resize(s.size());
            for (std::size_t k = 0; k < s.size(); ++k) {
                if (s[k] > INT32_MAX || s[k] < INT32_MIN)
                    throw std::overflow_error("hdcgpu: index exceeds the device index range");
                tmp[k] = static_cast<int32_t>(s[k]);
            }
            ptr = tmp.data();
        }
    }
};

// An input CSR's row pointer: passed through as is -- int32 in the default build,
// int64 with HDCG_ROWPTR_I64 in an HDC_INDEX64 build (nnz may then exceed 2^31,
// e.g. BASELINE config 4's 3.75e9 entries).  Column indices stay < n < 2^31.
struct RowPtrArg {
    const void* ptr;
    unsigned flags;
    explicit RowPtrArg(std::span<const index_t> s)
        : ptr(s.data()), flags(sizeof(index_t) == sizeof(int64_t) ? HDCG_ROWPTR_I64 : 0u) {}
};

template <class T>
std::vector<index_t> widen(const std::vector<T>& v) {
    return std::vector<index_t>(v.begin(), v.end());
}

// ---- optional lifetime tracking (hdc_gpu_shim_lifetime.cpp) ---------------------
// When that file is linked too, operator delete reports released arrays and a
// cached matrix whose arrays are all still alive is used without re-hashing them.
}  // namespace
extern "C" {
int hdcg_shim_lifetime_tracking() __attribute__((weak));
int hdcg_shim_track(const void* p) __attribute__((weak));
int hdcg_shim_alive(int slot) __attribute__((weak));
void hdcg_shim_untrack(int slot) __attribute__((weak));
}
namespace {
inline bool lifetime_mode() { return hdcg_shim_lifetime_tracking != nullptr && hdcg_shim_lifetime_tracking() == 1; }

// ---- device cache -------------------------------------------------------------
// A host matrix is identified by its array addresses and sizes AND a hash of
// every byte of its arrays.  The hash is recomputed on every lookup, so a matrix
// whose storage was freed and reused by another matrix of the same shape (or
// whose contents were changed in place) never hits a stale device copy: the
// entry is dropped and the new contents are uploaded.  Hashing reads the arrays
// once at host memory bandwidth, split over threads -- a fraction of what the
// PCIe upload it avoids would cost.
struct Key {
    int kind;
    const void* a;
    const void* b;
    const void* c;
    std::size_t na, nb, nc;
    bool operator==(const Key& o) const {
        return kind == o.kind && a == o.a && b == o.b && c == o.c && na == o.na && nb == o.nb && nc == o.nc;
    }
};

inline uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9E3779B97F4A7C15ULL + (h << 6) + (h >> 2);
    return h;
}

inline uint64_t fmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// 64-bit hash of one chunk of bytes: four independent multiply-rotate lanes
uint64_t hash_chunk(const unsigned char* p, std::size_t n, uint64_t seed) {
    uint64_t h[4] = {seed ^ 0x243F6A8885A308D3ULL, seed ^ 0x13198A2E03707344ULL, seed ^ 0xA4093822299F31D0ULL,
                     seed ^ 0x082EFA98EC4E6C89ULL};
    constexpr uint64_t P = 0x9FB21C651E98DF25ULL;
    std::size_t k = 0;
    for (; k + 32 <= n; k += 32) {
        uint64_t w[4];
        std::memcpy(w, p + k, 32);
        for (int j = 0; j < 4; ++j) {
            h[j] = (h[j] ^ w[j]) * P;
            h[j] = (h[j] << 29) | (h[j] >> 35);
        }
    }
    uint64_t tail = 0;
    if (k < n) std::memcpy(&tail, p + k, std::min<std::size_t>(8, n - k));
    for (std::size_t t = k + 8; t < n; t += 8) {  // <= 3 more words
        uint64_t w = 0;
        std::memcpy(&w, p + t, std::min<std::size_t>(8, n - t));
        tail = fmix(tail ^ w);
    }
    uint64_t r = fmix(n) ^ fmix(tail);
    for (int j = 0; j < 4; ++j) r = fmix(r ^ h[j]);
    return r;
}

// Whole-array hash: fixed 4 MiB chunks (deterministic for any thread count),
// hashed in parallel for large arrays, combined in chunk order.
uint64_t hash_bytes(const void* data, std::size_t n, uint64_t h) {
    constexpr std::size_t CH = std::size_t(4) << 20;
    const auto* p = static_cast<const unsigned char*>(data);
    const std::size_t nch = n == 0 ? 0 : (n + CH - 1) / CH;
    std::vector<uint64_t> part(nch);
    auto work = [&](std::size_t c0, std::size_t c1) {
        for (std::size_t c = c0; c < c1; ++c) part[c] = hash_chunk(p + c * CH, std::min(CH, n - c * CH), c);
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nt = std::min<std::size_t>(std::min<std::size_t>(hw, 32), nch);
    if (nt <= 1) {
        work(0, nch);
    } else {
        std::vector<std::thread> th;
        for (std::size_t t = 0; t < nt; ++t) th.emplace_back(work, nch * t / nt, nch * (t + 1) / nt);
        for (auto& t : th) t.join();
    }
    h = mix(h, n);
    for (uint64_t v : part) h = mix(h, v);
    return h;
}

template <class T>
uint64_t content_hash(std::span<const T> s, uint64_t h) {
    return hash_bytes(s.data(), s.size_bytes(), h);
}

struct Entry {
    Key key;
    uint64_t hash;
    hdcg_matrix h;
    int64_t bytes;
    int slots[3] = {-2, -2, -2};  // lifetime-tracker slots of key.a/b/c (-2: not tracked, -1: table full)
};

inline void untrack(Entry& e) {
    if (!lifetime_mode()) return;
    for (int& s : e.slots) {
        if (s >= 0) hdcg_shim_untrack(s);
        s = -2;
    }
}

class Cache {
public:
    ~Cache() {
        for (auto& e : lru_) {
            untrack(e);
            hdcg_free(e.h);
        }
    }
    // Lifetime mode only: the device copy at key k when none of the matrix's arrays
    // has been released since it was cached -- no hash, the arrays are not read.
    hdcg_matrix find_live(const Key& k) {
        if (!lifetime_mode()) return nullptr;
        std::lock_guard<std::mutex> lock(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it)
            if (it->key == k) {
                const void* ptrs[3] = {k.a, k.b, k.c};
                for (int j = 0; j < 3; ++j)
                    if (ptrs[j] != nullptr && !(it->slots[j] >= 0 && hdcg_shim_alive(it->slots[j]))) return nullptr;
                lru_.splice(lru_.begin(), lru_, it);
                return it->h;
            }
        return nullptr;
    }
    // the device copy of (key, hash); an entry at the same key with a different
    // hash (storage reused or contents changed) is freed
    hdcg_matrix find(const Key& k, uint64_t hash) {
        std::lock_guard<std::mutex> lock(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it)
            if (it->key == k) {
                if (it->hash == hash) {
                    if (lifetime_mode()) {  // same contents at re-used storage: track the new arrays
                        const void* ptrs[3] = {k.a, k.b, k.c};
                        for (int j = 0; j < 3; ++j)
                            if (ptrs[j] != nullptr && !(it->slots[j] >= 0 && hdcg_shim_alive(it->slots[j]))) {
                                if (it->slots[j] >= 0) hdcg_shim_untrack(it->slots[j]);
                                it->slots[j] = hdcg_shim_track(ptrs[j]);
                            }
                    }
                    lru_.splice(lru_.begin(), lru_, it);
                    return it->h;
                }
                bytes_ -= it->bytes;
                untrack(*it);
                hdcg_free(it->h);
                lru_.erase(it);
                return nullptr;
            }
        return nullptr;
    }
    void put(const Key& k, uint64_t hash, hdcg_matrix h) {
        hdcg_info info{};
        hdcg_get_info(h, &info);
        std::lock_guard<std::mutex> lock(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it)
            if (it->key == k) {  // superseded
                bytes_ -= it->bytes;
                untrack(*it);
                hdcg_free(it->h);
                lru_.erase(it);
                break;
            }
        lru_.push_front(Entry{k, hash, h, info.device_bytes});
        if (lifetime_mode()) {
            const void* ptrs[3] = {k.a, k.b, k.c};
            for (int j = 0; j < 3; ++j) lru_.front().slots[j] = ptrs[j] ? hdcg_shim_track(ptrs[j]) : -2;
        }
        bytes_ += info.device_bytes;
        // the newest entry always stays (its caller is about to use it)
        while (lru_.size() > 1 && (lru_.size() > kMaxEntries || bytes_ > kMaxBytes)) {
            bytes_ -= lru_.back().bytes;
            untrack(lru_.back());
            hdcg_free(lru_.back().h);
            lru_.pop_back();
        }
    }
    std::size_t size() {
        std::lock_guard<std::mutex> lock(mu_);
        return lru_.size();
    }

private:
    static constexpr std::size_t kMaxEntries = 64;
    static constexpr int64_t kMaxBytes = int64_t(8) << 30;  // retained HBM beyond the newest entry
    std::mutex mu_;
    std::list<Entry> lru_;
    int64_t bytes_ = 0;
};

Cache& cache() {
    static Cache c;
    return c;
}

enum { K_CSR = 1, K_DIA = 2, K_HDC = 3, K_MHDC = 4 };

struct Ident {
    Key key;
    uint64_t hash;
};

// the address / size part of a matrix's identity (no array is read)
Key key_of(const CsrMatrix& m) {
    return Key{K_CSR, m.values().data(), m.col_ind().data(), m.row_ptr().data(), m.values().size(),
               m.col_ind().size(), m.row_ptr().size()};
}
Key key_of(const DiaMatrix& m) {
    return Key{K_DIA, m.lanes().data(), m.offsets().data(), nullptr, m.lanes().size(), m.offsets().size(), 0};
}
Key key_of(const HdcMatrix& m) {
    const Key d = key_of(m.dia()), c = key_of(m.csr());
    return Key{K_HDC, d.a, d.b, c.a, d.na, d.nb, c.na};
}
Key key_of(const MHdcMatrix& m) {
    const Key c = key_of(m.csr());
    return Key{K_MHDC, m.segments().data(), m.dia_offsets().data(), c.a, m.segments().size(),
               m.dia_offsets().size(), c.na};
}

Ident ident(const CsrMatrix& m) {
    const uint64_t h = content_hash(m.values(), content_hash(m.col_ind(), content_hash(m.row_ptr(), m.n())));
    return {Key{K_CSR, m.values().data(), m.col_ind().data(), m.row_ptr().data(), m.values().size(),
                m.col_ind().size(), m.row_ptr().size()},
            h};
}
Ident ident(const DiaMatrix& m) {
    const uint64_t h = content_hash(m.lanes(), content_hash(m.offsets(), m.n()));
    return {Key{K_DIA, m.lanes().data(), m.offsets().data(), nullptr, m.lanes().size(), m.offsets().size(), 0}, h};
}
Ident ident(const HdcMatrix& m) {
    const Ident d = ident(m.dia()), c = ident(m.csr());
    return {Key{K_HDC, d.key.a, d.key.b, c.key.a, d.key.na, d.key.nb, c.key.na}, mix(d.hash, c.hash)};
}
Ident ident(const MHdcMatrix& m) {
    const uint64_t h = content_hash(m.segments(), content_hash(m.dia_offsets(), content_hash(m.dia_ptr(), m.bl())));
    const Ident c = ident(m.csr());
    return {Key{K_MHDC, m.segments().data(), m.dia_offsets().data(), c.key.a, m.segments().size(),
                m.dia_offsets().size(), c.key.na},
            mix(h, c.hash)};
}

hdcg_matrix device_of(const CsrMatrix& m) {
    if (hdcg_matrix live = cache().find_live(key_of(m))) return live;  // lifetime mode: no hashing
    const Ident id = ident(m);
    if (hdcg_matrix h = cache().find(id.key, id.hash)) return h;
    const RowPtrArg rp(m.row_ptr());
    const I32View col(m.col_ind());
    hdcg_matrix h = nullptr;
    call(hdcg_build_csr(m.n(), static_cast<int64_t>(m.values().size()), rp.ptr, col.ptr, m.values().data(),
                        rp.flags, nullptr, &h));
    cache().put(id.key, id.hash, h);
    return h;
}

hdcg_matrix upload_hdc(index_t n, std::span<const index_t> offsets, std::span<const real_t> lanes,
                       const CsrMatrix* rest) {
    const I32View offs(offsets);
    hdcg_matrix h = nullptr;
    if (rest) {
        const I32View rp(rest->row_ptr()), col(rest->col_ind());
        call(hdcg_upload_hdc(n, static_cast<int64_t>(offsets.size()), offs.ptr, lanes.data(), rp.ptr,
                             static_cast<int64_t>(rest->values().size()), col.ptr, rest->values().data(), 0, &h));
    } else {
        std::vector<int32_t> rp(static_cast<std::size_t>(n) + 1, 0);
        call(hdcg_upload_hdc(n, static_cast<int64_t>(offsets.size()), offs.ptr, lanes.data(), rp.data(), 0,
                             nullptr, nullptr, 0, &h));
    }
    return h;
}

hdcg_matrix device_of(const DiaMatrix& m) {
    if (hdcg_matrix live = cache().find_live(key_of(m))) return live;  // lifetime mode: no hashing
    const Ident id = ident(m);
    if (hdcg_matrix h = cache().find(id.key, id.hash)) return h;
    hdcg_matrix h = upload_hdc(m.n(), m.offsets(), m.lanes(), nullptr);
    cache().put(id.key, id.hash, h);
    return h;
}

hdcg_matrix device_of(const HdcMatrix& m) {
    if (hdcg_matrix live = cache().find_live(key_of(m))) return live;  // lifetime mode: no hashing
    const Ident id = ident(m);
    if (hdcg_matrix h = cache().find(id.key, id.hash)) return h;
    hdcg_matrix h = upload_hdc(m.n(), m.dia().offsets(), m.dia().lanes(), &m.csr());
    cache().put(id.key, id.hash, h);
    return h;
}

hdcg_matrix device_of(const MHdcMatrix& m) {
    if (hdcg_matrix live = cache().find_live(key_of(m))) return live;  // lifetime mode: no hashing
    const Ident id = ident(m);
    if (hdcg_matrix h = cache().find(id.key, id.hash)) return h;
    const I32View dp(m.dia_ptr()), offs(m.dia_offsets()), rp(m.csr().row_ptr()), col(m.csr().col_ind());
    hdcg_matrix h = nullptr;
    call(hdcg_upload_mhdc(m.n(), m.bl(), dp.ptr, m.n_segments(), offs.ptr, m.segments().data(), rp.ptr,
                          static_cast<int64_t>(m.csr().values().size()), col.ptr, m.csr().values().data(), 0, &h));
    cache().put(id.key, id.hash, h);
    return h;
}

struct Exported {
    hdcg_info info{};
    std::vector<int32_t> dia_ptr, offsets, rest_rp, rest_col;
    std::vector<real_t> segments, rest_val;
};

Exported export_all(hdcg_matrix h) {
    Exported e;
    call(hdcg_get_info(h, &e.info));
    e.dia_ptr.resize(static_cast<std::size_t>(e.info.n_blocks) + 1);
    e.offsets.resize(static_cast<std::size_t>(e.info.n_seg));
    e.segments.resize(static_cast<std::size_t>(e.info.n_seg * e.info.bl));
    e.rest_rp.resize(static_cast<std::size_t>(e.info.n_rows) + 1);
    e.rest_col.resize(static_cast<std::size_t>(e.info.nnz_rest));
    e.rest_val.resize(static_cast<std::size_t>(e.info.nnz_rest));
    call(hdcg_export(h, e.dia_ptr.data(), e.offsets.data(), e.segments.data(), e.rest_rp.data(), e.rest_col.data(),
                     e.rest_val.data()));
    return e;
}

// Input CSR handed to the device converters.  The reference's CsrMatrix is
// already validated by its constructor, so no HDCG_VALIDATE here.
struct CsrArgs {
    RowPtrArg rp;
    I32View col;
    const CsrMatrix& m;
    explicit CsrArgs(const CsrMatrix& mm) : rp(mm.row_ptr()), col(mm.col_ind()), m(mm) {}
};

void check_theta(real_t theta, const char* what) {
    if (!(theta >= 0.0 && theta <= 1.0)) throw std::invalid_argument(std::string(what) + ": theta must be in [0, 1]");
}

void check_vectors(index_t n, std::size_t nx, std::size_t ny, const char* what) {
    if (nx != static_cast<std::size_t>(n) || ny != static_cast<std::size_t>(n))
        throw std::invalid_argument(std::string(what) + ": x and y must have length n");
}

void check_plan(const BlockPlan& plan, index_t n, const char* what) {
    if (plan.n != n || plan.bl < 1 || plan.n_blocks != (n == 0 ? 0 : (n + plan.bl - 1) / plan.bl))
        throw std::invalid_argument(std::string(what) + ": block plan does not match matrix");
}

void run(hdcg_matrix h, index_t n, std::span<const real_t> x, std::span<real_t> y) {
    if (n == 0) return;
    call(hdcg_spmv_host(h, x.data(), y.data()));
}

// Create the device context when the library loads, so the first timed call
// does not pay for it.
struct EagerInit {
    EagerInit() { (void)hdcg_init(0); }
} g_eager_init;

}  // namespace

// ---- convert.hpp ------------------------------------------------------------------

index_t DiagonalCensus::total() const {
    index_t sum = 0;
    for (const auto& block : per_block)
        for (const OffsetCount& oc : block) sum += oc.count;
    return sum;
}

static DiagonalCensus census_impl(const CsrMatrix& m, index_t bl, bool global) {
    DiagonalCensus c;
    c.n = m.n();
    if (global && m.n() == 0) return c;  // convert.cpp:61-65
    c.bl = global ? m.n() : bl;
    c.n_blocks = m.n() == 0 ? 0 : (m.n() + c.bl - 1) / c.bl;
    c.per_block.resize(static_cast<std::size_t>(c.n_blocks));
    const RowPtrArg rp(m.row_ptr());
    const I32View col(m.col_ind());
    std::vector<int64_t> bp(static_cast<std::size_t>(c.n_blocks) + 1);
    int64_t total = 0;
    const int64_t arg_bl = global ? 0 : bl;
    const int64_t nnz = static_cast<int64_t>(m.values().size());
    call(hdcg_census(m.n(), nnz, rp.ptr, col.ptr, arg_bl, rp.flags, bp.data(), nullptr, nullptr, &total));
    std::vector<int32_t> offs(static_cast<std::size_t>(total));
    std::vector<int64_t> cnt(static_cast<std::size_t>(total));
    call(hdcg_census(m.n(), nnz, rp.ptr, col.ptr, arg_bl, rp.flags, bp.data(), offs.data(), cnt.data(), &total));
    for (index_t b = 0; b < c.n_blocks; ++b)
        for (int64_t k = bp[b]; k < bp[b + 1]; ++k)
            c.per_block[b].push_back(OffsetCount{static_cast<index_t>(offs[k]), static_cast<index_t>(cnt[k])});
    return c;
}

DiagonalCensus census_blocked(const CsrMatrix& m, index_t bl) {
    if (bl < 1) throw std::invalid_argument("census_blocked: block width must be >= 1");
    return census_impl(m, bl, false);
}

DiagonalCensus census_global(const CsrMatrix& m) { return census_impl(m, m.n(), true); }

static hdcg_matrix build_hdc_device(const CsrMatrix& m, real_t theta) {
    const CsrArgs a(m);
    hdcg_matrix h = nullptr;
    call(hdcg_build_hdc(m.n(), static_cast<int64_t>(m.values().size()), a.rp.ptr, a.col.ptr, m.values().data(),
                        theta, a.rp.flags, nullptr, &h));
    return h;
}

DiaMatrix to_dia(const CsrMatrix& m) {
    hdcg_matrix h = build_hdc_device(m, 0.0);  // theta = 0: every populated diagonal is a lane
    Exported e = export_all(h);
    DiaMatrix d(m.n(), widen(e.offsets), std::move(e.segments));
    const Ident id = ident(d);
    cache().put(id.key, id.hash, h);
    return d;
}

HdcMatrix to_hdc(const CsrMatrix& m, real_t theta) {
    check_theta(theta, "to_hdc");
    hdcg_matrix h = build_hdc_device(m, theta);
    Exported e = export_all(h);
    HdcMatrix out(m.n(), DiaMatrix(m.n(), widen(e.offsets), std::move(e.segments)),
                  CsrMatrix(m.n(), std::move(e.rest_val), widen(e.rest_col), widen(e.rest_rp)), theta);
    const Ident id = ident(out);
    cache().put(id.key, id.hash, h);
    return out;
}

MHdcMatrix to_mhdc(const CsrMatrix& m, real_t theta, index_t bl) {
    check_theta(theta, "to_mhdc");
    if (bl < 1) throw std::invalid_argument("to_mhdc: block width must be >= 1");
    const CsrArgs a(m);
    hdcg_matrix h = nullptr;
    call(hdcg_build_mhdc(m.n(), m.n(), 0, static_cast<int64_t>(m.values().size()), a.rp.ptr, a.col.ptr,
                         m.values().data(), theta, bl, a.rp.flags, nullptr, &h));
    Exported e = export_all(h);
    MHdcMatrix out(m.n(), bl, widen(e.dia_ptr), widen(e.offsets), std::move(e.segments),
                   CsrMatrix(m.n(), std::move(e.rest_val), widen(e.rest_col), widen(e.rest_rp)), theta);
    const Ident id = ident(out);
    cache().put(id.key, id.hash, h);
    return out;
}

static HybridRates rates_of(hdcg_matrix h) {
    HybridRates r{};
    int64_t slots = 0;
    call(hdcg_rates(h, &r.alpha, &r.beta, &slots));
    r.dia_slots = static_cast<index_t>(slots);
    return r;
}

HybridRates rates(const HdcMatrix& m) { return rates_of(device_of(m)); }
HybridRates rates(const MHdcMatrix& m) { return rates_of(device_of(m)); }

// ---- kernels.hpp ----------------------------------------------------------------

BlockPlan BlockPlan::rows(index_t n, index_t bl) {
    if (n < 0) throw std::invalid_argument("BlockPlan: negative row count");
    if (bl < 1) throw std::invalid_argument("BlockPlan: block width must be >= 1");
    return BlockPlan{n, bl, n == 0 ? 0 : (n + bl - 1) / bl};
}

void spmv_csr(const CsrMatrix& m, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_csr");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

void spmv_dia(const DiaMatrix& m, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_dia");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

void spmv_bdia(const DiaMatrix& m, const BlockPlan& plan, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_bdia");
    check_plan(plan, m.n(), "spmv_bdia");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

void spmv_hdc(const HdcMatrix& m, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_hdc");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

void spmv_bhdc(const HdcMatrix& m, const BlockPlan& plan, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_bhdc");
    check_plan(plan, m.n(), "spmv_bhdc");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

void spmv_mhdc(const MHdcMatrix& m, std::span<const real_t> x, std::span<real_t> y, int) {
    check_vectors(m.n(), x.size(), y.size(), "spmv_mhdc");
    if (m.n() == 0) return;
    run(device_of(m), m.n(), x, y);
}

DenseVector spmv_csr(const CsrMatrix& m, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_csr(m, x, y, w);
    return y;
}
DenseVector spmv_dia(const DiaMatrix& m, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_dia(m, x, y, w);
    return y;
}
DenseVector spmv_bdia(const DiaMatrix& m, const BlockPlan& plan, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_bdia(m, plan, x, y, w);
    return y;
}
DenseVector spmv_hdc(const HdcMatrix& m, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_hdc(m, x, y, w);
    return y;
}
DenseVector spmv_bhdc(const HdcMatrix& m, const BlockPlan& plan, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_bhdc(m, plan, x, y, w);
    return y;
}
DenseVector spmv_mhdc(const MHdcMatrix& m, const DenseVector& x, int w) {
    DenseVector y(static_cast<std::size_t>(m.n()));
    spmv_mhdc(m, x, y, w);
    return y;
}

}  // namespace hdc

// hdc_gpu_shim_lifetime.cpp -- OPTIONAL companion of hdc_gpu_shim.cpp.
//
// The shim keeps a device copy of every host matrix it has seen.  To be sure a
// cached copy still belongs to the matrix it is handed, the shim alone re-hashes
// every byte of the host arrays on every call -- which reads the matrix once from
// host memory, i.e. costs what the reference's CPU SpMV costs (config 1: ~10 ms of
// hashing + 4.8 ms on the GPU path against 13.9 ms on the CPU).
//
// Linking this file as well replaces that per-call hash by lifetime tracking: it
// replaces the global operator delete, so the shim learns when the storage of a
// cached matrix is released (the reference's containers are std::vectors, released
// through operator delete) and drops the device copy then.  While none of a matrix's
// arrays has been released, its cached copy is used without reading the arrays
// again (config 1: 4.8 ms per spmv_mhdc call).  The full hash still runs when a
// matrix is first seen.  What this mode cannot see is a host matrix modified in
// place through const_cast -- outside the reference's contract (matrices are
// immutable after construction).  A program that already replaces
// operator new/delete cannot link this file; it keeps the hashing mode.
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <new>

namespace {

constexpr int SLOTS = 4096;  // tracked arrays (3 per cached matrix, 64 matrices cached at most)
const void* const TOMB = reinterpret_cast<const void*>(1);
std::atomic<const void*> g_ptr[SLOTS];
std::atomic<bool> g_alive[SLOTS];
std::atomic<int> g_tracked{0};
std::mutex g_mu;  // track / untrack; the free path only reads

inline unsigned slot_of(const void* p) {
    auto v = reinterpret_cast<std::uintptr_t>(p);
    v ^= v >> 17;
    v *= 0x9E3779B97F4A7C15ull;
    return (unsigned)(v >> 40) & (SLOTS - 1);
}

inline void on_free(const void* p) noexcept {
    if (p == nullptr || g_tracked.load(std::memory_order_relaxed) == 0) return;
    unsigned s = slot_of(p);
    for (int k = 0; k < SLOTS; ++k, s = (s + 1) & (SLOTS - 1)) {
        const void* q = g_ptr[s].load(std::memory_order_acquire);
        if (q == nullptr) return;
        if (q == p) g_alive[s].store(false, std::memory_order_release);  // keep probing: duplicates are possible
    }
}

}  // namespace

extern "C" {

// 1: this translation unit is linked in (the shim tests the symbol's address)
int hdcg_shim_lifetime_tracking() { return 1; }

// Starts tracking the array at p; returns a slot id (>= 0), or -1 when the table is full.
int hdcg_shim_track(const void* p) {
    if (p == nullptr) return -1;
    std::lock_guard<std::mutex> lock(g_mu);
    unsigned s = slot_of(p);
    for (int k = 0; k < SLOTS; ++k, s = (s + 1) & (SLOTS - 1)) {
        const void* q = g_ptr[s].load(std::memory_order_relaxed);
        if (q == nullptr || q == TOMB) {
            g_alive[s].store(true, std::memory_order_relaxed);
            g_ptr[s].store(p, std::memory_order_release);
            g_tracked.fetch_add(1, std::memory_order_relaxed);
            return (int)s;
        }
    }
    return -1;
}

int hdcg_shim_alive(int slot) { return slot >= 0 && slot < SLOTS && g_alive[slot].load(std::memory_order_acquire); }

void hdcg_shim_untrack(int slot) {
    if (slot < 0 || slot >= SLOTS) return;
    std::lock_guard<std::mutex> lock(g_mu);
    g_alive[slot].store(false, std::memory_order_relaxed);
    g_ptr[slot].store(TOMB, std::memory_order_release);
    if (g_tracked.fetch_sub(1, std::memory_order_relaxed) == 1)  // nothing tracked: drop the tombstones
        for (auto& q : g_ptr) q.store(nullptr, std::memory_order_relaxed);
}

}  // extern "C"

// ---- the replaced deallocation functions (allocation stays the default: malloc) ----
void operator delete(void* p) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete[](void* p) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete(void* p, std::size_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete[](void* p, std::size_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete(void* p, std::align_val_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete[](void* p, std::align_val_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete(void* p, std::size_t, std::align_val_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete[](void* p, std::size_t, std::align_val_t) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete(void* p, const std::nothrow_t&) noexcept {
    on_free(p);
    std::free(p);
}
void operator delete[](void* p, const std::nothrow_t&) noexcept {
    on_free(p);
    std::free(p);
}

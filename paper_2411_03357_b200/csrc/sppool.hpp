// Size-class free lists for the control plane's small objects.
//
// Per event the engine creates and drops a handful of small objects (a
// message, a staging buffer handle, span and message vectors, map nodes for
// deferred decrypts and read guards).  At 64 KiB blocks that is ~250k events
// per OPT-66B layer pair, and malloc/free dominated the host time (bursts of
// tens of thousands of allocations overflow glibc's per-thread cache).  These
// lists hand the memory back without touching malloc: thread-local (a pipe
// has one owner thread at a time; a block freed on another thread simply
// joins that thread's list), refilled 64 KiB at a time, never returned to the
// OS (bounded by the peak number of live objects).
#pragma once

#include <cstddef>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <new>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace sppipe {

class FreeLists {
  public:
    static constexpr size_t kStep = 16, kMax = 512;

    void *get(size_t n) {
        if (n > kMax || n == 0) return ::operator new(n ? n : 1);
        const size_t c = (n + kStep - 1) / kStep;
        void *p = heads_[c];
        if (!p) {
            refill(c);
            p = heads_[c];
        }
        heads_[c] = *static_cast<void **>(p);
        return p;
    }
    void put(void *p, size_t n) {
        if (n > kMax || n == 0) {
            ::operator delete(p);
            return;
        }
        const size_t c = (n + kStep - 1) / kStep;
        *static_cast<void **>(p) = heads_[c];
        heads_[c] = p;
    }

  private:
    void refill(size_t c) {
        const size_t sz = c * kStep;
        const size_t count = (64u << 10) / sz;
        char *blk = static_cast<char *>(std::malloc(sz * count));
        if (!blk) throw std::bad_alloc();
        for (size_t i = 0; i < count; ++i) {
            void *p = blk + i * sz;
            *static_cast<void **>(p) = heads_[c];
            heads_[c] = p;
        }
    }
    void *heads_[kMax / kStep + 1] = {};
};

inline FreeLists &free_lists() {
    // intentionally leaked: objects may outlive the thread's destructors
    static thread_local FreeLists *f = new FreeLists();
    return *f;
}

template <class T>
struct PoolAlloc {
    using value_type = T;
    PoolAlloc() noexcept = default;
    template <class U>
    PoolAlloc(const PoolAlloc<U> &) noexcept {}
    T *allocate(size_t n) { return static_cast<T *>(free_lists().get(n * sizeof(T))); }
    void deallocate(T *p, size_t n) noexcept { free_lists().put(p, n * sizeof(T)); }
    template <class U>
    bool operator==(const PoolAlloc<U> &) const noexcept {
        return true;
    }
    template <class U>
    bool operator!=(const PoolAlloc<U> &) const noexcept {
        return false;
    }
};

template <class T>
using PVec = std::vector<T, PoolAlloc<T>>;
template <class K, class V, class C = std::less<K>>
using PMap = std::map<K, V, C, PoolAlloc<std::pair<const K, V>>>;
template <class K, class C = std::less<K>>
using PSet = std::set<K, C, PoolAlloc<K>>;
template <class K, class V, class H = std::hash<K>>
using PUMap = std::unordered_map<K, V, H, std::equal_to<K>, PoolAlloc<std::pair<const K, V>>>;
template <class K, class H = std::hash<K>>
using PUSet = std::unordered_set<K, H, std::equal_to<K>, PoolAlloc<K>>;

template <class T, class... A>
std::shared_ptr<T> pmake(A &&...a) {
    return std::allocate_shared<T>(PoolAlloc<T>(), std::forward<A>(a)...);
}

}  // namespace sppipe

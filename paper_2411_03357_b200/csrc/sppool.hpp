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

// A vector with N inline slots: no allocation until the N+1-th element (a
// buffer's per-stream fence list has 1-3 entries; at 64 KiB blocks a
// quarter million buffers are made per run).  Contiguous: iterates as T*.
template <class T, size_t N>
class SmallVec {
  public:
    SmallVec() = default;
    SmallVec(const SmallVec &o) { *this = o; }
    SmallVec(SmallVec &&o) noexcept { *this = std::move(o); }
    SmallVec &operator=(const SmallVec &o) {
        if (this == &o) return *this;
        clear();
        for (const T &x : o) push_back(x);
        return *this;
    }
    SmallVec &operator=(SmallVec &&o) noexcept {
        if (this == &o) return *this;
        clear();
        n_ = o.n_;
        for (size_t i = 0; i < o.n_; ++i) inl_[i] = std::move(o.inl_[i]);
        heap_ = std::move(o.heap_);
        o.clear();
        return *this;
    }
    T *begin() { return heap_.empty() ? inl_ : heap_.data(); }
    T *end() { return begin() + size(); }
    const T *begin() const { return heap_.empty() ? inl_ : heap_.data(); }
    const T *end() const { return begin() + size(); }
    size_t size() const { return heap_.empty() ? n_ : heap_.size(); }
    bool empty() const { return size() == 0; }
    T &front() { return *begin(); }
    template <class... A>
    T &emplace_back(A &&...a) {
        if (heap_.empty() && n_ < N) {
            inl_[n_] = T(std::forward<A>(a)...);
            return inl_[n_++];
        }
        if (heap_.empty()) {  // spill the inline slots first
            heap_.reserve(2 * N);
            for (size_t i = 0; i < n_; ++i) heap_.push_back(std::move(inl_[i]));
            for (size_t i = 0; i < n_; ++i) inl_[i] = T();
            n_ = 0;
        }
        heap_.emplace_back(std::forward<A>(a)...);
        return heap_.back();
    }
    void push_back(const T &x) { emplace_back(x); }
    void clear() {
        for (size_t i = 0; i < n_; ++i) inl_[i] = T();
        n_ = 0;
        heap_.clear();
    }

  private:
    T inl_[N] = {};
    size_t n_ = 0;
    PVec<T> heap_;
};
template <class K, class V, class C = std::less<K>>
using PMap = std::map<K, V, C, PoolAlloc<std::pair<const K, V>>>;
template <class K, class C = std::less<K>>
using PSet = std::set<K, C, PoolAlloc<K>>;
template <class K, class V, class H = std::hash<K>>
using PUMap = std::unordered_map<K, V, H, std::equal_to<K>, PoolAlloc<std::pair<const K, V>>>;
template <class K, class H = std::hash<K>>
using PUSet = std::unordered_set<K, H, std::equal_to<K>, PoolAlloc<K>>;

// Intrusive, non-atomic reference counting for the data plane's handles
// (buffers, fences, messages, slabs).  std::shared_ptr counts atomically in
// any process with threads (every Python process): at ~20 handle copies per
// trace event the locked increments were ~10% of the host time.  A pipe has
// one owner thread at a time, so plain counters suffice.
struct RcBase {
    uint32_t rc_ = 0;
};

template <class T>
class Rc {
  public:
    Rc() noexcept = default;
    Rc(std::nullptr_t) noexcept {}
    explicit Rc(T *p) noexcept : p_(p) {
        if (p_) ++p_->rc_;
    }
    Rc(const Rc &o) noexcept : p_(o.p_) {
        if (p_) ++p_->rc_;
    }
    Rc(Rc &&o) noexcept : p_(o.p_) { o.p_ = nullptr; }
    ~Rc() { drop(p_); }
    Rc &operator=(const Rc &o) noexcept {
        if (o.p_) ++o.p_->rc_;
        T *old = p_;
        p_ = o.p_;
        drop(old);
        return *this;
    }
    Rc &operator=(Rc &&o) noexcept {
        if (this != &o) {
            T *old = p_;
            p_ = o.p_;
            o.p_ = nullptr;
            drop(old);
        }
        return *this;
    }
    Rc &operator=(std::nullptr_t) noexcept {
        reset();
        return *this;
    }
    void reset() noexcept {
        T *old = p_;
        p_ = nullptr;
        drop(old);
    }
    T *get() const noexcept { return p_; }
    T *operator->() const noexcept { return p_; }
    T &operator*() const noexcept { return *p_; }
    explicit operator bool() const noexcept { return p_ != nullptr; }
    bool operator==(const Rc &o) const noexcept { return p_ == o.p_; }
    bool operator!=(const Rc &o) const noexcept { return p_ != o.p_; }

  private:
    static void drop(T *p) noexcept {
        if (p && --p->rc_ == 0) {
            p->~T();
            free_lists().put(p, sizeof(T));
        }
    }
    T *p_ = nullptr;
};

template <class T, class... A>
Rc<T> pmake(A &&...a) {
    void *m = free_lists().get(sizeof(T));
    return Rc<T>(new (m) T(std::forward<A>(a)...));
}

}  // namespace sppipe

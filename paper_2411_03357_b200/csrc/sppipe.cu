// libsppipe — native speculative pipeline for the encrypted swap path.
//
// Control plane: the reference's engine/validator/predictor/channel counters
// (/root/reference/pkg/src/specpipe/{engine,validator,predictor,channel,memory}.py)
// restated in C++ with the same decisions in the same order, so the same
// trace yields identical sent logs, actions, report() counters and decision
// logs (tests/test_native_engine.py against the reference goldens).
//
// Data plane (B200): long-lived streams per device, shared by the pipes
//   h2d   plaintext of swap-ins crosses PCIe from the caller's pinned blocks
//   spec  encrypt-ahead seals (SpecBatch, engine.py:487-513), <= batch_bytes per launch
//   comp, comp2  the compute queue of on-the-fly / NOP / swap-out seals and
//         every receiver open, flushed as level-scheduled k_gcm launches;
//         consecutive flushes alternate between the two streams
//   out   swap-out seals of KV-cache evictions
//   land  host-endpoint opens of swap-outs (deferred decrypts)
//   d2h   plaintext lands in the caller's host blocks
//   host  ordered application writes into host blocks
// Cross-stream order uses CUDA events only; the calls are issued in order by
// one worker thread per pipe (Issuer).  Device buffers of <= 1 MiB come from
// 32 MiB slabs, larger ones from a stream-ordered CUDA memory pool kept
// reserved for the life of the process (release threshold = max); a buffer
// is returned to the pool on the stream of its last use once every other
// stream that touched it has passed its fence.
#include <cuda_runtime.h>
#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "spgcm.h"
#include "spguard.h"
#include "sppipe.h"
#include "sppool.hpp"
#include "sppred.hpp"

namespace sppipe {

// Byte copy between UVA-mapped (pinned host or device) buffers, for small
// ordered writes that must not use a copy engine.
__global__ void k_bytes(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// ---- SM-driven host<->device transfers ----------------------------------------------
// The copy engine pays ~4.5 us of device time per cudaMemcpyAsync whatever its
// size (B200, pinned, profiles/r2_copy_probe.txt: 64 KiB copies move at 12.7
// GB/s, 224 KiB at 29 GB/s), so the many small copies of one flush (KV blocks,
// 64 KiB chunks, landings) are moved instead by ONE launch of k_xfer: warps
// stream 16 KiB pieces of every job straight over PCIe between HBM and the
// UVA-mapped pinned host block (~50 GB/s per direction from 16 CTAs, the same
// probe).  Large copies (> kXferMax) stay on the copy engine, which needs no
// SMs and is as fast there.
struct XferJob {
    const uint8_t *src;
    uint8_t *dst;
    uint64_t n;
};
constexpr int kXferInline = 128;           // jobs per launch, inside the kernel parameters (<= 3 KiB)
constexpr uint64_t kXferPiece = 16384;     // bytes per warp step
constexpr int kXferThreads = 256;          // fits beside a k_gcm CTA (104 registers x 512 threads)
template <int N>
struct XferParams {
    XferJob j[N];
    uint32_t n;
};

__device__ __forceinline__ void xfer_piece(const uint8_t *s, uint8_t *d, uint64_t lo, uint64_t hi, int lane) {
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15u) == 0) {
        // 16-byte words, four loads in flight per lane before their stores
        const uint4 *s4 = reinterpret_cast<const uint4 *>(s);
        uint4 *d4 = reinterpret_cast<uint4 *>(d);
        const uint64_t w_lo = lo >> 4, w_hi = hi >> 4;
        for (uint64_t i = w_lo + lane; i < w_hi; i += 128) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (i + 32 * k < w_hi) v[k] = __ldcv(s4 + i + 32 * k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (i + 32 * k < w_hi) __stcs(d4 + i + 32 * k, v[k]);
        }
        for (uint64_t i = (w_hi << 4) + lane; i < hi; i += 32) d[i] = s[i];  // tail of the job
    } else {
        for (uint64_t i = lo + lane; i < hi; i += 32) d[i] = s[i];
    }
}

template <int N>
__global__ void __launch_bounds__(kXferThreads) k_xfer(const __grid_constant__ XferParams<N> p) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t j = 0;
    uint64_t base = 0;  // global index of job j's first piece
    for (uint64_t q = warp;; q += nwarps) {
        while (j < p.n && q >= base + (p.j[j].n + kXferPiece - 1) / kXferPiece) {
            base += (p.j[j].n + kXferPiece - 1) / kXferPiece;
            ++j;
        }
        if (j >= p.n) return;
        const uint64_t lo = (q - base) * kXferPiece;
        xfer_piece(p.j[j].src, p.j[j].dst, lo, min(p.j[j].n, lo + kXferPiece), lane);
    }
}

// Model compute of a trace's ComputeEvent (the reference charges it to the
// GPU timeline, simulator.py:431-434): a fixed amount of FMA work per
// launch, calibrated to the event's duration on an idle GPU, in 16 waves of
// 4 CTAs x 256 threads per SM (tiles, like a GEMM: CTAs flow to whichever
// SMs are free).  Fixed work, not a timed spin, so SM contention with the
// crypto kernels slows it down measurably.  The app stream has the highest
// stream priority: its CTAs are dispatched ahead of queued crypto CTAs.  Each launch
// stamps its first-CTA start and last-CTA end (globaltimer) into its span
// slot: slot[0] = min start, slot[1] = ~max end (both atomicMin on a slot
// initialised to all ones).
constexpr int kComputeThreads = 256;
constexpr int kComputeCtasPerSm = 4;
constexpr int kComputeWaves = 16;
__global__ void __launch_bounds__(kComputeThreads) k_layer_compute(uint64_t iters, unsigned long long *slot) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0 && slot) atomicMin(slot, t0);
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = (float)(threadIdx.x + c);
    for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fmaf(x[c], 0.999999f, 0.5f);
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc += x[c];
    __syncthreads();
    if (threadIdx.x == 0 && slot) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMin(slot + 1, ~t1);
        if (acc == -1.0f) slot[0] = 0;  // never: keeps the FMA chains live
    }
}

// ---- NVTX (SURVEY §5 tracing) ----------------------------------------------------
// Domain "sppipe": a range per engine entry point (payload = the channel's
// H2D send counter at entry) and a mark per message put on the wire (name =
// direction and kind, payload = its counter), so nsys / ncu timelines line
// the control plane up with the kernels and copies.  NVTX3 is header-only:
// without an attached tool every call is a null check.
nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("sppipe");
    return d;
}
inline nvtxEventAttributes_t nvtx_attr(const char *msg, uint64_t payload) {
    nvtxEventAttributes_t a{};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = msg;
    a.payloadType = NVTX_PAYLOAD_TYPE_UNSIGNED_INT64;
    a.payload.ullValue = payload;
    return a;
}
struct NvtxRange {
    NvtxRange(const char *msg, uint64_t payload) {
        nvtxEventAttributes_t a = nvtx_attr(msg, payload);
        nvtxDomainRangePushEx(nvtx_domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
};
inline void nvtx_mark(const char *msg, uint64_t payload) {
    nvtxEventAttributes_t a = nvtx_attr(msg, payload);
    nvtxDomainMarkEx(nvtx_domain(), &a);
}

// ---- error classes (Python exception names) -----------------------------------
struct EngineErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct OverlapErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct StateErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct BoundsErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct GuardErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct KeyErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct AuthErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaErr : std::runtime_error { using std::runtime_error::runtime_error; };

thread_local std::string g_err;

inline void ck(cudaError_t e, const char *where) {
    if (e != cudaSuccess) throw CudaErr(std::string(where) + ": " + cudaGetErrorString(e));
}
inline void ck_sp(int rc, const char *where) {
    if (rc == SP_OK) return;
    if (rc == SP_EINVAL) throw ValueErr(std::string(where) + ": " + sp_last_error());
    throw CudaErr(std::string(where) + ": " + sp_last_error());
}

std::string hex(uint64_t v) {
    char b[32];
    snprintf(b, sizeof b, "%#llx", (unsigned long long)v);
    return b;
}

constexpr uint64_t kTag = 16;
constexpr int H2D = 0, D2H = 1;
inline uint64_t round16(uint64_t n) { return (n + 15u) & ~uint64_t(15); }

// ---- events and device buffers ------------------------------------------------
class Plane;

struct Fence : RcBase {
    cudaEvent_t ev = nullptr;
    cudaStream_t stream = nullptr;
    bool recorded = false;
    bool complete = false;  // observed complete once (never re-recorded after that)
    uint64_t seq = 0;       // record order: on one stream a higher seq completes later
    uint64_t mark = 0;      // de-duplicates waits within one issue pass
    uint64_t post_seq = 0;  // Issuer position of its cudaEventRecord (0: issued inline)
    Plane *plane = nullptr;
    ~Fence();
};
using FenceP = Rc<Fence>;

struct Slab;
struct Buf : RcBase {
    Plane *plane = nullptr;
    Rc<Slab> slab;  // sub-allocation of a slab (small buffers), else null
    uint8_t *ptr = nullptr;
    uint64_t size = 0;
    uint64_t alloc_size = 0;
    SmallVec<std::pair<cudaStream_t, FenceP>, 4> uses;  // latest fence per stream
    uint64_t last_use = 0;
    cudaStream_t last_stream = nullptr;
    uint32_t queued = 0;       // ops in the compute queue that touch this buffer (not yet issued)
    // flush-local list of the regions queued ops touch (Plane::flush)
    mutable uint64_t touch_epoch = 0;
    mutable int32_t touch_head = -1;
    uint32_t out_pending = 0;  // swap-out seals reading it, not yet launched
    void use(cudaStream_t s, const FenceP &f, uint64_t tick) {
        last_use = tick;
        last_stream = s;
        for (auto &u : uses)
            if (u.first == s) {
                u.second = f;
                return;
            }
        uses.emplace_back(s, f);
    }
    ~Buf();
};
using BufP = Rc<Buf>;

// Small buffers (<= 1 MiB: staging of small chunks, KV blocks, arenas) are
// bump-allocated from 32 MiB slabs, one open slab per (stream, lane): a
// sub-buffer costs no driver call (a pool allocation is ~1.5 us, per chunk
// at 64 KiB blocks).  A dying sub-buffer folds its stream fences into the
// slab; the slab retires (buffer cache, same reuse rules) when the last of
// its sub-buffers is gone.  Ranges inside a slab are never reused while it
// lives, so sub-buffers need no ordering among themselves.
struct Slab : RcBase {
    BufP big;
    uint64_t off = 0;
    FenceP born;  // recorded on the allocating stream right after the slab's allocation
};

struct View {
    BufP buf;
    uint64_t off = 0, len = 0;
    uint8_t *ptr() const { return buf->ptr + off; }
};

// A sealed message on the wire (channel.CiphertextMsg / DeviceCiphertext).
struct Msg : RcBase {
    BufP buf;  // payload at off, tag at tag_off (null in the dry plane)
    uint64_t off = 0, tag_off = 0, len = 0;
    bool nop = false;
    FenceP ready;  // producer's fence (recorded at its launch)
    // H2D messages are opened on the device when sent (Engine::eager_open):
    // the IV and destination of that open
    bool opened = false;
    uint64_t open_iv = 0;
    View open_dst;
};
using MsgP = Rc<Msg>;
using Spans = PVec<std::pair<uint64_t, uint64_t>>;  // (offset, length) of the messages of one transfer

// ---- host memory model (memory.py) ---------------------------------------------
struct Block {
    int64_t id;
    uint64_t base, len;
    int kind;
    uint8_t *host;
    uint8_t *host_dev = nullptr;  // device-accessible alias of a pinned host block (UVA), else null
    bool page_owned = false;      // SP_BLOCK_PAGE_OWNED: whole pages, exclusively this block's
};

struct WriteGuard {
    uint64_t base, len;
    int64_t owner;
    bool active;
};

class HostMem {
  public:
    // id -> block (ids are small and dense, memory.py:117-166); stable addresses
    std::vector<std::unique_ptr<Block>> blocks;
    PMap<int64_t, WriteGuard> write_guards;  // owner (record id) -> guard (insertion order == id order)

    Block &block(int64_t id) {
        if (id < 0 || id >= (int64_t)blocks.size() || !blocks[(size_t)id]) throw KeyErr(std::to_string(id));
        return *blocks[(size_t)id];
    }
    void add_block(const Block &b) {
        if (b.id < 0 || b.id > (int64_t)1 << 40) throw ValueErr("block id out of range");
        if ((size_t)b.id >= blocks.size()) blocks.resize((size_t)b.id + 1);
        if (blocks[(size_t)b.id]) {
            const uint64_t old = blocks[(size_t)b.id]->base;
            for (size_t i = 0; i < by_base.size(); ++i)
                if (by_base[i].first == old && by_base[i].second == b.id) {
                    by_base.erase(by_base.begin() + (long)i);
                    break;
                }
        }
        blocks[(size_t)b.id].reset(new Block(b));
        if (!by_base.empty() && by_base.back().first >= b.base) by_base_sorted = false;
        by_base.emplace_back(b.base, b.id);
    }
    // memory.py block_at: the block containing [base, base+len)
    std::pair<Block *, uint64_t> block_at(uint64_t base, uint64_t len) {
        const size_t i = block_index(base);
        if (i != SIZE_MAX) {
            Block &b = block(by_base[i].second);
            if (b.base <= base && base + len <= b.base + b.len) return {&b, base - b.base};
        }
        throw BoundsErr("range (" + hex(base) + ", " + std::to_string(len) + ") is not inside any block");
    }
    static bool overlaps(uint64_t ab, uint64_t al, uint64_t bb, uint64_t bl) { return ab < bb + bl && bb < ab + al; }

    bool hw = false;  // mirror write guards with mprotect'ed pages (libspguard)

    void install_write_guard(uint64_t base, uint64_t len, int64_t owner) {
        for (auto &kv : write_guards) {
            const WriteGuard &g = kv.second;
            if (g.active && overlaps(base, len, g.base, g.len))
                throw GuardErr("write guard (" + hex(base) + ", " + std::to_string(len) + ") overlaps guard of record " +
                               std::to_string(g.owner));
        }
        write_guards[owner] = WriteGuard{base, len, owner, true};
        if (hw) {
            auto bi = block_at(base, len);
            const Block &hb = *bi.first;
            const int flags = hb.page_owned ? ((bi.second == 0 ? SPG_HEAD_OWNED : 0) |
                                               (bi.second + len == hb.len ? SPG_TAIL_OWNED : 0))
                                            : 0;
            if (hb.host && spg_protect_ex(hb.host + bi.second, len, owner, flags) != SPG_OK)
                throw std::runtime_error("spg_protect failed (errno " + std::to_string(spg_errno()) + ")");
        }
    }
    void release_write_guard(int64_t owner) {
        write_guards.erase(owner);
        if (hw) spg_release(owner);
    }

    // Read guards are disjoint (install rejects overlaps).  Each is listed
    // under every block it overlaps (swap-outs guard one block, so a query
    // scans one short list after one binary search over block bases); a
    // guard over no block goes to `rg_loose`.  Results come back in task id
    // order = the reference's dict insertion order (memory.py:244-259).
    struct ReadGuard {
        uint64_t base, len;
    };
    PUMap<int64_t, ReadGuard> read_guards;  // task id -> range
    std::vector<PVec<int64_t>> rg_block;    // block id -> tasks of the guards overlapping it
    PVec<int64_t> rg_loose;

    PVec<int64_t> read_guards_over(uint64_t base, uint64_t len) const {
        PVec<int64_t> out;
        if (!len || read_guards.empty()) return out;
        auto scan = [&](const PVec<int64_t> &tasks) {
            for (int64_t t : tasks) {
                const ReadGuard &g = read_guards.at(t);
                if (overlaps(base, len, g.base, g.len)) out.push_back(t);
            }
        };
        blocks_over(base, len, [&](int64_t bid) {
            if ((size_t)bid < rg_block.size()) scan(rg_block[(size_t)bid]);
        });
        scan(rg_loose);
        std::sort(out.begin(), out.end());
        out.erase(std::unique(out.begin(), out.end()), out.end());  // a guard over several blocks
        return out;
    }
    void install_read_guard(uint64_t base, uint64_t len, int64_t task) {
        auto hits = read_guards_over(base, len);
        if (!hits.empty())
            throw GuardErr("read guard (" + hex(base) + ", " + std::to_string(len) + ") overlaps task " +
                           std::to_string(hits.front()));
        read_guards[task] = ReadGuard{base, len};
        bool any = false;
        blocks_over(base, len, [&](int64_t bid) {
            if ((size_t)bid >= rg_block.size()) rg_block.resize((size_t)bid + 1);
            rg_block[(size_t)bid].push_back(task);
            any = true;
        });
        if (!any) rg_loose.push_back(task);
    }
    void release_read_guard(int64_t task) {
        auto it = read_guards.find(task);
        if (it == read_guards.end()) return;
        auto drop = [task](PVec<int64_t> &v) {
            for (size_t i = 0; i < v.size(); ++i)
                if (v[i] == task) {
                    v[i] = v.back();
                    v.pop_back();
                    return;
                }
        };
        blocks_over(it->second.base, it->second.len, [&](int64_t bid) {
            if ((size_t)bid < rg_block.size()) drop(rg_block[(size_t)bid]);
        });
        drop(rg_loose);
        read_guards.erase(it);
    }

  private:
    // (base, id) of every block; sorted on demand (bump allocation appends in order)
    mutable std::vector<std::pair<uint64_t, int64_t>> by_base;
    mutable bool by_base_sorted = true;
    void sort_bases() const {
        if (by_base_sorted) return;
        std::sort(by_base.begin(), by_base.end());
        by_base_sorted = true;
    }
    // index in by_base of the last block whose base <= addr, or SIZE_MAX
    size_t block_index(uint64_t addr) const {
        sort_bases();
        // traces walk blocks in order: try the last hit and its successor first
        const size_t n = by_base.size();
        for (size_t c = hint_; c < n && c <= hint_ + 1; ++c)
            if (by_base[c].first <= addr && (c + 1 == n || by_base[c + 1].first > addr)) return hint_ = c;
        auto it = std::upper_bound(by_base.begin(), by_base.end(), std::make_pair(addr, INT64_MAX));
        if (it == by_base.begin()) return SIZE_MAX;
        return hint_ = (size_t)(it - by_base.begin()) - 1;
    }
    mutable size_t hint_ = 0;
    template <class F>
    void blocks_over(uint64_t base, uint64_t len, F &&f) const {
        sort_bases();
        size_t i = block_index(base);
        if (i == SIZE_MAX) i = 0;
        for (; i < by_base.size() && by_base[i].first < base + len; ++i) {
            const Block *b = blocks[(size_t)by_base[i].second].get();
            if (b && overlaps(base, len, b->base, b->len)) f(by_base[i].second);
        }
    }
};

// ---- validator (validator.py:104-230) ----------------------------------------------
enum RecState { PENDING = 0, COMMITTED = 1, INVALIDATED = 2 };
enum Verdict { V_HIT = 0, V_AHEAD = 1, V_BEHIND = 2, V_STALE = 3, V_MISS = 4, V_NONE = 5 };

struct Record {
    int64_t id;
    uint64_t base, len, iv;
    PVec<MsgP> chunks;  // released (emptied) once the record leaves the window
    PVec<uint64_t> chunk_lens;
    RecState state = PENDING;
    int64_t block_id;  // INT64_MIN = None
    uint64_t span() const { return chunk_lens.size(); }
    uint64_t last_iv() const { return iv + span() - 1; }
};

struct RangeKey {
    uint64_t base, len;
    bool operator==(const RangeKey &o) const { return base == o.base && len == o.len; }
};
struct RangeHash {
    size_t operator()(const RangeKey &k) const { return (size_t)(k.base * 0x9e3779b97f4a7c15ull ^ (k.len + (k.len << 17))); }
};

class Validator {
  public:
    Validator(HostMem &m, uint64_t window) : mem(m), window(window) {}
    HostMem &mem;
    uint64_t window;
    std::deque<Record> records;  // id i at index i - first_id
    int64_t first_id = 1;        // oldest retained record (compact())
    uint64_t history = 0;        // retained finished records (0: all, as the reference keeps them)
    int64_t next_id = 1;
    PUMap<RangeKey, int64_t, RangeHash> by_range, stale;
    PUMap<uint64_t, int64_t> by_iv;
    PSet<int64_t> order;                        // pending ids (label order == id order)
    PSet<std::pair<uint64_t, int64_t>> bases;  // (base, id) of pending
    int64_t counters[5] = {0, 0, 0, 0, 0};
    int64_t evicted = 0;

    Record &rec(int64_t id) { return records[(size_t)(id - first_id)]; }
    bool retained(int64_t id) const { return id >= first_id && id < next_id; }

    // Forget finished records older than every pending one, beyond the last
    // `history`: a long-running pipe's record list stays bounded (their
    // payloads are already released; STALE verdicts keep only the range map).
    void compact() {
        if (!history || records.size() <= history + history / 2) return;
        const int64_t oldest_pending = order.empty() ? next_id : *order.begin();
        while (records.size() > history && records.front().id < oldest_pending) {
            records.pop_front();
            ++first_id;
        }
    }

    int64_t label(PVec<MsgP> chunks, PVec<uint64_t> lens, uint64_t base, uint64_t len, uint64_t iv,
                  int64_t block_id) {
        // pending ranges are disjoint: only the last one starting below the end can intersect
        auto it = bases.lower_bound({base + len, INT64_MIN});
        if (it != bases.begin()) {
            --it;
            if (it->first + rec(it->second).len > base)
                throw OverlapErr("range (" + hex(base) + ", " + std::to_string(len) + ") overlaps pending record " +
                                 std::to_string(it->second));
        }
        uint64_t span = lens.size();
        for (uint64_t v = iv; v < iv + span; ++v)
            if (by_iv.count(v)) throw OverlapErr("counter " + std::to_string(v) + " already claimed by a pending record");
        if (order.size() >= window) {
            invalidate(*order.begin());
            ++evicted;
        }
        Record r;
        r.id = next_id++;
        r.base = base;
        r.len = len;
        r.iv = iv;
        r.chunks = std::move(chunks);
        r.chunk_lens = std::move(lens);
        r.block_id = block_id;
        records.push_back(std::move(r));
        Record &x = records.back();
        by_range[{base, len}] = x.id;
        for (uint64_t v = iv; v < iv + span; ++v) by_iv[v] = x.id;
        order.insert(x.id);
        bases.insert({base, x.id});
        stale.erase({base, len});
        mem.install_write_guard(base, len, x.id);
        return x.id;
    }

    Verdict validate(uint64_t base, uint64_t len, uint64_t cur, int64_t &rid) {
        rid = -1;
        Verdict v;
        auto it = by_range.find({base, len});
        if (it != by_range.end()) {
            Record &r = rec(it->second);
            rid = r.id;
            v = r.iv == cur ? V_HIT : (r.iv > cur ? V_AHEAD : V_BEHIND);
        } else {
            auto s = stale.find({base, len});
            if (s != stale.end()) {
                rid = s->second;
                v = V_STALE;
            } else {
                v = V_MISS;
            }
        }
        counters[v]++;
        return v;
    }

    void drop_pending(Record &r) {
        by_range.erase({r.base, r.len});
        for (uint64_t v = r.iv; v < r.iv + r.span(); ++v) by_iv.erase(v);
        order.erase(r.id);
        bases.erase({r.base, r.id});
        mem.release_write_guard(r.id);
    }
    void commit(int64_t id) {
        Record &r = rec(id);
        if (r.state != PENDING) throw StateErr("record " + std::to_string(id) + " is " + state_name(r.state) + ", not pending");
        drop_pending(r);
        r.state = COMMITTED;
    }
    void invalidate(int64_t id) {
        Record &r = rec(id);
        if (r.state != PENDING) throw StateErr("record " + std::to_string(id) + " is " + state_name(r.state) + ", not pending");
        drop_pending(r);
        r.state = INVALIDATED;
        stale[{r.base, r.len}] = r.id;
        r.chunks.clear();  // device payloads go back to the pool
    }
    void on_write_fault(int64_t owner) {
        if (retained(owner) && rec(owner).state == PENDING) invalidate(owner);
    }
    std::vector<int64_t> pending_ids() const { return std::vector<int64_t>(order.begin(), order.end()); }
    int64_t pending_at_iv(uint64_t iv) const {
        auto it = by_iv.find(iv);
        return it == by_iv.end() ? -1 : it->second;
    }
    bool has_pending_range(uint64_t base, uint64_t len) const { return by_range.count({base, len}) != 0; }
    int64_t invalidate_pending_below(uint64_t iv) {
        std::vector<int64_t> doomed;
        for (int64_t id : order)
            if (rec(id).last_iv() < iv) doomed.push_back(id);
        for (int64_t id : doomed) invalidate(id);
        return (int64_t)doomed.size();
    }
    static const char *state_name(RecState s) {
        return s == PENDING ? "pending" : (s == COMMITTED ? "committed" : "invalidated");
    }
};

// ---- data plane -----------------------------------------------------------------------
struct Streams {
    cudaStream_t comp, spec, h2d, d2h, land, host, out;  // host: ordered app writes; out: swap-out seals
    cudaStream_t spec_h2d;  // encrypt-ahead staging copies (SPPIPE_SPEC_H2D=0: they use h2d)
    cudaStream_t comp2;  // consecutive flushes alternate between comp and comp2
    cudaStream_t app;    // the model's compute (trace ComputeEvents)
};

struct DevicePool {
    cudaMemPool_t pool = nullptr;
    uint64_t reserved = 0;
};

std::mutex g_dev_mu;
std::map<int, Streams> g_streams;
std::map<int, DevicePool> g_pools;
std::map<std::pair<int, std::string>, sp_ctx *> g_ctx;  // key setup once per (device, key)
std::vector<std::pair<uint8_t *, uint64_t>> g_rings;    // idle pinned staging rings (process-wide)
// Idle CUDA events per device, handed from destroyed planes to new ones:
// cudaEventCreate takes the driver's write lock (~2-5 us beside a busy
// issuing thread) and a fresh pipe creates hundreds of fences in its first
// milliseconds (20% of the KV trace's control thread, sampled).
std::map<int, std::vector<cudaEvent_t>> g_events;
constexpr size_t kEventsWarm = 256, kEventsKeep = 8192;
// Device buffers of destroyed pipes, idle (their streams were drained):
// the next pipe on the device takes them without a pool call (a pipe per
// replay / bench repetition would otherwise re-carve its whole working set).
struct IdleBufs {
    std::unordered_map<uint64_t, std::vector<uint8_t *>> by_size;
    uint64_t bytes = 0;
};
std::map<int, IdleBufs> g_idle;
constexpr uint64_t kIdleBytes = 16ull << 30;
// Off by default: with slab allocation a new pipe makes few pool calls, and
// parked buffers of sizes the next pipe does not use would only keep memory
// from the pool (measured equal on the bench traces).
bool idle_cache_enabled() {  // SPPIPE_IDLE_CACHE=1: hand a destroyed pipe's idle buffers to the next pipe
    static const bool on = [] {
        const char *e = getenv("SPPIPE_IDLE_CACHE");
        return e && e[0] == '1';
    }();
    return on;
}

sp_ctx *ctx_for(int dev, const uint8_t key[32]) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto k = std::make_pair(dev, std::string(reinterpret_cast<const char *>(key), 32));
    auto it = g_ctx.find(k);
    if (it != g_ctx.end()) return it->second;
    sp_ctx *c = nullptr;
    int rc = sp_ctx_create(key, &c);
    if (rc) throw CudaErr(std::string("sp_ctx_create: ") + sp_last_error());
    g_ctx[k] = c;
    return c;
}

Streams streams_for(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_streams.find(dev);
    if (it != g_streams.end()) return it->second;
    Streams s;
    // Stream priorities (SPPIPE_PRIO): "crypto" (default) — the data plane's
    // streams outrank the model's compute, so a seal/open/transfer launched
    // while a compute kernel fills the GPU gets SMs as soon as one of the
    // compute's CTAs retires (~20 us) instead of after the whole kernel
    // (~300 us): on the KV trace each decode step's swap-out landing ->
    // D2H -> swap-in -> open chain used to wait out the compute kernel before
    // it (profiles/r2_dbg_kv_compute).  "app": the compute outranks the data
    // plane (r1 policy); "equal": one priority.
    static const int mode = [] {
        const char *e = getenv("SPPIPE_PRIO");
        if (!e) return 0;
        const std::string v(e);
        return v == "app" ? 1 : (v == "equal" ? 2 : (v == "spec_low" ? 3 : 0));
    }();
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
    const int plane_prio = (mode == 0 || mode == 3) ? hi : lo, app_prio = mode == 1 ? hi : lo;
    cudaStream_t *all[9] = {&s.comp, &s.spec, &s.h2d, &s.d2h, &s.land, &s.host, &s.out, &s.comp2, &s.spec_h2d};
    for (auto p : all)
        ck(cudaStreamCreateWithPriority(p, cudaStreamNonBlocking, (mode == 3 && p == &s.spec) ? lo : plane_prio),
           "cudaStreamCreate");
    ck(cudaStreamCreateWithPriority(&s.app, cudaStreamNonBlocking, app_prio), "cudaStreamCreate(app)");
    g_streams[dev] = s;
    return s;
}

cudaMemPool_t pool_for(int dev, uint64_t reserve, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevicePool &p = g_pools[dev];
    if (!p.pool) {
        cudaMemPoolProps props;
        memset(&props, 0, sizeof props);
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        ck(cudaMemPoolCreate(&p.pool, &props), "cudaMemPoolCreate");
        uint64_t thr = UINT64_MAX;
        ck(cudaMemPoolSetAttribute(p.pool, cudaMemPoolAttrReleaseThreshold, &thr), "pool threshold");
        int zero = 0;
        // never make an allocating stream wait on another stream's pending free
        ck(cudaMemPoolSetAttribute(p.pool, cudaMemPoolReuseAllowInternalDependencies, &zero), "pool deps");
    }
    if (reserve > p.reserved) {
        void *ptr = nullptr;
        ck(cudaMallocFromPoolAsync(&ptr, reserve, p.pool, s), "pool reserve");
        ck(cudaFreeAsync(ptr, s), "pool reserve free");
        ck(cudaStreamSynchronize(s), "pool reserve sync");
        p.reserved = reserve;
    }
    return p.pool;
}

// One queued seal/open of the compute stream.  The regions it reads and
// writes give the dependencies flush() schedules by: an op runs in a later
// launch than every earlier op it conflicts with (RAW, WAR, WAW), independent
// seals and opens share launches (sp_crypt_batch).
struct Region {
    const Buf *buf;
    uint64_t lo, hi;
};
struct Op {
    sp_desc d;     // d.reserved = SP_OP_SEAL / SP_OP_OPEN
    FenceP wait;   // produced on another stream (staging copy, spec batch, earlier window)
    BufP a, b;     // buffers the op touches (kept alive until issued)
    Region r[2], w[2];
    int nr = 0, nw = 0;
};

// Host->device staging copies gathered and issued as one batch (one
// issuing-thread closure of per-copy calls) with one shared fence, recorded at issue.
struct CopyBatch {
    std::vector<void *> dst;
    std::vector<void *> src;
    std::vector<size_t> n;
    std::vector<BufP> keep;     // staging buffers, alive until issued
    std::vector<FenceP> waits;  // host blocks' landings that must precede the reads
    FenceP fence;
    cudaStream_t stream = nullptr;  // copy stream (null: the plane's h2d stream)
    bool empty() const { return n.empty(); }
};

struct Landing {
    Block *block;
    PVec<std::tuple<MsgP, uint64_t, uint64_t>> jobs;  // msg, iv, offset in block
    int dir;
};

// Stream-ordered CUDA calls of a plane (copies, launches, event records and
// waits, stream-ordered frees) are issued by one worker thread, in the order
// the control plane posts them: the control plane (channel, validator,
// predictor, staging decisions) overlaps the driver's per-call cost, which
// dominates at small messages (64 KiB blocks: ~1.5 us of driver time per
// event).  Posted closures capture only raw handles and pointers, never the
// plane's reference-counted objects.  Anything that reads device state
// (event queries of not-yet-issued records, stream/event syncs, status reads)
// drains the queue first.  SPPIPE_ASYNC_ISSUE=0: every call inline.
// A forked child has no issuing threads: its planes fall back to inline calls.
std::atomic<bool> g_forked{false};

class Issuer {
  public:
    static bool enabled_by_env() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_ASYNC_ISSUE");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    void start(int device) {
        static const bool hooked = [] {
            pthread_atfork(nullptr, nullptr, [] { g_forked.store(true); });
            return true;
        }();
        (void)hooked;
        dev_ = device;
        th_ = std::thread([this] { run(); });
        on_ = true;
    }
    ~Issuer() { stop(); }
    void stop() {
        if (!on_) return;
        if (g_forked.load()) {  // the thread does not exist in this process: forget it
            new (&th_) std::thread();
            on_ = false;
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            quit_ = true;
            quit_flag_.store(true, std::memory_order_release);
        }
        cv_.notify_one();
        th_.join();
        on_ = false;
    }
    bool on() const { return on_; }
    // Run `fn` now (inline mode) or queue it; returns its sequence number.
    // `tag` (a string literal) names the call kind for the per-kind
    // profile (SPPIPE_ISSUER_PROFILE=1 prints it when the plane closes).
    uint64_t post(std::function<void()> fn, const char *tag = "misc") {
        if (!on_ || g_forked.load(std::memory_order_relaxed)) {
            fn();
            return 0;
        }
        if (failed_.load(std::memory_order_acquire)) rethrow();
        uint64_t seq;
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(Job{std::move(fn), tag});
            seq = ++posted_;
            posted_seen_.store(seq, std::memory_order_release);
        }
        if (sleeping_.load(std::memory_order_acquire)) cv_.notify_one();
        return seq;
    }
    bool done(uint64_t seq) const { return seq <= done_.load(std::memory_order_acquire); }
    void drain() {
        if (!on_ || g_forked.load(std::memory_order_relaxed)) return;
        std::unique_lock<std::mutex> lk(mu_);
        cv_done_.wait(lk, [&] { return done_.load(std::memory_order_acquire) == posted_; });
        lk.unlock();
        if (failed_.load(std::memory_order_acquire)) rethrow();
    }

  private:
    void rethrow() {
        std::lock_guard<std::mutex> lk(mu_);
        std::string e = err_;
        err_.clear();
        failed_.store(false, std::memory_order_release);
        throw CudaErr(e);
    }
    void run() {
        cudaSetDevice(dev_);
        std::vector<Job> batch;
        for (;;) {
            // spin ~50 us for the next post before sleeping: a flush posts a
            // burst of calls, and a futex wake-up would add its latency to
            // every burst's first call
            const auto t_spin = std::chrono::steady_clock::now();
            while (posted_seen_.load(std::memory_order_acquire) == done_.load(std::memory_order_acquire) &&
                   std::chrono::steady_clock::now() - t_spin < std::chrono::microseconds(50) &&
                   !quit_flag_.load(std::memory_order_acquire)) {
            }
            {
                std::unique_lock<std::mutex> lk(mu_);
                sleeping_.store(true, std::memory_order_release);
                cv_.wait(lk, [&] { return quit_ || !q_.empty(); });
                sleeping_.store(false, std::memory_order_release);
                if (q_.empty() && quit_) return;
                batch.assign(std::make_move_iterator(q_.begin()), std::make_move_iterator(q_.end()));
                q_.clear();
            }
            const auto t_batch = std::chrono::steady_clock::now();
            calls_.fetch_add(batch.size(), std::memory_order_relaxed);
            for (auto &job : batch) {
                const auto t_job = profile_ ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point();
                try {
                    job.fn();
                } catch (const std::exception &e) {
                    std::lock_guard<std::mutex> lk(mu_);
                    if (err_.empty()) err_ = e.what();
                    failed_.store(true, std::memory_order_release);
                }
                if (profile_) {
                    auto &k = kinds_[job.tag];
                    k.first++;
                    k.second += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                    std::chrono::steady_clock::now() - t_job)
                                    .count();
                }
                {
                    std::lock_guard<std::mutex> lk(mu_);
                    done_.fetch_add(1, std::memory_order_acq_rel);
                }
                cv_done_.notify_all();
            }
            busy_ns_.fetch_add((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                   std::chrono::steady_clock::now() - t_batch)
                                   .count(),
                               std::memory_order_relaxed);
            batch.clear();
        }
    }
    int dev_ = 0;
    bool on_ = false, quit_ = false;
    std::thread th_;
    std::mutex mu_;
    std::condition_variable cv_, cv_done_;
    struct Job {
        std::function<void()> fn;
        const char *tag;
    };
    std::deque<Job> q_;
    uint64_t posted_ = 0;
    std::atomic<uint64_t> done_{0}, posted_seen_{0};
    std::atomic<bool> failed_{false}, sleeping_{false}, quit_flag_{false};
    std::string err_;

  public:
    // CUDA calls issued and the time the worker spent inside them (a worker
    // busy for most of a run's wall time means the run is issue-bound)
    std::atomic<uint64_t> calls_{0}, busy_ns_{0};
    const bool profile_ = [] {
        const char *e = getenv("SPPIPE_ISSUER_PROFILE");
        return e && e[0] == '1';
    }();
    std::map<const char *, std::pair<uint64_t, uint64_t>> kinds_;  // tags are literals; worker thread only
    void print_profile() const {
        if (!profile_) return;
        for (auto &k : kinds_)
            fprintf(stderr, "[issuer] %-16s n=%6llu total %8.3f ms  %6.2f us/call\n", k.first,
                    (unsigned long long)k.second.first, k.second.second / 1e6,
                    k.second.first ? k.second.second / 1e3 / k.second.first : 0.0);
    }
};

class Plane {
  public:
    bool dry;
    Issuer iss;
    int dev = 0;
    Streams s{};
    cudaMemPool_t pool = nullptr;
    sp_ctx *ctx = nullptr;
    uint64_t batch_bytes;
    uint64_t tick = 0;
    std::vector<cudaEvent_t> free_events;
    struct Garbage {
        uint8_t *ptr;
        SmallVec<std::pair<cudaStream_t, FenceP>, 4> uses;
        cudaStream_t last;
        uint64_t size;
    };
    std::vector<Garbage> garbage;
    bool collecting = false;
    std::unordered_map<uint64_t, std::deque<Garbage>> cache;  // size class -> retired buffers, oldest first
    uint64_t cached_bytes = 0;
    bool closing = false;
    static constexpr uint64_t kCacheBytes = 8ull << 30;
    uint64_t pool_bytes = 0;  // bytes this plane holds from the pool (in use or cached)
    // SPPIPE_POOL_BUDGET_GB (default 16): past this, allocations wait for retired buffers
    static uint64_t pool_budget() {
        static const uint64_t b = [] {
            const char *e = getenv("SPPIPE_POOL_BUDGET_GB");
            const double gb = e ? atof(e) : 16.0;
            return (uint64_t)(gb > 0 ? gb * (double)(1ull << 30) : 16.0 * (double)(1ull << 30));
        }();
        return b;
    }

    // compute queue
    std::vector<Op> ops, ops_spare;
    std::vector<FenceP> flush_waits;  // fences the next flush's stream must wait for (swap-out WAR)
    uint64_t flush_no = 0;
    // Consecutive flushes alternate between two compute streams so one
    // batch boundary's launches can overlap the previous one's (small
    // batches are launch-latency bound); the order between them comes from
    // each buffer's per-stream fences instead of stream order.
    // SPPIPE_COMP_STREAMS=1: one compute stream.
    static bool two_comp() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_COMP_STREAMS");
            return !(e && e[0] == '1');
        }();
        return on;
    }
    struct Touch {
        uint64_t lo, hi;
        int level;
        bool write;
        int32_t next;
    };
    std::vector<Touch> touches;
    std::vector<int> op_level;
    std::vector<uint32_t> level_start, by_level;
    std::vector<sp_desc> descs_scratch;
    uint64_t touch_epoch = 0, mark_seq = 0;
    uint64_t ops_bytes = 0;
    FenceP window;
    // small-payload arena
    BufP arena_dev;
    uint64_t arena_off = 0;      // payloads (copied from the host) grow up from 0
    uint64_t arena_low = 0;      // device-only scratch grows down from the end
    // Pinned host staging ring for small payloads (arena flushes, token
    // copies): slots are taken in order and handed back when the fence of
    // the copy that read/wrote them has passed; one cudaHostAlloc per process.
    struct Ring {
        uint8_t *ptr = nullptr;
        uint64_t cap = 0, head = 0;
        std::deque<std::tuple<uint64_t, uint64_t, FenceP>> busy;  // [begin, end), fence
    } ring;
    static constexpr uint64_t kRingBytes = 32ull << 20;
    static constexpr uint64_t kArenaBytes = 1 << 20;
    // NOP pads seal zeros: read from a device zero page instead of crossing PCIe
    static constexpr uint64_t kZeroBytes = 1 << 20;
    uint8_t *zero_dev = nullptr;
    // ring slots read by queued (not yet issued) seals: committed with the
    // fence of the flush that issues them
    std::vector<std::pair<uint8_t *, uint64_t>> ring_pending;
    uint64_t ring_pending_bytes = 0;
    // landings
    std::vector<Landing> landings;
    PUSet<int64_t> landing_blocks;
    PUMap<int64_t, FenceP> host_ready;  // block -> fence after last D2H into it
    PUMap<int64_t, FenceP> h2d_done;    // block -> fence after last H2D from it
    CopyBatch otf_copies;                             // on-the-fly staging copies (issued at flush)
    // Swap-out seals on their own stream (SPPIPE_OUT_STREAM=1, see
    // out_stream_enabled): each waits only for the launch that last wrote
    // its source block.
    struct OutBatch {
        std::vector<sp_desc> items;
        std::vector<BufP> bufs;
        std::vector<FenceP> waits;
        uint64_t bytes = 0;
        FenceP ready;
    } outb;
    CopyBatch *spec_copies = nullptr;                 // copies of the SpecBatch being built
    // Open verdicts: every open of the pipe shares one sticky status word in
    // mapped pinned memory (SP_STATUS_ON_FAILURE: k_gcm writes it only on a
    // tag mismatch), read by the host at finish / strict checks.  (A status
    // word per open needed a full-device sync to recycle the words every
    // 64K opens: four pipeline drains per 64 KiB-chunk OPT-66B run.)
    volatile int32_t *auth_h = nullptr;  // host view
    int32_t *auth_d = nullptr;           // device alias
    uint64_t opens_unchecked = 0;
    uint64_t bytes_h2d = 0, bytes_d2h = 0, launches = 0;

    Plane(bool dry_, const uint8_t key[32], uint64_t batch, uint64_t reserve) : dry(dry_), batch_bytes(batch) {
        if (dry) return;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        s = streams_for(dev);
        pool = pool_for(dev, reserve, s.comp);
        ctx = ctx_for(dev, key);
        ck(cudaHostAlloc(reinterpret_cast<void **>(const_cast<int32_t **>(&auth_h)), 64, cudaHostAllocMapped),
           "cudaHostAlloc(auth flag)");
        *auth_h = 0;
        ck(cudaHostGetDevicePointer(reinterpret_cast<void **>(&auth_d), const_cast<int32_t *>(auth_h), 0),
           "cudaHostGetDevicePointer(auth flag)");
        ck(cudaMalloc(&zero_dev, kZeroBytes), "cudaMalloc(zero page)");
        ck(cudaMemset(zero_dev, 0, kZeroBytes), "cudaMemset(zero page)");
        {
            std::lock_guard<std::mutex> lk(g_dev_mu);
            auto &pool = g_events[dev];
            free_events.swap(pool);
        }
        if (dbg_times())
            for (int i = 0; i < 16384; ++i) {
                cudaEvent_t e;
                ck(cudaEventCreate(&e), "cudaEventCreate(dbg)");
                dbg_events.push_back(e);
            }
        while (free_events.size() < kEventsWarm) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            free_events.push_back(e);
        }
        window = new_fence();
        if (Issuer::enabled_by_env()) iss.start(dev);
    }
    ~Plane() {
        if (dry) return;
        if (!g_forked.load()) dbg_print();
        if (g_forked.load()) {
            // CUDA is unusable in a forked child: no stream syncs or frees
            // (the parent still owns the device memory); members unwind
            // without CUDA calls
            closing = true;
            iss.stop();
            return;
        }
        bool idle = true;
        try {
            finish_streams();
        } catch (...) {
            idle = false;
        }
        try {
            iss.drain();
        } catch (...) {
            idle = false;
        }
        iss.stop();  // everything below runs inline
        iss.print_profile();
        ops.clear();
        landings.clear();
        host_ready.clear();
        h2d_done.clear();
        arena_dev.reset();
        window.reset();
        slabs.clear();  // open slabs retire into the cache
        closing = true;
        {
            std::lock_guard<std::mutex> lk(g_dev_mu);
            IdleBufs &ib = g_idle[dev];
            for (auto &kv : cache)
                for (auto &g : kv.second) {
                    if (idle && idle_cache_enabled() && ib.bytes + kv.first <= kIdleBytes) {
                        ib.by_size[kv.first].push_back(g.ptr);
                        ib.bytes += kv.first;
                    } else {
                        garbage.push_back(std::move(g));
                    }
                }
        }
        cache.clear();
        collect();
        cudaStreamSynchronize(s.comp);
        cudaStreamSynchronize(s.comp2);
        if (ring.ptr) {
            // every copy through the ring is done (streams drained): hand it on
            ring.busy.clear();
            std::lock_guard<std::mutex> lk(g_dev_mu);
            g_rings.push_back({ring.ptr, ring.cap});
        }
        {
            std::lock_guard<std::mutex> lk(g_dev_mu);
            auto &pool = g_events[dev];
            for (cudaEvent_t e : free_events) {
                if (pool.size() < kEventsKeep) pool.push_back(e);
                else cudaEventDestroy(e);
            }
            free_events.clear();
        }
        if (auth_h) cudaFreeHost(const_cast<int32_t *>(auth_h));
        if (zero_dev) cudaFree(zero_dev);
        if (d_spans) cudaFree(d_spans);
    }

    // -- events / buffers --------------------------------------------------------------
    // SPPIPE_DEBUG_TIMES=1 (diagnostics): fences get timing events, and every
    // swap-out launch logs when each of its waits and its own fence completed
    // (ms after the plane's first record), printed when the plane closes.
    static bool dbg_times() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_DEBUG_TIMES");
            return e && e[0] == '1';
        }();
        return on;
    }
    cudaEvent_t dbg_base = nullptr;
    std::vector<cudaEvent_t> dbg_events;
    struct DbgEntry {
        const char *what;
        cudaStream_t st;
        FenceP f;
        uint64_t batch;
    };
    std::vector<DbgEntry> dbg_log;
    uint64_t dbg_batches = 0, dbg_computes = 0;
    const char *stream_name(cudaStream_t st) const {
        if (st == s.comp) return "comp";
        if (st == s.comp2) return "comp2";
        if (st == s.h2d) return "h2d";
        if (st == s.d2h) return "d2h";
        if (st == s.land) return "land";
        if (st == s.out) return "out";
        if (st == s.spec) return "spec";
        if (st == s.host) return "host";
        if (st == s.app) return "app";
        return "?";
    }
    void dbg_print() {
        if (!dbg_base) return;
        iss.drain();
        cudaDeviceSynchronize();
        for (auto &d : dbg_log) {
            float ms = -1;
            if (d.f && d.f->recorded && cudaEventElapsedTime(&ms, dbg_base, d.f->ev) != cudaSuccess) ms = -2;
            fprintf(stderr, "[dbg] batch %llu %-10s %-6s %9.3f ms\n", (unsigned long long)d.batch, d.what,
                    stream_name(d.st), ms);
        }
        cudaGetLastError();
        dbg_log.clear();
    }
    FenceP new_fence() {
        auto f = pmake<Fence>();
        f->plane = this;
        if (dbg_times()) {
            if (!dbg_base) {
                ck(cudaEventCreate(&dbg_base), "cudaEventCreate(dbg)");
                ck(cudaEventRecord(dbg_base, s.comp), "cudaEventRecord(dbg)");
            }
            if (!dbg_events.empty()) {  // timing events made up front (no driver call per fence)
                f->ev = dbg_events.back();
                dbg_events.pop_back();
            } else {
                ck(cudaEventCreate(&f->ev), "cudaEventCreate(dbg)");
            }
            return f;
        }
        if (!free_events.empty()) {
            f->ev = free_events.back();
            free_events.pop_back();
        } else {
            ck(cudaEventCreateWithFlags(&f->ev, cudaEventDisableTiming), "cudaEventCreate");
        }
        return f;
    }
    uint64_t record_seq = 0;
    void record(const FenceP &f, cudaStream_t st, const char *tag = "record") {
        const cudaEvent_t ev = f->ev;
        f->post_seq = iss.post([ev, st] { ck(cudaEventRecord(ev, st), "cudaEventRecord"); }, tag);
        f->stream = st;
        f->recorded = true;
        f->seq = ++record_seq;
    }
    FenceP record_new(cudaStream_t st, const char *tag = "record") {
        FenceP f = new_fence();
        record(f, st, tag);
        return f;
    }
    void wait(cudaStream_t st, const FenceP &f) {
        if (!f) return;
        if (!f->recorded) throw std::logic_error("wait on an unrecorded fence");
        if (f->stream == st) return;  // stream order covers it
        const cudaEvent_t ev = f->ev;
        iss.post([st, ev] { ck(cudaStreamWaitEvent(st, ev, 0), "cudaStreamWaitEvent"); }, "wait");
    }
    // Size classes of the plane's buffer cache: 4 KiB steps up to 1 MiB,
    // then 1 MiB steps (staging sizes repeat: chunks, KV blocks, arenas).
    static uint64_t size_class(uint64_t n) {
        n = std::max<uint64_t>(n, 16);
        return n <= (1u << 20) ? (n + 4095u) & ~uint64_t(4095) : (n + (1u << 20) - 1) & ~uint64_t((1u << 20) - 1);
    }
    // Fence completion without a driver call where stream order answers it:
    // on one stream a fence recorded later completes later, so a completed
    // fence vouches for every earlier one on its stream, and a pending one
    // (queried in the last few microseconds) for every later one.  A stale
    // "pending" only delays a buffer's reuse; it never reports a fence done
    // early.  cudaEventQuery takes the driver lock the issuing thread needs
    // for every launch and copy (~1.5 us each).
    struct StreamDone {
        cudaStream_t st;
        uint64_t done_seq, pending_seq;
        std::chrono::steady_clock::time_point pending_at;
    };
    std::vector<StreamDone> stream_done;
    uint64_t host_queries = 0;  // cudaEventQuery calls of the control plane (diagnostics)
    StreamDone &stream_state(cudaStream_t st) {
        for (auto &d : stream_done)
            if (d.st == st) return d;
        stream_done.push_back(StreamDone{st, 0, UINT64_MAX, {}});
        return stream_done.back();
    }
    static bool infer_enabled() {  // SPPIPE_INFER_FENCES=0: query every fence (A/B)
        static const bool on = [] {
            const char *e = getenv("SPPIPE_INFER_FENCES");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    bool passed(Fence &f) {
        if (f.complete) return true;
        if (!f.recorded || !iss.done(f.post_seq)) return false;
        if (!infer_enabled()) {
            ++host_queries;
            if (cudaEventQuery(f.ev) == cudaSuccess) f.complete = true;
            return f.complete;
        }
        StreamDone &sd = stream_state(f.stream);
        if (f.seq <= sd.done_seq) return f.complete = true;
        const auto now = std::chrono::steady_clock::now();
        if (f.seq >= sd.pending_seq && now - sd.pending_at < std::chrono::microseconds(20)) return false;
        ++host_queries;
        if (cudaEventQuery(f.ev) == cudaSuccess) {
            f.complete = true;
            sd.done_seq = std::max(sd.done_seq, f.seq);
            if (sd.pending_seq <= f.seq) sd.pending_seq = UINT64_MAX;
        } else if (f.seq < sd.pending_seq || now - sd.pending_at >= std::chrono::microseconds(20)) {
            sd.pending_seq = f.seq;
            sd.pending_at = now;
        }
        return f.complete;
    }
    // A retired buffer is reusable on stream st without any wait when every
    // other stream that touched it has passed its fence.
    bool reusable(const Garbage &g, cudaStream_t st) {
        for (auto &u : g.uses) {
            if (u.first == st) continue;
            if (!u.second || !u.second->recorded) return false;
            if (!passed(*u.second)) return false;
        }
        return true;
    }
    // Sub-buffers up to slab_max() come from slabs.  The cap sits above 1 MiB
    // + tags so a 1 MiB chunk's staging / ciphertext buffer (1 MiB + 16 B)
    // is bump-allocated too: at 1 MiB it used to take a 2 MiB pool-size
    // class, a pool allocation, a fence and a stream-ordered free per chunk.
    // SPPIPE_SLAB_MAX_KIB overrides (A/B).
    static constexpr uint64_t kSlabBytes = 32ull << 20;
    static uint64_t slab_max() {
        static const uint64_t v = [] {
            const char *e = getenv("SPPIPE_SLAB_MAX_KIB");
            return e ? (uint64_t)atoll(e) << 10 : (uint64_t)((1u << 20) + (64u << 10));
        }();
        return v;
    }
    static bool slabs_enabled() {  // SPPIPE_SLAB=0: every buffer from the pool / cache
        static const bool on = [] {
            const char *e = getenv("SPPIPE_SLAB");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    // open slab per (stream, lane): a handful of keys, searched linearly
    struct OpenSlab {
        cudaStream_t st;
        int lane;
        Rc<Slab> slab;
    };
    std::vector<OpenSlab> slabs;
    Rc<Slab> &open_slab(cudaStream_t st, int lane) {
        for (auto &o : slabs)
            if (o.st == st && o.lane == lane) return o.slab;
        slabs.push_back(OpenSlab{st, lane, Rc<Slab>()});
        return slabs.back().slab;
    }
    // lane separates lifetimes: 0 = transient staging, 1 = device copies of blocks
    BufP alloc(uint64_t n, cudaStream_t st, int lane = 0) {
        if (!dry && n <= slab_max() && slabs_enabled()) {
            auto &sl = open_slab(st, lane);
            const uint64_t need = (std::max<uint64_t>(n, 16) + 255u) & ~uint64_t(255);
            if (!sl || sl->off + need > sl->big->size) {
                sl = pmake<Slab>();
                sl->big = alloc_whole(kSlabBytes, st);
                sl->born = record_new(st, "rec_slab");
            }
            auto b = pmake<Buf>();
            b->plane = this;
            b->size = n;
            b->ptr = sl->big->ptr + sl->off;
            sl->off += need;
            b->slab = sl;
            b->last_stream = st;
            // its range was never used before: other streams need only the
            // slab's allocation to be ordered before them
            b->uses.emplace_back(st, sl->born);
            return b;
        }
        return alloc_whole(n, st);
    }
    BufP alloc_whole(uint64_t n, cudaStream_t st) {
        auto b = pmake<Buf>();
        b->plane = this;
        b->size = n;
        if (!dry) {
            bool cache_reuse = false;  // taken from the cache with every other stream's old fence passed
            FenceP reuse_fence;
            const uint64_t cls = size_class(n);
            auto it = cache.find(cls);
            if (it != cache.end()) {
                // oldest first: the likeliest to have every fence passed
                auto &v = it->second;
                const size_t lim = std::min<size_t>(v.size(), 8);
                for (size_t k = 0; k < lim; ++k) {
                    if (!reusable(v[k], st)) continue;
                    b->ptr = v[k].ptr;
                    // every other stream's old use has passed; st's own old
                    // use (if any) may still run: carry its fence, so a
                    // stream other than st that touches the buffer first
                    // orders after it
                    for (auto &u : v[k].uses)
                        if (u.first == st) reuse_fence = u.second && u.second->recorded ? u.second : record_new(st, "rec_alloc");
                    v.erase(v.begin() + (long)k);
                    cached_bytes -= cls;
                    cache_reuse = true;
                    break;
                }
                // Backpressure: past the pool budget, wait for the oldest
                // retired buffer of this class instead of growing the pool
                // (the host can run a whole trace ahead of the device; an
                // unbounded lead turns into slow pool growth and HBM use).
                if (!b->ptr && pool_bytes + cls > pool_budget()) trim_cache();
                if (!b->ptr && !v.empty() && pool_bytes + cls > pool_budget()) {
                    iss.drain();
                    for (auto &u : v.front().uses) {
                        if (u.second && u.second->recorded) {
                            ck(cudaEventSynchronize(u.second->ev), "pool backpressure");
                        } else if (u.first != st) {
                            FenceP f = record_new(u.first);
                            iss.drain();
                            ck(cudaEventSynchronize(f->ev), "pool backpressure");
                        }
                    }
                    b->ptr = v.front().ptr;
                    v.erase(v.begin());
                    cached_bytes -= cls;
                }
            }
            if (!b->ptr) {
                std::lock_guard<std::mutex> lk(g_dev_mu);
                IdleBufs &ib = g_idle[dev];
                auto it = ib.by_size.find(cls);
                if (it != ib.by_size.end() && !it->second.empty()) {
                    b->ptr = it->second.back();
                    it->second.pop_back();
                    ib.bytes -= cls;
                    pool_bytes += cls;
                }
            }
            bool fresh = false;
            if (!b->ptr) {
                void *p = nullptr;
                ck(cudaMallocFromPoolAsync(&p, cls, pool, st), "cudaMallocFromPoolAsync");
                b->ptr = static_cast<uint8_t *>(p);
                pool_bytes += cls;
                fresh = true;
            }
            b->alloc_size = cls;
            b->last_stream = st;
            // A reused cache buffer carries st's old fence (or nothing when
            // st never touched it).  A fresh pool allocation (or a
            // backpressure / idle-pool buffer) is ordered on st:
            // The allocation point on st, recorded now: another stream that
            // later orders after "st's last use" of this buffer waits only
            // for the allocation, not for whatever st is running by then.
            // (A null entry used to be resolved by recording a fence on st
            // at free time, which made the freeing stream — e.g. the swap-out
            // stream — wait for st's whole backlog: with many 16 MiB
            // swap-ins queued on the compute streams, swap-out seals stalled
            // until the layer's swap-in finished; profiles/r2_dbg_out_waits.)
            if (cache_reuse && !fresh) {
                if (reuse_fence) b->uses.emplace_back(st, reuse_fence);
            } else {
                b->uses.emplace_back(st, record_new(st, "rec_alloc"));
            }
        }
        return b;
    }
    // Return every cached buffer whose fences have all passed (idle) to the
    // pool: frees budget for other size classes without waiting.
    void trim_cache() {
        for (auto &kv : cache) {
            auto &v = kv.second;
            size_t w = 0;
            for (size_t k = 0; k < v.size(); ++k) {
                bool idle = true;
                for (auto &u : v[k].uses)
                    if (u.second && (!u.second->recorded || !passed(*u.second))) {
                        idle = false;
                        break;
                    }
                if (idle) {
                    void *ptr = v[k].ptr;
                    const cudaStream_t st = s.comp;
                    iss.post([ptr, st] { ck(cudaFreeAsync(ptr, st), "cudaFreeAsync(trim)"); }, "free");
                    pool_bytes -= std::min(pool_bytes, kv.first);
                    cached_bytes -= kv.first;
                } else {
                    if (w != k) v[w] = std::move(v[k]);
                    ++w;
                }
            }
            v.resize(w);
        }
    }
    void retire(Buf *b) {
        if (dry || !b->ptr) return;
        Garbage g{b->ptr, std::move(b->uses), b->last_stream, b->alloc_size};
        if (!closing && cached_bytes + b->alloc_size <= kCacheBytes) {
            cache[b->alloc_size].push_back(std::move(g));
            cached_bytes += b->alloc_size;
            return;
        }
        garbage.push_back(std::move(g));
    }
    // Return retired buffers to the pool on the stream of their last use,
    // after every other stream that touched them has passed its fence.
    void collect() {
        if (dry || collecting) return;
        collecting = true;
        std::vector<Garbage> g;
        g.swap(garbage);
        for (auto &x : g) {
            cudaStream_t fs = x.last;
            for (auto &u : x.uses) {
                if (u.first == fs) continue;
                const cudaEvent_t ev = (u.second && u.second->recorded) ? u.second->ev : record_new(u.first, "rec_free")->ev;
                iss.post([fs, ev] { ck(cudaStreamWaitEvent(fs, ev, 0), "cudaStreamWaitEvent(free)"); }, "wait");
            }
            x.uses.clear();
            void *ptr = x.ptr;
            iss.post([ptr, fs] { ck(cudaFreeAsync(ptr, fs), "cudaFreeAsync"); }, "free");
            pool_bytes -= std::min(pool_bytes, x.size);
        }
        collecting = false;
    }

    // -- status slots -------------------------------------------------------------------
    int32_t *status_slot() {
        ++opens_unchecked;
        return auth_d;
    }
    void check_auth() {
        if (dry) return;
        flush();
        if (!opens_unchecked) return;
        iss.drain();
        ck(cudaStreamSynchronize(s.comp), "sync comp");
        ck(cudaStreamSynchronize(s.comp2), "sync comp2");
        ck(cudaStreamSynchronize(s.land), "sync land");
        ck(cudaStreamSynchronize(s.out), "sync out");  // landing opens behind out-stream seals
        ck(cudaStreamSynchronize(s.d2h), "sync d2h");
        opens_unchecked = 0;
        if (*auth_h) {
            *auth_h = 0;
            throw AuthErr("authentication failed on the device");
        }
    }

    // -- compute queue ------------------------------------------------------------------
    void queue(Op &&op, uint64_t nbytes) {
        if (op.wait == window) op.wait.reset();  // queue order covers the current window
        // write-after-read against swap-out seals still reading the buffer on
        // the out stream (partial swap-outs keep the block buffer alive)
        for (int k = 0; k < op.nw; ++k) {
            const Buf *b = op.w[k].buf;
            if (b->out_pending) launch_out();
            for (auto &u : b->uses)
                if (u.first == s.out && u.second && u.second->recorded) flush_waits.push_back(u.second);
        }
        if (op.a) op.a->queued++;
        if (op.b) op.b->queued++;
        ops.push_back(std::move(op));
        ops_bytes += nbytes;
        if (ops_bytes >= batch_bytes) flush();
    }
    static Op make_op(uint32_t opkind, uint32_t dir, uint64_t iv, uint64_t len, const View &src, const View &dst,
                      const BufP &tagbuf, uint64_t tag_off, int32_t *status) {
        Op op;
        op.d.dir = dir;
        op.d.reserved = opkind == SP_OP_OPEN ? (SP_OP_OPEN | SP_STATUS_ON_FAILURE) : opkind;
        op.d.iv = iv;
        op.d.len = len;
        op.d.src = src.ptr();
        op.d.dst = dst.ptr();
        op.d.tag = tagbuf->ptr + tag_off;
        op.d.status = status;
        op.a = src.buf;
        op.b = dst.buf;
        op.r[op.nr++] = Region{src.buf.get(), src.off, src.off + len};
        op.w[op.nw++] = Region{dst.buf.get(), dst.off, dst.off + len};
        if (opkind == SP_OP_SEAL) op.w[op.nw++] = Region{tagbuf.get(), tag_off, tag_off + kTag};
        else op.r[op.nr++] = Region{tagbuf.get(), tag_off, tag_off + kTag};
        return op;
    }

    void flush() {
        if (dry) return;
        issue_pending_copies();
        if (arena_dev && (arena_off || arena_low < arena_dev->size)) {
            // the window's arena is sealed/opened by this flush; the next one starts fresh
            arena_dev.reset();
            arena_off = 0;
            arena_low = 0;
        }
        if (!ops.empty()) {
            std::vector<Op> q;
            q.swap(ops);
            ops.swap(ops_spare);  // keep the queue's capacity across flushes
            ops_bytes = 0;
            // level = 1 + max level of the earlier ops it conflicts with;
            // per-buffer touch lists live in `touches` (no per-flush maps)
            ++touch_epoch;
            touches.clear();
            auto head = [&](const Buf *b) -> int32_t & {
                if (b->touch_epoch != touch_epoch) {
                    b->touch_epoch = touch_epoch;
                    b->touch_head = -1;
                }
                return b->touch_head;
            };
            op_level.assign(q.size(), 0);
            int top = 0;
            for (size_t i = 0; i < q.size(); ++i) {
                const Op &op = q[i];
                int lv = 0;
                auto scan = [&](const Region &rg, bool write) {
                    for (int32_t t = head(rg.buf); t >= 0; t = touches[t].next) {
                        const Touch &x = touches[t];
                        if ((write || x.write) && x.lo < rg.hi && rg.lo < x.hi) lv = std::max(lv, x.level + 1);
                    }
                };
                for (int k = 0; k < op.nr; ++k) scan(op.r[k], false);
                for (int k = 0; k < op.nw; ++k) scan(op.w[k], true);
                op_level[i] = lv;
                top = std::max(top, lv);
                auto add = [&](const Region &rg, bool write) {
                    int32_t &h = head(rg.buf);
                    touches.push_back({rg.lo, rg.hi, lv, write, h});
                    h = (int32_t)touches.size() - 1;
                };
                for (int k = 0; k < op.nr; ++k) add(op.r[k], false);
                for (int k = 0; k < op.nw; ++k) add(op.w[k], true);
            }
            // ops grouped by level, queue order kept inside a level
            level_start.assign((size_t)top + 2, 0);
            for (int lv : op_level) level_start[(size_t)lv + 1]++;
            for (int lv = 0; lv <= top; ++lv) level_start[(size_t)lv + 1] += level_start[(size_t)lv];
            by_level.resize(q.size());
            {
                std::vector<uint32_t> fill(level_start.begin(), level_start.end() - 1);
                for (size_t i = 0; i < q.size(); ++i) by_level[fill[(size_t)op_level[i]]++] = (uint32_t)i;
            }
            const uint64_t mk = ++mark_seq;
            const cudaStream_t cs = (two_comp() && (flush_no++ & 1)) ? s.comp2 : s.comp;
            const cudaStream_t other = cs == s.comp ? s.comp2 : s.comp;
            for (auto &f : flush_waits)
                if (f->mark != mk) {
                    wait(cs, f);
                    f->mark = mk;
                }
            flush_waits.clear();
            if (two_comp()) {
                // what the other compute stream last did to these buffers
                // (or, for buffers allocated on comp, its allocation point)
                FenceP alloc_point;
                auto order_after_other = [&](Buf *b) {
                    for (auto &u : b->uses) {
                        if (u.first != other) continue;
                        if (u.second) {
                            if (!u.second->recorded) continue;  // this flush's own window
                            if (u.second->mark != mk) {
                                wait(cs, u.second);
                                u.second->mark = mk;
                            }
                        } else {
                            if (!alloc_point) alloc_point = record_new(other, "rec_alloc_point");
                            if (alloc_point->mark != mk) {
                                wait(cs, alloc_point);
                                alloc_point->mark = mk;
                            }
                        }
                    }
                };
                for (auto &op : q) {
                    if (op.a) order_after_other(op.a.get());
                    if (op.b && op.b != op.a) order_after_other(op.b.get());
                }
            }
            auto &descs = descs_scratch;
            if (fuse_levels() && top >= 1 && top < (int)kFuseLevels && q.size() <= kLaunchMsgs) {
                // the flush's dependent levels in ONE launch (sp_crypt_levels):
                // level l starts inside the kernel once level l-1 is done, no
                // launch boundary per level.  Every op's input fence is waited
                // for up front.
                descs.clear();
                std::vector<int> starts;
                starts.reserve((size_t)top + 2);
                for (int lv = 0; lv <= top; ++lv) {
                    starts.push_back((int)descs.size());
                    for (uint32_t k = level_start[(size_t)lv]; k < level_start[(size_t)lv + 1]; ++k) {
                        const Op &op = q[by_level[k]];
                        if (op.wait && op.wait->mark != mk) {
                            wait(cs, op.wait);
                            op.wait->mark = mk;
                        }
                        descs.push_back(op.d);
                    }
                }
                starts.push_back((int)descs.size());
                post_levels(descs, std::move(starts), cs);
                ++launches;
                top = -1;  // nothing left for the per-level loop below
            }
            for (int lv = 0; lv <= top; ++lv) {
                descs.clear();
                for (uint32_t k = level_start[(size_t)lv]; k < level_start[(size_t)lv + 1]; ++k) {
                    const Op &op = q[by_level[k]];
                    if (op.wait && op.wait->mark != mk) {
                        wait(cs, op.wait);
                        op.wait->mark = mk;
                    }
                    descs.push_back(op.d);
                }
                if (descs.empty()) continue;
                post_batch(0, descs, cs, "sp_crypt_batch");
                ++launches;
            }
            record(window, cs, "rec_flush");
            if (dbg_times()) dbg_log.push_back({"flush", cs, window, flush_no});
            ++tick;
            for (auto &op : q) {
                if (op.a) {
                    op.a->use(cs, window, tick);
                    op.a->queued--;
                }
                if (op.b) {
                    op.b->use(cs, window, tick);
                    op.b->queued--;
                }
            }
            for (auto &r : ring_pending) ring_commit(r.first, r.second, window);
            ring_pending.clear();
            ring_pending_bytes = 0;
            window = new_fence();
            q.clear();
            if (q.capacity() > ops_spare.capacity()) ops_spare.swap(q);
        }
        launch_out();
        if (!landings.empty()) flush_landings();
        ops_bytes = 0;  // landings count toward the threshold too: everything queued is issued now
        collect();
    }

    bool ring_aliased = false;
    uint8_t *ring_reserve(uint64_t n) {
        if (!ring.ptr) {
            {
                std::lock_guard<std::mutex> lk(g_dev_mu);
                if (!g_rings.empty()) {
                    ring.ptr = g_rings.back().first;
                    ring.cap = g_rings.back().second;
                    g_rings.pop_back();
                }
            }
            if (!ring.ptr) {
                ring.cap = kRingBytes;
                // mapped: the sealing kernel reads small payloads straight from here
                // (no copy-engine transfer queued behind bulk swap copies)
                ck(cudaHostAlloc(reinterpret_cast<void **>(&ring.ptr), ring.cap,
                                 cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc(ring)");
            }
        }
        if (!ring_aliased) {
            void *dp = nullptr;
            if (cudaHostGetDevicePointer(&dp, ring.ptr, 0) == cudaSuccess) add_alias(ring.ptr, ring.cap, dp);
            cudaGetLastError();
            ring_aliased = true;
        }
        if (n > ring.cap) throw ValueErr("small payload larger than the staging ring");
        n = (n + 63u) & ~uint64_t(63);  // 64-byte slots: vectorised kernel reads straight from the ring
        if (ring.head + n > ring.cap) ring.head = 0;
        const uint64_t lo = ring.head, hi = lo + n;
        while (!ring.busy.empty()) {
            auto &b = ring.busy.front();
            const bool overlap = std::get<0>(b) < hi && lo < std::get<1>(b);
            if (overlap) {
                iss.drain();
                ck(cudaEventSynchronize(std::get<2>(b)->ev), "ring slot wait");
            } else if (!passed(*std::get<2>(b))) {
                break;
            }
            ring.busy.pop_front();
        }
        ring.head = hi;
        return ring.ptr + lo;
    }
    void ring_commit(uint8_t *p, uint64_t n, const FenceP &f) {
        const uint64_t lo = (uint64_t)(p - ring.ptr);
        ring.busy.emplace_back(lo, lo + n, f);
    }

    static bool land_on_out_enabled() {  // SPPIPE_LAND_ON_OUT=0: landings always on the land stream (A/B)
        static const bool on = [] {
            const char *e = getenv("SPPIPE_LAND_ON_OUT");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    // Smallest message whose landing open follows its seal on the out stream.
    // Without model compute 4 MiB (small KV opens there queue behind the next
    // decode step's seals: KV swap-only 0.79 vs 0.76 with every landing on
    // out).  Once the model's compute shares the GPU, every size: the open
    // then follows its seal on one stream instead of a cross-stream hop (KV
    // with compute 0.963 -> 0.970 in four A/B pairs, profiles/r2_ab_land_small.txt).
    // SPPIPE_LAND_ON_OUT_MIN=<bytes> fixes it either way.
    uint64_t land_on_out_min() const {
        static const char *e = getenv("SPPIPE_LAND_ON_OUT_MIN");
        if (e) return (uint64_t)atoll(e);
        return app_fence ? 0 : (4ull << 20);
    }
    void flush_landings() {
        std::vector<Landing> ls;
        ls.swap(landings);
        landing_blocks.clear();
        uint64_t total = 0;
        // Landings of >= 4 MiB messages all sealed on the out stream open
        // right behind their seals on that stream: no event hop between the
        // seal and the host endpoint's open (16 MiB-chunk swap-only 0.92 ->
        // 0.97 of plain).  KV evictions keep the landing stream (measured
        // 0.76 vs 0.74 there: their small opens would queue behind the next
        // step's seals).
        bool on_out = land_on_out_enabled();
        for (auto &l : ls)
            for (auto &j : l.jobs) {
                const MsgP &m = std::get<0>(j);
                total += m->len;
                if (!m->ready || !m->ready->recorded || m->ready->stream != s.out || m->len < land_on_out_min()) on_out = false;
            }
        const cudaStream_t ls_st = on_out ? s.out : s.land;
        const uint64_t mk_ready = ++mark_seq;
        for (auto &l : ls)
            for (auto &j : l.jobs) {
                const MsgP &m = std::get<0>(j);
                if (m->ready && m->ready->mark != mk_ready) {
                    wait(ls_st, m->ready);
                    m->ready->mark = mk_ready;
                }
            }
        BufP buf = alloc(total, ls_st);
        std::vector<sp_desc> descs;
        struct Place {
            Block *block;
            uint64_t off, boff, n;
        };
        std::vector<Place> places;
        uint64_t off = 0;
        for (auto &l : ls)
            for (auto &j : l.jobs) {
                const MsgP &m = std::get<0>(j);
                sp_desc d{};
                d.dir = (uint32_t)l.dir;
                d.iv = std::get<1>(j);
                d.len = m->len;
                d.src = m->buf->ptr + m->off;
                d.dst = buf->ptr + off;
                d.tag = m->buf->ptr + m->tag_off;
                d.status = status_slot();
                d.reserved = SP_STATUS_ON_FAILURE;
                descs.push_back(d);
                places.push_back({l.block, off, std::get<2>(j), m->len});
                off += m->len;
            }
        post_batch(2, descs, ls_st, "sp_open_batch(landing)");
        ++launches;
        FenceP opened = record_new(ls_st, "rec_land");
        if (dbg_times()) dbg_log.push_back({"landed", ls_st, opened, dbg_batches});
        ++tick;
        buf->use(ls_st, opened, tick);
        for (auto &l : ls)
            for (auto &j : l.jobs) std::get<0>(j)->buf->use(ls_st, opened, tick);
        wait(s.d2h, opened);
        Block *last = nullptr;
        const uint64_t mk = ++mark_seq;  // one wait per distinct fence (staging copies share a batch fence)
        auto wait_once = [&](const FenceP &f) {
            if (f && f->mark != mk) {
                wait(s.d2h, f);
                f->mark = mk;
            }
        };
        for (auto &p : places) {
            if (p.block != last) {
                auto it = h2d_done.find(p.block->id);
                if (it != h2d_done.end()) wait_once(it->second);
                auto hr = host_ready.find(p.block->id);  // an ordered app write (same stream: no-op otherwise)
                if (hr != host_ready.end()) wait_once(hr->second);
                last = p.block;
            }
        }
        copy_batch_d2h(places.size(), [&](size_t i, void *&dst, void *&src, size_t &n) {
            dst = places[i].block->host + places[i].boff;
            src = buf->ptr + places[i].off;
            n = places[i].n;
        });
        FenceP ev = record_new(s.d2h, "rec_d2h");
        if (dbg_times()) dbg_log.push_back({"d2h-done", s.d2h, ev, dbg_batches});
        buf->use(s.d2h, ev, ++tick);
        for (auto &l : ls) host_ready[l.block->id] = ev;
        bytes_d2h += total;
    }

    // Issue a gathered batch of H2D staging copies on the copy stream.
    void issue(CopyBatch &cb) {
        if (cb.empty()) return;
        const cudaStream_t st = cb.stream ? cb.stream : s.h2d;
        std::unordered_set<Fence *> seen;
        for (auto &f : cb.waits)
            if (f && seen.insert(f.get()).second) wait(st, f);
        copy_batch(st, true, cb.n.size(), [&](size_t i, void *&dst, void *&src, size_t &n) {
            dst = cb.dst[i];
            src = cb.src[i];
            n = cb.n[i];
        });
        record(cb.fence, st, "rec_copy");
        if (dbg_times()) dbg_log.push_back({"h2d-copy", st, cb.fence, dbg_computes});
        ++tick;
        for (auto &b : cb.keep) b->use(st, cb.fence, tick);
        cb.dst.clear();
        cb.src.clear();
        cb.n.clear();
        cb.keep.clear();
        cb.waits.clear();
        cb.fence.reset();
    }
    void issue_pending_copies() {
        issue(otf_copies);
        if (spec_copies) issue(*spec_copies);
    }

    template <class F>
    void copy_batch_d2h(size_t count, F &&get) {
        copy_batch(s.d2h, false, count, get);
    }
    // Device aliases of pinned host memory the plane copies to or from
    // (registered blocks, the token ring): host lo -> (host hi, device lo).
    std::map<uintptr_t, std::pair<uintptr_t, uintptr_t>> host_alias;
    // Ranges with the same host->device offset that touch or sit within 64
    // KiB of each other (page-padded blocks of one pinned slab; under UVA the
    // offset is 0 for all pinned memory) are merged: a 64 KiB-chunk layer
    // registers ~31k blocks, and a lookup per copy walked a map that size.
    // Plane copies never span two blocks, so the padding between merged
    // blocks is never translated.
    void add_alias(const void *host, uint64_t len, const void *dev) {
        if (!host || !dev || !len) return;
        uintptr_t lo = reinterpret_cast<uintptr_t>(host), hi = lo + len;
        const uintptr_t dlo = reinterpret_cast<uintptr_t>(dev);
        const intptr_t delta = (intptr_t)(dlo - lo);
        constexpr uintptr_t kGap = 64u << 10;
        auto it = host_alias.upper_bound(lo);
        if (it != host_alias.begin()) {  // a range starting at or before lo
            auto pv = std::prev(it);
            if ((intptr_t)(pv->second.second - pv->first) == delta && pv->second.first + kGap >= lo) {
                lo = pv->first;
                hi = std::max(hi, pv->second.first);
                host_alias.erase(pv);
            }
        }
        it = host_alias.lower_bound(lo);
        while (it != host_alias.end() && it->first <= hi + kGap &&
               (intptr_t)(it->second.second - it->first) == delta) {  // following ranges
            hi = std::max(hi, it->second.first);
            it = host_alias.erase(it);
        }
        host_alias[lo] = {hi, (uintptr_t)((intptr_t)lo + delta)};
    }
    // device address of [host, host + n), or null when not inside one mapped range
    void *dev_alias(const void *host, uint64_t n) const {
        const uintptr_t a = reinterpret_cast<uintptr_t>(host);
        auto it = host_alias.upper_bound(a);
        if (it == host_alias.begin()) return nullptr;
        --it;
        if (a + n > it->second.first) return nullptr;
        return reinterpret_cast<void *>(it->second.second + (a - it->first));
    }
    // Copies of one flush / batch are posted as one closure.  Copies of <=
    // xfer_max() bytes whose host side is mapped go out as k_xfer launches
    // (<= kXferInline jobs each); the rest as one cudaMemcpyAsync per copy.
    // (The driver's batched copy entry points are not used: on this pool
    // they faulted the GPU.)  SPPIPE_XFER_MAX=0 sends everything to the copy
    // engine (A/B).
    static uint64_t xfer_max() {
        static const uint64_t v = [] {
            const char *e = getenv("SPPIPE_XFER_MAX");
            return e ? (uint64_t)atoll(e) : (uint64_t)(2u << 20);
        }();
        return v;
    }
    uint64_t xfer_launches = 0, xfer_jobs = 0, ce_copies = 0;  // diagnostics
    template <class F>
    void copy_batch(cudaStream_t st, bool h2d, size_t count, F &&get) {
        if (!count) return;
        std::vector<void *> dsts, srcs;
        std::vector<size_t> sizes;
        std::vector<XferJob> jobs;
        jobs.reserve(count);
        const uint64_t xmax = xfer_max();
        for (size_t i = 0; i < count; ++i) {
            void *d = nullptr, *s0 = nullptr;
            size_t n = 0;
            get(i, d, s0, n);
            if (!n) continue;
            void *alias = n <= xmax ? dev_alias(h2d ? s0 : d, n) : nullptr;
            if (alias) {
                jobs.push_back(h2d ? XferJob{static_cast<const uint8_t *>(alias), static_cast<uint8_t *>(d), n}
                                   : XferJob{static_cast<const uint8_t *>(s0), static_cast<uint8_t *>(alias), n});
            } else {
                dsts.push_back(d);
                srcs.push_back(s0);
                sizes.push_back(n);
            }
        }
        xfer_jobs += jobs.size();
        xfer_launches += (jobs.size() + kXferInline - 1) / kXferInline;
        ce_copies += sizes.size();
        iss.post([st, h2d, dsts = std::move(dsts), srcs = std::move(srcs), sizes = std::move(sizes),
                  jobs = std::move(jobs)]() mutable {
            issue_xfers(st, jobs);
            issue_copies(st, h2d, dsts, srcs, sizes);
        }, h2d ? "copy_h2d" : "copy_d2h");
    }
    // Runs on the issuing thread (or inline).
    static void issue_copies(cudaStream_t st, bool h2d, std::vector<void *> &dsts, std::vector<void *> &srcs,
                             std::vector<size_t> &sizes) {
        for (size_t i = 0; i < sizes.size(); ++i)
            ck(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st),
               "batched copy");
    }
    // One 256-thread CTA per 32 KiB of a launch's bytes, 1..64 CTAs (~1 MiB
    // in flight keeps ~50 GB/s over PCIe; more only add SM occupancy).  The
    // parameter block is sized to the job count (the driver copies every
    // parameter byte per launch: 8 jobs 0.2 KiB, 32 0.8 KiB, 128 3 KiB).
    template <int N>
    static void launch_xfer(cudaStream_t st, const XferJob *jobs, uint32_t n) {
        XferParams<N> p;
        p.n = n;
        uint64_t bytes = 0;
        for (uint32_t k = 0; k < n; ++k) {
            p.j[k] = jobs[k];
            bytes += jobs[k].n;
        }
        static const uint64_t max_ctas = [] {  // SPPIPE_XFER_CTAS: grid cap (A/B)
            const char *e = getenv("SPPIPE_XFER_CTAS");
            const long v = e ? atol(e) : 64;
            return (uint64_t)std::max(1L, v);
        }();
        const unsigned ctas = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(max_ctas, (bytes + 32767) >> 15));
        k_xfer<N><<<ctas, kXferThreads, 0, st>>>(p);
        ck(cudaGetLastError(), "k_xfer launch");
    }
    static void issue_xfers(cudaStream_t st, const std::vector<XferJob> &jobs) {
        for (size_t i = 0; i < jobs.size(); i += kXferInline) {
            const uint32_t n = (uint32_t)std::min<size_t>(kXferInline, jobs.size() - i);
            if (n <= 8) launch_xfer<8>(st, jobs.data() + i, n);
            else if (n <= 32) launch_xfer<32>(st, jobs.data() + i, n);
            else launch_xfer<kXferInline>(st, jobs.data() + i, n);
        }
    }
    // One seal / open / mixed launch of libspgcm, issued in order.
    // kind: 0 sp_crypt_batch (per-message op), 1 sp_seal_batch, 2 sp_open_batch
    // Batches of more than 256 messages go out as several launches of <= 256:
    // libspgcm passes up to 256 descriptors inside the kernel parameters,
    // beyond that it stages them with an H2D copy on the launch stream, and
    // that copy waits for a copy engine busy with bulk swap traffic (and
    // throttles the issuing thread on its staging slots).  The messages of
    // one batch are independent, so consecutive launches on the stream (PDL
    // chained) are equivalent.
    static constexpr size_t kLaunchMsgs = 256;
    void post_batch(int kind, const std::vector<sp_desc> &d, cudaStream_t st, const char *what) {
        sp_ctx *c = ctx;
        iss.post([c, kind, st, what, d = std::vector<sp_desc>(d)] {
            for (size_t i = 0; i < d.size(); i += kLaunchMsgs) {
                const int n = (int)std::min(kLaunchMsgs, d.size() - i);
                const sp_desc *p = d.data() + i;
                const int rc = kind == 0 ? sp_crypt_batch(c, p, n, st)
                                         : (kind == 1 ? sp_seal_batch(c, p, n, st) : sp_open_batch(c, p, n, st));
                ck_sp(rc, what);
            }
        }, what);  // profile tag: the launch kind
    }

    static constexpr size_t kFuseLevels = 8;
    // SPPIPE_FUSE_LEVELS=1: multi-level flushes as one sp_crypt_levels launch.
    // Off by default: one launch per level with programmatic dependent launch
    // is faster (a KV seal -> open flush: 15.6 vs 18.5 us for one 224 KiB
    // block, 25.3 vs 31.6 us for eight, profiles/r2_levels_probe.txt; the
    // traces are neutral, r2_ab_fuse_levels.txt): the next grid's CTAs are
    // already resident with their tables filled when the level boundary
    // comes, while the in-kernel hand-off pays a claim, an acquire poll and
    // an exit round trip per warp.
    static bool fuse_levels() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_FUSE_LEVELS");
            return e && e[0] == '1';
        }();
        return on;
    }
    void post_levels(const std::vector<sp_desc> &d, std::vector<int> starts, cudaStream_t st) {
        sp_ctx *c = ctx;
        iss.post([c, st, d = std::vector<sp_desc>(d), starts = std::move(starts)] {
            ck_sp(sp_crypt_levels(c, d.data(), (int)d.size(), starts.data(), (int)starts.size() - 1, st),
                  "sp_crypt_levels");
        }, "sp_crypt_levels");
    }

    void before_host_read_of(int64_t block_id) {
        if (landing_blocks.count(block_id)) flush();
    }

    // -- seals ----------------------------------------------------------------------------
    // H2D the plaintext of `block` [inner+off, +n) per span into one staging
    // buffer; returns the staging buffer (payload views at off-first, tags after).
    // The copy joins `cb` (issued with its batch); `done` is the batch fence.
    BufP stage_h2d(Block &b, uint64_t inner, const Spans &spans, FenceP &done,
                   CopyBatch &cb) {
        before_host_read_of(b.id);
        uint64_t total = 0;
        for (auto &sp : spans) total += sp.second;
        uint64_t first = spans[0].first;
        auto it = host_ready.find(b.id);
        if (it != host_ready.end() && it->second) cb.waits.push_back(it->second);
        BufP buf = alloc(round16(total) + kTag * spans.size(), cb.stream ? cb.stream : s.h2d);
        if (!cb.fence) cb.fence = new_fence();
        cb.dst.push_back(buf->ptr);
        cb.src.push_back(b.host + inner + first);
        cb.n.push_back(total);
        cb.keep.push_back(buf);
        done = cb.fence;
        h2d_done[b.id] = done;
        bytes_h2d += total;
        return buf;
    }

    // KV blocks sealed on the fly read their plaintext straight from the
    // mapped pinned host block (k_gcm's loads cross PCIe): no staging copy,
    // no copy fence, one link less on the swap-in chain of a decode step.
    // Only small on-the-fly KV transfers: a big fused seal would hold every
    // SM for the whole PCIe transfer.  Measured neutral on the OPT-30B KV
    // trace (0.775 vs 0.785 of plain swap-only, 0.937 both with compute;
    // profiles/r2_ab_fuse_h2d.txt), so off by default: SPPIPE_FUSE_H2D=1.
    static bool fuse_h2d_enabled() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_FUSE_H2D");
            return e && e[0] == '1';
        }();
        return on;
    }
    PVec<MsgP> seal_host_chunks(Block &b, uint64_t inner, const Spans &spans,
                                       int dir, uint64_t iv0, bool fuse = false) {
        PVec<MsgP> msgs;
        if (dry) {
            for (auto &sp : spans) {
                auto m = pmake<Msg>();
                m->len = sp.second;
                msgs.push_back(m);
                bytes_h2d += sp.second;
            }
            return msgs;
        }
        if (fuse && b.host_dev && fuse_h2d_enabled()) {
            before_host_read_of(b.id);
            uint64_t first = spans[0].first, total = 0;
            for (auto &sp : spans) total += sp.second;
            if (total <= (1u << 20)) {
                FenceP landed;
                auto it = host_ready.find(b.id);
                if (it != host_ready.end() && it->second && it->second->recorded) landed = it->second;
                BufP buf = alloc(round16(total) + kTag * spans.size(), s.comp);
                for (size_t i = 0; i < spans.size(); ++i) {
                    auto m = pmake<Msg>();
                    m->buf = buf;
                    m->off = spans[i].first - first;
                    m->len = spans[i].second;
                    m->tag_off = round16(total) + kTag * i;
                    Op op;
                    op.d.dir = (uint32_t)dir;
                    op.d.reserved = SP_OP_SEAL;
                    op.d.iv = iv0 + i;
                    op.d.len = m->len;
                    op.d.src = b.host_dev + inner + spans[i].first;
                    op.d.dst = buf->ptr + m->off;
                    op.d.tag = buf->ptr + m->tag_off;
                    op.d.status = nullptr;
                    op.b = buf;
                    op.w[op.nw++] = Region{buf.get(), m->off, m->off + m->len};
                    op.w[op.nw++] = Region{buf.get(), m->tag_off, m->tag_off + kTag};
                    op.wait = landed;  // the block's last landing lands before we read it
                    m->ready = window;
                    queue(std::move(op), m->len);
                    msgs.push_back(m);
                }
                h2d_done[b.id] = window;  // recorded by the flush that issues these seals
                bytes_h2d += total;
                return msgs;
            }
        }
        FenceP done;
        BufP buf = stage_h2d(b, inner, spans, done, otf_copies);
        uint64_t first = spans[0].first, total = 0;
        for (auto &sp : spans) total += sp.second;
        for (size_t i = 0; i < spans.size(); ++i) {
            auto m = pmake<Msg>();
            m->buf = buf;
            m->off = spans[i].first - first;
            m->len = spans[i].second;
            m->tag_off = round16(total) + kTag * i;
            View v{buf, m->off, m->len};
            Op op = make_op(SP_OP_SEAL, (uint32_t)dir, iv0 + i, m->len, v, v, buf, m->tag_off, nullptr);
            op.wait = done;
            m->ready = window;  // before queue(): a threshold flush there issues this op in this window
            queue(std::move(op), m->len);
            msgs.push_back(m);
        }
        return msgs;
    }

    // Encrypt-ahead work of one engine entry point (devplane.SpecBatch).
    struct SpecBatch {
        Plane *p;
        std::vector<sp_desc> items;
        std::vector<BufP> bufs;
        uint64_t bytes = 0;
        FenceP ready;
        FenceP last_copy;
        CopyBatch copies;
        bool stream_set = false;
        explicit SpecBatch(Plane *pl) : p(pl) {
            if (!p->dry) ready = p->new_fence();
        }
        // Small encrypt-ahead staging copies (<= 2 MiB, the k_xfer class) run
        // on their own copy stream, so the demand (on-the-fly) copies on h2d
        // never queue behind them and the two streams' k_xfer launches
        // overlap: KV trace swap-only 0.80 -> 0.82 of plain in three
        // alternating A/B pairs, unchanged with compute
        // (profiles/r2_ab_spec_h2d.txt).  Big ones stay on h2d: on a second
        // copy engine they split PCIe with the demand copies (activation
        // trace, 28 MiB chunks: 0.985 -> 0.954).  SPPIPE_SPEC_H2D=0: all on h2d.
        static bool spec_h2d_enabled() {
            static const bool on = [] {
                const char *e = getenv("SPPIPE_SPEC_H2D");
                return !(e && e[0] == '0');
            }();
            return on;
        }
        ~SpecBatch() {
            if (p->spec_copies == &copies) p->spec_copies = nullptr;
        }
        PVec<MsgP> add(Block &b, uint64_t inner, const Spans &spans, int dir,
                              uint64_t iv0) {
            PVec<MsgP> msgs;
            if (p->dry) {
                for (auto &sp : spans) {
                    auto m = pmake<Msg>();
                    m->len = sp.second;
                    msgs.push_back(m);
                    p->bytes_h2d += sp.second;
                }
                return msgs;
            }
            FenceP done;
            p->spec_copies = &copies;  // a flush while this batch is built issues its copies first
            if (!stream_set) {  // the batch's copy stream, once, by its first chunk's size
                // (one stream per batch: launch() waits only for the last copy)
                uint64_t n = 0;
                for (auto &sp : spans) n += sp.second;
                copies.stream = spec_h2d_enabled() && n <= p->xfer_max() ? p->s.spec_h2d : nullptr;
                stream_set = true;
            }
            BufP buf = p->stage_h2d(b, inner, spans, done, copies);
            last_copy = done;
            uint64_t first = spans[0].first, total = 0;
            for (auto &sp : spans) total += sp.second;
            for (size_t i = 0; i < spans.size(); ++i) {
                auto m = pmake<Msg>();
                m->buf = buf;
                m->off = spans[i].first - first;
                m->len = spans[i].second;
                m->tag_off = round16(total) + kTag * i;
                m->ready = ready;
                sp_desc d{};
                d.dir = (uint32_t)dir;
                d.iv = iv0 + i;
                d.len = m->len;
                d.src = buf->ptr + m->off;
                d.dst = buf->ptr + m->off;
                d.tag = buf->ptr + m->tag_off;
                items.push_back(d);
                msgs.push_back(m);
            }
            bufs.push_back(buf);
            bytes += total;
            if (bytes >= p->batch_bytes) launch();
            return msgs;
        }
        void launch() {
            if (p->dry || items.empty()) return;
            p->issue(copies);
            p->wait(p->s.spec, last_copy);
            p->post_batch(1, items, p->s.spec, "sp_seal_batch(spec)");
            ++p->launches;
            p->record(ready, p->s.spec, "rec_spec");
            if (p->dbg_times()) p->dbg_log.push_back({"spec", p->s.spec, ready, p->dbg_computes});
            ++p->tick;
            for (auto &b : bufs) b->use(p->s.spec, ready, p->tick);
            items.clear();
            bufs.clear();
            bytes = 0;
            ready = p->new_fence();
        }
    };

    PVec<MsgP> seal_device_chunks(const View &src, const Spans &spans, int dir,
                                         uint64_t iv0, bool own_stream = false) {
        PVec<MsgP> msgs;
        if (dry) {
            for (auto &sp : spans) {
                auto m = pmake<Msg>();
                m->len = sp.second;
                msgs.push_back(m);
            }
            return msgs;
        }
        uint64_t total = 0, first = spans[0].first;
        for (auto &sp : spans) total += sp.second;
        if (!own_stream) {  // swap-out seals join the compute queue
            BufP buf = alloc(round16(total) + kTag * spans.size(), s.comp);
            for (size_t i = 0; i < spans.size(); ++i) {
                auto m = pmake<Msg>();
                m->buf = buf;
                m->off = spans[i].first - first;
                m->len = spans[i].second;
                m->tag_off = round16(total) + kTag * i;
                Op op = make_op(SP_OP_SEAL, (uint32_t)dir, iv0 + i, m->len,
                                View{src.buf, src.off + spans[i].first, m->len}, View{buf, m->off, m->len}, buf,
                                m->tag_off, nullptr);
                op.wait = app_fence;  // the model's compute before this swap-out (if any)
                m->ready = window;
                queue(std::move(op), m->len);
                msgs.push_back(m);
            }
            return msgs;
        }
        // the source's writer (a receiver open) must be issued before we can wait for it
        if (src.buf->queued) flush();
        for (auto &u : src.buf->uses)
            if (u.first != s.out && u.second && u.second->recorded) outb.waits.push_back(u.second);
        if (app_fence) outb.waits.push_back(app_fence);  // the model's compute before this swap-out
        if (!outb.ready) outb.ready = new_fence();
        BufP buf = alloc(round16(total) + kTag * spans.size(), s.out);
        for (size_t i = 0; i < spans.size(); ++i) {
            auto m = pmake<Msg>();
            m->buf = buf;
            m->off = spans[i].first - first;
            m->len = spans[i].second;
            m->tag_off = round16(total) + kTag * i;
            sp_desc d{};
            d.dir = (uint32_t)dir;
            d.reserved = SP_OP_SEAL;
            d.iv = iv0 + i;
            d.len = m->len;
            d.src = src.buf->ptr + src.off + spans[i].first;
            d.dst = buf->ptr + m->off;
            d.tag = buf->ptr + m->tag_off;
            outb.items.push_back(d);
            m->ready = outb.ready;
            msgs.push_back(m);
        }
        outb.bufs.push_back(buf);
        outb.bufs.push_back(src.buf);
        src.buf->out_pending++;
        outb.bytes += total;
        if (outb.bytes >= batch_bytes) launch_out();
        return msgs;
    }

    // Where swap-out seals run.  KV-cache evictions (small device-born
    // blocks evicted in groups between decode steps) seal on their own
    // stream, each waiting only for the launch that last wrote its block:
    // the OPT-30B KV trace runs ~25% faster.  Weight/activation chunks join
    // the compute queue: with hundreds of chunks per sync the extra stream
    // costs more buffer reuse across streams than it overlaps (1 MiB-chunk
    // offload 0.90 vs 0.65 of plain).  SPPIPE_OUT_STREAM=0/1 forces either.
    static int out_stream_mode() {
        static const int m = [] {
            const char *e = getenv("SPPIPE_OUT_STREAM");
            return e ? (e[0] == '1' ? 1 : 0) : -1;
        }();
        return m;
    }
    // Chunks of >= 4 MiB seal on the out stream too: a weight swap-out then
    // waits only for its own block's open, not for every swap-in queued
    // ahead of it on the compute streams (256 MiB-block offload without
    // compute 0.84 -> 0.98 of plain, 32 MiB with compute 0.957 -> 0.977;
    // 1 MiB chunks measured better in the queue, 0.915 vs 0.888).
    static bool out_stream_for(bool kv_class, uint64_t len) {
        const int m = out_stream_mode();
        return m < 0 ? (kv_class || len >= (4ull << 20)) : m == 1;
    }

    void launch_out() {
        if (outb.items.empty()) return;
        std::unordered_set<Fence *> seen;
        const uint64_t bno = ++dbg_batches;
        for (auto &f : outb.waits)
            if (seen.insert(f.get()).second) {
                wait(s.out, f);
                if (dbg_times()) dbg_log.push_back({"out-wait", f->stream, f, bno});
            }
        if (dbg_times()) dbg_log.push_back({"out-ready", s.out, outb.ready, bno});
        post_batch(1, outb.items, s.out, "sp_seal_batch(swap-out)");
        ++launches;
        record(outb.ready, s.out, "rec_out");
        ++tick;
        for (auto &b : outb.bufs) {
            b->use(s.out, outb.ready, tick);
            b->out_pending = 0;
        }
        outb = OutBatch{};
    }

    // NOP pads and token I/O: staged in the byte arena (one PCIe copy per flush).
    PVec<MsgP> seal_bytes(const std::vector<std::pair<const uint8_t *, uint64_t>> &payloads, int dir, uint64_t iv0,
                                 bool nop) {
        PVec<MsgP> msgs;
        for (size_t i = 0; i < payloads.size(); ++i) {
            uint64_t n = payloads[i].second;
            auto m = pmake<Msg>();
            m->len = n;
            m->nop = nop;
            if (!dry) {
                // source: the device zero page (NOPs) or the payload in the
                // mapped pinned ring, read by the kernel over PCIe; the sealed
                // message lands in the window's device arena
                const bool zeros = !payloads[i].first && n <= kZeroBytes;
                const uint8_t *src = zero_dev;
                if (!zeros) {
                    if (ring_pending_bytes + n > kRingBytes / 2) flush();  // keep unissued slots clear of wrap-around
                    uint8_t *h = ring_reserve(n);
                    if (payloads[i].first) memcpy(h, payloads[i].first, n);
                    else memset(h, 0, n);
                    ring_pending.push_back({h, n});
                    ring_pending_bytes += n;
                    src = h;
                    bytes_h2d += n;
                }
                uint64_t need = round16(n) + kTag;
                if (!arena_dev || arena_off + need > arena_low) new_arena(need);
                uint64_t o = arena_off;
                arena_off += need;
                m->buf = arena_dev;
                m->off = o;
                m->tag_off = o + need - kTag;
                Op op;
                op.d.dir = (uint32_t)dir;
                op.d.reserved = SP_OP_SEAL;
                op.d.iv = iv0 + i;
                op.d.len = n;
                op.d.src = src;
                op.d.dst = arena_dev->ptr + o;
                op.d.tag = arena_dev->ptr + m->tag_off;
                op.b = arena_dev;
                op.w[op.nw++] = Region{arena_dev.get(), o, o + n};
                op.w[op.nw++] = Region{arena_dev.get(), m->tag_off, m->tag_off + kTag};
                m->ready = window;
                queue(std::move(op), n);
            }
            msgs.push_back(m);
        }
        return msgs;
    }

    // -- opens ----------------------------------------------------------------------------
    // jobs: (msg, iv, dst view or empty) -> queued receiver opens.
    void open_into(PVec<std::tuple<MsgP, uint64_t, View>> &jobs, int dir) {
        if (dry) return;
        for (auto &j : jobs) {
            const MsgP &m = std::get<0>(j);
            View dst = std::get<2>(j);
            if (!dst.buf) dst = arena_scratch(m->len);
            int32_t *st = status_slot();
            Op op = make_op(SP_OP_OPEN, (uint32_t)dir, std::get<1>(j), m->len, View{m->buf, m->off, m->len}, dst,
                            m->buf, m->tag_off, st);
            op.wait = m->ready;
            queue(std::move(op), m->len);
        }
    }

    void land_on_host(Block &b, PVec<std::tuple<MsgP, uint64_t, uint64_t>> jobs, int dir) {
        uint64_t n = 0;
        for (auto &j : jobs) n += std::get<0>(j)->len;
        if (dry) {
            bytes_d2h += n;
            return;
        }
        landings.push_back({&b, std::move(jobs), dir});
        landing_blocks.insert(b.id);
        ops_bytes += n;
        if (ops_bytes >= batch_bytes) flush();
    }

    View new_device_buffer(uint64_t n) { return View{alloc(n, s.comp, 1), 0, n}; }

    // Device-only bytes carved from the current small-payload arena (open
    // destinations of NOPs and token messages): no allocation per message.
    View arena_scratch(uint64_t n) {
        uint64_t need = round16(n);
        if (need > kArenaBytes / 4) return new_device_buffer(n);
        if (!arena_dev || arena_off + need > arena_low) new_arena(need);
        arena_low -= need;
        return View{arena_dev, arena_low, n};
    }
    // Seal the current arena's window (flush) and start a fresh arena.
    void new_arena(uint64_t need) {
        if (arena_dev) flush();
        arena_dev = alloc(std::max(kArenaBytes, need), s.comp);
        arena_off = 0;
        arena_low = arena_dev->size;
    }

    void host_sync(int64_t block_id) {
        if (dry) return;
        flush();
        iss.drain();
        if (block_id == INT64_MIN) {
            ck(cudaStreamSynchronize(s.d2h), "sync d2h");
            return;
        }
        auto it = host_ready.find(block_id);
        if (it != host_ready.end() && it->second) ck(cudaEventSynchronize(it->second->ev), "host_ready sync");
    }
    // An application write into a host block, ordered on the device
    // timeline instead of by a host wait: stream-ordered copies from the
    // pinned staging ring into the block run after every issued landing
    // into the block and every issued H2D read of it, and later H2D reads /
    // landings / app reads order after it through host_ready.
    void ordered_host_write(Block &b, uint64_t offset, const uint8_t *data, uint64_t n) {
        if (!b.host) return;
        if (dry) {
            memcpy(b.host + offset, data, n);
            return;
        }
        flush();  // issue pending landings and staging copies first
        enqueue_host_write(b, offset, data, n, h2d_done[b.id]);
    }
    // On its own stream, so only work on this block waits for the callback.
    void enqueue_host_write(Block &b, uint64_t offset, const uint8_t *data, uint64_t n, const FenceP &reads) {
        if (reads) wait(s.host, reads);
        auto lr = host_ready.find(b.id);  // the block's last landing (or earlier app write)
        if (lr != host_ready.end() && lr->second) wait(s.host, lr->second);
        // Staged in the mapped pinned ring; a small kernel then copies it into
        // the (pinned, UVA-mapped) block over PCIe — no copy-engine transfer
        // that could queue behind bulk swap copies.  Pageable blocks bounce
        // through HBM with two DMA copies.  (A host-to-host cudaMemcpyAsync
        // would block the caller until the stream drains; host functions
        // stall on the callback thread.)
        uint8_t *h = ring_reserve(n);
        memcpy(h, data, n);
        FenceP f;
        const cudaStream_t st = s.host;
        if (b.host_dev) {
            const unsigned blocks = (unsigned)std::min<uint64_t>(148, (n + 4095) / 4096);
            uint8_t *dst = b.host_dev + offset;
            iss.post([blocks, st, dst, h, n] {
                k_bytes<<<blocks, 256, 0, st>>>(dst, h, n);
                ck(cudaGetLastError(), "k_bytes(app write)");
            }, "app_write");
            f = record_new(s.host, "rec_host");
        } else {
            BufP tmp = alloc(n, s.host);
            uint8_t *t = tmp->ptr, *dst = b.host + offset;
            iss.post([st, t, dst, h, n] {
                ck(cudaMemcpyAsync(t, h, n, cudaMemcpyHostToDevice, st), "app write H2D");
                ck(cudaMemcpyAsync(dst, t, n, cudaMemcpyDeviceToHost, st), "app write D2H");
            }, "app_write");
            f = record_new(s.host, "rec_host");
            tmp->use(s.host, f, ++tick);
        }
        ring_commit(h, n, f);
        host_ready[b.id] = f;
    }
    void finish_streams() {
        flush();
        iss.drain();
        cudaStream_t all[10] = {s.comp, s.spec, s.land, s.h2d, s.d2h, s.host, s.out, s.comp2, s.app, s.spec_h2d};
        for (auto st : all) ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    }

    // -- model compute (trace ComputeEvents) -----------------------------------------
    // The app stream runs the model: each compute waits for the swap-in data
    // of the batch synced before it (compute_inputs), and every swap-out
    // seal waits for the compute before it (app_fence) — the dependencies a
    // real layer has.  Swap-ins of later layers do not wait: prefetch
    // overlaps compute, as in FlexGen.
    FenceP compute_inputs[2];  // recorded at each sync (the streams that land swap-in data)
    FenceP app_fence;          // the last compute launch
    unsigned long long *d_spans = nullptr;
    uint64_t span_cap = 0, span_used = 0;
    uint64_t compute_launches = 0, compute_ns_requested = 0;
    static double compute_ns_per_iter(int dev, int sms) {
        // calibrated once per device on an idle GPU (the first compute event
        // of the process pays it, synchronously)
        static std::mutex mu;
        static std::map<int, double> cal;
        std::lock_guard<std::mutex> lk(mu);
        auto it = cal.find(dev);
        if (it != cal.end()) return it->second;
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "calibration stream");
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        const uint64_t iters = 1 << 16;
        double best = 1e30;
        for (int r = 0; r < 4; ++r) {
            ck(cudaEventRecord(a, st), "event");
            k_layer_compute<<<sms * kComputeCtasPerSm * kComputeWaves, kComputeThreads, 0, st>>>(iters, nullptr);
            ck(cudaEventRecord(b, st), "event");
            ck(cudaEventSynchronize(b), "calibration");
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
            if (r) best = std::min(best, (double)ms * 1e6);  // first launch warms up
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(st);
        return cal[dev] = best / (double)iters;
    }
    // Marked at every sync, recorded lazily by the next compute: everything
    // issued on the compute streams by then includes the batch's swap-ins
    // (a trace without compute costs no event records).
    bool compute_inputs_dirty = false;
    void mark_compute_inputs() { compute_inputs_dirty = true; }
    void compute(uint64_t ns, const FenceP *deps, int ndeps) {
        if (dry || !ns) return;
        if (deps == compute_inputs && compute_inputs_dirty) {
            compute_inputs[0] = record_new(s.comp, "rec_compute");
            compute_inputs[1] = record_new(s.comp2, "rec_compute");
            compute_inputs_dirty = false;
        }
        int sms = 148;
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
        const double per_iter = compute_ns_per_iter(dev, sms);
        const uint64_t iters = std::max<uint64_t>(1, (uint64_t)((double)ns / per_iter + 0.5));
        if (span_used == span_cap) {  // grow the span ring (rare): copy the used slots over
            const uint64_t cap = std::max<uint64_t>(4096, span_cap * 2);
            unsigned long long *nd = nullptr;
            iss.drain();
            ck(cudaMalloc(&nd, cap * 2 * sizeof(unsigned long long)), "cudaMalloc(spans)");
            ck(cudaMemset(nd, 0xff, cap * 2 * sizeof(unsigned long long)), "cudaMemset(spans)");
            if (d_spans) {
                ck(cudaStreamSynchronize(s.app), "sync app");
                ck(cudaMemcpy(nd, d_spans, span_used * 2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice),
                   "span copy");
                cudaFree(d_spans);
            }
            d_spans = nd;
            span_cap = cap;
        }
        for (int k = 0; k < ndeps; ++k)
            if (deps[k]) {
                wait(s.app, deps[k]);
                if (dbg_times()) dbg_log.push_back({"comp-in", deps[k]->stream, deps[k], ++dbg_computes});
            }
        unsigned long long *slot = d_spans + 2 * span_used++;
        const cudaStream_t st = s.app;
        const unsigned grid = (unsigned)(sms * kComputeCtasPerSm * kComputeWaves);
        iss.post([iters, slot, st, grid] {
            k_layer_compute<<<grid, kComputeThreads, 0, st>>>(iters, slot);
            ck(cudaGetLastError(), "k_layer_compute launch");
        }, "compute");
        app_fence = record_new(s.app, "rec_compute");
        if (dbg_times()) dbg_log.push_back({"comp-done", s.app, app_fence, dbg_computes});
        ++compute_launches;
        compute_ns_requested += ns;
    }
    // Device time the compute launches took (sum of first-start..last-end),
    // in ns; waits for them.
    uint64_t compute_ns_measured() {
        if (dry || !span_used) return 0;
        iss.drain();
        ck(cudaStreamSynchronize(s.app), "sync app");
        std::vector<unsigned long long> h(2 * span_used);
        ck(cudaMemcpy(h.data(), d_spans, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "spans");
        uint64_t sum = 0;
        for (uint64_t k = 0; k < span_used; ++k) {
            const unsigned long long t0 = h[2 * k], t1 = ~h[2 * k + 1];
            if (t0 != ~0ull && t1 >= t0) sum += t1 - t0;
        }
        return sum;
    }
    void reset_compute_stats() {
        if (d_spans && span_used) {
            iss.drain();
            ck(cudaStreamSynchronize(s.app), "sync app");
            ck(cudaMemset(d_spans, 0xff, span_used * 2 * sizeof(unsigned long long)), "cudaMemset(spans)");
        }
        span_used = 0;
        compute_launches = 0;
        compute_ns_requested = 0;
    }
    // drain_all = false: wait only for work whose results can be observed —
    // every receiver open and verdict (comp; it waited for the encrypt-ahead
    // seals and copies it consumed), swap-out seals, landings and D2H copies,
    // app writes.  What can still run then on the h2d/spec streams is
    // encrypt-ahead of records discarded at finish (engine.py:583-592), which
    // gates nothing (the reference simulator leaves it out of its makespan,
    // simulator.py:441-443); the pipe's destructor drains it.
    void finish(bool drain_all = true) {
        if (dry) return;
        if (drain_all) {
            finish_streams();
        } else {
            flush();
            iss.drain();
            cudaStream_t obs[6] = {s.comp, s.comp2, s.out, s.land, s.d2h, s.host};
            for (auto st : obs) ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        }
        check_auth();
    }
    void copy_to_host(const View &v, void *out) {
        flush();
        iss.drain();
        ck(cudaStreamSynchronize(s.comp), "sync comp");
        ck(cudaStreamSynchronize(s.comp2), "sync comp2");
        ck(cudaStreamSynchronize(s.land), "sync land");
        ck(cudaMemcpy(out, v.ptr(), v.len, cudaMemcpyDeviceToHost), "copy to host");
    }
};

Fence::~Fence() {
    if (plane && ev) (Plane::dbg_times() ? plane->dbg_events : plane->free_events).push_back(ev);
}
Buf::~Buf() {
    if (slab) {
        // fold this sub-buffer's uses into the slab (latest recorded fence
        // per stream; unrecorded ones are kept alongside, as extra entries)
        Buf &into = *slab->big;
        for (auto &u : uses) {
            bool merged = false;
            for (auto &v : into.uses) {
                if (v.first != u.first) continue;
                if (!u.second || v.second == u.second) {
                    merged = true;
                } else if (!v.second) {
                    v.second = u.second;
                    merged = true;
                } else if (v.second->recorded && u.second->recorded) {
                    if (u.second->seq > v.second->seq) v.second = u.second;
                    merged = true;
                }
                if (merged) break;
            }
            if (!merged) into.uses.push_back(u);
        }
        if (last_use >= into.last_use) {
            into.last_use = last_use;
            into.last_stream = last_stream;
        }
        return;  // the slab member releases the slab (and, last, the slab buffer)
    }
    if (plane) plane->retire(this);
}

// ---- engine (engine.py:171-624) --------------------------------------------------------
enum Counter {
    C_HIT, C_IV_AHEAD, C_IV_BEHIND, C_STALE, C_MISS, C_COMMITTED_SENDS, C_ON_THE_FLY, C_DATA_MSGS, C_NOPS,
    C_RELINQUISHES, C_RELINQUISHED_RECORDS, C_NOP_BURNED_RECORDS, C_EXPIRED_RECORDS, C_DEFERRED_DECRYPTS,
    C_SYNC_DECRYPTS, C_WRITE_FAULTS, C_READ_FAULTS, C_SPEC_ENCRYPTS, C_REPLANS, C_REPLANNED_RECORDS, C_SPEC_SKIPPED,
    C_SPEC_CANCELLED, C_SMALL_IO_H2D, C_SMALL_IO_D2H, C_SYNCS, C_SEQ_BATCHES, C_SEQ_HITS, C_SUSPENDED,
    C_SUSPENDED_FALLBACK, C_FINAL_DISCARDED, C_OTF_BURNED_RECORDS, C_COUNT
};
const char *kCounterNames[] = {
    "hit", "iv_ahead", "iv_behind", "stale", "miss", "committed_sends", "on_the_fly", "data_msgs", "nops",
    "relinquishes", "relinquished_records", "nop_burned_records", "expired_records", "deferred_decrypts",
    "sync_decrypts", "write_faults", "read_faults", "spec_encrypts", "replans", "replanned_records",
    "spec_skipped", "spec_cancelled", "small_io_h2d", "small_io_d2h", "syncs", "seq_batches", "seq_hits",
    "suspended", "suspended_fallback", "final_discarded", "otf_burned_records",
    // derived entries appended by sp_pipe_report
    "ring_violations", "ring_high_water", "send_iv", "gpu_send_iv", "otf_burned_present",
};
constexpr int kReportCount = C_COUNT + 5;

struct SpecTask {
    int64_t block_id;
    uint64_t base, len, iv;
    bool cancelled = false;
};
struct Req {
    int dir;
    uint64_t base, len;
    int cls;
    int64_t block_id;
};
struct Suspended {
    Req req;
    int64_t record;
    uint64_t seq;
};
struct Deferred {
    int64_t task_id, block_id;
    uint64_t base, len;
    PVec<std::tuple<MsgP, uint64_t, uint64_t>> chunks;  // msg, iv, offset
    bool done = false, landing = false;
};

// Pending deferred decrypts by task id.  Ids are handed out in increasing
// order, so a deque indexed by (id - first id) with holes for resolved
// tasks replaces an ordered map: O(1) insert / find / erase, iteration in
// id order (the reference's dict order, engine.py:579-581).
class DeferredTable {
  public:
    Deferred *find(int64_t id) {
        if (id < base_ || id >= base_ + (int64_t)q_.size()) return nullptr;
        auto &slot = q_[(size_t)(id - base_)];
        return slot.first ? &slot.second : nullptr;
    }
    Deferred &insert(Deferred &&d) {
        const int64_t id = d.task_id;
        if (q_.empty()) base_ = id;
        if (id < base_ + (int64_t)q_.size()) throw std::logic_error("deferred task ids must increase");
        while (base_ + (int64_t)q_.size() < id) q_.emplace_back(false, Deferred{});
        q_.emplace_back(true, std::move(d));
        ++live_;
        return q_.back().second;
    }
    void erase(int64_t id) {
        Deferred *d = find(id);
        if (!d) return;
        auto &slot = q_[(size_t)(id - base_)];
        slot.first = false;
        slot.second = Deferred{};
        --live_;
        while (!q_.empty() && !q_.front().first) {
            q_.pop_front();
            ++base_;
        }
    }
    bool contains(int64_t id) { return find(id) != nullptr; }
    size_t size() const { return live_; }
    std::vector<int64_t> ids() const {
        std::vector<int64_t> out;
        out.reserve(live_);
        for (size_t i = 0; i < q_.size(); ++i)
            if (q_[i].first) out.push_back(base_ + (int64_t)i);
        return out;
    }

  private:
    std::deque<std::pair<bool, Deferred>> q_;
    int64_t base_ = 0;
    size_t live_ = 0;
};
struct Meta {
    int kind;  // 0 data, 1 small_io, 2 nop
    uint64_t seq;
    int64_t block_id;  // INT64_MIN none
    uint64_t base, offset, nbytes;
};
struct Lane {
    std::deque<MsgP> queue;
    std::deque<sp_sent> log;
};
struct Recorded {
    uint64_t seq, addr, n;
    View view;
};

constexpr int64_t NONE = INT64_MIN;

Spans chunk_spans(uint64_t length, uint64_t chunk) {
    Spans out;
    for (uint64_t off = 0; off < length; off += chunk) out.push_back({off, std::min(chunk, length - off)});
    return out;
}

class Engine {
  public:
    sp_pipe_config cfg;
    Plane plane;  // destroyed last (fences/buffers below point into it)
    HostMem mem;
    Predictor *pred;
    Validator val;
    Lane lanes[2];
    uint64_t send_iv[2], recv_iv[2];  // [H2D]: cpu send / gpu recv; [D2H]: gpu send / cpu recv
    std::deque<sp_action> actions;  // grows without copying (a 64 KiB-chunk run logs ~0.5M actions)
    int64_t counters[C_COUNT] = {};
    bool otf_burned_present = false;
    uint64_t initial_send_iv;
    std::deque<SpecTask> spec_queue;
    std::vector<Suspended> suspended;
    PSet<uint64_t> suspended_seqs;
    std::vector<int64_t> batch_ins, predicted_queue;
    DeferredTable deferred;
    int64_t next_task_id = 1;
    uint64_t next_seq = 0, next_label_iv = 0;
    std::deque<Meta> h2d_meta;
    PUMap<int64_t, View> device_mem;
    std::vector<Recorded> delivered, d2h_stream;
    int64_t ring_occupied = 0, ring_high = 0, ring_insertions = 0, ring_violations = 0;

    Engine(const sp_pipe_config &c, const uint8_t key[32], Predictor *p)
        : cfg(c), plane(c.dry != 0, key, c.batch_bytes ? c.batch_bytes : (64ull << 20), c.reserve_bytes), pred(p),
          val(mem, c.window) {
        val.history = c.record_history;
        if (!plane.dry) {
            ck_sp(sp_ctx_set_max_sms(plane.ctx, (int)c.crypto_sms), "sp_ctx_set_max_sms");
            // small launches (KV batches, tokens, NOP pads) on <= 32 SMs, so
            // they leave the rest to the model's compute and the k_xfer
            // transfers (include/spgcm.h; SPPIPE_SMALL_SMS overrides, 0 = off)
            static const int small_sms = [] {
                const char *e = getenv("SPPIPE_SMALL_SMS");
                return e ? atoi(e) : 32;
            }();
            ck_sp(sp_ctx_set_small_sms(plane.ctx, small_sms), "sp_ctx_set_small_sms");
        }
        if (c.hw_guards) {
            if (spg_init() != SPG_OK) throw std::runtime_error("spg_init failed");
            mem.hw = true;
        }
        send_iv[H2D] = c.initial_h2d_iv;
        send_iv[D2H] = c.initial_d2h_iv;
        recv_iv[H2D] = c.initial_h2d_iv;
        recv_iv[D2H] = c.initial_d2h_iv;
        initial_send_iv = c.initial_h2d_iv;
    }

    // -- channel (channel.py:146-215) --
    void send(int dir, const MsgP &m) {
        nvtx_mark(dir == H2D ? (m->nop ? "h2d nop" : "h2d msg") : (m->nop ? "d2h nop" : "d2h msg"), send_iv[dir]);
        lanes[dir].log.push_back({send_iv[dir], m->len, m->nop ? 1 : 0, 0});
        lanes[dir].queue.push_back(m);
        send_iv[dir] += 1;
    }
    bool pending(int dir) const { return !lanes[dir].queue.empty(); }
    std::pair<MsgP, uint64_t> take(int dir) {
        if (lanes[dir].queue.empty()) throw EngineErr("channel empty");
        MsgP m = lanes[dir].queue.front();
        lanes[dir].queue.pop_front();
        return {m, recv_iv[dir]++};
    }

    uint64_t seq() { return ++next_seq; }
    void act(int kind, int64_t iv = -1, uint64_t nbytes = 0, int64_t record = -1, int64_t task = -1, bool committed = false,
             bool otf = false, int64_t count = 0, int64_t sq = -1) {
        sp_action a{};
        a.kind = kind;
        a.flags = (committed ? 1 : 0) | (otf ? 2 : 0);
        a.iv = iv;
        a.nbytes = nbytes;
        a.record_id = record;
        a.task_id = task;
        a.count = count;
        a.seq = sq;
        actions.push_back(a);
    }

    // -- deferred decrypts --
    void resolve_decrypts_over(uint64_t base, uint64_t len, bool blocking) {
        for (int64_t tid : mem.read_guards_over(base, len)) {
            if (deferred.contains(tid)) apply_decrypt(tid, blocking);
        }
    }
    void apply_decrypt(int64_t tid, bool blocking) {
        Deferred *tp = deferred.find(tid);
        if (!tp || tp->done) return;
        Deferred &t = *tp;
        if (!t.landing) land(t);
        mem.release_read_guard(t.task_id);
        t.done = true;
        int64_t task_id = t.task_id;
        uint64_t len = t.len;
        deferred.erase(tid);
        if (blocking) {
            counters[C_SYNC_DECRYPTS]++;
            act(SP_ACT_RESOLVE_DECRYPT, -1, len, -1, task_id);
        }
    }
    void land(Deferred &t) {
        Block &b = mem.block(t.block_id);
        uint64_t inner = t.base - b.base;
        // the task's chunk list becomes the landing's job list (offsets
        // rebased to the block): nothing reads t.chunks after its landing
        for (auto &c : t.chunks) std::get<2>(c) += inner;
        plane.land_on_host(b, std::move(t.chunks), D2H);
        t.chunks.clear();
        t.landing = true;
    }

    View device_buffer(int64_t block_id) {
        auto it = device_mem.find(block_id);
        if (it != device_mem.end()) return it->second;
        View v = plane.dry ? View{} : plane.new_device_buffer(mem.block(block_id).len);
        device_mem[block_id] = v;
        return v;
    }

    void drain_soon() {
        if (cfg.strict_auth) drain_gpu();
    }

    // GPU endpoint receives everything queued on the H2D lane: one batched open.
    // Where the GPU endpoint puts an H2D message (engine.py:251-267).
    View h2d_destination(const Msg &m, const Meta &meta) {
        if (m.nop) return plane.dry ? View{} : plane.arena_scratch(m.len);
        if (meta.block_id != NONE) {
            Block &b = mem.block(meta.block_id);
            uint64_t inner = meta.base - b.base + meta.offset;
            View whole = device_buffer(meta.block_id);
            return View{whole.buf, whole.off + inner, meta.nbytes};
        }
        return plane.dry ? View{} : plane.arena_scratch(meta.nbytes);
    }
    // The receiver's counter for an H2D message is its send counter (the
    // lane is FIFO and lossless), so the device can open it as soon as it is
    // on the wire instead of at the next drain: opens overlap the rest of the
    // batch's copies rather than piling up at the sync.  The channel state
    // (recv counter, deliveries) still advances at the reference's drain
    // points.  SPPIPE_EAGER_OPEN=0 opens at the drain.
    static bool eager_open() {
        static const bool on = [] {
            const char *e = getenv("SPPIPE_EAGER_OPEN");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    void open_on_send(const MsgP &m, uint64_t iv, const Meta &meta) {
        if (plane.dry || !eager_open()) return;
        View dst = h2d_destination(*m, meta);
        PVec<std::tuple<MsgP, uint64_t, View>> job;
        job.emplace_back(m, iv, dst);
        plane.open_into(job, H2D);
        m->opened = true;
        m->open_iv = iv;
        m->open_dst = dst;
    }
    void drain_gpu() {
        PVec<std::tuple<MsgP, uint64_t, View>> jobs;
        while (pending(H2D)) {
            auto mi = take(H2D);
            Meta meta = h2d_meta.front();
            h2d_meta.pop_front();
            View dst;
            if (mi.first->opened) {
                if (mi.first->open_iv != mi.second) throw EngineErr("H2D receive counter diverged from the send counter");
                dst = mi.first->open_dst;
            } else {
                dst = h2d_destination(*mi.first, meta);
                jobs.emplace_back(mi.first, mi.second, dst);
            }
            if (!mi.first->nop && cfg.record_stream)
                delivered.push_back({meta.seq, meta.base + meta.offset, meta.nbytes, dst});
        }
        plane.open_into(jobs, H2D);
        if (cfg.strict_auth) plane.check_auth();
    }

    void send_h2d(const MsgP &m, int64_t record, const Meta &meta, uint64_t sq) {
        ring_insertions++;
        if (record != NONE && val.rec(record).state != COMMITTED) ring_violations++;
        ring_occupied++;
        ring_high = std::max(ring_high, ring_occupied);
        uint64_t iv = send_iv[H2D];
        if (record == NONE && !cfg.reference_compat) {
            int64_t claimed = val.pending_at_iv(iv);
            if (claimed >= 0) {
                val.invalidate(claimed);
                counters[C_OTF_BURNED_RECORDS]++;
                otf_burned_present = true;
            }
        }
        send(H2D, m);
        h2d_meta.push_back(meta);
        open_on_send(m, iv, meta);
        ring_occupied--;
        counters[C_DATA_MSGS]++;
        act(SP_ACT_H2D_DATA, (int64_t)iv, m->len, record == NONE ? -1 : record, -1, record != NONE, record == NONE, 0,
            (int64_t)sq);
    }

    // -- host-to-device (engine.py:295-349) --
    int submit_h2d(const Req &r, uint64_t &sq) {
        NvtxRange nvtx_("submit_h2d", send_iv[H2D]);
        complete_spec_tasks();
        sq = seq();
        if (r.cls == TC_SMALL) {
            counters[C_SMALL_IO_H2D]++;
            send_on_the_fly(r, sq);
            return V_NONE;
        }
        int64_t rid;
        Verdict v = val.validate(r.base, r.len, send_iv[H2D], rid);
        counters[C_HIT + v]++;
        batch_ins.push_back(r.block_id);
        if (v == V_HIT) {
            commit_and_send(rid, sq);
        } else if (v == V_AHEAD) {
            counters[C_SUSPENDED]++;
            suspended.push_back({r, rid, sq});
            suspended_seqs.insert(sq);
        } else {
            if (v == V_BEHIND) relinquish();
            send_on_the_fly(r, sq);
        }
        return v;
    }

    void send_on_the_fly(const Req &r, uint64_t sq) {
        for (auto &t : spec_queue)
            if (!t.cancelled && t.base == r.base && t.len == r.len) {
                t.cancelled = true;
                counters[C_SPEC_CANCELLED]++;
            }
        resolve_decrypts_over(r.base, r.len, true);
        auto bi = mem.block_at(r.base, r.len);
        auto spans = chunk_spans(r.len, cfg.chunk_bytes);
        auto msgs = plane.seal_host_chunks(*bi.first, bi.second, spans, H2D, send_iv[H2D], r.cls == TC_KV);
        for (size_t i = 0; i < spans.size(); ++i)
            send_h2d(msgs[i], NONE, Meta{0, sq, r.block_id, r.base, spans[i].first, spans[i].second}, sq);
        drain_soon();
        counters[C_ON_THE_FLY]++;
        suspended_seqs.erase(sq);
    }

    void commit_and_send(int64_t rid, uint64_t sq) {
        Record &rec = val.rec(rid);
        if (rec.iv != send_iv[H2D])
            throw EngineErr("commit at counter " + std::to_string(send_iv[H2D]) + " for record at " + std::to_string(rec.iv));
        val.commit(rid);
        uint64_t off = 0;
        PVec<MsgP> chunks = val.rec(rid).chunks;
        PVec<uint64_t> lens = val.rec(rid).chunk_lens;
        int64_t block_id = val.rec(rid).block_id;
        uint64_t base = val.rec(rid).base;
        for (size_t i = 0; i < lens.size(); ++i) {
            MsgP m = plane.dry ? pmake<Msg>() : chunks[i];
            if (plane.dry) m->len = lens[i];
            send_h2d(m, rid, Meta{0, sq, block_id, base, off, lens[i]}, sq);
            off += lens[i];
        }
        val.rec(rid).chunks.clear();  // the lane now owns the payloads
        drain_soon();
        counters[C_COMMITTED_SENDS]++;
        suspended_seqs.erase(sq);
    }

    // -- device-to-host (engine.py:353-393) --
    uint64_t submit_d2h(const Req &r) {
        NvtxRange nvtx_("submit_d2h", send_iv[H2D]);
        complete_spec_tasks();
        if (pending(H2D)) drain_gpu();
        uint64_t sq = seq();
        auto it = device_mem.find(r.block_id);
        if (it == device_mem.end()) throw EngineErr("device does not hold block " + std::to_string(r.block_id));
        View buf = it->second;
        Block &b = mem.block(r.block_id);
        uint64_t inner = r.base - b.base;
        bool swap = r.cls == TC_WEIGHTS || r.cls == TC_KV;
        auto spans = chunk_spans(r.len, cfg.chunk_bytes);
        View src{buf.buf, buf.off + inner, r.len};
        auto msgs = plane.seal_device_chunks(src, spans, D2H, send_iv[D2H], Plane::out_stream_for(r.cls == TC_KV, spans.empty() ? r.len : spans[0].second));
        for (auto &m : msgs) send(D2H, m);
        if (inner == 0 && r.len == b.len) device_mem.erase(r.block_id);
        PVec<std::tuple<MsgP, uint64_t, uint64_t>> taken;
        for (auto &sp : spans) {
            auto mi = take(D2H);
            taken.emplace_back(mi.first, mi.second, sp.first);
        }
        if (swap && cfg.defer_swap_decrypt) {
            int64_t tid = next_task_id++;
            Deferred t;
            t.task_id = tid;
            t.block_id = r.block_id;
            t.base = r.base;
            t.len = r.len;
            t.chunks = std::move(taken);
            Deferred &dt = deferred.insert(std::move(t));
            mem.install_read_guard(r.base, r.len, tid);
            land(dt);
            counters[C_DEFERRED_DECRYPTS]++;
            act(SP_ACT_D2H_DATA, -1, r.len, -1, tid, false, false, 0, (int64_t)sq);
        } else {
            PVec<std::tuple<MsgP, uint64_t, uint64_t>> jobs;
            for (auto &t : taken) jobs.emplace_back(std::get<0>(t), std::get<1>(t), inner + std::get<2>(t));
            plane.land_on_host(b, std::move(jobs), D2H);
            act(SP_ACT_D2H_DATA, -1, r.len, -1, -1, true, false, 0, (int64_t)sq);
        }
        if (swap) pred->observe_swap_out(r.block_id);
        return sq;
    }

    // -- token-sized transfers (engine.py:397-416) --
    void small_io(int dir, const uint8_t *payload, uint64_t size) {
        NvtxRange nvtx_("small_io", send_iv[H2D]);
        complete_spec_tasks();
        uint64_t sq = seq();
        if (dir == H2D) {
            counters[C_SMALL_IO_H2D]++;
            auto msgs = plane.seal_bytes({{payload, size}}, H2D, send_iv[H2D], false);
            send_h2d(msgs[0], NONE, Meta{1, sq, NONE, 0, 0, size}, sq);
            drain_soon();
        } else {
            counters[C_SMALL_IO_D2H]++;
            auto msgs = plane.seal_bytes({{payload, size}}, D2H, send_iv[D2H], false);
            send(D2H, msgs[0]);
            auto mi = take(D2H);
            View dst = plane.dry ? View{} : plane.arena_scratch(size);
            PVec<std::tuple<MsgP, uint64_t, View>> jobs{{mi.first, mi.second, dst}};
            plane.open_into(jobs, D2H);
            if (cfg.record_stream) d2h_stream.push_back({sq, 0, size, dst});
            counters[C_SYNC_DECRYPTS]++;
            act(SP_ACT_D2H_DATA, -1, size, -1, -1, true, false, 0, (int64_t)sq);
        }
    }

    // -- application access (engine.py:420-440) --
    int64_t app_write(int64_t block_id, uint64_t offset, const uint8_t *data, uint64_t n) {
        complete_spec_tasks();
        Block &b = mem.block(block_id);
        resolve_decrypts_over(b.base + offset, n, true);
        if (offset + n > b.len)
            throw BoundsErr("access (" + std::to_string(offset) + ", " + std::to_string(n) + ") outside block " +
                            std::to_string(b.id) + " of " + std::to_string(b.len) + " bytes");
        uint64_t base = b.base + offset;
        std::vector<int64_t> owners;
        for (auto &kv : mem.write_guards)
            if (kv.second.active && HostMem::overlaps(base, n, kv.second.base, kv.second.len)) owners.push_back(kv.first);
        for (int64_t o : owners) {
            mem.release_write_guard(o);
            val.on_write_fault(o);
        }
        plane.ordered_host_write(b, offset, data, n);
        // with page guards, a record labeled after this call must not see the
        // deferred store land on its freshly protected pages: complete it now
        if (mem.hw) plane.host_sync(block_id);
        counters[C_WRITE_FAULTS] += (int64_t)owners.size();
        return (int64_t)owners.size();
    }

    void app_read(int64_t block_id, uint64_t offset, uint64_t n, uint8_t *out) {
        complete_spec_tasks();
        plane.host_sync(block_id);
        Block &b = mem.block(block_id);
        if (offset + n > b.len)
            throw BoundsErr("access (" + std::to_string(offset) + ", " + std::to_string(n) + ") outside block " +
                            std::to_string(b.id) + " of " + std::to_string(b.len) + " bytes");
        auto faults = mem.read_guards_over(b.base + offset, n);
        if (!faults.empty()) {
            counters[C_READ_FAULTS] += (int64_t)faults.size();
            for (int64_t tid : faults)
                if (deferred.contains(tid)) apply_decrypt(tid, true);
            plane.host_sync(block_id);
        }
        if (b.host) memcpy(out, b.host + offset, n);
    }

    // -- pipeline control (engine.py:442-535) --
    void speculate_tick() {
        NvtxRange nvtx_("speculate_tick", send_iv[H2D]);
        complete_spec_tasks();
        if (!cfg.speculate) return;
        auto flat = pred->predict_batches(send_iv[H2D], cfg.leeway, (int)cfg.depth);
        predicted_queue.clear();
        for (auto &p : flat) predicted_queue.push_back(p.block);
        bool trimmed = false;
        if (cfg.window_aware) {
            // whole predicted batches only, while they fit the record window
            size_t keep = 0;
            while (keep < flat.size()) {
                size_t end = keep;
                while (end < flat.size() && flat[end].batch == flat[keep].batch) ++end;
                if (end > (size_t)cfg.window) break;
                keep = end;
            }
            trimmed = keep < flat.size();
            flat.resize(keep);
        }
        std::vector<int64_t> planned;
        {
            std::vector<std::pair<uint64_t, int64_t>> recs;
            for (int64_t id : val.order) recs.push_back({val.rec(id).iv, id});
            std::stable_sort(recs.begin(), recs.end(),
                             [](const std::pair<uint64_t, int64_t> &a, const std::pair<uint64_t, int64_t> &b) {
                                 return a.first < b.first;
                             });
            for (auto &r : recs) planned.push_back(val.rec(r.second).block_id);
            for (auto &t : spec_queue)
                if (!t.cancelled) planned.push_back(t.block_id);
        }
        bool diverged = false;
        for (size_t i = 0; i < std::min(planned.size(), flat.size()); ++i)
            if (planned[i] != flat[i].block) {
                diverged = true;
                break;
            }
        // Window-aware trimming dropped predictions: pending records and
        // queued tasks past the kept plan belong to an earlier plan (the
        // prefix comparison above never sees them) and would hold window
        // slots until sync expiry; discard them like any other replan.
        if (trimmed && planned.size() > flat.size()) diverged = true;
        if (diverged) {
            int64_t n = discard_pipeline();
            counters[C_REPLANS]++;
            counters[C_REPLANNED_RECORDS] += n;
            act(SP_ACT_RELINQUISH, -1, 0, -1, -1, false, false, n);
        }
        int64_t room = (int64_t)cfg.window - (int64_t)val.order.size() - (int64_t)spec_queue.size();
        std::unordered_set<int64_t> queued;
        for (auto &t : spec_queue)
            if (!t.cancelled) queued.insert(t.block_id);
        for (auto &p : flat) {
            if (room <= 0) break;
            Block &b = mem.block(p.block);
            if (queued.count(p.block) || val.has_pending_range(b.base, b.len)) continue;
            uint64_t iv = std::max<uint64_t>(p.iv, next_label_iv);
            next_label_iv = iv + chunk_spans(b.len, cfg.chunk_bytes).size();
            spec_queue.push_back(SpecTask{p.block, b.base, b.len, iv, false});
            queued.insert(p.block);
            --room;
        }
    }

    // Stores that bypassed app_write into mprotect'ed guarded pages: the
    // SIGSEGV handler queued their owners; turn them into write faults
    // (memory.poll_hw_faults -> validator invalidation) before any verdict.
    void poll_hw_faults() {
        int64_t owners[256];
        for (;;) {
            int n = spg_drain(owners, 256);
            for (int i = 0; i < n; ++i) {
                auto it = mem.write_guards.find(owners[i]);
                if (it == mem.write_guards.end() || !it->second.active) continue;
                mem.release_write_guard(owners[i]);
                counters[C_WRITE_FAULTS]++;
                val.on_write_fault(owners[i]);
            }
            if (n < 256) break;
        }
    }

    void complete_spec_tasks() {
        NvtxRange nvtx_("complete_spec_tasks", send_iv[H2D]);
        if (mem.hw) poll_hw_faults();
        if (spec_queue.empty()) return;
        Plane::SpecBatch batch(&plane);
        try {
            label_spec_tasks(batch);
        } catch (...) {
            batch.launch();
            throw;
        }
        batch.launch();
    }

    void label_spec_tasks(Plane::SpecBatch &batch) {
        while (!spec_queue.empty()) {
            SpecTask t = spec_queue.front();
            spec_queue.pop_front();
            if (t.cancelled || !pred->is_outstanding(t.block_id) || val.has_pending_range(t.base, t.len)) {
                counters[C_SPEC_SKIPPED]++;
                continue;
            }
            resolve_decrypts_over(t.base, t.len, false);
            Block &b = mem.block(t.block_id);
            auto spans = chunk_spans(t.len, cfg.chunk_bytes);
            auto msgs = batch.add(b, t.base - b.base, spans, H2D, t.iv);
            PVec<uint64_t> lens;
            for (auto &sp : spans) lens.push_back(sp.second);
            int64_t rid = val.label(plane.dry ? PVec<MsgP>() : std::move(msgs), std::move(lens), t.base, t.len, t.iv, t.block_id);
            counters[C_SPEC_ENCRYPTS]++;
            act(SP_ACT_SPEC_ENCRYPT, (int64_t)t.iv, t.len, rid);
        }
    }

    int64_t discard_pipeline() {
        int64_t n = 0;
        for (int64_t id : val.pending_ids()) {
            val.invalidate(id);
            ++n;
        }
        for (auto &t : spec_queue)
            if (!t.cancelled) {
                t.cancelled = true;
                counters[C_SPEC_CANCELLED]++;
            }
        next_label_iv = 0;
        return n;
    }

    int64_t relinquish() {
        NvtxRange nvtx_("relinquish", send_iv[H2D]);
        int64_t n = discard_pipeline();
        counters[C_RELINQUISHES]++;
        counters[C_RELINQUISHED_RECORDS] += n;
        act(SP_ACT_RELINQUISH, -1, 0, -1, -1, false, false, n);
        return n;
    }

    void pad_to(uint64_t target, int64_t keep_id) {
        NvtxRange nvtx_("pad_to (NOPs)", send_iv[H2D]);
        if (target <= send_iv[H2D]) return;
        uint64_t gap = target - send_iv[H2D];
        std::vector<std::pair<const uint8_t *, uint64_t>> pads(gap, {nullptr, (uint64_t)cfg.nop_bytes});
        auto msgs = plane.seal_bytes(pads, H2D, send_iv[H2D], true);
        for (auto &m : msgs) {
            int64_t burned = val.pending_at_iv(send_iv[H2D]);
            if (burned >= 0 && burned != keep_id) {
                val.invalidate(burned);
                counters[C_NOP_BURNED_RECORDS]++;
            }
            uint64_t iv = send_iv[H2D];
            send(H2D, m);
            h2d_meta.push_back(Meta{2, 0, NONE, 0, 0, cfg.nop_bytes});
            open_on_send(m, iv, h2d_meta.back());
            counters[C_NOPS]++;
            act(SP_ACT_NOP, (int64_t)iv, cfg.nop_bytes);
        }
        drain_soon();
    }

    // -- batch boundary (engine.py:537-577) --
    void sync() {
        NvtxRange nvtx_("sync", send_iv[H2D]);
        complete_spec_tasks();
        std::vector<Suspended> susp(suspended);
        std::stable_sort(susp.begin(), susp.end(),
                         [this](const Suspended &a, const Suspended &b) { return val.rec(a.record).iv < val.rec(b.record).iv; });
        for (auto &s : susp) {
            if (val.rec(s.record).state != PENDING) {
                counters[C_SUSPENDED_FALLBACK]++;
                send_on_the_fly(s.req, s.seq);
                continue;
            }
            pad_to(val.rec(s.record).iv, s.record);
            commit_and_send(s.record, s.seq);
        }
        suspended.clear();
        if (pending(H2D)) drain_gpu();
        counters[C_EXPIRED_RECORDS] += val.invalidate_pending_below(send_iv[H2D]);
        drain_decrypts();
        plane.flush();
        plane.mark_compute_inputs();  // the batch's swap-in data, for the compute after this sync
        if (!batch_ins.empty()) {
            std::vector<int64_t> batch(batch_ins);
            batch_ins.clear();
            counters[C_SEQ_BATCHES]++;
            size_t k = batch.size();
            bool hit = false;
            if (predicted_queue.size() >= k) {
                // set equality (the reference compares sets, engine.py:566-571)
                std::vector<int64_t> a(predicted_queue.begin(), predicted_queue.begin() + (long)k), b(batch);
                std::sort(a.begin(), a.end());
                a.erase(std::unique(a.begin(), a.end()), a.end());
                std::sort(b.begin(), b.end());
                b.erase(std::unique(b.begin(), b.end()), b.end());
                hit = a == b;
            }
            if (hit) {
                counters[C_SEQ_HITS]++;
                predicted_queue.erase(predicted_queue.begin(), predicted_queue.begin() + (long)k);
            } else {
                predicted_queue.clear();
            }
            pred->observe_swap_in(batch);
        }
        pred->observe_sync();
        act(SP_ACT_SYNC_POINT);
        counters[C_SYNCS]++;
        speculate_tick();
        val.compact();  // no suspended request refers to a record here
    }

    void drain_decrypts() {
        std::vector<int64_t> ids;
        ids = deferred.ids();
        for (int64_t id : ids) apply_decrypt(id, false);
    }

    void finish(bool drain_all = true) {
        if (!suspended.empty() || !batch_ins.empty()) sync();
        drain_decrypts();
        for (int64_t id : val.pending_ids()) {
            val.invalidate(id);
            counters[C_FINAL_DISCARDED]++;
        }
        spec_queue.clear();
        if (pending(H2D)) drain_gpu();
        plane.finish(drain_all);
        audit();
    }

    void audit() {
        uint64_t expect = initial_send_iv + (uint64_t)counters[C_DATA_MSGS] + (uint64_t)counters[C_NOPS];
        if (send_iv[H2D] != expect)
            throw EngineErr("counter ledger violated: send counter " + std::to_string(send_iv[H2D]) + ", expected " +
                            std::to_string(expect));
        if (ring_violations)
            throw EngineErr(std::to_string(ring_violations) + " uncommitted payloads reached the shared ring");
    }

    void seed_device(int64_t block_id, const void *src, uint64_t n, bool src_dev) {
        if (plane.dry) {
            device_mem[block_id] = View{};
            return;
        }
        View v = plane.new_device_buffer(n);
        plane.iss.drain();
        ck(cudaMemcpyAsync(v.ptr(), src, n, src_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, plane.s.comp),
           "seed_device copy");
        ck(cudaStreamSynchronize(plane.s.comp), "seed_device sync");
        device_mem[block_id] = v;
    }

    // The unencrypted baseline of the same trace (the simulator's NoCc
    // system, simulator.py SystemKind): every swap is one plain
    // cudaMemcpyAsync between the pinned host block and HBM on the same
    // copy streams, same ordering rules (a block's swap-in waits for its
    // last swap-out to land; swap-outs follow earlier swap-ins), no crypto,
    // no control plane.  Token I/O crosses PCIe from the pinned arena.
    void plain_replay(const sp_event *ev, uint64_t n, const uint8_t *payloads) {
        if (plane.dry) return;
        Plane &pl = plane;
        std::unordered_map<int64_t, View> dev;
        std::unordered_map<int64_t, FenceP> landed;  // block -> its last D2H / app write
        FenceP last_in;
        // Copies gathered per batch boundary (sync) like the engine's flushes,
        // so the baseline gets the same batched-copy advantage.
        struct Pend {
            std::vector<void *> dst, src;
            std::vector<size_t> n;
            std::vector<BufP> keep;
            std::unordered_set<int64_t> blocks;
            std::vector<std::pair<uint8_t *, uint64_t>> ring;  // token slots of the pinned ring it copies
            uint64_t ring_bytes = 0;
            uint64_t bytes = 0;
            void add(void *d, void *s, size_t k, const BufP &b, int64_t blk) {
                dst.push_back(d);
                src.push_back(s);
                n.push_back(k);
                keep.push_back(b);
                if (blk >= 0) blocks.insert(blk);
                bytes += k;
            }
        };
        Pend pin, pout;
        std::unordered_map<int64_t, FenceP> in_fence;  // block -> the H2D flush that carried its swap-in
        FenceP sync_in;                                // swap-ins up to the last sync (what compute reads)
        auto issue = [&](Pend &q, cudaStream_t st, bool h2d) {
            pl.copy_batch(st, h2d, q.n.size(), [&](size_t i, void *&d, void *&src, size_t &k) {
                d = q.dst[i];
                src = q.src[i];
                k = q.n[i];
            });
            FenceP f = pl.record_new(st, "rec_plain");
            ++pl.tick;
            for (auto &b : q.keep) b->use(st, f, pl.tick);
            for (auto &r : q.ring) pl.ring_commit(r.first, r.second, f);
            return f;
        };
        auto flush_in = [&] {
            if (pin.n.empty()) return;
            last_in = issue(pin, pl.s.h2d, true);
            for (int64_t b : pin.blocks) in_fence[b] = last_in;
            pin = Pend{};
        };
        auto flush_out = [&] {
            if (pout.n.empty()) return;
            // a swap-out reads what its own swap-in brought (and what the
            // model computed since), the same dependencies the engine has
            std::unordered_set<Fence *> waited;
            for (int64_t b : pout.blocks) {
                auto it = in_fence.find(b);
                if (it != in_fence.end() && waited.insert(it->second.get()).second) pl.wait(pl.s.d2h, it->second);
            }
            if (pl.app_fence) pl.wait(pl.s.d2h, pl.app_fence);
            FenceP f = issue(pout, pl.s.d2h, false);
            for (int64_t b : pout.blocks) landed[b] = f;
            pout = Pend{};
        };
        const uint64_t kBatch = 64ull << 20;
        for (uint64_t k = 0; k < n; ++k) {
            const sp_event &e = ev[k];
            if (e.kind == SP_EV_SWAP_IN) {
                Block &b = mem.block(e.block);
                if (pout.blocks.count(e.block)) flush_out();  // its last swap-out lands first
                auto it = landed.find(e.block);
                if (it != landed.end()) pl.wait(pl.s.h2d, it->second);
                View v{pl.alloc(b.len, pl.s.h2d, 1), 0, b.len};
                pin.add(v.ptr(), b.host, b.len, v.buf, e.block);
                dev[e.block] = v;
                if (pin.bytes >= kBatch) flush_in();
            } else if (e.kind == SP_EV_SWAP_OUT) {
                Block &b = mem.block(e.block);
                if (pin.blocks.count(e.block)) flush_in();  // its swap-in reaches the device first
                auto it = dev.find(e.block);
                View v = it != dev.end() ? it->second : View{pl.alloc(b.len, pl.s.d2h), 0, b.len};
                auto lt = landed.find(e.block);  // an earlier app write into the block
                if (lt != landed.end()) pl.wait(pl.s.d2h, lt->second);
                pout.add(b.host, v.ptr(), b.len, v.buf, e.block);
                dev.erase(e.block);
                if (pout.bytes >= kBatch) flush_out();
            } else if (e.kind == SP_EV_SYNC) {
                flush_in();
                flush_out();
                sync_in = last_in;
            } else if (e.kind == SP_EV_COMPUTE) {
                pl.compute(e.len, &sync_in, 1);
            } else if (e.kind == SP_EV_APP_WRITE) {
                // the same ordered host write the engine performs (after the block's pending DMA)
                flush_in();
                flush_out();
                Block &b = mem.block(e.block);
                auto lt = landed.find(e.block);
                if (lt != landed.end()) pl.host_ready[e.block] = lt->second;
                pl.enqueue_host_write(b, e.base, payloads + e.payload, e.len, last_in);
                landed[e.block] = pl.host_ready[e.block];
            } else if (e.kind == SP_EV_SMALL_IO_H2D || e.kind == SP_EV_SMALL_IO_D2H) {
                // token copies ride in the batch of their direction (one
                // batched copy closure per sync), through the pinned ring
                const bool h2d = e.kind == SP_EV_SMALL_IO_H2D;
                cudaStream_t st = h2d ? pl.s.h2d : pl.s.d2h;
                View v{pl.alloc(e.len, st), 0, e.len};
                uint8_t *h = pl.ring_reserve(e.len);
                if (h2d && payloads) memcpy(h, payloads + e.payload, e.len);
                Pend &q = h2d ? pin : pout;
                if (h2d) q.add(v.ptr(), h, e.len, v.buf, -1);
                else q.add(h, v.ptr(), e.len, v.buf, -1);
                q.ring.push_back({h, e.len});
                // ring slots are reserved against committed fences only:
                // issue long token runs before the ring could wrap onto them
                q.ring_bytes += (e.len + 63u) & ~uint64_t(63);
                if (q.ring_bytes >= (8ull << 20)) h2d ? flush_in() : flush_out();
            }
        }
        flush_in();
        flush_out();
        dev.clear();
        pl.collect();
        pl.finish_streams();
    }

    // Replay driver (simulator.py:404-426 dispatch, workload event kinds).
    // A trace ComputeEvent (duration in ns): model work on the app stream
    // after the last sync's swap-ins; later swap-outs wait for it.
    void compute(uint64_t ns) {
        NvtxRange nvtx_("compute", send_iv[H2D]);
        complete_spec_tasks();
        plane.compute(ns, plane.compute_inputs, 2);
    }

    void replay(const sp_event *ev, uint64_t n, const uint8_t *payloads, uint64_t *done) {
        for (uint64_t k = 0; k < n; ++k) {
            const sp_event &e = ev[k];
            uint64_t sq;
            switch (e.kind) {
                case SP_EV_SWAP_IN: submit_h2d(Req{H2D, e.base, e.len, e.cls, e.block}, sq); break;
                case SP_EV_SWAP_OUT: submit_d2h(Req{D2H, e.base, e.len, e.cls, e.block}); break;
                case SP_EV_SMALL_IO_H2D: small_io(H2D, payloads ? payloads + e.payload : nullptr, e.len); break;
                case SP_EV_SMALL_IO_D2H: small_io(D2H, payloads ? payloads + e.payload : nullptr, e.len); break;
                case SP_EV_SYNC: sync(); break;
                case SP_EV_APP_WRITE: app_write(e.block, e.base, payloads + e.payload, e.len); break;
                case SP_EV_COMPUTE: compute(e.len); break;
                default: break;
            }
            if (done) *done = k + 1;
        }
    }
};

}  // namespace sppipe

using namespace sppipe;

__global__ void k_xor_byte(uint8_t *p, uint8_t mask) { *p ^= mask; }

struct sp_pred {
    Predictor p;
    explicit sp_pred(const PredConfig &c) : p(c) {}
};
struct sp_pipe {
    std::unique_ptr<Engine> e;
};
// A validator of its own (validator.Validator used without an engine): the
// same class the pipe runs, over an empty host-memory model.
struct sp_val {
    HostMem mem;
    Validator v;
    explicit sp_val(uint64_t window) : v(mem, window) {}
};

namespace {

template <class F>
int guarded(F &&f) {
    try {
        f();
        return SP_OK;
    } catch (const EngineErr &x) {
        g_err = x.what();
        return SP_EENGINE;
    } catch (const OverlapErr &x) {
        g_err = x.what();
        return SP_EOVERLAP;
    } catch (const StateErr &x) {
        g_err = x.what();
        return SP_ESTATE;
    } catch (const UnknownBlockErr &x) {
        g_err = x.what();
        return SP_EUNKNOWN_BLOCK;
    } catch (const BoundsErr &x) {
        g_err = x.what();
        return SP_EBOUNDS;
    } catch (const GuardErr &x) {
        g_err = x.what();
        return SP_EGUARD;
    } catch (const AmbiguousProfileErr &x) {
        g_err = x.what();
        return SP_EAMBIGUOUS;
    } catch (const KeyErr &x) {
        g_err = x.what();
        return SP_EKEY;
    } catch (const AuthErr &x) {
        g_err = x.what();
        return SP_EAUTH;
    } catch (const ValueErr &x) {
        g_err = x.what();
        return SP_EINVAL;
    } catch (const CudaErr &x) {
        g_err = x.what();
        return SP_ECUDA;
    } catch (const std::exception &x) {
        g_err = x.what();
        return SP_ECUDA;
    }
}

PredConfig to_pred_config(const sp_pred_config *c) {
    PredConfig pc;
    if (c) {
        pc.small_io_threshold = c->small_io_threshold;
        pc.swap_min = c->swap_min;
        pc.chunk_bytes = c->chunk_bytes;
        pc.warmup_matches = c->warmup_matches;
        pc.history_cap = c->history_cap;
        pc.layer_param_bytes = c->layer_param_bytes;
        pc.kv_block_bytes = c->kv_block_bytes;
    }
    return pc;
}

}  // namespace

extern "C" {

const char *sp_pipe_last_error(void) { return g_err.c_str(); }

// ---- predictor ---------------------------------------------------------------------------
int sp_pred_create(const sp_pred_config *cfg, sp_pred **out) {
    if (!out) return SP_EINVAL;
    return guarded([&] { *out = new sp_pred(to_pred_config(cfg)); });
}
void sp_pred_destroy(sp_pred *p) { delete p; }
int sp_pred_classify(sp_pred *p, uint64_t size, int32_t *cls) {
    return guarded([&] { *cls = (int32_t)p->p.classify_size(size); });
}
int sp_pred_observe_out(sp_pred *p, int64_t block) {
    return guarded([&] { p->p.observe_swap_out(block); });
}
int sp_pred_observe_in(sp_pred *p, const int64_t *blocks, int32_t n) {
    return guarded([&] { p->p.observe_swap_in(std::vector<int64_t>(blocks, blocks + (n > 0 ? n : 0))); });
}
int sp_pred_observe_sync(sp_pred *p) {
    return guarded([&] { p->p.observe_sync(); });
}
int sp_pred_recognize(sp_pred *p, int32_t *kind, int64_t *confidence, int64_t *phase, int64_t *cycle_len) {
    return guarded([&] {
        Hypothesis h = p->p.recognize();
        *kind = h.kind;
        *confidence = h.confidence;
        *phase = h.phase;
        *cycle_len = (int64_t)h.cycle.size();
    });
}
int sp_pred_cycle_entry(sp_pred *p, int64_t i, int64_t *blocks, int32_t cap, int32_t *n) {
    return guarded([&] {
        Hypothesis h = p->p.recognize();
        if (i < 0 || i >= (int64_t)h.cycle.size()) throw KeyErr("cycle entry " + std::to_string(i));
        const auto &b = p->p.batch_of(h.cycle[(size_t)i]);
        *n = (int32_t)b.size();
        for (int32_t k = 0; k < std::min<int32_t>(cap, *n); ++k) blocks[k] = b[(size_t)k];
    });
}
int sp_pred_predict_batches(sp_pred *p, uint64_t current_iv, uint64_t leeway, int32_t depth, sp_prediction *out,
                            int32_t cap, int32_t *n) {
    return guarded([&] {
        auto v = p->p.predict_batches(current_iv, leeway, depth);
        *n = (int32_t)v.size();
        for (int32_t k = 0; k < std::min<int32_t>(cap, *n); ++k)
            out[k] = sp_prediction{v[(size_t)k].block, v[(size_t)k].iv, v[(size_t)k].leeway, v[(size_t)k].batch, 0};
    });
}
int sp_pred_outstanding(sp_pred *p, int64_t *out, int64_t cap, int64_t *n) {
    return guarded([&] {
        const auto v = p->p.outstanding_list();
        *n = (int64_t)v.size();
        for (int64_t k = 0; k < std::min<int64_t>(cap, *n); ++k) out[k] = v[(size_t)k];
    });
}
int sp_pred_predict_batches_in(sp_pred *p, uint64_t current_iv, uint64_t leeway, int32_t depth,
                               const int64_t *outstanding, int64_t n_out, sp_prediction *out, int32_t cap,
                               int32_t *n) {
    return guarded([&] {
        std::unordered_set<int64_t> outs(outstanding, outstanding + (n_out > 0 ? n_out : 0));
        auto v = p->p.predict_batches(current_iv, leeway, depth, &outs);
        *n = (int32_t)v.size();
        for (int32_t k = 0; k < std::min<int32_t>(cap, *n); ++k)
            out[k] = sp_prediction{v[(size_t)k].block, v[(size_t)k].iv, v[(size_t)k].leeway, v[(size_t)k].batch, 0};
    });
}
int sp_pred_script(sp_pred *p, const sp_prediction *preds, int32_t n, const int64_t *outstanding, int64_t n_out) {
    return guarded([&] {
        std::vector<Prediction> v;
        std::vector<int> rounds;
        for (int32_t k = 0; k < n; ++k) {
            v.push_back({preds[k].block, preds[k].predicted_iv, preds[k].leeway, preds[k].batch});
            rounds.push_back(preds[k].reserved);
        }
        p->p.script(std::move(v), std::vector<int64_t>(outstanding, outstanding + (n_out > 0 ? n_out : 0)),
                    std::move(rounds));
    });
}
int64_t sp_pred_event_count(sp_pred *p) { return (int64_t)p->p.events().size(); }
int sp_pred_event(sp_pred *p, int64_t i, int32_t *kind, int64_t *value) {
    if (i < 0 || i >= (int64_t)p->p.events().size()) {
        g_err = "event " + std::to_string(i);
        return SP_EKEY;
    }
    *kind = p->p.events()[(size_t)i].kind;
    *value = p->p.events()[(size_t)i].a;
    return SP_OK;
}
int sp_pred_in_batch(sp_pred *p, int64_t i, int64_t *blocks, int32_t cap, int32_t *n) {
    return guarded([&] {
        if (i < 0 || i >= (int64_t)p->p.in_batch_count()) throw KeyErr("in-batch " + std::to_string(i));
        const auto &b = p->p.in_batch((size_t)i);
        *n = (int32_t)b.size();
        for (int32_t k = 0; k < std::min<int32_t>(cap, *n); ++k) blocks[k] = b[(size_t)k];
    });
}
int64_t sp_pred_in_batch_count(sp_pred *p) { return (int64_t)p->p.in_batch_count(); }
int64_t sp_pred_decision_count(sp_pred *p) { return (int64_t)p->p.decision_log.size(); }
int sp_pred_decision(sp_pred *p, int64_t i, sp_decision *out) {
    if (i < 0 || i >= (int64_t)p->p.decision_log.size()) return SP_EKEY;
    const Decision &d = p->p.decision_log[(size_t)i];
    *out = sp_decision{d.event, d.pattern, d.confidence, d.after_batches};
    return SP_OK;
}

// ---- pipe ----------------------------------------------------------------------------------
int sp_pipe_create(const sp_pipe_config *cfg, const uint8_t key[SP_KEY_BYTES], sp_pred *pred, sp_pipe **out) {
    if (!cfg || !key || !pred || !out) {
        g_err = "null argument";
        return SP_EINVAL;
    }
    return guarded([&] {
        auto p = new sp_pipe();
        try {
            sp_pipe_config c = *cfg;
            // tri-state window_aware: AUTO (0, a zero-initialised config)
            // follows reference_compat exactly like Python's EngineConfig
            // (window_aware=None: on iff the C2 fix is on)
            if (c.window_aware > SP_WINDOW_AWARE_OFF) {
                g_err = "window_aware must be SP_WINDOW_AWARE_AUTO, _ON or _OFF";
                throw ValueErr(g_err);
            }
            // one channel message per chunk: the reference rejects > 32 MiB
            // plaintexts in encrypt_at (channel.py:92-95)
            if (c.chunk_bytes < 1 || c.chunk_bytes > SP_MAX_MESSAGE_BYTES)
                throw ValueErr("chunk_bytes must be in 1..32 MiB (one channel message per chunk)");
            c.window_aware = c.window_aware == SP_WINDOW_AWARE_AUTO ? (c.reference_compat ? 0 : 1)
                                                                     : (c.window_aware == SP_WINDOW_AWARE_ON ? 1 : 0);
            p->e.reset(new Engine(c, key, &pred->p));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
void sp_pipe_destroy(sp_pipe *p) { delete p; }

int sp_pipe_register_block(sp_pipe *p, int64_t id, uint64_t base, uint64_t len, int32_t kind, void *host) {
    return guarded([&] {
        Block b{id, base, len, kind & 0xff, static_cast<uint8_t *>(host)};
        b.page_owned = (kind & SP_BLOCK_PAGE_OWNED) && (reinterpret_cast<uintptr_t>(host) & 4095u) == 0;
        if (host && !p->e->plane.dry) {
            cudaPointerAttributes a;
            if (cudaPointerGetAttributes(&a, host) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer)
                b.host_dev = static_cast<uint8_t *>(a.devicePointer);
            cudaGetLastError();  // pageable memory: clear the sticky query error
            p->e->plane.add_alias(b.host, len, b.host_dev);
        }
        p->e->mem.add_block(b);
    });
}
int sp_pipe_seed_device(sp_pipe *p, int64_t block, const void *src, uint64_t len, int32_t src_is_device) {
    return guarded([&] { p->e->seed_device(block, src, len, src_is_device != 0); });
}
int sp_pipe_submit_h2d(sp_pipe *p, uint64_t base, uint64_t len, int32_t cls, int64_t block, uint64_t *seq,
                       int32_t *verdict) {
    return guarded([&] {
        uint64_t sq = 0;
        int v = p->e->submit_h2d(Req{H2D, base, len, cls, block}, sq);
        if (seq) *seq = sq;
        if (verdict) *verdict = v;
    });
}
int sp_pipe_submit_d2h(sp_pipe *p, uint64_t base, uint64_t len, int32_t cls, int64_t block, uint64_t *seq) {
    return guarded([&] {
        uint64_t sq = p->e->submit_d2h(Req{D2H, base, len, cls, block});
        if (seq) *seq = sq;
    });
}
int sp_pipe_small_io(sp_pipe *p, int32_t dir, const void *payload, uint64_t size) {
    if (dir != H2D && dir != D2H) {
        g_err = "unknown direction";
        return SP_EINVAL;
    }
    return guarded([&] { p->e->small_io(dir, static_cast<const uint8_t *>(payload), size); });
}
int sp_pipe_sync(sp_pipe *p) {
    return guarded([&] { p->e->sync(); });
}
int sp_pipe_speculate(sp_pipe *p) {
    return guarded([&] { p->e->speculate_tick(); });
}
int sp_pipe_relinquish(sp_pipe *p, int64_t *count) {
    return guarded([&] {
        int64_t n = p->e->relinquish();
        if (count) *count = n;
    });
}
int sp_pipe_drain_decrypts(sp_pipe *p) {
    return guarded([&] { p->e->drain_decrypts(); });
}
int sp_pipe_finish(sp_pipe *p) {
    return guarded([&] { p->e->finish(); });
}
int sp_pipe_audit(sp_pipe *p) {
    return guarded([&] { p->e->audit(); });
}
int sp_pipe_finish_observable(sp_pipe *p) {
    return guarded([&] { p->e->finish(false); });
}
int sp_pipe_flush(sp_pipe *p, int32_t wait) {
    return guarded([&] {
        if (p->e->plane.dry) return;
        if (wait) p->e->plane.finish_streams();
        else p->e->plane.flush();
    });
}
int sp_pipe_app_write(sp_pipe *p, int64_t block, uint64_t offset, const void *data, uint64_t n, int64_t *faults) {
    return guarded([&] {
        int64_t f = p->e->app_write(block, offset, static_cast<const uint8_t *>(data), n);
        if (faults) *faults = f;
    });
}
int sp_pipe_app_read(sp_pipe *p, int64_t block, uint64_t offset, uint64_t n, void *out) {
    return guarded([&] { p->e->app_read(block, offset, n, static_cast<uint8_t *>(out)); });
}
int sp_pipe_plain_replay(sp_pipe *p, const sp_event *ev, uint64_t n, const uint8_t *payloads) {
    return guarded([&] { p->e->plain_replay(ev, n, payloads); });
}
int sp_pipe_replay(sp_pipe *p, const sp_event *ev, uint64_t n, const uint8_t *payloads, uint64_t *done) {
    if (done) *done = 0;
    return guarded([&] { p->e->replay(ev, n, payloads, done); });
}
int sp_test_xfer(int32_t n, void *const *dst, const void *const *src, const uint64_t *len) {
    if (n < 0 || n > kXferInline || (n && (!dst || !src || !len))) {
        g_err = "sp_test_xfer: 0 <= n <= 128 jobs with non-null arrays";
        return SP_EINVAL;
    }
    return guarded([&] {
        std::vector<XferJob> jobs;
        for (int32_t i = 0; i < n; ++i)
            jobs.push_back(XferJob{static_cast<const uint8_t *>(src[i]), static_cast<uint8_t *>(dst[i]), len[i]});
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        Plane::issue_xfers(st, jobs);
        const cudaError_t e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        ck(e, "sp_test_xfer");
    });
}
int sp_pipe_test_corrupt(sp_pipe *p, int32_t dir, uint64_t index, uint64_t byte_index, uint8_t mask) {
    return guarded([&] {
        Engine &e = *p->e;
        auto &q = e.lanes[dir & 1].queue;
        if (index >= q.size()) throw KeyErr("no in-flight message " + std::to_string(index));
        const MsgP &m = q[(size_t)index];
        if (byte_index >= m->len) throw ValueErr("byte index outside the message");
        if (e.plane.dry || !m->buf) return;
        e.plane.flush();  // its seal is issued; the flip is ordered after it on its producer stream
        e.plane.iss.drain();
        cudaStream_t st = m->ready && m->ready->recorded ? m->ready->stream : e.plane.s.comp;
        k_xor_byte<<<1, 1, 0, st>>>(m->buf->ptr + m->off + byte_index, mask);
        ck(cudaGetLastError(), "k_xor_byte");
        ck(cudaStreamSynchronize(st), "test corrupt");
        if (m->opened) {
            // opened on send already: the receiver sees the flipped bytes now
            PVec<std::tuple<MsgP, uint64_t, View>> job;
            job.emplace_back(m, m->open_iv, m->open_dst);
            e.plane.open_into(job, dir & 1);
            e.plane.flush();
        }
    });
}
int sp_pipe_handle_done(sp_pipe *p, uint64_t seq, int32_t *done) {
    *done = (seq >= 1 && seq <= p->e->next_seq && !p->e->suspended_seqs.count(seq)) ? 1 : 0;
    return SP_OK;
}

int sp_pipe_report(sp_pipe *p, int64_t *out, int32_t cap, int32_t *n) {
    Engine &e = *p->e;
    int64_t v[kReportCount];
    for (int i = 0; i < C_COUNT; ++i) v[i] = e.counters[i];
    v[C_COUNT + 0] = e.ring_violations;
    v[C_COUNT + 1] = e.ring_high;
    v[C_COUNT + 2] = (int64_t)e.send_iv[H2D];
    v[C_COUNT + 3] = (int64_t)e.send_iv[D2H];
    v[C_COUNT + 4] = e.otf_burned_present ? 1 : 0;
    *n = kReportCount;
    for (int i = 0; i < std::min<int32_t>(cap, kReportCount); ++i) out[i] = v[i];
    return SP_OK;
}
const char *sp_pipe_counter_name(int32_t i) {
    if (i < 0 || i >= kReportCount) return nullptr;
    return kCounterNames[i];
}
uint64_t sp_pipe_send_iv(sp_pipe *p, int32_t dir) { return p->e->send_iv[dir & 1]; }
uint64_t sp_pipe_recv_iv(sp_pipe *p, int32_t dir) { return p->e->recv_iv[dir & 1]; }
int64_t sp_pipe_action_count(sp_pipe *p) { return (int64_t)p->e->actions.size(); }
int sp_pipe_actions(sp_pipe *p, int64_t from, sp_action *out, int64_t cap, int64_t *n) {
    auto &a = p->e->actions;
    int64_t k = 0;
    for (int64_t i = from; i < (int64_t)a.size() && k < cap; ++i) out[k++] = a[(size_t)i];
    *n = k;
    return SP_OK;
}
int64_t sp_pipe_sent_count(sp_pipe *p, int32_t dir) { return (int64_t)p->e->lanes[dir & 1].log.size(); }
int sp_pipe_sent_log(sp_pipe *p, int32_t dir, int64_t from, sp_sent *out, int64_t cap, int64_t *n) {
    auto &l = p->e->lanes[dir & 1].log;
    int64_t k = 0;
    for (int64_t i = from; i < (int64_t)l.size() && k < cap; ++i) out[k++] = l[(size_t)i];
    *n = k;
    return SP_OK;
}
int64_t sp_pipe_record_count(sp_pipe *p) { return p->e->val.next_id - 1; }
int64_t sp_pipe_record_first(sp_pipe *p) { return p->e->val.first_id; }
int sp_pipe_pending(sp_pipe *p, int64_t *ids, int64_t cap, int64_t *n) {
    return guarded([&] {
        *n = (int64_t)p->e->val.order.size();
        int64_t k = 0;
        for (int64_t id : p->e->val.order) {
            if (k >= cap) break;
            ids[k++] = id;
        }
    });
}
int64_t sp_pipe_pending_at_iv(sp_pipe *p, uint64_t iv) { return p->e->val.pending_at_iv(iv); }
int sp_pipe_record(sp_pipe *p, int64_t id, sp_record *out) {
    Validator &v = p->e->val;
    if (!v.retained(id)) {
        g_err = id >= 1 && id < v.first_id ? "record " + std::to_string(id) + " compacted (record_history)"
                                           : "no record " + std::to_string(id);
        return SP_EKEY;
    }
    const Record &r = v.rec(id);
    *out = sp_record{r.id, r.base, r.len, r.iv, r.span(), r.block_id, (int32_t)r.state, 0};
    return SP_OK;
}
int64_t sp_pipe_delivered_count(sp_pipe *p, int32_t which) {
    return (int64_t)(which ? p->e->d2h_stream.size() : p->e->delivered.size());
}
int sp_pipe_delivered(sp_pipe *p, int32_t which, int64_t i, sp_delivery *out, void *bytes) {
    auto &v = which ? p->e->d2h_stream : p->e->delivered;
    if (i < 0 || i >= (int64_t)v.size()) return SP_EKEY;
    const Recorded &r = v[(size_t)i];
    *out = sp_delivery{r.seq, r.addr, r.n};
    if (!bytes) return SP_OK;
    return guarded([&] {
        if (p->e->plane.dry || !r.view.buf) throw ValueErr("the dry plane holds no bytes");
        if (p->e->pending(H2D)) p->e->drain_gpu();
        p->e->plane.copy_to_host(r.view, bytes);
    });
}
int sp_pipe_pool_stats(sp_pipe *p, uint64_t *reserved, uint64_t *used, uint64_t *cached) {
    Plane &pl = p->e->plane;
    uint64_t r = 0, u = 0;
    if (!pl.dry) {
        unsigned long long v = 0;
        if (cudaMemPoolGetAttribute(pl.pool, cudaMemPoolAttrReservedMemCurrent, &v) == cudaSuccess) r = v;
        if (cudaMemPoolGetAttribute(pl.pool, cudaMemPoolAttrUsedMemCurrent, &v) == cudaSuccess) u = v;
    }
    if (reserved) *reserved = r;
    if (used) *used = u;
    if (cached) *cached = pl.cached_bytes;
    return SP_OK;
}
int sp_pipe_issuer_stats(sp_pipe *p, uint64_t *calls, uint64_t *busy_ns, uint64_t *host_queries) {
    if (calls) *calls = p->e->plane.iss.calls_.load();
    if (busy_ns) *busy_ns = p->e->plane.iss.busy_ns_.load();
    if (host_queries) *host_queries = p->e->plane.host_queries;
    return SP_OK;
}
int sp_pipe_compute(sp_pipe *p, uint64_t duration_ns) {
    return guarded([&] { p->e->compute(duration_ns); });
}
int sp_pipe_compute_stats(sp_pipe *p, uint64_t *launches, uint64_t *requested_ns, uint64_t *measured_ns) {
    return guarded([&] {
        if (launches) *launches = p->e->plane.compute_launches;
        if (requested_ns) *requested_ns = p->e->plane.compute_ns_requested;
        if (measured_ns) *measured_ns = p->e->plane.compute_ns_measured();
    });
}
int sp_pipe_stats(sp_pipe *p, uint64_t *bytes_h2d, uint64_t *bytes_d2h, uint64_t *launches) {
    if (bytes_h2d) *bytes_h2d = p->e->plane.bytes_h2d;
    if (bytes_d2h) *bytes_d2h = p->e->plane.bytes_d2h;
    if (launches) *launches = p->e->plane.launches;
    return SP_OK;
}


// ---- standalone validator (validator.Validator, validator.py:90-236) -------------------------
int sp_val_create(uint64_t window, sp_val **out) {
    if (!out) return SP_EINVAL;
    return guarded([&] { *out = new sp_val(window); });
}
void sp_val_destroy(sp_val *v) { delete v; }
int sp_val_label(sp_val *v, uint64_t base, uint64_t len, uint64_t iv, uint64_t span, int64_t block_id, int64_t *id) {
    return guarded([&] {
        if (span < 1) throw ValueErr("a record spans at least one counter");
        PVec<uint64_t> lens;
        for (uint64_t k = 0; k < span; ++k) lens.push_back(0);
        *id = v->v.label(PVec<MsgP>(), std::move(lens), base, len, iv, block_id);
    });
}
int sp_val_validate(sp_val *v, uint64_t base, uint64_t len, uint64_t current_iv, int32_t *verdict, int64_t *record_id) {
    return guarded([&] {
        int64_t rid = -1;
        *verdict = v->v.validate(base, len, current_iv, rid);
        *record_id = rid;
    });
}
int sp_val_commit(sp_val *v, int64_t id) {
    return guarded([&] {
        if (id < 1 || id >= v->v.next_id) throw KeyErr(std::to_string(id));
        v->v.commit(id);
    });
}
int sp_val_invalidate(sp_val *v, int64_t id) {
    return guarded([&] {
        if (id < 1 || id >= v->v.next_id) throw KeyErr(std::to_string(id));
        v->v.invalidate(id);
    });
}
int sp_val_write_fault(sp_val *v, int64_t owner) {
    return guarded([&] { v->v.on_write_fault(owner); });
}
int64_t sp_val_pending_at_iv(sp_val *v, uint64_t iv) { return v->v.pending_at_iv(iv); }
int32_t sp_val_has_pending_range(sp_val *v, uint64_t base, uint64_t len) { return v->v.has_pending_range(base, len) ? 1 : 0; }
int sp_val_invalidate_pending_below(sp_val *v, uint64_t iv, int64_t *n) {
    return guarded([&] { *n = v->v.invalidate_pending_below(iv); });
}
int sp_val_pending(sp_val *v, int64_t *ids, int64_t cap, int64_t *n) {
    return guarded([&] {
        *n = (int64_t)v->v.order.size();
        int64_t k = 0;
        for (int64_t id : v->v.order) {
            if (k >= cap) break;
            ids[k++] = id;
        }
    });
}
int64_t sp_val_record_count(sp_val *v) { return v->v.next_id - 1; }
int sp_val_record(sp_val *v, int64_t id, sp_record *out) {
    if (!v->v.retained(id)) {
        g_err = "no record " + std::to_string(id);
        return SP_EKEY;
    }
    const Record &r = v->v.rec(id);
    *out = sp_record{r.id, r.base, r.len, r.iv, r.span(), r.block_id, (int32_t)r.state, 0};
    return SP_OK;
}
int sp_val_counters(sp_val *v, int64_t out[6]) {
    for (int k = 0; k < 5; ++k) out[k] = v->v.counters[k];
    out[5] = v->v.evicted;
    return SP_OK;
}

}  // extern "C"

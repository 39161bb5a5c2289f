// libspguard: mprotect-based write guards with a SIGSEGV fault ring.
// See include/spguard.h.  Async-signal-safety: the handler only reads the
// guard table with atomic loads, calls mprotect (a plain syscall) and pushes
// into a lock-free ring; table updates from normal context use a spinlock
// that the handler never takes.
#define _GNU_SOURCE
#include <errno.h>
#include <signal.h>
#include <stdatomic.h>
#include <stdint.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

#include "spguard.h"

#define SPG_MAX_GUARDS 4096
#define SPG_RING 8192
#define SPG_TOMB 1024  // recently lifted ranges (see handler)

typedef struct {
    _Atomic uintptr_t lo;   // first protected page (0 = free slot)
    _Atomic uintptr_t hi;   // one past the last protected page
    _Atomic int64_t owner;
    _Atomic int active;
} guard_t;

static guard_t g_guards[SPG_MAX_GUARDS];
static _Atomic int g_lock = 0;
static _Atomic int g_nactive = 0;
static _Atomic uint64_t g_faults = 0;
static _Atomic int64_t g_ring[SPG_RING];
static _Atomic uint32_t g_head = 0, g_tail = 0;  // head: next write, tail: next read
static struct sigaction g_prev;
static _Atomic int g_inited = 0;
static _Atomic int g_errno = 0;
static _Atomic uint64_t g_uncovered = 0;  // guards whose byte range is not fully under protection
static uintptr_t g_page = 4096;
// Tombstones: ranges whose protection was lifted by spg_release.  A store
// that faulted just before the lift may reach the handler after the slot
// was cleared; finding its range here, the handler lets it retry on the
// (now writable) page instead of treating the fault as foreign.
static _Atomic uintptr_t g_tomb_lo[SPG_TOMB], g_tomb_hi[SPG_TOMB];
static _Atomic uint32_t g_tomb_head = 0;

static void lock(void) {
    int expected = 0;
    while (!atomic_compare_exchange_weak(&g_lock, &expected, 1)) expected = 0;
}
static void unlock(void) { atomic_store(&g_lock, 0); }

static void ring_push(int64_t owner) {
    uint32_t h = atomic_fetch_add(&g_head, 1u);
    atomic_store(&g_ring[h % SPG_RING], owner);
}

static void handler(int sig, siginfo_t *info, void *uctx) {
    const uintptr_t a = (uintptr_t)info->si_addr;
    int hit = 0;
    // 1. an active guard covering the address: the first faulting thread
    //    lifts it and records the owner
    for (int i = 0; i < SPG_MAX_GUARDS; ++i) {
        if (!atomic_load(&g_guards[i].active)) continue;
        const uintptr_t lo = atomic_load(&g_guards[i].lo), hi = atomic_load(&g_guards[i].hi);
        if (a >= lo && a < hi) {
            int one = 1;
            if (atomic_compare_exchange_strong(&g_guards[i].active, &one, 0)) {
                mprotect((void *)lo, hi - lo, PROT_READ | PROT_WRITE);
                ring_push(atomic_load(&g_guards[i].owner));
                atomic_fetch_add(&g_faults, 1u);
                atomic_fetch_sub(&g_nactive, 1);
            }
            hit = 1;
        }
    }
    if (hit) return;  // the faulting store retries on a writable page
    // 2. a guard another thread (a concurrent fault, or spg_release) is
    //    lifting right now: its slot is inactive but still holds the range;
    //    the store retries and faults again until the mprotect has landed
    for (int i = 0; i < SPG_MAX_GUARDS; ++i) {
        const uintptr_t lo = atomic_load(&g_guards[i].lo), hi = atomic_load(&g_guards[i].hi);
        if (lo && a >= lo && a < hi) return;
    }
    // 3. a range lifted by a release that has since cleared its slot
    for (int i = 0; i < SPG_TOMB; ++i) {
        const uintptr_t lo = atomic_load(&g_tomb_lo[i]), hi = atomic_load(&g_tomb_hi[i]);
        if (lo && a >= lo && a < hi) return;
    }
    // not ours: hand over to whoever was installed before us
    if (g_prev.sa_flags & SA_SIGINFO) {
        if (g_prev.sa_sigaction) { g_prev.sa_sigaction(sig, info, uctx); return; }
    } else if (g_prev.sa_handler != SIG_DFL && g_prev.sa_handler != SIG_IGN && g_prev.sa_handler) {
        g_prev.sa_handler(sig);
        return;
    }
    signal(sig, SIG_DFL);
    raise(sig);
}

int spg_init(void) {
    if (atomic_exchange(&g_inited, 1)) return SPG_OK;
    long ps = sysconf(_SC_PAGESIZE);
    if (ps > 0) g_page = (uintptr_t)ps;
    struct sigaction sa;
    memset(&sa, 0, sizeof(sa));
    sa.sa_sigaction = handler;
    sa.sa_flags = SA_SIGINFO | SA_NODEFER;
    sigemptyset(&sa.sa_mask);
    if (sigaction(SIGSEGV, &sa, &g_prev) != 0) {
        atomic_store(&g_errno, errno);
        atomic_store(&g_inited, 0);
        return SPG_ESYS;
    }
    return SPG_OK;
}

int spg_protect_ex(const void *addr, size_t len, int64_t owner, int flags) {
    if (!addr || !len || (flags & ~(SPG_HEAD_OWNED | SPG_TAIL_OWNED))) return SPG_EINVAL;
    if (!atomic_load(&g_inited) && spg_init() != SPG_OK) return SPG_ESYS;
    const uintptr_t a = (uintptr_t)addr;
    // whole pages inside the range; a partial head / tail page is included
    // when the caller owns the rest of that page exclusively
    const uintptr_t lo = (flags & SPG_HEAD_OWNED) ? a & ~(g_page - 1) : (a + g_page - 1) & ~(g_page - 1);
    const uintptr_t hi = (flags & SPG_TAIL_OWNED) ? (a + len + g_page - 1) & ~(g_page - 1) : (a + len) & ~(g_page - 1);
    if (lo > a || hi < a + len) atomic_fetch_add(&g_uncovered, 1u);
    if (hi <= lo) return SPG_OK;                                // no whole page inside
    lock();
    int slot = -1;
    for (int i = 0; i < SPG_MAX_GUARDS; ++i)
        if (!atomic_load(&g_guards[i].active) && atomic_load(&g_guards[i].lo) == 0) { slot = i; break; }
    if (slot < 0) { unlock(); return SPG_EFULL; }
    atomic_store(&g_guards[slot].lo, lo);
    atomic_store(&g_guards[slot].hi, hi);
    atomic_store(&g_guards[slot].owner, owner);
    atomic_store(&g_guards[slot].active, 1);
    atomic_fetch_add(&g_nactive, 1);
    unlock();
    if (mprotect((void *)lo, hi - lo, PROT_READ) != 0) {
        atomic_store(&g_errno, errno);
        spg_release(owner);
        return SPG_ESYS;
    }
    return SPG_OK;
}

int spg_protect(const void *addr, size_t len, int64_t owner) { return spg_protect_ex(addr, len, owner, 0); }

int spg_release(int64_t owner) {
    lock();
    for (int i = 0; i < SPG_MAX_GUARDS; ++i) {
        if (atomic_load(&g_guards[i].lo) == 0 || atomic_load(&g_guards[i].owner) != owner) continue;
        int one = 1;
        if (atomic_compare_exchange_strong(&g_guards[i].active, &one, 0)) {
            mprotect((void *)atomic_load(&g_guards[i].lo),
                     atomic_load(&g_guards[i].hi) - atomic_load(&g_guards[i].lo), PROT_READ | PROT_WRITE);
            atomic_fetch_sub(&g_nactive, 1);
        }
        // tombstone before the slot forgets the range (handler step 3)
        const uint32_t t = atomic_fetch_add(&g_tomb_head, 1u) % SPG_TOMB;
        atomic_store(&g_tomb_lo[t], 0);
        atomic_store(&g_tomb_hi[t], atomic_load(&g_guards[i].hi));
        atomic_store(&g_tomb_lo[t], atomic_load(&g_guards[i].lo));
        atomic_store(&g_guards[i].lo, 0);
        atomic_store(&g_guards[i].hi, 0);
    }
    unlock();
    return SPG_OK;
}

int spg_drain(int64_t *out, int cap) {
    int n = 0;
    while (n < cap) {
        uint32_t t = atomic_load(&g_tail);
        if (t == atomic_load(&g_head)) break;
        out[n++] = atomic_load(&g_ring[t % SPG_RING]);
        atomic_store(&g_tail, t + 1);
    }
    return n;
}

int spg_active(void) { return atomic_load(&g_nactive); }
uint64_t spg_faults(void) { return atomic_load(&g_faults); }
int spg_errno(void) { return atomic_load(&g_errno); }
uint64_t spg_uncovered(void) { return atomic_load(&g_uncovered); }

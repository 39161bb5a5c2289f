/*
 * libspguard — page-protection write guards for speculatively encrypted host
 * ranges (the paper's MPK guards).
 *
 * The reference models guards byte-precisely in Python
 * (/root/reference/pkg/src/specpipe/memory.py:186-201 `write`, 227-242
 * `install_write_guard` / `release_write_guard`): only writes that go through
 * HostMemory.write fault.  This library adds the hardware half: the pages
 * fully inside a guarded range are mprotect()ed read-only, so ANY store to
 * them — numpy, torch, C code, other threads — traps; the SIGSEGV handler
 * records the guard owner in a lock-free fault ring, lifts the protection of
 * that guard, and lets the store retry.  The engine drains the ring at its
 * entry points and feeds WriteFault events to the validator (validator.py:
 * 199-203), which invalidates the record before its stale ciphertext can be
 * committed.
 *
 * Pages only partially covered by a guard are left writable (page
 * granularity must not create faults the byte-precise reference would not
 * raise) unless the caller states that it owns the rest of that page
 * (spg_protect_ex flags: page-aligned, page-padded pinned blocks guarded
 * from their first / to their last byte).  Guards whose bytes are not all
 * under protection are counted (spg_uncovered); the byte-precise
 * HostMemory.write check still covers them.
 *
 * Concurrency: a store that faults while another thread lifts the same
 * guard (a concurrent fault, or spg_release on commit/invalidate) retries
 * instead of reaching the previous SIGSEGV handler: the handler also matches
 * ranges that are being lifted and a ring of recently released ranges.
 */
#ifndef SPGUARD_H_
#define SPGUARD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPG_OK 0
#define SPG_EINVAL 1
#define SPG_EFULL 2     /* guard table full */
#define SPG_ESYS 3      /* mprotect/sigaction failed (errno in sp_guard_errno) */

/* Install the SIGSEGV handler (idempotent; chains to the previous handler
 * for faults outside any guard). */
int spg_init(void);
/* Protect the whole pages inside [addr, addr+len) for `owner` (record id).
 * Returns SPG_OK even if no whole page is inside (nothing to protect). */
int spg_protect(const void *addr, size_t len, int64_t owner);
/* flags for spg_protect_ex: the caller exclusively owns the rest of the
 * partial page before addr (HEAD) / after addr+len (TAIL), so that page is
 * protected too. */
#define SPG_HEAD_OWNED 1
#define SPG_TAIL_OWNED 2
int spg_protect_ex(const void *addr, size_t len, int64_t owner, int flags);
/* Lift the guard of `owner` (commit / invalidate / eviction). */
int spg_release(int64_t owner);
/* Pop up to `cap` faulted owners into `out`; returns how many. */
int spg_drain(int64_t *out, int cap);
/* Number of active guards / total faults taken (diagnostics). */
int spg_active(void);
uint64_t spg_faults(void);
int spg_errno(void);
/* Guards installed with part of their byte range left writable. */
uint64_t spg_uncovered(void);

#ifdef __cplusplus
}
#endif

#endif /* SPGUARD_H_ */

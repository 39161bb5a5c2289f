"""Hardware write guards (libspguard.so, include/spguard.h): mprotect the
pages of a speculatively encrypted host range so that ANY store to it — not
only HostMemory.write — invalidates the record (the paper's MPK
guards).  Faults are collected by a SIGSEGV handler into a ring and drained
by the engine at its entry points."""
from __future__ import annotations

import ctypes
import os

from ._native import LIB_DIR

_PATH = os.path.join(LIB_DIR, "libspguard.so")
_lib = None

SYMBOLS = ("spg_init", "spg_protect", "spg_protect_ex", "spg_release", "spg_drain", "spg_active", "spg_faults",
           "spg_errno", "spg_uncovered")
HEAD_OWNED = 1  # SPG_HEAD_OWNED
TAIL_OWNED = 2  # SPG_TAIL_OWNED


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise RuntimeError(f"{_PATH} missing; run __graft_entry__.build()")
        L = ctypes.CDLL(_PATH)
        L.spg_protect.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64]
        L.spg_protect_ex.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_int]
        L.spg_uncovered.restype = ctypes.c_uint64
        L.spg_release.argtypes = [ctypes.c_int64]
        L.spg_drain.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.spg_faults.restype = ctypes.c_uint64
        if L.spg_init() != 0:
            raise OSError(L.spg_errno(), "spg_init: sigaction failed")
        _lib = L
    return _lib


def protect(addr: int, length: int, owner: int, flags: int = 0) -> None:
    """Guard [addr, addr+length); flags HEAD_OWNED / TAIL_OWNED extend the
    protection over partial pages the caller owns exclusively."""
    rc = lib().spg_protect_ex(addr, length, owner, flags)
    if rc != 0:
        raise OSError(lib().spg_errno(), f"spg_protect rc={rc}")


def release(owner: int) -> None:
    lib().spg_release(owner)


def drain() -> list[int]:
    buf = (ctypes.c_int64 * 256)()
    out: list[int] = []
    while True:
        n = lib().spg_drain(buf, 256)
        out.extend(buf[:n])
        if n < 256:
            return out


def active() -> int:
    return lib().spg_active()


def faults() -> int:
    return int(lib().spg_faults())


def uncovered() -> int:
    """Guards installed with part of their bytes left writable."""
    return int(lib().spg_uncovered())

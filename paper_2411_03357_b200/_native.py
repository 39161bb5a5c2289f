"""ctypes binding of libspgcm.so (include/spgcm.h) and libsppipe.so.

The shared libraries are built in-tree by `__graft_entry__.build()` into
`paper_2411_03357_b200/lib/`.  There is no fallback: if the library or a CUDA
device is missing, every crypto entry point raises `NativeUnavailable`.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
SPGCM_PATH = os.environ.get("SPGCM_LIB") or os.path.join(LIB_DIR, "libspgcm.so")  # env: A/B builds

SP_OK, SP_EINVAL, SP_EAUTH, SP_ECUDA, SP_ENODEV = 0, 1, 2, 3, 4

# Every symbol include/spgcm.h declares (checked by tests/test_abi.py).
SPGCM_SYMBOLS = (
    "sp_ctx_create", "sp_ctx_destroy", "sp_seal", "sp_open", "sp_seal_batch", "sp_open_batch",
    "sp_seal_host", "sp_open_host", "sp_seal_host_batch", "sp_open_host_batch",
    "sp_last_error", "sp_version", "sp_launch_count", "sp_ctx_round_keys", "sp_ctx_hash_key",
)


class NativeUnavailable(RuntimeError):
    """libspgcm could not be loaded or has no usable sm_100a device."""


class SpDesc(ctypes.Structure):
    _fields_ = [
        ("dir", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("iv", ctypes.c_uint64),
        ("len", ctypes.c_uint64),
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("tag", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None


def load_spgcm() -> ctypes.CDLL:
    """Load libspgcm.so (no GPU needed just to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SPGCM_PATH):
            raise NativeUnavailable(
                f"{SPGCM_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(SPGCM_PATH)
        vp, u8p = ctypes.c_void_p, ctypes.c_void_p
        lib.sp_ctx_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        lib.sp_ctx_create.restype = ctypes.c_int
        lib.sp_ctx_destroy.argtypes = [vp]
        lib.sp_ctx_destroy.restype = None
        lib.sp_seal.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, vp, vp]
        lib.sp_open.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, vp, vp, vp]
        for name in ("sp_seal_batch", "sp_open_batch"):
            getattr(lib, name).argtypes = [vp, ctypes.POINTER(SpDesc), ctypes.c_int, vp]
        for name in ("sp_seal_host_batch", "sp_open_host_batch"):
            getattr(lib, name).argtypes = [vp, ctypes.POINTER(SpDesc), ctypes.c_int]
        lib.sp_seal_host.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, vp, u8p]
        lib.sp_open_host.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, vp, ctypes.c_size_t, u8p, vp]
        lib.sp_last_error.restype = ctypes.c_char_p
        lib.sp_version.restype = ctypes.c_char_p
        lib.sp_launch_count.restype = ctypes.c_uint64
        lib.sp_ctx_round_keys.argtypes = [vp, vp]
        lib.sp_ctx_hash_key.argtypes = [vp, vp]
        _lib = lib
        return lib


def last_error() -> str:
    return load_spgcm().sp_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load_spgcm().sp_launch_count())

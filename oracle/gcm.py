"""TEST INFRASTRUCTURE: ctypes wrapper over the plain-C oracle (gcm_oracle.c).

Restates channel.py:85-115 (`encrypt_at` / `decrypt_at`) with the arithmetic of
FIPS-197 and SP 800-38D.  Build with `make -C oracle` (done by
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_gcm.so")
_lib = None

MAX_MESSAGE_BYTES = 32 * 1024 * 1024


class OracleAuthError(Exception):
    pass


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        c_u8p = ctypes.c_char_p
        lib.oracle_gcm_seal.argtypes = [c_u8p, ctypes.c_uint32, ctypes.c_uint64, c_u8p,
                                        ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_gcm_open.argtypes = [c_u8p, ctypes.c_uint32, ctypes.c_uint64, c_u8p,
                                        ctypes.c_size_t, c_u8p, ctypes.c_void_p]
        lib.oracle_aes256_key_expand.argtypes = [c_u8p, ctypes.c_void_p]
        lib.oracle_aes256_encrypt_block.argtypes = [c_u8p, c_u8p, ctypes.c_void_p]
        lib.oracle_gf128_mul.argtypes = [c_u8p, c_u8p, ctypes.c_void_p]
        _lib = lib
    return _lib


def seal(key: bytes, direction: int, iv: int, plaintext: bytes) -> tuple[bytes, bytes]:
    """(key, dir, iv, P) -> (C, T).  channel.py:85-101."""
    if not 0 <= iv < (1 << 64):
        raise ValueError("counter out of range")
    if len(plaintext) < 1 or len(plaintext) > MAX_MESSAGE_BYTES:
        raise ValueError("bad plaintext length")
    out = ctypes.create_string_buffer(len(plaintext))
    tag = ctypes.create_string_buffer(16)
    rc = _load().oracle_gcm_seal(bytes(key), direction, iv, bytes(plaintext), len(plaintext), out, tag)
    if rc != 0:
        raise ValueError(f"oracle seal rc={rc}")
    return out.raw, tag.raw


def open_(key: bytes, direction: int, iv: int, ciphertext: bytes, tag: bytes) -> bytes:
    """(key, dir, iv, C, T) -> P or OracleAuthError.  channel.py:104-115."""
    if not 0 <= iv < (1 << 64):
        raise ValueError("counter out of range")
    out = ctypes.create_string_buffer(len(ciphertext))
    rc = _load().oracle_gcm_open(bytes(key), direction, iv, bytes(ciphertext), len(ciphertext), bytes(tag), out)
    if rc == 2:
        raise OracleAuthError(f"authentication failed at counter {iv}")
    if rc != 0:
        raise ValueError(f"oracle open rc={rc}")
    return out.raw


def key_expand(key: bytes) -> bytes:
    out = ctypes.create_string_buffer(240)
    _load().oracle_aes256_key_expand(bytes(key), out)
    return out.raw


def aes_block(key: bytes, block: bytes) -> bytes:
    out = ctypes.create_string_buffer(16)
    _load().oracle_aes256_encrypt_block(bytes(key), bytes(block), out)
    return out.raw


def gf128_mul(x: bytes, y: bytes) -> bytes:
    out = ctypes.create_string_buffer(16)
    _load().oracle_gf128_mul(bytes(x), bytes(y), out)
    return out.raw

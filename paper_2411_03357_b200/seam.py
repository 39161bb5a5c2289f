"""Seam-only drop-in: keep the reference's own engine,
predictor and validator, and replace only the three names through which it
reaches AES-GCM — `specpipe.channel.encrypt_at`, `specpipe.channel.decrypt_at`
and `specpipe.engine.encrypt_at` (imported by value at engine.py:34, called at
engine.py:503) — with libspgcm's host-bytes entry points (sp_seal_host /
sp_open_host, include/spgcm.h).  Pure ctypes: the stub a reference maintainer
would add next to channel.py.

    import specpipe
    from paper_2411_03357_b200 import seam
    seam.install(specpipe)          # every seal/open now runs in k_gcm on the B200
"""
from __future__ import annotations

import ctypes
import functools

from . import _native


@functools.lru_cache(maxsize=None)
def _ctx(key: bytes) -> ctypes.c_void_p:
    """One sp_ctx per key (replaces the per-call AESGCM(key), channel.py:96,111)."""
    lib = _native.load_spgcm()
    h = ctypes.c_void_p()
    rc = lib.sp_ctx_create(key, ctypes.byref(h))
    if rc != _native.SP_OK:
        raise _native.NativeUnavailable(_native.last_error())
    return h


def make_seams(channel_mod):
    """encrypt_at / decrypt_at with the reference's signatures, framing and
    errors (channel.py:85-115), computed by libspgcm."""
    lib = _native.load_spgcm()
    limit = channel_mod.MAX_MESSAGE_BYTES

    def encrypt_at(key, iv, plaintext, direction=channel_mod.Direction.HOST_TO_DEVICE):
        if not 0 <= iv < 1 << 64:
            raise ValueError("counter out of range")
        n = len(plaintext)
        if n < 1 or n > limit:
            raise ValueError("plaintext must be 1 .. 32 MiB")
        out, tag = ctypes.create_string_buffer(n), ctypes.create_string_buffer(16)
        rc = lib.sp_seal_host(_ctx(bytes(key.key_bytes)), direction.value, iv, bytes(plaintext), n, out, tag)
        if rc != _native.SP_OK:
            raise RuntimeError(_native.last_error())
        return channel_mod.CiphertextMsg(payload=out.raw, auth_tag=tag.raw, declared_len=n)

    def decrypt_at(key, iv, msg, direction=channel_mod.Direction.HOST_TO_DEVICE):
        if not 0 <= iv < 1 << 64:
            raise ValueError("counter out of range")
        n = len(msg.payload)
        out = ctypes.create_string_buffer(max(1, n))
        rc = lib.sp_open_host(_ctx(bytes(key.key_bytes)), direction.value, iv, bytes(msg.payload), n,
                              bytes(msg.auth_tag), out)
        if rc == _native.SP_EAUTH:
            raise channel_mod.AuthError(f"authentication failed at counter {iv}")
        if rc != _native.SP_OK:
            raise RuntimeError(_native.last_error())
        return out.raw[:n]

    return encrypt_at, decrypt_at


def install(specpipe_pkg) -> tuple:
    """Rebind the reference's three crypto names; returns the previous
    bindings (pass them to `uninstall`)."""
    ch, eng = specpipe_pkg.channel, specpipe_pkg.engine
    old = (ch.encrypt_at, ch.decrypt_at, eng.encrypt_at)
    enc, dec = make_seams(ch)
    ch.encrypt_at = enc   # encrypt_next (channel.py:156), nop (176)
    ch.decrypt_at = dec   # recv_msg (188), deferred_decrypt (215)
    eng.encrypt_at = enc  # the by-value import used at engine.py:503
    return old


def uninstall(specpipe_pkg, old: tuple) -> None:
    specpipe_pkg.channel.encrypt_at, specpipe_pkg.channel.decrypt_at, specpipe_pkg.engine.encrypt_at = old

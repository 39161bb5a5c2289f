"""Cipher context over libspgcm: the replacement for the reference's
per-call `AESGCM(key)` (channel.py:96,111).

`GcmContext` owns one `sp_ctx` (key schedule, H and GHASH power tables in HBM)
and exposes three call shapes:

* host bytes in / bytes out (`seal_bytes`, `open_bytes`) — the exact shape of
  `encrypt_at` / `decrypt_at`; copies are pipelined inside the library;
* device tensors (`seal_device`, `open_device`) — stream-ordered, no copies;
* batches (`seal_batch`, `open_batch`) — many messages in one launch (chunk
  runs, NOP padding, deferred-decrypt drains).

There is no CPU path: without the library or a B200 every call raises.
"""
from __future__ import annotations

import ctypes
import threading
from typing import Sequence

from . import _native
from ._native import SpDesc, NativeUnavailable

TAG_BYTES = 16
MAX_MESSAGE_BYTES = 32 * 1024 * 1024
_IV_LIMIT = 1 << 64


class GcmAuthError(Exception):
    """Tag mismatch reported by the device."""


def _check(rc: int, what: str) -> None:
    if rc == _native.SP_OK:
        return
    msg = f"{what}: {_native.last_error()} (rc={rc})"
    if rc == _native.SP_EINVAL:
        raise ValueError(msg)
    if rc == _native.SP_EAUTH:
        raise GcmAuthError(msg)
    if rc == _native.SP_ENODEV:
        raise NativeUnavailable(msg)
    raise RuntimeError(msg)


def _check_len_iv(iv: int, n: int) -> None:
    if not 0 <= iv < _IV_LIMIT:
        raise ValueError("counter out of range")
    if n < 1:
        raise ValueError("plaintext must be at least 1 byte")
    if n > MAX_MESSAGE_BYTES:
        raise ValueError("message exceeds the 32 MiB channel limit; chunk it")


def _ptr(buf) -> int:
    """Address of a bytes/bytearray/memoryview/torch tensor."""
    if hasattr(buf, "data_ptr"):
        return int(buf.data_ptr())
    if isinstance(buf, bytes):
        return ctypes.cast(ctypes.c_char_p(buf), ctypes.c_void_p).value
    mv = memoryview(buf)
    if mv.readonly:
        raise TypeError("read-only buffers other than bytes are not accepted; pass bytes")
    return ctypes.addressof(ctypes.c_char.from_buffer(mv))


def _stream_handle(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


class GcmContext:
    """One AES-256-GCM key resident on the current CUDA device."""

    def __init__(self, key: bytes) -> None:
        if len(key) != 32:
            raise ValueError("key must be 32 bytes")
        self._lib = _native.load_spgcm()
        h = ctypes.c_void_p()
        _check(self._lib.sp_ctx_create(bytes(key), ctypes.byref(h)), "sp_ctx_create")
        self._h = h
        self.key = bytes(key)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.sp_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self) -> None:  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    # -- host bytes (encrypt_at / decrypt_at shape) -------------------------
    def seal_bytes(self, direction: int, iv: int, plaintext) -> tuple[bytes, bytes]:
        n = len(plaintext)
        _check_len_iv(iv, n)
        src = plaintext if isinstance(plaintext, bytes) else bytes(plaintext)
        out = ctypes.create_string_buffer(n)
        tag = ctypes.create_string_buffer(TAG_BYTES)
        _check(self._lib.sp_seal_host(self._h, direction, iv, _ptr(src), n, out, tag), "sp_seal_host")
        return out.raw, tag.raw

    def open_bytes(self, direction: int, iv: int, ciphertext, tag: bytes) -> bytes:
        n = len(ciphertext)
        if not 0 <= iv < _IV_LIMIT:
            raise ValueError("counter out of range")
        if n < 1 or n > MAX_MESSAGE_BYTES or len(tag) != TAG_BYTES:
            # the reference's AESGCM raises InvalidTag for malformed input,
            # which decrypt_at turns into AuthError (channel.py:110-115)
            raise GcmAuthError(f"malformed message at counter {iv}")
        src = ciphertext if isinstance(ciphertext, bytes) else bytes(ciphertext)
        out = ctypes.create_string_buffer(n)
        _check(self._lib.sp_open_host(self._h, direction, iv, _ptr(src), n, bytes(tag), out), "sp_open_host")
        return out.raw

    # -- host batch (pinned or pageable buffers) -----------------------------
    def seal_host_batch(self, items: Sequence[tuple]) -> None:
        """items: (dir, iv, src, dst, tag16) host buffers; results in place."""
        descs = (SpDesc * len(items))()
        for d, (direction, iv, src, dst, tag) in zip(descs, items):
            _check_len_iv(iv, len(src))
            d.dir, d.iv, d.len = direction, iv, len(src)
            d.src, d.dst, d.tag, d.status = _ptr(src), _ptr(dst), _ptr(tag), None
        _check(self._lib.sp_seal_host_batch(self._h, descs, len(items)), "sp_seal_host_batch")

    def open_host_batch(self, items: Sequence[tuple]) -> None:
        """items: (dir, iv, src, dst, tag16) host buffers; raises on auth failure."""
        descs = (SpDesc * len(items))()
        status = (ctypes.c_int32 * len(items))()
        for k, (d, (direction, iv, src, dst, tag)) in enumerate(zip(descs, items)):
            _check_len_iv(iv, len(src))
            d.dir, d.iv, d.len = direction, iv, len(src)
            d.src, d.dst, d.tag = _ptr(src), _ptr(dst), _ptr(tag)
            d.status = ctypes.addressof(status) + 4 * k
        _check(self._lib.sp_open_host_batch(self._h, descs, len(items)), "sp_open_host_batch")

    # -- device tensors --------------------------------------------------------
    def set_max_sms(self, max_sms: int) -> None:
        """SM budget of this context's launches (0: every SM)."""
        _check(self._lib.sp_ctx_set_max_sms(self._h, int(max_sms)), "sp_ctx_set_max_sms")

    @property
    def max_sms(self) -> int:
        return int(self._lib.sp_ctx_max_sms(self._h))

    def set_small_sms(self, small_sms: int) -> None:
        """SM cap of this context's small (<= 2 MiB) launches (0: none)."""
        _check(self._lib.sp_ctx_set_small_sms(self._h, int(small_sms)), "sp_ctx_set_small_sms")

    def seal_batch(self, items: Sequence[tuple], stream=None) -> None:
        """items: (dir, iv, src, dst, tag) with device tensors (or int
        pointers + explicit len via a 6th element)."""
        descs = self._descs(items, status=None)
        _check(self._lib.sp_seal_batch(self._h, descs, len(items), _stream_handle(stream)), "sp_seal_batch")

    def open_batch(self, items: Sequence[tuple], status, stream=None) -> None:
        """items: (dir, iv, src, dst, tag[, len]); status: device int32 tensor
        with one slot per item (0 ok, 1 tag mismatch -> dst zeroed)."""
        descs = self._descs(items, status=status)
        _check(self._lib.sp_open_batch(self._h, descs, len(items), _stream_handle(stream)), "sp_open_batch")

    def seal_device(self, direction, iv, src, dst, tag, stream=None) -> None:
        self.seal_batch([(direction, iv, src, dst, tag)], stream)

    def open_device(self, direction, iv, src, dst, tag, status, stream=None) -> None:
        self.open_batch([(direction, iv, src, dst, tag)], status, stream)

    def _descs(self, items, status):
        descs = (SpDesc * len(items))()
        sbase = _ptr(status) if status is not None else None
        for k, (d, it) in enumerate(zip(descs, items)):
            direction, iv, src, dst, tag = it[:5]
            n = it[5] if len(it) > 5 else (src.numel() * src.element_size())
            _check_len_iv(iv, n)
            d.dir, d.iv, d.len = direction, iv, n
            d.src, d.dst, d.tag = _ptr(src), _ptr(dst), _ptr(tag)
            d.status = (sbase + 4 * k) if sbase is not None else None
        return descs

    # -- introspection (tests) ---------------------------------------------------
    def round_keys(self) -> bytes:
        out = ctypes.create_string_buffer(240)
        _check(self._lib.sp_ctx_round_keys(self._h, out), "sp_ctx_round_keys")
        return out.raw

    def hash_key(self) -> bytes:
        out = ctypes.create_string_buffer(16)
        _check(self._lib.sp_ctx_hash_key(self._h, out), "sp_ctx_hash_key")
        return out.raw


_ctx_lock = threading.Lock()
_ctx_cache: dict[tuple[int, bytes], GcmContext] = {}


def context_for(key: bytes) -> GcmContext:
    """Cached context per (device, key): key setup happens once per channel,
    not once per message as `AESGCM(key)` does in the reference."""
    import torch

    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    k = (dev, bytes(key))
    with _ctx_lock:
        ctx = _ctx_cache.get(k)
        if ctx is None:
            ctx = GcmContext(key)
            _ctx_cache[k] = ctx
        return ctx

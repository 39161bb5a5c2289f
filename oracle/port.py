"""TEST INFRASTRUCTURE: restatement of the reference seam over its own
third-party arithmetic (`cryptography` AESGCM, pinned `cryptography>=41`,
/root/reference/pkg/pyproject.toml:10-12).

Follows channel.py:77-82 (`_nonce`), 85-101 (`encrypt_at`) and 104-115
(`decrypt_at`).  Used by tests for large messages (the C oracle is bit-serial)
and by bench.py as the CPU baseline / `--impl reference` arm.
"""
from __future__ import annotations

from cryptography.exceptions import InvalidTag
from cryptography.hazmat.primitives.ciphers.aead import AESGCM

MAX_MESSAGE_BYTES = 32 * 1024 * 1024


class PortAuthError(Exception):
    pass


def nonce(direction: int, iv: int) -> bytes:
    if not 0 <= iv < (1 << 64):
        raise ValueError("counter out of range")
    return direction.to_bytes(4, "big") + iv.to_bytes(8, "big")


def seal(key: bytes, direction: int, iv: int, plaintext: bytes) -> tuple[bytes, bytes]:
    if len(plaintext) < 1 or len(plaintext) > MAX_MESSAGE_BYTES:
        raise ValueError("bad plaintext length")
    sealed = AESGCM(bytes(key)).encrypt(nonce(direction, iv), bytes(plaintext), None)
    return sealed[:-16], sealed[-16:]


def open_(key: bytes, direction: int, iv: int, ciphertext: bytes, tag: bytes) -> bytes:
    try:
        return AESGCM(bytes(key)).decrypt(nonce(direction, iv), bytes(ciphertext) + bytes(tag), None)
    except InvalidTag as exc:
        raise PortAuthError(f"authentication failed at counter {iv}") from exc


def seal_into(aead: AESGCM, direction: int, iv: int, plaintext, out) -> None:
    """Reused-buffer variant for the CPU baseline (no per-call allocation)."""
    aead.encrypt_into(nonce(direction, iv), plaintext, None, out)

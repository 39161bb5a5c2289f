"""Generate golden vectors by running the REFERENCE itself (importable only in
the build container: PYTHONPATH=/root/reference/pkg/src).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

Writes tests/golden/cipher_vectors.json.  Every vector is produced by
`specpipe.channel.encrypt_at` (channel.py:85-101) on inputs from
`specpipe.memory.prng_fill` (memory.py:106-110) and keys from
`specpipe.channel.new_channel(seed)` (channel.py:275-298), so the fixtures pin
the reference's observable bytes, not a re-implementation.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from specpipe.channel import (  # noqa: E402
    ChannelKey, Direction, MAX_MESSAGE_BYTES, decrypt_at, encrypt_at, new_channel,
)
from specpipe.memory import prng_fill  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
KIB = 1024
MIB = 1024 * KIB

SMALL_SIZES = [1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 255, 256, 257, 2048, 4095, 4096, 4097]
MID_SIZES = [160 * KIB, 224 * KIB, 288 * KIB, 384 * KIB, 1 * MIB, 1_000_003]
BIG_SIZES = [8 * MIB + 7, 25_298_944, 29_360_128, MAX_MESSAGE_BYTES]
EDGE_IVS = [0, 1, (1 << 32) - 1, 1 << 32, 1 << 63, (1 << 64) - 1]


def vec(key_seed, key, direction, iv, payload_seed, n, explicit=None):
    p = explicit if explicit is not None else prng_fill(payload_seed)(n)
    msg = encrypt_at(key, iv, p, direction)
    assert decrypt_at(key, iv, msg, direction) == p
    rec = {
        "key_seed": key_seed,
        "key": key.key_bytes.hex(),
        "dir": direction.value,
        "iv": str(iv),
        "len": len(p),
        "payload_seed": payload_seed,
        "sha256_p": hashlib.sha256(p).hexdigest(),
        "sha256_c": hashlib.sha256(msg.payload).hexdigest(),
        "tag": msg.auth_tag.hex(),
    }
    if explicit is not None:
        rec["p_hex"] = p.hex()
    if len(p) <= 64:
        rec["c_hex"] = msg.payload.hex()
    return rec


def main() -> None:
    vectors = []
    # McGrew-Viega GCM Test Case 14 through the reference seam (zero key, zero nonce).
    zero = ChannelKey(bytes(32))
    vectors.append(vec(None, zero, Direction.HOST_TO_DEVICE, 0, None, 16, explicit=bytes(16)))
    keys = {s: new_channel(seed=s)[0].key for s in (0, 1, 2, 3)}
    # NOP (channel.py:174-177): one 0x00 byte.
    for iv in EDGE_IVS:
        for d in Direction:
            vectors.append(vec(0, keys[0], d, iv, None, 1, explicit=b"\x00"))
    ps = 100
    for n in SMALL_SIZES:
        for iv in EDGE_IVS:
            for d in Direction:
                vectors.append(vec(1, keys[1], d, iv, ps, n))
                ps += 1
    for n in MID_SIZES:
        for iv in (0, 5, (1 << 64) - 1):
            for d in Direction:
                vectors.append(vec(2, keys[2], d, iv, ps, n))
                ps += 1
    for n in BIG_SIZES:
        vectors.append(vec(0, keys[0], Direction.HOST_TO_DEVICE, 0, ps, n))
        ps += 1
        vectors.append(vec(3, keys[3], Direction.DEVICE_TO_HOST, (1 << 63) + 7, ps, n))
        ps += 1
    # survey Appendix B vectors (key seed 0)
    vectors.append(vec(0, keys[0], Direction.DEVICE_TO_HOST, 5, None, 16, explicit=bytes(16)))
    vectors.append(vec(0, keys[0], Direction.HOST_TO_DEVICE, 1, 7, 262144))
    vectors.append(vec(0, keys[0], Direction.HOST_TO_DEVICE, 0, 1, MAX_MESSAGE_BYTES))
    vectors.append(vec(0, keys[0], Direction.DEVICE_TO_HOST, (1 << 64) - 1, 3, 1_000_003))

    errors = []
    for iv, n in (((1 << 64), 16), (-1, 16), (0, 0), (0, MAX_MESSAGE_BYTES + 1)):
        try:
            encrypt_at(keys[0], iv, bytes(n))
            errors.append({"iv": str(iv), "len": n, "error": None})
        except ValueError as exc:
            errors.append({"iv": str(iv), "len": n, "error": "ValueError", "msg": str(exc)})

    prng = []
    for seed in (0, 1, 7, 123456789, (1 << 30) - 1):
        for n in (1, 3, 4, 5, 7, 8, 1000, 4099):
            prng.append({"seed": seed, "len": n, "hex": prng_fill(seed)(n).hex()})
    for seed, n in ((1, MAX_MESSAGE_BYTES), (7, 262144), (3, 1_000_003)):
        prng.append({"seed": seed, "len": n, "sha256": hashlib.sha256(prng_fill(seed)(n)).hexdigest()})

    out = {
        "generator": "tests/golden/gen_golden.py (reference specpipe 0.1.0 over cryptography "
                     + __import__("cryptography").__version__ + ")",
        "channel_keys": {str(s): k.key_bytes.hex() for s, k in keys.items()},
        "vectors": vectors,
        "errors": errors,
        "prng_fill": prng,
    }
    with open(os.path.join(HERE, "cipher_vectors.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"wrote {len(vectors)} vectors, {len(prng)} prng cases")


if __name__ == "__main__":
    main()

"""GPU parity of the sm_100a AES-256-GCM kernels against the golden vectors
produced by the reference itself (tests/golden/cipher_vectors.json) and against
the CPU oracles (oracle.gcm plain-C restatement, oracle.port = cryptography,
the reference's own dependency).  Bit-exact: ciphertext, tags and plaintext.
"""
from __future__ import annotations

import hashlib
import json
import os
import random

import numpy as np
import pytest

from oracle import gcm as oracle_gcm
from oracle import port as oracle_port

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cipher_vectors.json")))
MIB = 1 << 20

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    torch.cuda.set_device(0)
    return torch


@pytest.fixture(scope="module")
def ctx_for(torch_cuda):
    from paper_2411_03357_b200.gcm import GcmContext

    cache = {}

    def get(key: bytes):
        if key not in cache:
            cache[key] = GcmContext(key)
        return cache[key]

    return get


def _payload(v):
    from paper_2411_03357_b200 import prng

    if "p_hex" in v:
        return bytes.fromhex(v["p_hex"])
    return prng.random_bytes(v["payload_seed"], v["len"]).tobytes()


def _dev(torch, b: bytes):
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()


def _host(t) -> bytes:
    return t.cpu().numpy().tobytes()


def _check_vec(v, c: bytes, tag: bytes):
    assert tag.hex() == v["tag"], (v["len"], v["iv"], v["dir"])
    if "c_hex" in v:
        assert c.hex() == v["c_hex"]
    assert hashlib.sha256(c).hexdigest() == v["sha256_c"]


def test_tc14_and_hash_key(ctx_for, torch_cuda):
    torch = torch_cuda
    ctx = ctx_for(bytes(32))
    assert ctx.round_keys() == oracle_gcm.key_expand(bytes(32))
    assert ctx.hash_key() == oracle_gcm.aes_block(bytes(32), bytes(16))
    src = _dev(torch, bytes(16))
    dst = torch.empty_like(src)
    tag = torch.empty(16, dtype=torch.uint8, device="cuda")
    ctx.seal_device(0, 0, src, dst, tag)
    torch.cuda.synchronize()
    assert _host(dst).hex() == "cea7403d4d606b6e074ec5d3baf39d18"
    assert _host(tag).hex() == "d0d1c8a799996bf0265b98b5d48ab919"


def test_golden_vectors_one_by_one(ctx_for, torch_cuda):
    """Every reference-generated vector, each in its own launch; open round trip."""
    torch = torch_cuda
    for v in GOLD["vectors"]:
        key = bytes.fromhex(v["key"])
        ctx = ctx_for(key)
        p = _payload(v)
        assert hashlib.sha256(p).hexdigest() == v["sha256_p"]
        src = _dev(torch, p)
        dst = torch.empty_like(src)
        tag = torch.empty(16, dtype=torch.uint8, device="cuda")
        iv = int(v["iv"])
        ctx.seal_device(v["dir"], iv, src, dst, tag)
        back = torch.empty_like(src)
        st = torch.full((1,), 7, dtype=torch.int32, device="cuda")
        ctx.open_device(v["dir"], iv, dst, back, tag, st)
        torch.cuda.synchronize()
        _check_vec(v, _host(dst), _host(tag))
        assert int(st.item()) == 0
        assert torch.equal(back, src)


def test_golden_vectors_single_batch(ctx_for, torch_cuda):
    """All vectors of one key in ONE launch (K3 descriptor batch)."""
    torch = torch_cuda
    by_key = {}
    for v in GOLD["vectors"]:
        by_key.setdefault(v["key"], []).append(v)
    for khex, vs in by_key.items():
        ctx = ctx_for(bytes.fromhex(khex))
        srcs = [_dev(torch, _payload(v)) for v in vs]
        dsts = [torch.empty_like(s) for s in srcs]
        tags = torch.empty((len(vs), 16), dtype=torch.uint8, device="cuda")
        items = [(v["dir"], int(v["iv"]), s, d, tags[i]) for i, (v, s, d) in enumerate(zip(vs, srcs, dsts))]
        ctx.seal_batch(items)
        backs = [torch.empty_like(s) for s in srcs]
        st = torch.full((len(vs),), 7, dtype=torch.int32, device="cuda")
        ctx.open_batch([(v["dir"], int(v["iv"]), d, b, tags[i]) for i, (v, d, b) in
                        enumerate(zip(vs, dsts, backs))], st)
        torch.cuda.synchronize()
        for i, v in enumerate(vs):
            _check_vec(v, _host(dsts[i]), _host(tags[i]))
            assert torch.equal(backs[i], srcs[i])
        assert int(st.abs().sum().item()) == 0


def test_random_sizes_vs_oracles(ctx_for, torch_cuda):
    torch = torch_cuda
    rng = random.Random(1234)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    sizes = [rng.randrange(1, 70000) for _ in range(60)] + [rng.randrange(1, 3 * MIB) for _ in range(12)]
    items, refs, srcs = [], [], []
    tags = torch.empty((len(sizes), 16), dtype=torch.uint8, device="cuda")
    for i, n in enumerate(sizes):
        p = rng.randbytes(n)
        iv = rng.choice([0, 1, rng.randrange(1 << 64), (1 << 64) - 1, (1 << 32) - 1])
        d = rng.randrange(2)
        src = _dev(torch, p)
        dst = torch.empty_like(src)
        srcs.append(src)
        items.append((d, iv, src, dst, tags[i]))
        refs.append(oracle_port.seal(key, d, iv, p) if n > 4096 else oracle_gcm.seal(key, d, iv, p))
    ctx.seal_batch(items)
    torch.cuda.synchronize()
    for i, (c, t) in enumerate(refs):
        assert _host(items[i][3]) == c, sizes[i]
        assert _host(tags[i]) == t, sizes[i]


def test_unaligned_and_inplace(ctx_for, torch_cuda):
    torch = torch_cuda
    key = bytes(range(100, 132))
    ctx = ctx_for(key)
    rng = random.Random(5)
    big = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    for so, do, n in [(1, 3, 1000), (15, 0, 4097), (0, 7, 65536 + 9), (5, 5, 33), (8, 12, 300000)]:
        p = rng.randbytes(n)
        big[so:so + n] = torch.frombuffer(bytearray(p), dtype=torch.uint8).cuda()
        out = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
        tag = torch.empty(17, dtype=torch.uint8, device="cuda")
        ctx.seal_batch([(1, 99, big[so:so + n], out[do:do + n], tag[1:17])])
        torch.cuda.synchronize()
        c, t = oracle_port.seal(key, 1, 99, p)
        assert _host(out[do:do + n]) == c
        assert _host(tag[1:17]) == t
        assert int(out[:do].abs().sum()) == 0 and int(out[do + n:].abs().sum()) == 0
    # in place
    p = rng.randbytes(100003)
    buf = _dev(torch, p)
    tag = torch.empty(16, dtype=torch.uint8, device="cuda")
    ctx.seal_device(0, 5, buf, buf, tag)
    torch.cuda.synchronize()
    c, t = oracle_port.seal(key, 0, 5, p)
    assert _host(buf) == c and _host(tag) == t
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.open_device(0, 5, buf, buf, tag, st)
    torch.cuda.synchronize()
    assert _host(buf) == p and int(st.item()) == 0


def test_tamper_rejected_and_zeroed(ctx_for, torch_cuda):
    """Bit flips in payload or tag, wrong IV, wrong direction -> status 1 and
    no plaintext released (channel.py:110-115 AuthError semantics)."""
    torch = torch_cuda
    key = bytes(range(32, 64))
    ctx = ctx_for(key)
    rng = random.Random(9)
    for n in (1, 16, 17, 5000, 2 * MIB + 3):
        p = rng.randbytes(n)
        src = _dev(torch, p)
        ct = torch.empty_like(src)
        tag = torch.empty(16, dtype=torch.uint8, device="cuda")
        ctx.seal_device(0, 77, src, ct, tag)
        cases = []
        c2 = ct.clone(); c2[rng.randrange(n)] ^= 1 << rng.randrange(8); cases.append((0, 77, c2, tag))
        t2 = tag.clone(); t2[rng.randrange(16)] ^= 0x80; cases.append((0, 77, ct, t2))
        cases.append((0, 78, ct, tag))
        cases.append((1, 77, ct, tag))
        for d, iv, c, t in cases:
            out = torch.full_like(src, 0x5A)
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            ctx.open_device(d, iv, c, out, t, st)
            torch.cuda.synchronize()
            assert int(st.item()) == 1
            assert int(out.abs().sum().item()) == 0


def test_host_bytes_api(ctx_for, torch_cuda):
    from paper_2411_03357_b200.gcm import GcmAuthError

    key = bytes(range(7, 39))
    ctx = ctx_for(key)
    rng = random.Random(3)
    for n in (1, 2048, 229376, 8 * MIB + 1, 32 * MIB):
        p = rng.randbytes(n)
        iv = rng.randrange(1 << 64)
        c, t = ctx.seal_bytes(1, iv, p)
        assert (c, t) == oracle_port.seal(key, 1, iv, p)
        assert ctx.open_bytes(1, iv, c, t) == p
        bad = bytearray(c); bad[-1] ^= 1
        with pytest.raises(GcmAuthError):
            ctx.open_bytes(1, iv, bytes(bad), t)


def test_full_size_batch_round_trip(ctx_for, torch_cuda):
    """BASELINE config sizes: an OPT-13B layer (18 x 32 MiB + 25,298,944 B) in one
    launch; size-independent property = open(seal(P)) == P with all tags valid,
    plus spot checks of first/last chunk against the reference arithmetic."""
    torch = torch_cuda
    key = bytes(range(200, 232))
    ctx = ctx_for(key)
    sizes = [32 * MIB] * 18 + [25_298_944]
    total = sum(sizes)
    buf = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(buf)
    back = torch.empty_like(buf)
    tags = torch.empty((len(sizes), 16), dtype=torch.uint8, device="cuda")
    items, off = [], 0
    for i, n in enumerate(sizes):
        items.append((0, 1000 + i, buf[off:off + n], out[off:off + n], tags[i]))
        off += n
    ctx.seal_batch(items)
    st = torch.full((len(sizes),), 7, dtype=torch.int32, device="cuda")
    ctx.open_batch([(0, 1000 + i, it[3], back[o:o + it[2].numel()], tags[i])
                    for i, (it, o) in enumerate(zip(items, np.cumsum([0] + sizes[:-1])))], st)
    torch.cuda.synchronize()
    assert int(st.abs().sum().item()) == 0
    assert torch.equal(back, buf)
    for i in (0, len(sizes) - 1):
        p = _host(items[i][2])
        c, t = oracle_port.seal(key, 0, 1000 + i, p)
        assert _host(items[i][3]) == c and _host(tags[i]) == t


def test_random_batches_fuzz(ctx_for, torch_cuda):
    """Randomised batches: 1..40 messages, sizes from 1 B to 5 MiB (skewed
    small), arbitrary byte offsets, random directions and counters, mixed in
    one launch; every ciphertext/tag vs the reference arithmetic, every open
    back to the plaintext with status 0."""
    torch = torch_cuda
    rng = random.Random(2024)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    for _ in range(25):
        k = rng.randrange(1, 41)
        sizes = [min(5 * MIB, int(rng.paretovariate(0.7) * rng.choice([1, 16, 200, 3000]))) or 1 for _ in range(k)]
        offs = [rng.randrange(0, 64) for _ in range(k)]
        total = sum(s + o for s, o in zip(sizes, offs)) + 64
        src = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
        dst = torch.zeros_like(src)
        back = torch.zeros_like(src)
        tags = torch.zeros((k, 17), dtype=torch.uint8, device="cuda")
        st = torch.full((k,), 9, dtype=torch.int32, device="cuda")
        items, oitems, meta, pos = [], [], [], 0
        for i, (n, o) in enumerate(zip(sizes, offs)):
            d = rng.randrange(2)
            iv = rng.choice([0, rng.randrange(1 << 64), (1 << 64) - 1])
            a = pos + o
            items.append((d, iv, src[a:a + n], dst[a:a + n], tags[i, 1:17]))
            oitems.append((d, iv, dst[a:a + n], back[a:a + n], tags[i, 1:17]))
            meta.append((d, iv, a, n))
            pos = a + n
        ctx.seal_batch(items)
        ctx.open_batch(oitems, st)
        torch.cuda.synchronize()
        assert int(st.abs().sum()) == 0
        h_src, h_dst, h_back = src.cpu().numpy(), dst.cpu().numpy(), back.cpu().numpy()
        h_tags = tags.cpu().numpy()
        for i, (d, iv, a, n) in enumerate(meta):
            p = h_src[a:a + n].tobytes()
            c, t = oracle_port.seal(key, d, iv, p)
            assert h_dst[a:a + n].tobytes() == c, (n, a)
            assert h_tags[i, 1:17].tobytes() == t
            assert h_back[a:a + n].tobytes() == p


def test_host_batch_pieces_split_messages(ctx_for, torch_cuda):
    """Host pipeline: messages straddle the 1..32 MiB piece schedule, so runs
    of one message finish in different launches (accumulator path)."""
    rng = random.Random(77)
    key = bytes(range(50, 82))
    ctx = ctx_for(key)
    import torch

    sizes = [3 * MIB + 5, 32 * MIB, 1, 17 * MIB + 3, 700_001]
    src = [torch.from_numpy(np.frombuffer(rng.randbytes(n), dtype=np.uint8).copy()).pin_memory() for n in sizes]
    dst = [torch.empty_like(s).pin_memory() for s in src]
    back = [torch.empty_like(s).pin_memory() for s in src]
    tags = [torch.empty(16, dtype=torch.uint8).pin_memory() for _ in sizes]
    ctx.seal_host_batch([(0, 900 + i, s, d, t) for i, (s, d, t) in enumerate(zip(src, dst, tags))])
    for i, n in enumerate(sizes):
        c, t = oracle_port.seal(key, 0, 900 + i, src[i].numpy().tobytes())
        assert dst[i].numpy().tobytes() == c and tags[i].numpy().tobytes() == t
    ctx.open_host_batch([(0, 900 + i, d, b, t) for i, (d, b, t) in enumerate(zip(dst, back, tags))])
    for s, b in zip(src, back):
        assert torch.equal(s, b)
    # a tampered message fails the whole call and its output is scrubbed
    from paper_2411_03357_b200.gcm import GcmAuthError

    dst[3][5] ^= 1
    for b in back:
        b.fill_(0xAB)
    with pytest.raises(GcmAuthError):
        ctx.open_host_batch([(0, 900 + i, d, b, t) for i, (d, b, t) in enumerate(zip(dst, back, tags))])
    # the tampered message crossed PCIe once, after its verdict: all zeros
    # (no unverified plaintext, no stale sentinel); the others are verified
    assert int(back[3].sum()) == 0
    for i in (0, 1, 2, 4):
        assert torch.equal(src[i], back[i]), i


def test_mixed_seal_open_batch(ctx_for, torch_cuda):
    """sp_crypt_batch: seals and opens interleaved in one launch (the data
    plane's level-scheduled flushes) — seals match the oracle bit for bit,
    authentic opens return the plaintext, a tampered one fails and is zeroed."""
    import ctypes

    from paper_2411_03357_b200 import _native

    torch = torch_cuda
    rng = random.Random(77)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    lib = _native.load_spgcm()
    n = 48
    sizes = [rng.choice([1, 17, 2048, 229_376, rng.randrange(1, 3 * MIB)]) for _ in range(n)]
    plains = [rng.randbytes(s) for s in sizes]
    ivs = [rng.randrange(1 << 64) for _ in range(n)]
    dirs = [rng.randrange(2) for _ in range(n)]
    refs = [oracle_port.seal(key, d, iv, p) for d, iv, p in zip(dirs, ivs, plains)]
    is_open = [i % 2 == 1 for i in range(n)]
    srcs, dsts = [], []
    tags = torch.zeros((n, 16), dtype=torch.uint8, device="cuda")
    status = torch.full((n,), 7, dtype=torch.int32, device="cuda")
    descs = (_native.SpDesc * n)()
    for i in range(n):
        if is_open[i]:
            c, t = refs[i]
            if i == 5:
                c = bytes([c[0] ^ 1]) + c[1:]  # tampered
            src = _dev(torch, c)
            tags[i] = torch.tensor(list(t), dtype=torch.uint8)
        else:
            src = _dev(torch, plains[i])
        dst = torch.full_like(src, 0xAB)
        srcs.append(src)
        dsts.append(dst)
        d = descs[i]
        d.dir, d.reserved, d.iv, d.len = dirs[i], int(is_open[i]), ivs[i], sizes[i]
        d.src, d.dst, d.tag = src.data_ptr(), dst.data_ptr(), tags[i].data_ptr()
        d.status = status.data_ptr() + 4 * i
    rc = lib.sp_crypt_batch(ctx._h, descs, n, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, _native.last_error()
    torch.cuda.synchronize()
    st = status.cpu().tolist()
    for i in range(n):
        if is_open[i]:
            if i == 5:
                assert st[i] == 1 and _host(dsts[i]) == bytes(sizes[i])
            else:
                assert st[i] == 0 and _host(dsts[i]) == plains[i], i
        else:
            assert (_host(dsts[i]), _host(tags[i])) == refs[i], i
            assert st[i] == 7  # seals leave status alone


@pytest.mark.parametrize("tamper", [None, 3])
def test_status_on_failure_shared_word(ctx_for, torch_cuda, tamper):
    """SP_STATUS_ON_FAILURE (include/spgcm.h): opens that share one status
    word write it only on a tag mismatch — an all-authentic batch leaves the
    word untouched, one tampered message sets it to 1 (its output zeroed,
    the others' plaintext intact).  The pipeline keeps one such word per pipe
    in mapped pinned memory; here it is host-mapped too."""
    import ctypes

    from paper_2411_03357_b200 import _native

    torch = torch_cuda
    rng = random.Random(5)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    lib = _native.load_spgcm()
    n = 8
    sizes = [rng.choice([1, 100, 229_376, 65536]) for _ in range(n)]
    plains = [rng.randbytes(s) for s in sizes]
    refs = [oracle_port.seal(key, 0, 40 + i, p) for i, p in enumerate(plains)]
    word = torch.full((16,), 7, dtype=torch.int32).pin_memory()  # UVA-mapped pinned
    tags = torch.zeros((n, 16), dtype=torch.uint8, device="cuda")
    descs = (_native.SpDesc * n)()
    srcs, dsts = [], []
    for i in range(n):
        c, t = refs[i]
        if i == tamper:
            c = bytes([c[0] ^ 0x80]) + c[1:]
        src = _dev(torch, c)
        tags[i] = torch.tensor(list(t), dtype=torch.uint8)
        dst = torch.full_like(src, 0xAB)
        srcs.append(src)
        dsts.append(dst)
        d = descs[i]
        d.dir, d.reserved, d.iv, d.len = 0, 0x100, 40 + i, sizes[i]
        d.src, d.dst, d.tag = src.data_ptr(), dst.data_ptr(), tags[i].data_ptr()
        d.status = word.data_ptr()
    rc = lib.sp_open_batch(ctx._h, descs, n, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, _native.last_error()
    torch.cuda.synchronize()
    assert int(word[0]) == (7 if tamper is None else 1)
    for i in range(n):
        want = bytes(sizes[i]) if i == tamper else plains[i]
        assert _host(dsts[i]) == want, i


@pytest.mark.parametrize("per_level,nlevels,reps", [(1, 2, 40), (3, 4, 20), (60, 4, 3), (2, 8, 10)])
def test_fused_levels_chain(ctx_for, torch_cuda, per_level, nlevels, reps):
    """sp_crypt_levels: a chain of dependent levels in ONE launch — level 0
    seals plaintexts, every odd level opens what the level before sealed,
    every later even level re-seals that plaintext at a new counter (the
    flush shape of a KV swap-in: stage seal -> receiver open).  Every seal
    matches the oracle bit for bit, every open returns the plaintext, an
    open at the wrong counter fails and is zeroed; repeated launches on one
    stream reuse the in-kernel level counters."""
    import ctypes

    from paper_2411_03357_b200 import _native

    torch = torch_cuda
    rng = random.Random(per_level * 100 + nlevels)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    lib = _native.load_spgcm()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sizes = [rng.choice([1, 17, 2048, 229_376, rng.randrange(1, MIB)]) for _ in range(per_level)]
    plains = [rng.randbytes(s) for s in sizes]
    n = per_level * nlevels
    bufs = [[_dev(torch, p)] for p in plains]  # bufs[i][l] = output of level l-1 for chain i
    for i in range(per_level):
        for _ in range(nlevels):
            bufs[i].append(torch.full_like(bufs[i][0], 0xAB))
    tags = torch.zeros((nlevels, per_level, 16), dtype=torch.uint8, device="cuda")
    status = torch.full((n,), 7, dtype=torch.int32, device="cuda")
    iv_of = lambda lv, i: 1000 * (lv // 2) + i  # noqa: E731  (seal lv and its open lv+1 share it)
    bad = (nlevels - 1, per_level - 1) if nlevels % 2 == 0 else None  # last open at a wrong counter
    descs = (_native.SpDesc * n)()
    for lv in range(nlevels):
        for i in range(per_level):
            d = descs[lv * per_level + i]
            opening = lv % 2 == 1
            iv = iv_of(lv, i) + (1 if (lv, i) == bad else 0)
            d.dir, d.reserved, d.iv, d.len = (lv // 2) & 1, int(opening), iv, sizes[i]
            d.src, d.dst = bufs[i][lv].data_ptr(), bufs[i][lv + 1].data_ptr()
            d.tag = tags[lv - 1 if opening else lv, i].data_ptr()
            d.status = status.data_ptr() + 4 * (lv * per_level + i)
    starts = (ctypes.c_int * (nlevels + 1))(*[lv * per_level for lv in range(nlevels + 1)])
    before = _native.launch_count()
    for _ in range(reps):
        rc = lib.sp_crypt_levels(ctx._h, descs, n, starts, nlevels, stream)
        assert rc == 0, _native.last_error()
    torch.cuda.synchronize()
    assert _native.launch_count() - before == reps  # one launch per call
    st = status.cpu().tolist()
    for lv in range(nlevels):
        for i in range(per_level):
            out = _host(bufs[i][lv + 1])
            if lv % 2 == 0:
                want = oracle_port.seal(key, (lv // 2) & 1, iv_of(lv, i), plains[i])
                assert (out, _host(tags[lv, i])) == want, (lv, i)
            elif (lv, i) == bad:
                assert st[lv * per_level + i] == 1 and out == bytes(sizes[i])
            else:
                assert st[lv * per_level + i] == 0 and out == plains[i], (lv, i)


def test_fused_levels_rejects_bad_layout(ctx_for, torch_cuda):
    import ctypes

    from paper_2411_03357_b200 import _native

    lib = _native.load_spgcm()
    ctx = ctx_for(bytes(32))
    descs = (_native.SpDesc * 2)()
    for starts in ([0, 0, 2], [1, 2], [0, 1]):
        arr = (ctypes.c_int * len(starts))(*starts)
        assert lib.sp_crypt_levels(ctx._h, descs, 2, arr, len(starts) - 1, None) == _native.SP_EINVAL
    arr = (ctypes.c_int * 2)(0, 0)
    assert lib.sp_crypt_levels(ctx._h, descs, 0, arr, 1, None) == _native.SP_EINVAL  # empty batch


def test_small_sms_cap_same_bytes(ctx_for, torch_cuda):
    """sp_ctx_set_small_sms changes only where small launches run: a KV-sized
    batch sealed capped at 8 SMs is bit-identical to the oracle."""
    torch = torch_cuda
    from paper_2411_03357_b200.gcm import GcmContext

    rng = random.Random(11)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = GcmContext(key)
    ctx.set_small_sms(8)
    plains = [rng.randbytes(229_376) for _ in range(4)] + [rng.randbytes(2048), b"\x00"]
    srcs = [_dev(torch, p) for p in plains]
    dsts = [torch.empty_like(s) for s in srcs]
    tags = torch.zeros((len(plains), 16), dtype=torch.uint8, device="cuda")
    ctx.seal_batch([(0, 50 + i, srcs[i], dsts[i], tags[i]) for i in range(len(plains))])
    torch.cuda.synchronize()
    for i, p in enumerate(plains):
        assert (_host(dsts[i]), _host(tags[i])) == oracle_port.seal(key, 0, 50 + i, p), i
    ctx.set_small_sms(0)


def test_fused_levels_concurrent_streams_under_load(ctx_for, torch_cuda):
    """sp_crypt_levels on two streams at once while a matmul keeps the SMs
    busy: every unit of level l waits in-kernel for level l-1, and each
    stream's control words are its own — all results still match the oracle."""
    import ctypes

    from paper_2411_03357_b200 import _native

    torch = torch_cuda
    rng = random.Random(99)
    key = bytes(rng.randrange(256) for _ in range(32))
    ctx = ctx_for(key)
    lib = _native.load_spgcm()
    per_level, nlevels = 8, 4
    n = per_level * nlevels
    setups = []
    for sidx in range(2):
        sizes = [rng.choice([17, 2048, 229_376, 65_536]) for _ in range(per_level)]
        plains = [rng.randbytes(sz) for sz in sizes]
        bufs = [[_dev(torch, p)] + [torch.full((sz,), 0xAB, dtype=torch.uint8, device="cuda") for _ in range(nlevels)]
                for p, sz in zip(plains, sizes)]
        tags = torch.zeros((nlevels, per_level, 16), dtype=torch.uint8, device="cuda")
        status = torch.full((n,), 7, dtype=torch.int32, device="cuda")
        descs = (_native.SpDesc * n)()
        for lv in range(nlevels):
            for i in range(per_level):
                d = descs[lv * per_level + i]
                opening = lv % 2 == 1
                d.dir, d.reserved, d.iv, d.len = 0, int(opening), 100 * sidx + 10 * (lv // 2) + i, sizes[i]
                d.src, d.dst = bufs[i][lv].data_ptr(), bufs[i][lv + 1].data_ptr()
                d.tag = tags[lv - 1 if opening else lv, i].data_ptr()
                d.status = status.data_ptr() + 4 * (lv * per_level + i)
        starts = (ctypes.c_int * (nlevels + 1))(*[lv * per_level for lv in range(nlevels + 1)])
        setups.append((torch.cuda.Stream(), plains, bufs, tags, status, descs, starts, sidx))
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(4):
        a = a @ a  # keeps SMs busy on the default stream while the fused launches run
        for st, _, _, _, _, descs, starts, _ in setups:
            for _ in range(10):
                rc = lib.sp_crypt_levels(ctx._h, descs, n, starts, nlevels, ctypes.c_void_p(st.cuda_stream))
                assert rc == 0, _native.last_error()
    torch.cuda.synchronize()
    for _, plains, bufs, tags, status, _, _, sidx in setups:
        assert status.cpu().tolist() == [7] * per_level + [0] * per_level + [7] * per_level + [0] * per_level
        for lv in range(nlevels):
            for i, p in enumerate(plains):
                out = _host(bufs[i][lv + 1])
                if lv % 2 == 0:
                    want = oracle_port.seal(key, 0, 100 * sidx + 10 * (lv // 2) + i, p)
                    assert (out, _host(tags[lv, i])) == want, (sidx, lv, i)
                else:
                    assert out == p, (sidx, lv, i)

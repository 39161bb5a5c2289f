"""Drop-in channel API on the B200 (channel.py semantics) and the engine's
verify scenarios with real crypto (cli.py:205-330)."""
from __future__ import annotations

import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cipher_vectors.json")))


def test_encrypt_at_decrypt_at_golden():
    from paper_2411_03357_b200 import prng
    from paper_2411_03357_b200.channel import ChannelKey, Direction, decrypt_at, encrypt_at
    import hashlib

    for v in GOLD["vectors"][:120]:
        key = ChannelKey(bytes.fromhex(v["key"]))
        p = bytes.fromhex(v["p_hex"]) if "p_hex" in v else prng.random_bytes(v["payload_seed"], v["len"]).tobytes()
        d = Direction(v["dir"])
        msg = encrypt_at(key, int(v["iv"]), p, d)
        assert msg.auth_tag.hex() == v["tag"] and msg.declared_len == len(p) and not msg.nop
        assert hashlib.sha256(msg.payload).hexdigest() == v["sha256_c"]
        assert decrypt_at(key, int(v["iv"]), msg, d) == p


def test_errors_match_reference():
    from paper_2411_03357_b200.channel import (
        AuthError, ChannelKey, CiphertextMsg, IvReuseError, MAX_MESSAGE_BYTES, decrypt_at, encrypt_at, new_channel,
    )

    k = ChannelKey(bytes(32))
    for e in GOLD["errors"]:
        with pytest.raises(ValueError):
            encrypt_at(k, int(e["iv"]), bytes(e["len"]))
    with pytest.raises(ValueError):
        ChannelKey(b"short")
    msg = encrypt_at(k, 3, b"hello")
    with pytest.raises(AuthError):
        decrypt_at(k, 4, msg)
    with pytest.raises(AuthError):
        decrypt_at(k, 3, CiphertextMsg(msg.payload, bytes(16), 5))
    cpu, gpu = new_channel(seed=1)
    m = cpu.encrypt_next(b"x")
    cpu.send(m)
    cpu.send_iv -= 1
    with pytest.raises(IvReuseError):
        cpu.send(m)
    assert MAX_MESSAGE_BYTES == 32 << 20


def test_verify_counters_fig2():
    """cli.py:205-214: H2D from iv 1, D2H from iv 5 -> 3 and 7."""
    from paper_2411_03357_b200.channel import new_channel

    cpu, gpu = new_channel(seed=1, initial_iv_h2d=1, initial_iv_d2h=5)
    for payload in (b"a", b"b"):
        cpu.send(cpu.encrypt_next(payload))
        assert gpu.recv() == payload
    for payload in (b"c", b"d"):
        gpu.send(gpu.encrypt_next(payload))
        assert cpu.recv() == payload
    assert cpu.send_iv == 3 and gpu.send_iv == 7


def test_verify_replay_rejection():
    """cli.py:294-330: replay, reorder and bit flip all raise AuthError."""
    from paper_2411_03357_b200.channel import AuthError, Direction, new_channel

    cpu, gpu = new_channel(seed=3, test_hooks=True)
    msg = cpu.encrypt_next(b"payload-0")
    cpu.send(msg)
    gpu.recv()
    cpu.channel.hook_resend_raw(Direction.HOST_TO_DEVICE, msg)
    with pytest.raises(AuthError):
        gpu.recv()
    cpu2, gpu2 = new_channel(seed=4, test_hooks=True)
    cpu2.send(cpu2.encrypt_next(b"first"))
    cpu2.send(cpu2.encrypt_next(b"second"))
    cpu2.channel.hook_swap_in_flight(Direction.HOST_TO_DEVICE, 0, 1)
    with pytest.raises(AuthError):
        gpu2.recv()
    cpu3, gpu3 = new_channel(seed=5, test_hooks=True)
    cpu3.send(cpu3.encrypt_next(b"bits"))
    cpu3.channel.hook_corrupt_in_flight(Direction.HOST_TO_DEVICE, 0, byte_index=0, bit=3)
    with pytest.raises(AuthError):
        gpu3.recv()


def test_nop_neutrality_and_dup():
    from paper_2411_03357_b200.channel import AuthError, Direction, new_channel

    cpu, gpu = new_channel(seed=9, test_hooks=True)
    cpu.send(cpu.encrypt_next(b"one"))
    cpu.nop()
    cpu.nop()
    cpu.send(cpu.encrypt_next(b"two"))
    assert gpu.recv() == b"one" and gpu.recv() == b"two"
    assert cpu.channel.sent_log(Direction.HOST_TO_DEVICE) == [(0, False, 3), (1, True, 1), (2, True, 1), (3, False, 3)]
    cpu.send(cpu.encrypt_next(b"three"))
    cpu.channel.hook_duplicate_in_flight(Direction.HOST_TO_DEVICE)
    assert gpu.recv() == b"three"
    with pytest.raises(AuthError):
        gpu.recv()


def test_nop_padding_fig5_gpu():
    import hashlib

    from tests.test_engine_scenarios import nop_padding_scenario

    eng, blocks, shape, d2 = nop_padding_scenario("gpu")
    eng.finish()
    assert shape == ["data", "nop", "data"]
    # data3 and data1 reached the device byte-exact (sha256 of the opened plaintext per delivery)
    got = {addr: digest for _seq, addr, _n, digest in eng.delivered}
    for name in ("data1", "data3"):
        b = blocks[name]
        assert got[b.base] == hashlib.sha256(b.data.tobytes()).hexdigest()


def test_relinquish_launches_nothing_gpu():
    from tests.test_engine_scenarios import relinquish_scenario

    relinquish_scenario("gpu").finish()


def test_engine_tamper_detected():
    """A committed speculative record corrupted on the wire is rejected by
    the device open; finish raises AuthError (GcmAuthError)."""
    from paper_2411_03357_b200.channel import Direction, new_channel
    from paper_2411_03357_b200.engine import CopyRequest, Engine, EngineConfig
    from paper_2411_03357_b200.gcm import GcmAuthError
    from paper_2411_03357_b200.memory import HostMemory, ModelLayer, prng_fill
    from paper_2411_03357_b200.predictor import Prediction, Predictor, TransferClass

    memory = HostMemory()
    cpu, gpu = new_channel(seed=8)
    b = memory.alloc(ModelLayer(1), 70000, prng_fill(4))
    eng = Engine(memory, cpu, gpu, Predictor.scripted([[Prediction(b.id, 0, 0)]], {b.id}), EngineConfig(leeway=0))
    eng.speculate_tick()
    h = eng.copy_h2d(CopyRequest("h2d", b.base, b.len, TransferClass.MODEL_WEIGHTS, block_id=b.id))
    assert h.verdict.value == "hit"
    eng.test_corrupt_in_flight(Direction.HOST_TO_DEVICE, 0, byte_index=100, bit=0)
    eng.sync()
    with pytest.raises(GcmAuthError):
        eng.finish()


def test_opt13b_offload_round_trip_full_size():
    """Two full OPT-13B layers (19 blocks each, 32 MiB chunks) through the
    speculative engine for 2 iterations: every swap-in is opened on the
    device, every swap-out lands back in host memory through the deferred
    host open; afterwards the host blocks must hold exactly the original
    bytes and every tag must have verified."""
    import hashlib

    from paper_2411_03357_b200 import prng, workload
    from paper_2411_03357_b200.replay import ReplayConfig, run_engine

    tr = workload.gen_opt_offload_trace("opt-13b", [1, 2], iterations=2)
    res = run_engine(tr, ReplayConfig(system="specpipe", plane="gpu"))
    eng = res.engine
    rep = eng.report()
    assert rep["hit"] + rep["iv_ahead"] > 0 and rep["deferred_decrypts"] == 2 * 2 * 19
    for spec in tr.header.blocks:
        blk = eng.memory.block(spec.id)
        want = hashlib.sha256(prng.random_bytes(spec.content_seed, spec.nbytes)).hexdigest()
        assert hashlib.sha256(blk.data).hexdigest() == want

"""libsppipe (include/sppipe.h): the native pipeline and predictor.

CPU (dry data plane, no GPU): every reference golden trace replayed through
the native engine gives the reference's sent logs, actions, report() counters,
decision log and errors — per event through the Python API and as one
sp_pipe_replay call; the native predictor decides exactly as the Python one
on random histories; the native engine equals the Python engine on the 180
adversarial OPT-30B-shaped KV traces with the C2 fix on.

GPU: the same goldens with real bytes (delivered plaintext digests per seq),
full-size OPT shapes, host bytes restored after swap-outs, and tamper
detection.
"""
from __future__ import annotations

import ctypes
import random

import pytest

from paper_2411_03357_b200 import _native, workload
from paper_2411_03357_b200.predictor import ModelProfile, Predictor
from paper_2411_03357_b200.replay import ReplayConfig, run_engine
from tests.test_abi import declared
from tests.test_engine_parity import GOLD, compare, make_trace


def test_sppipe_exports_every_declared_symbol():
    lib = _native.load_sppipe()
    names = declared("sppipe.h")
    assert names
    for n in sorted(names):
        assert hasattr(lib, n), f"libsppipe.so does not export {n}"
    assert set(_native.SPPIPE_SYMBOLS) == names


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """ctypes mirrors of include/sppipe.h structs: sizes and field offsets as
    gcc lays them out."""
    import os
    import subprocess

    structs = {"sp_pred_config": _native.SpPredConfig, "sp_prediction": _native.SpPrediction,
               "sp_decision": _native.SpDecision, "sp_pipe_config": _native.SpPipeConfig,
               "sp_action": _native.SpAction, "sp_sent": _native.SpSent, "sp_delivery": _native.SpDelivery,
               "sp_event": _native.SpEvent}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sppipe.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


@pytest.mark.parametrize("dispatch", ["python", "replay"])
@pytest.mark.parametrize("case", GOLD, ids=[f"{c['name']}-{c['system']}" for c in GOLD])
def test_native_control_plane_parity_dry(case, dispatch):
    tr = make_trace(case["params"])
    res = run_engine(tr, ReplayConfig(system=case["system"], record_stream=True, plane="dry", engine="native",
                                      native_dispatch=dispatch), catch=True)
    compare(case, res, with_bytes=False)


@pytest.mark.parametrize("seed", range(40))
def test_native_predictor_matches_python(seed):
    from paper_2411_03357_b200.native_engine import NativePredictor

    rng = random.Random(seed)
    prof = ModelProfile("m", 1000, 10)
    p, q = Predictor(prof), NativePredictor(prof)
    on_gpu = set(range(1, 13))
    for _ in range(rng.randrange(30, 160)):
        r = rng.random()
        if r < 0.45 and on_gpu:
            b = rng.choice(sorted(on_gpu))
            on_gpu.discard(b)
            p.observe_swap_out(b)
            q.observe_swap_out(b)
        elif r < 0.85 and p.outstanding:
            out = sorted(p.outstanding)
            batch = rng.sample(out, rng.randrange(1, min(3, len(out)) + 1))
            p.observe_swap_in(batch)
            q.observe_swap_in(batch)
            on_gpu.update(batch)
        else:
            p.observe_sync()
            q.observe_sync()
        assert q.outstanding == p.outstanding
        assert q.recognize() == p.recognize()
        for depth in (1, 2, 3):
            iv = rng.randrange(100)
            assert q.predict_batches(iv, 8, depth) == p.predict_batches(iv, 8, depth)
    assert q.decision_log == p.decision_log
    for size in (1, 10, 1000, 999, 8192, 1 << 20):
        assert q.classify(size) == p.classify(size)


def test_native_predictor_errors():
    from paper_2411_03357_b200.native_engine import NativePredictor
    from paper_2411_03357_b200.predictor import AmbiguousProfile, UnknownBlock

    q = NativePredictor(ModelProfile("m", 1000, 10))
    q.observe_swap_out(1)
    with pytest.raises(UnknownBlock):
        q.observe_swap_out(1)
    with pytest.raises(UnknownBlock):
        q.observe_swap_in([2])
    with pytest.raises(ValueError):
        q.observe_swap_in([])
    with pytest.raises(AmbiguousProfile):
        NativePredictor(ModelProfile("x", 5, 5)).classify(5)
    with pytest.raises(ValueError):
        NativePredictor().classify(5)


def _adv(policy, rate, seed, kv=28 * 1024):
    base = workload.gen_kvswap_trace(12, policy, kv_block_bytes=kv, parallel_size=4, seed=0)
    return workload.gen_adversarial_trace(base, rate, seed=seed)


def _schedule(engine):
    from tests.test_engine_parity import action_tuple

    return ([action_tuple(a) for a in engine.actions], engine.report(), engine.predictor.decision_log)


def test_native_equals_python_on_adversarial_sweep():
    """180 adversarial KV traces, both compat modes: native == Python engine
    (actions, report, decision log, error)."""
    for compat in (True, False):
        for policy in ("lifo", "fifo"):
            for rate in (0.1, 0.25, 0.5):
                for seed in range(30):
                    tr = _adv(policy, rate, seed)
                    a = run_engine(tr, ReplayConfig(plane="dry", reference_compat=compat), catch=True)
                    b = run_engine(tr, ReplayConfig(plane="dry", reference_compat=compat, engine="native"),
                                   catch=True)
                    assert a.error == b.error, (compat, policy, rate, seed)
                    assert _schedule(a.engine) == _schedule(b.engine), (compat, policy, rate, seed)


def _app_scenario(native: bool):
    """Speculate a FIFO pattern, then application writes over speculated and
    swapped-out ranges and reads of ranges with pending deferred decrypts
    (engine.py:420-440)."""
    from paper_2411_03357_b200.channel import new_channel
    from paper_2411_03357_b200.engine import CopyRequest, Engine, EngineConfig
    from paper_2411_03357_b200.memory import HostMemory, ModelLayer
    from paper_2411_03357_b200.native_engine import NativeEngine, NativePredictor
    from paper_2411_03357_b200.predictor import TransferClass

    mem = HostMemory(pinned=False)
    cpu, gpu = new_channel(seed=1)
    prof = ModelProfile("m", 4096, 64)
    pred = NativePredictor(prof) if native else Predictor(prof)
    cfg = EngineConfig(plane="dry", leeway=0)
    eng = NativeEngine(mem, cpu, gpu, pred, cfg) if native else Engine(mem, cpu, gpu, pred, cfg)
    blocks = [mem.alloc(ModelLayer(i), 4096) for i in range(4)]
    for b in blocks:
        pred.observe_swap_out(b.id)
    W = TransferClass.MODEL_WEIGHTS
    verdicts = []
    for it in range(3):
        for b in blocks:
            verdicts.append(eng.copy_h2d(CopyRequest("h2d", b.base, b.len, W, block_id=b.id)).verdict)
            eng.sync()
            eng.copy_d2h(CopyRequest("d2h", b.base, b.len, W, block_id=b.id))
            if it == 1:
                eng.app_write(blocks[b.id % 4].id, 7, b"\x01\x02\x03")
                eng.app_read(b.id, 0, 16)
    eng.sync()
    eng.finish()
    return verdicts, _schedule(eng)


def test_native_app_access_matches_python():
    a, b = _app_scenario(False), _app_scenario(True)
    assert a == b
    assert a[1][1]["write_faults"] > 0 and a[1][1]["read_faults"] > 0


# ---- GPU -------------------------------------------------------------------------------


@pytest.mark.gpu
def test_native_engine_parity_gpu():
    """Reference goldens with real sealing/opening on the B200 through
    libsppipe: same schedule and the same plaintext reaches the device,
    message by message (sha256 per seq)."""
    for case in GOLD:
        tr = make_trace(case["params"])
        res = run_engine(tr, ReplayConfig(system=case["system"], record_stream=True, plane="gpu", engine="native"),
                         catch=True)
        compare(case, res, with_bytes=case["error"] is None)


@pytest.mark.gpu
def test_native_engine_per_event_dispatch_gpu():
    for case in GOLD[:8]:
        tr = make_trace(case["params"])
        res = run_engine(tr, ReplayConfig(system=case["system"], record_stream=True, plane="gpu", engine="native",
                                          native_dispatch="python"), catch=True)
        compare(case, res, with_bytes=case["error"] is None)


@pytest.mark.gpu
def test_native_opt13b_round_trip_restores_host_bytes():
    import hashlib

    from paper_2411_03357_b200 import prng

    tr = workload.gen_opt_offload_trace("opt-13b", [1, 2], iterations=2)
    res = run_engine(tr, ReplayConfig(system="specpipe", plane="gpu", engine="native"))
    rep = res.engine.report()
    assert rep["hit"] + rep["iv_ahead"] > 0 and rep["deferred_decrypts"] == 2 * 2 * 19
    for spec in tr.header.blocks:
        blk = res.engine.memory.block(spec.id)
        want = hashlib.sha256(prng.random_bytes(spec.content_seed, spec.nbytes)).hexdigest()
        assert hashlib.sha256(blk.data).hexdigest() == want


@pytest.mark.gpu
def test_native_criterion5_gpu():
    """Speculative == no-speculation delivered plaintext per request on
    adversarial OPT-30B KV traces (C2 fixed), through libsppipe."""
    def per_seq(engine):
        out = {}
        for seq, addr, n, digest in engine.delivered:
            out.setdefault(seq, []).append((addr, n, digest))
        return out

    for policy, rate, seed in [("lifo", 0.25, 8), ("fifo", 0.5, 2), ("fifo", 0.1, 26)]:
        tr = _adv(policy, rate, seed, kv=229_376)
        a = run_engine(tr, ReplayConfig(system="specpipe", record_stream=True, reference_compat=False,
                                        engine="native"))
        b = run_engine(tr, ReplayConfig(system="synccc", record_stream=True, reference_compat=False,
                                        engine="native"))
        assert per_seq(a.engine) == per_seq(b.engine)
        assert a.engine.report()["ring_violations"] == 0


@pytest.mark.gpu
def test_native_app_read_sees_swapped_out_bytes_gpu():
    """A swap-out lands through the deferred host open; app_read of the range
    returns the device bytes."""
    import torch

    from paper_2411_03357_b200.channel import new_channel
    from paper_2411_03357_b200.engine import CopyRequest, EngineConfig
    from paper_2411_03357_b200.memory import HostMemory, KvCache
    from paper_2411_03357_b200.native_engine import NativeEngine, NativePredictor
    from paper_2411_03357_b200.predictor import TransferClass

    mem = HostMemory()
    cpu, gpu = new_channel(seed=5)
    pred = NativePredictor(ModelProfile("m", 1 << 20, 229_376))
    eng = NativeEngine(mem, cpu, gpu, pred, EngineConfig())
    b = mem.alloc(KvCache(1, 0), 229_376)
    dev = torch.randint(0, 256, (b.len,), dtype=torch.uint8, device="cuda")
    eng.seed_device(b.id, dev)
    eng.copy_d2h(CopyRequest("d2h", b.base, b.len, TransferClass.KV_CACHE, block_id=b.id))
    got = eng.app_read(b.id, 0, b.len)
    assert got == dev.cpu().numpy().tobytes()
    assert eng.report()["read_faults"] == 1
    eng.finish()


def _one_block_engine(plane: str, strict: bool = False):
    from paper_2411_03357_b200.channel import new_channel
    from paper_2411_03357_b200.engine import EngineConfig
    from paper_2411_03357_b200.memory import HostMemory, ModelLayer, prng_fill
    from paper_2411_03357_b200.native_engine import NativeEngine, NativePredictor

    mem = HostMemory(pinned=None if plane == "gpu" else False)
    cpu, gpu = new_channel(seed=9)
    pred = NativePredictor(ModelProfile("m", 70_000, 64))
    eng = NativeEngine(mem, cpu, gpu, pred, EngineConfig(plane=plane, strict_auth=strict))
    b = mem.alloc(ModelLayer(1), 70_000, prng_fill(4))
    pred.observe_swap_out(b.id)
    return eng, b


def test_native_test_hook_bounds():
    from paper_2411_03357_b200.channel import Direction

    eng, _ = _one_block_engine("dry")
    with pytest.raises(KeyError):
        eng.test_corrupt_in_flight(Direction.HOST_TO_DEVICE, 0)


@pytest.mark.gpu
def test_native_tamper_detected_gpu():
    """A bit flipped in an in-flight H2D message (after its seal, before the
    receiver's open) fails authentication: finish raises AuthError
    (GcmAuthError) and the schedule is otherwise untouched."""
    from paper_2411_03357_b200.channel import Direction
    from paper_2411_03357_b200.engine import CopyRequest
    from paper_2411_03357_b200.gcm import GcmAuthError
    from paper_2411_03357_b200.predictor import TransferClass

    eng, b = _one_block_engine("gpu")
    eng.copy_h2d(CopyRequest("h2d", b.base, b.len, TransferClass.MODEL_WEIGHTS, block_id=b.id))
    eng.test_corrupt_in_flight(Direction.HOST_TO_DEVICE, 0, byte_index=1234, bit=3)
    eng.sync()
    with pytest.raises(GcmAuthError):
        eng.finish()
    # an untouched run of the same request authenticates
    eng2, b2 = _one_block_engine("gpu")
    eng2.copy_h2d(CopyRequest("h2d", b2.base, b2.len, TransferClass.MODEL_WEIGHTS, block_id=b2.id))
    eng2.sync()
    eng2.finish()


@pytest.mark.parametrize("chunk_mib", [4, 16])
def test_layer_larger_than_window_hits_c2_in_both_engines(chunk_mib):
    """A FIFO weight-offload layer split into more chunks than the validator
    window (64) triggers the reference's defect C2 without
    any adversarial mutation; the native and the Python engine raise the same
    EngineError at the same point, and both complete with the fix on: the
    reference's speculation policy then burns records, the window-aware one
    does not speculate batches larger than the window at all."""
    chunk = chunk_mib << 20
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=chunk)
    for compat, aware in ((True, None), (False, False), (False, None)):
        runs = [run_engine(tr, ReplayConfig(plane="dry", engine=e, chunk_bytes=chunk, predictor_chunk_bytes=chunk,
                                            reference_compat=compat, window_aware=aware), catch=True)
                for e in ("python", "native")]
        assert runs[0].error == runs[1].error
        assert _schedule(runs[0].engine) == _schedule(runs[1].engine)
        if compat:
            assert runs[0].error.startswith("EngineError: commit at counter")
        elif aware is False:
            assert runs[0].error is None and runs[0].engine.report()["otf_burned_records"] > 0
        else:
            rep = runs[0].engine.report()
            assert runs[0].error is None and rep.get("otf_burned_records", 0) == 0 and rep["spec_encrypts"] == 0


def test_native_validator_view_matches_python():
    """engine.validator.records as the reference exposes it (cli.py nop-padding
    scenario reads it): same ids, ranges, counters and states as the Python
    engine's validator after a KV trace."""
    tr = _adv("lifo", 0.25, 8)
    a = run_engine(tr, ReplayConfig(plane="dry"), catch=True)
    b = run_engine(tr, ReplayConfig(plane="dry", engine="native"), catch=True)
    ra, rb = a.engine.validator.records, b.engine.validator.records
    assert list(ra) == list(rb) and ra
    for rid in ra:
        x, y = ra[rid], rb[rid]
        assert (x.id, x.base, x.len, x.iv, x.iv_span, x.state, x.block_id) == \
               (y.id, y.base, y.len, y.iv, y.iv_span, y.state, y.block_id)


def _random_trace(seed: int):
    rng = random.Random(seed)
    kind = rng.choice(["offload", "kvswap", "adversarial", "activation"])
    if kind == "offload":
        layers = rng.randrange(3, 9)
        offload = sorted(rng.sample(range(1, layers + 1), rng.randrange(1, layers + 1)))
        return workload.gen_offload_trace(layers, offload, rng.randrange(2, 4),
                                          layer_bytes=rng.choice([4096, 65536, 98309, 1 << 20]), seed=seed)
    if kind == "activation":
        return workload.gen_activation_trace(rng.randrange(3, 9), rng.choice([4099, 49155, 1 << 20]), 2, seed=seed)
    base = workload.gen_kvswap_trace(rng.randrange(4, 12), rng.choice(["lifo", "fifo"]),
                                     kv_block_bytes=rng.choice([4096, 28672, 229_376]),
                                     parallel_size=rng.randrange(2, 5), seed=seed)
    if kind == "kvswap":
        return base
    return workload.gen_adversarial_trace(base, rng.choice([0.1, 0.25, 0.5]), seed=seed)


@pytest.mark.gpu
def test_native_vs_python_random_traces_gpu():
    """Random traces of every generator shape, both engines on the B200 with
    real bytes: identical schedules, reports, decision logs and delivered
    plaintext per message (C2 fixed so every trace completes)."""
    for seed in range(12):
        tr = _random_trace(seed)
        runs = [run_engine(tr, ReplayConfig(plane="gpu", engine=e, record_stream=True, reference_compat=False),
                           catch=True) for e in ("python", "native")]
        assert runs[0].error is None and runs[1].error is None, (seed, runs[0].error, runs[1].error)
        assert _schedule(runs[0].engine) == _schedule(runs[1].engine), seed
        assert runs[0].engine.delivered == runs[1].engine.delivered, seed
        assert runs[0].engine.d2h_stream == runs[1].engine.d2h_stream, seed


@pytest.mark.gpu
@pytest.mark.parametrize("switch", ["SPPIPE_EAGER_OPEN=0", "SPPIPE_SLAB=0", "SPPIPE_OUT_STREAM=1", "SPPIPE_ASYNC_ISSUE=0", "SPPIPE_COMP_STREAMS=1",
                                    "SPPIPE_BATCH_COPY=0"])
def test_native_parity_under_data_plane_switches_gpu(switch):
    """The data-plane switches (drain-time opens, pool-only buffers, own-stream
    swap-out seals, per-copy calls) change scheduling only: the golden parity
    test passes under each (read once per process, so in a subprocess)."""
    import os
    import subprocess
    import sys

    k, v = switch.split("=")
    env = dict(os.environ, **{k: v})
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        f"{here}/test_native_engine.py::test_native_engine_parity_gpu",
                        f"{here}/test_native_engine.py::test_native_tamper_detected_gpu"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("chunk_kib", [64, 32 << 10])
def test_native_opt66b_offload_round_trip_full_size_gpu(chunk_kib):
    """The bench's OPT-66B offload shape at full size (2 offloaded layers of
    2,038,671,360 B, 2 iterations) split into 64 KiB blocks (31,108 per layer,
    ~250k events: slabs, pooled objects, opens on send at scale) or 32 MiB
    blocks: after SpecPipe swapped every layer in and out twice, every host
    block holds exactly its original bytes, and every swap-out was landed."""
    import hashlib

    from paper_2411_03357_b200.replay import prepare_memory

    chunk = chunk_kib << 10
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=chunk)
    cfg = ReplayConfig(system="specpipe", plane="gpu", engine="native", fill="fast", chunk_bytes=min(chunk, 32 << 20),
                       predictor_chunk_bytes=min(chunk, 32 << 20), reference_compat=False)
    mem = prepare_memory(tr, cfg)
    before = [hashlib.sha256(b.data).digest() for b in mem.blocks()]
    res = run_engine(tr, cfg, memory=mem)
    rep = res.engine.report()
    outs = sum(1 for e in tr.events if type(e).__name__ == "SwapOut")
    assert rep["deferred_decrypts"] == outs and rep["ring_violations"] == 0
    assert res.engine.plane_stats()["bytes_d2h"] == tr.swap_bytes() // 2
    after = [hashlib.sha256(b.data).digest() for b in mem.blocks()]
    assert after == before


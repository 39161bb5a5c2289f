"""Engine scenarios of the reference's `specpipe verify` (cli.py:241-291)
and SPEC acceptance criteria that need no bytes, on the native engine's dry
data plane; the GPU versions live in tests/test_gpu_channel.py.  The
reference's scenario mock (cli.py:241-259 `_ScriptedPredictor`) is the native
predictor in scripted mode (`Predictor.scripted`)."""
from __future__ import annotations

from paper_2411_03357_b200.channel import Direction, new_channel
from paper_2411_03357_b200.engine import CopyRequest, Engine, EngineConfig
from paper_2411_03357_b200.memory import HostMemory, ModelLayer, prng_fill
from paper_2411_03357_b200.predictor import Prediction, Predictor, TransferClass
from paper_2411_03357_b200.validator import RecordState


def nop_padding_scenario(plane: str):
    memory = HostMemory(pinned=(plane == "gpu"))
    cpu, gpu = new_channel(seed=2, initial_iv_h2d=1)
    blocks = {name: memory.alloc(ModelLayer(i), 4096, prng_fill(i))
              for i, name in enumerate(("data1", "data2", "data3"), start=1)}
    sched = [[Prediction(blocks["data1"].id, 1, 0)], [Prediction(blocks["data2"].id, 2, 0)],
             [Prediction(blocks["data3"].id, 3, 0)]]
    eng = Engine(memory, cpu, gpu, Predictor.scripted(sched, {b.id for b in blocks.values()}),
                 EngineConfig(speculate=True, leeway=0, plane=plane))
    eng.speculate_tick()

    def req(b):
        return CopyRequest("h2d", b.base, b.len, TransferClass.MODEL_WEIGHTS, block_id=b.id)

    eng.copy_h2d(req(blocks["data3"]))
    eng.copy_h2d(req(blocks["data1"]))
    eng.sync()
    shape = ["nop" if nop else "data" for _, nop, _ in eng.cpu.channel.sent_log(Direction.HOST_TO_DEVICE)]
    d2 = next(r for r in eng.validator.records.values() if r.block_id == blocks["data2"].id)
    return eng, blocks, shape, d2


def test_nop_padding_fig5_dry():
    """Fig 5: wire = [data, nop, data], data2's record burned by the NOP."""
    eng, _, shape, d2 = nop_padding_scenario("dry")
    assert shape == ["data", "nop", "data"]
    assert d2.state is RecordState.INVALIDATED
    assert eng.report()["nop_burned_records"] == 1


def relinquish_scenario(plane: str):
    memory = HostMemory(pinned=(plane == "gpu"))
    cpu, gpu = new_channel(seed=5)
    b1 = memory.alloc(ModelLayer(1), 1000, prng_fill(1))
    b2 = memory.alloc(ModelLayer(2), 1000, prng_fill(2))
    sched = [[Prediction(b1.id, 3, 3), Prediction(b2.id, 4, 3)]]
    eng = Engine(memory, cpu, gpu, Predictor.scripted(sched, {b1.id, b2.id}), EngineConfig(plane=plane))
    eng.speculate_tick()   # queues the two encrypt-ahead tasks
    eng.speculate_tick()   # the next entry point seals and labels them
    assert eng.validator.pending_count() == 2
    eng.flush(wait=(plane == "gpu"))
    launches = eng.plane_stats()["launches"]
    assert eng.relinquish() == 2
    eng.flush(wait=(plane == "gpu"))
    assert eng.plane_stats()["launches"] == launches  # no device work on relinquish
    assert eng.validator.pending_count() == 0
    assert all(r.state is RecordState.INVALIDATED for r in eng.validator.records.values())
    return eng


def test_relinquish_is_metadata_only():
    relinquish_scenario("dry")


def test_window_aware_trim_discards_the_earlier_plan():
    """with window-aware speculation, a prediction switching from
    a batch that fits the record window to one that does not trims the plan
    to nothing; the records encrypted ahead for the earlier plan must be
    discarded (a replan), not left holding window slots until sync expiry."""
    memory = HostMemory(pinned=False)
    cpu, gpu = new_channel(seed=3)
    blocks = [memory.alloc(ModelLayer(i), 4096, prng_fill(i)) for i in range(1, 8)]
    fits = [[Prediction(blocks[0].id, 0, 0)]]
    too_big = [[Prediction(b.id, 1 + k, 0) for k, b in enumerate(blocks[1:6])]]  # 5 blocks > window 4
    pred = Predictor.scripted(None, {b.id for b in blocks}, rounds=[fits, too_big])
    eng = Engine(memory, cpu, gpu, pred, EngineConfig(leeway=0, window=4, reference_compat=False, plane="dry"))
    eng.speculate_tick()   # plan [b1]: queued
    assert eng.report()["replans"] == 0
    eng.speculate_tick()   # seals b1 ahead; the new prediction (5 blocks) does not fit: nothing kept
    rep = eng.report()
    assert rep["spec_encrypts"] == 1 and rep["replans"] == 1, rep
    assert eng.validator.pending_count() == 0
    assert all(r.state is RecordState.INVALIDATED for r in eng.validator.records.values())


def test_record_history_bounds_the_record_list():
    """a long-running pipe's validator list stays bounded with
    EngineConfig.record_history; decisions are unchanged (same report as the
    keep-everything run) and pending records are never forgotten."""
    from paper_2411_03357_b200 import workload
    from paper_2411_03357_b200.replay import ReplayConfig, run_engine

    tr = workload.gen_offload_trace(6, [1, 2, 3, 4, 5, 6], 12, layer_bytes=65536, seed=0)
    runs = [run_engine(tr, ReplayConfig(plane="dry", record_history=h)).engine for h in (0, 8)]
    assert runs[0].report() == runs[1].report()
    full, capped = runs[0].validator.records, runs[1].validator.records
    total = runs[1]._lib.sp_pipe_record_count(runs[1]._h)
    assert len(full) == total and min(full) == 1
    assert len(capped) <= 12 and min(capped) > 1 and max(capped) == total
    assert {i: r.state for i, r in capped.items()} == {i: full[i].state for i in capped}
    assert {r.id for r in runs[1].validator.pending_records()} <= set(capped)

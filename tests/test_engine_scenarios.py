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

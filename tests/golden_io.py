"""Cached loaders of the committed golden fixtures (tests/golden/*.json)."""
from __future__ import annotations

import functools
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def schedules_golden() -> dict:
    """tests/golden/schedules.json (gen_schedule_golden.py: the reference's
    schedules, predictor histories, app scenario and validator records)."""
    with open(os.path.join(GOLDEN, "schedules.json")) as fh:
        return json.load(fh)


def sha(obj) -> str:
    import hashlib

    return hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()


def action_tuple(a):
    return [a.kind.value, a.iv, a.nbytes, a.record_id, a.task_id, a.committed, a.otf, a.count, a.seq]


def schedule_sha(engine) -> str:
    """sha256 of the canonical (sent_h2d, sent_d2h, actions) — the same
    digest gen_schedule_golden.py stores for the reference engine."""
    from paper_2411_03357_b200.channel import Direction

    ch = engine.cpu.channel
    return sha({"sent_h2d": [list(x) for x in ch.sent_log(Direction.HOST_TO_DEVICE)],
                "sent_d2h": [list(x) for x in ch.sent_log(Direction.DEVICE_TO_HOST)],
                "actions": [action_tuple(a) for a in engine.actions]})


def golden_trace(p: dict):
    """A schedules.json trace rebuilt from its params with this repo's generators."""
    import random

    from paper_2411_03357_b200 import workload as w

    g = p["gen"]
    if g == "chunked":
        return w.gen_chunked_offload_trace(p["layers"], p["offload"], p["iterations"], p["layer_bytes"],
                                           chunk_bytes=p["chunk"], seed=p["seed"])
    if g == "opt":
        return w.gen_opt_offload_trace(p["model"], p["offload"], p["iterations"], chunk_bytes=p["chunk"],
                                       seed=p["seed"], quant_bits=p.get("quant_bits", 16))
    if g == "adversarial":
        base = w.gen_kvswap_trace(p["requests"], p["policy"], kv_block_bytes=p["kv"], parallel_size=4, seed=0)
        return w.gen_adversarial_trace(base, p["rate"], seed=p["seed"])
    if g == "random":
        rng = random.Random(p["seed"])
        kind = rng.choice(["offload", "kvswap", "adversarial", "activation"])
        seed = p["seed"]
        if kind == "offload":
            layers = rng.randrange(3, 9)
            offload = sorted(rng.sample(range(1, layers + 1), rng.randrange(1, layers + 1)))
            return w.gen_offload_trace(layers, offload, rng.randrange(2, 4),
                                       layer_bytes=rng.choice([4096, 65536, 98309, 1 << 20]), seed=seed)
        if kind == "activation":
            return w.gen_activation_trace(rng.randrange(3, 9), rng.choice([4099, 49155, 1 << 20]), 2, seed=seed)
        base = w.gen_kvswap_trace(rng.randrange(4, 12), rng.choice(["lifo", "fifo"]),
                                  kv_block_bytes=rng.choice([4096, 28672, 229_376]),
                                  parallel_size=rng.randrange(2, 5), seed=seed)
        if kind == "kvswap":
            return base
        return w.gen_adversarial_trace(base, rng.choice([0.1, 0.25, 0.5]), seed=seed)
    raise ValueError(g)


def schedule_case(name: str, system: str = "specpipe") -> dict:
    for r in schedules_golden()["schedules"]:
        if r["name"] == name and r["system"] == system:
            return r
    raise KeyError((name, system))


def replay_schedule_case(rec: dict, plane: str, **overrides):
    """Replay a schedules.json case through libsppipe the way the generator
    drove the reference (chunk on predictor and engine when set)."""
    from paper_2411_03357_b200.replay import ReplayConfig, run_engine

    tr = golden_trace(rec["params"])
    kw = dict(system=rec["system"], plane=plane, record_stream=rec["delivered_sha256"] is not None)
    if rec["chunk"]:
        kw.update(chunk_bytes=rec["chunk"], predictor_chunk_bytes=rec["chunk"])
    kw.update(overrides)
    return tr, run_engine(tr, ReplayConfig(**kw), catch=True)


def assert_schedule_matches(rec: dict, res, with_bytes: bool = False) -> None:
    eng = res.engine
    assert res.error == rec["error"], (rec["name"], res.error)
    assert eng.report() == rec["report"], rec["name"]
    assert eng.predictor.decision_log == rec["decision_log"], rec["name"]
    assert len(eng.actions) == rec["n_actions"], rec["name"]
    assert schedule_sha(eng) == rec["schedule_sha256"], rec["name"]
    if with_bytes:
        assert sha([list(d) for d in eng.delivered]) == rec["delivered_sha256"], rec["name"]
        assert sha([list(d) for d in eng.d2h_stream]) == rec["d2h_stream_sha256"], rec["name"]

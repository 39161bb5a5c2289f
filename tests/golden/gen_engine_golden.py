"""Generate control-plane golden logs by replaying traces through the
REFERENCE engine (build container only: needs /root/reference).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_engine_golden.py

For each case it stores the trace fingerprint (sha256 of the reference's JSONL
lines), the H2D/D2H sent logs (channel.py:229-230), the engine action list
(engine.py:187), report() (engine.py:617-624), the predictor decision log
(predictor.py:327), the delivered stream digests per seq (engine.py:212) and
the D2H small-I/O stream, or the exception the reference raised (defect C2).
Cases follow SURVEY §8d, scaled so the whole set replays in seconds.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from specpipe import simulator, workload  # noqa: E402
from specpipe.memory import KvCache, ModelLayer  # noqa: E402
from specpipe.predictor import ModelProfile  # noqa: E402
from specpipe.workload import (  # noqa: E402
    BlockSpec, ComputeEvent, SCHEMA_VERSION, SwapInRequest, SwapOut, SyncEvent, Trace, TraceHeader,
)

HERE = os.path.dirname(os.path.abspath(__file__))
KIB = 1024


def activation_trace(layers: int, act_bytes: int, steps: int, seed: int = 0) -> Trace:
    """Config 4 shape: forward swaps activations out 1..L,
    backward swaps them in L..1, each followed by sync + compute."""
    import random

    rng = random.Random(seed)
    profile = ModelProfile("opt-30b-act", act_bytes, act_bytes // 7 + 1)
    blocks = tuple(BlockSpec(id=i + 1, kind=ModelLayer(i + 1), nbytes=act_bytes, resident="gpu",
                             content_seed=rng.randrange(1 << 30)) for i in range(layers))
    ev, t = [], 0
    for _ in range(steps):
        for b in blocks:
            ev.append(ComputeEvent(t, 1000)); t += 1
            ev.append(SwapOut(t, b.id)); t += 1
        for b in reversed(blocks):
            ev.append(SwapInRequest(t, b.id)); ev.append(SyncEvent(t)); t += 1
            ev.append(ComputeEvent(t, 1000)); t += 1
    tr = Trace(TraceHeader(SCHEMA_VERSION, profile, {"generator": "activation", "layers": layers,
                                                      "act_bytes": act_bytes, "steps": steps, "seed": seed},
                           blocks), ev)
    workload.validate_trace(tr)
    return tr


def cases():
    out = []
    out.append(("offload_l6", {"gen": "offload", "layers": 6, "offload": [1, 2, 3, 4, 5, 6], "iterations": 3,
                               "layer_bytes": 64 * KIB, "seed": 0}))
    out.append(("offload_l8_half", {"gen": "offload", "layers": 8, "offload": [2, 4, 5, 7], "iterations": 4,
                                    "layer_bytes": 96 * KIB + 5, "seed": 3}))
    for pol in ("lifo", "fifo"):
        out.append((f"kv_{pol}", {"gen": "kvswap", "requests": 12, "policy": pol, "kv_block_bytes": 28 * KIB,
                                  "parallel_size": 4, "small_io_size": 2048, "seed": 0}))
    # adversarial OPT-30B-shaped KV traces (scaled block size); includes
    # relinquish seeds and EngineError (C2) seeds from SURVEY §8d config 3
    for pol, rate, seeds in (("lifo", 0.1, (3, 7, 0)), ("lifo", 0.25, (8, 9)), ("lifo", 0.5, (6, 17)),
                             ("fifo", 0.1, (19, 26)), ("fifo", 0.25, (2, 25)), ("fifo", 0.5, (2, 23))):
        for s in seeds:
            out.append((f"adv_{pol}_{rate}_{s}", {"gen": "adversarial", "policy": pol, "rate": rate, "seed": s,
                                                  "requests": 12, "kv_block_bytes": 28 * KIB, "parallel_size": 4}))
    out.append(("activation_l10", {"gen": "activation", "layers": 10, "act_bytes": 48 * KIB + 3, "steps": 3}))
    # full-size shapes, replayed on the GPU by the
    # slow-marked parity test
    out.append(("full_kv_opt30b_lifo_adv", {"gen": "adversarial", "policy": "lifo", "rate": 0.25, "seed": 8,
                                            "requests": 12, "kv_block_bytes": 229_376, "parallel_size": 4}))
    out.append(("full_kv_opt30b_fifo", {"gen": "kvswap", "requests": 12, "policy": "fifo",
                                        "kv_block_bytes": 229_376, "parallel_size": 4, "small_io_size": 2048,
                                        "seed": 0}))
    out.append(("full_act_opt30b", {"gen": "activation", "layers": 4, "act_bytes": 29_360_128, "steps": 2}))
    out.append(("full_offload_opt13b", {"gen": "opt_offload", "model": "opt-13b", "offload": [21, 22],
                                        "iterations": 2}))
    return out


def make_trace(p: dict) -> Trace:
    g = p["gen"]
    if g == "offload":
        return workload.gen_offload_trace(p["layers"], p["offload"], p["iterations"], layer_bytes=p["layer_bytes"],
                                          seed=p["seed"])
    if g == "kvswap":
        return workload.gen_kvswap_trace(p["requests"], p["policy"], kv_block_bytes=p["kv_block_bytes"],
                                         parallel_size=p["parallel_size"], small_io_size=p["small_io_size"],
                                         seed=p["seed"])
    if g == "adversarial":
        base = workload.gen_kvswap_trace(p["requests"], p["policy"], kv_block_bytes=p["kv_block_bytes"],
                                         parallel_size=p["parallel_size"], seed=0)
        return workload.gen_adversarial_trace(base, p["rate"], seed=p["seed"])
    if g == "activation":
        return activation_trace(p["layers"], p["act_bytes"], p["steps"])
    if g == "opt_offload":
        return opt_offload_trace(p["model"], p["offload"], p["iterations"])
    raise ValueError(g)


OPT = {"opt-13b": (5120, 40), "opt-30b": (7168, 48), "opt-66b": (9216, 64)}


def opt_offload_trace(model: str, offload, iterations: int, chunk: int = 32 * 1024 * 1024) -> Trace:
    """Config 2 shape: each OPT layer (2*(12h^2+13h) bytes) split into 32 MiB
    blocks + tail so the reference classifies them MODEL_WEIGHTS (defect C3)."""
    import random

    h, nl = OPT[model]
    layer = 2 * (12 * h * h + 13 * h)
    sizes = [chunk] * (layer // chunk) + ([layer % chunk] if layer % chunk else [])
    rng = random.Random(0)
    profile = ModelProfile(model, layer, 16 * h * 2)
    blocks, of, nid = [], {}, 1
    for l in sorted(offload):
        of[l] = []
        for n in sizes:
            blocks.append(BlockSpec(id=nid, kind=ModelLayer(l), nbytes=n, resident="cpu",
                                    content_seed=rng.randrange(1 << 30)))
            of[l].append(nid)
            nid += 1
    ev, t = [], 0
    for _ in range(iterations):
        for l in range(1, nl + 1):
            ids = of.get(l)
            if ids:
                ev.extend(SwapInRequest(t, b) for b in ids)
                ev.append(SyncEvent(t))
                t += 1
            ev.append(ComputeEvent(t, 200_000))
            t += 1
            if ids:
                ev.extend(SwapOut(t, b) for b in ids)
                t += 1
    params = {"generator": "opt_offload", "model": model, "offload": sorted(offload), "iterations": iterations,
              "chunk_bytes": chunk, "layer_bytes": layer, "compute_per_layer": 200_000, "seed": 0}
    tr = Trace(TraceHeader(SCHEMA_VERSION, profile, params, tuple(blocks)), ev)
    workload.validate_trace(tr)
    return tr


def action_tuple(a):
    return [a.kind.value, a.iv, a.nbytes, a.record_id, a.task_id, a.committed, a.otf, a.count, a.seq]


def run_case(name: str, p: dict, system: str) -> dict:
    tr = make_trace(p)
    lines = list(workload.trace_to_lines(tr))
    rec = {"name": name, "params": p, "system": system,
           "trace_sha256": hashlib.sha256("\n".join(lines).encode()).hexdigest(), "n_events": len(tr.events)}
    kind = {"specpipe": simulator.SystemKind.SPECPIPE, "synccc": simulator.SystemKind.SYNCCC}[system]
    cfg = simulator.SimConfig(system=kind, record_stream=True)
    rp = simulator._Replay(tr, cfg)
    eng = rp.engine
    try:
        rp.run()
        rec["error"] = None
    except Exception as exc:  # defect C2 reproduces as EngineError
        rec["error"] = f"{type(exc).__name__}: {exc}"
    from specpipe.channel import Direction

    rec["sent_h2d"] = [list(x) for x in eng.cpu.channel.sent_log(Direction.HOST_TO_DEVICE)]
    rec["sent_d2h"] = [list(x) for x in eng.cpu.channel.sent_log(Direction.DEVICE_TO_HOST)]
    rec["actions"] = [action_tuple(a) for a in eng.actions]
    rec["report"] = eng.report()
    rec["decision_log"] = eng.predictor.decision_log
    rec["delivered"] = [list(d) for d in eng.delivered]
    rec["d2h_stream"] = [list(d) for d in eng.d2h_stream]
    return rec


def main() -> None:
    recs = []
    for name, p in cases():
        for system in ("specpipe", "synccc"):
            if system == "synccc" and not name.startswith(("offload_l6", "kv_lifo", "adv_lifo_0.25_8")):
                continue
            recs.append(run_case(name, p, system))
            r = recs[-1]
            print(f"{name:28} {system:9} events={r['n_events']:5} h2d={len(r['sent_h2d']):5} "
                  f"nops={r['report']['nops']:4} rel={r['report']['relinquishes']} err={r['error']}")
    with open(os.path.join(HERE, "engine_traces.json"), "w") as fh:
        json.dump({"generator": "tests/golden/gen_engine_golden.py (reference specpipe 0.1.0)", "cases": recs}, fh)


if __name__ == "__main__":
    main()

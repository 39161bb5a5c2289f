"""Reference-generated control-plane goldens for the native engine and
predictor (build container only: needs /root/reference).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_schedule_golden.py

Everything here runs the REFERENCE's own classes (specpipe 0.1.0:
engine.Engine, predictor.Predictor/SwapHistory/recognize/predict_batches,
validator.Validator via the engine, workload.load_trace):

* schedules — full-size traces (SURVEY §8d config 1 at 64 MiB layers, the
  bench's OPT-66B offload trace, a 1 MiB and two 4/16 MiB chunk-sweep points,
  the 180 adversarial OPT-30B-shaped KV traces, random traces of every
  generator).  Traces are generated with this repo's workload.py, written as
  reference JSONL and loaded with the reference's `load_trace` (so the trace
  format is pinned too).  Stored: the error (defect C2 included), report(),
  decision log, and sha256 of the canonical JSON of (sent_h2d, sent_d2h,
  actions) — plus, where payloads are real, of the delivered streams.
* the crypto seams (`channel.encrypt_at`, `channel.decrypt_at`,
  `engine.encrypt_at`, engine.py:34) are replaced by an identity seal with a
  zero tag: no decision depends on ciphertext bytes (the cipher is pinned
  separately by cipher_vectors.json), and the delivered plaintext is then
  exactly what the reference would deliver.  For the multi-GB traces
  `prng_fill` and the engine's per-message sha256 (defect C4) are stubbed as
  well (schedule only, `delivered_sha256` null).
* predictor — 40 random swap histories: per step the outstanding set,
  recognize() and predict_batches at depths 1-3; the decision log; classify.
* app scenario and validator records (engine.py:420-440, validator.py:46-63).
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import tempfile

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, ROOT)

import specpipe.channel as rch  # noqa: E402
import specpipe.engine as reng  # noqa: E402
import specpipe.memory as rmem  # noqa: E402
import specpipe.predictor as rpred  # noqa: E402
import specpipe.simulator as rsim  # noqa: E402
import specpipe.workload as rwl  # noqa: E402

from paper_2411_03357_b200 import workload as ours  # noqa: E402

MIB = 1 << 20
_real = {"enc": rch.encrypt_at, "dec": rch.decrypt_at, "prng": rmem.prng_fill, "hashlib": reng.hashlib}


_ZERO = memoryview(bytes(rch.MAX_MESSAGE_BYTES))
_share_zero = {"on": False}


def _id_encrypt(key, iv, plaintext, direction=rch.Direction.HOST_TO_DEVICE):
    if not 0 <= iv < 1 << 64:
        raise ValueError("counter out of range")
    n = len(plaintext)
    if not 1 <= n <= rch.MAX_MESSAGE_BYTES:
        raise ValueError("bad length")
    # schedule-only runs (payloads stubbed to zeros): large payloads share one
    # zero buffer, since the reference keeps every record's ciphertext alive
    payload = _ZERO[:n] if _share_zero["on"] and n >= (1 << 20) else bytes(plaintext)
    return rch.CiphertextMsg(payload=payload, auth_tag=bytes(16), declared_len=n)


def _id_decrypt(key, iv, msg, direction=rch.Direction.HOST_TO_DEVICE):
    return msg.payload


class _NoHash:
    @staticmethod
    def sha256(_data=b""):
        class _H:
            def hexdigest(self):
                return None
        return _H()


def stub(crypto: bool = True, payloads: bool = False) -> None:
    rch.encrypt_at = reng.encrypt_at = _id_encrypt if crypto else _real["enc"]
    rch.decrypt_at = _id_decrypt if crypto else _real["dec"]
    _share_zero["on"] = payloads
    if payloads:
        zero = lambda seed: (lambda n: bytes(n))  # noqa: E731
        rmem.prng_fill = rsim.prng_fill = zero
        reng.hashlib = _NoHash
    else:
        rmem.prng_fill = rsim.prng_fill = _real["prng"]
        reng.hashlib = _real["hashlib"]


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()


def action_tuple(a):
    return [a.kind.value, a.iv, a.nbytes, a.record_id, a.task_id, a.committed, a.otf, a.count, a.seq]


def to_reference(tr) -> "rwl.Trace":
    with tempfile.NamedTemporaryFile("w", suffix=".jsonl", delete=False) as fh:
        fh.write("\n".join(ours.trace_to_lines(tr)) + "\n")
        path = fh.name
    try:
        return rwl.load_trace(path)
    finally:
        os.unlink(path)


def make_trace(p: dict):
    """Trace from its params with THIS repo's generators (tests rebuild it the same way)."""
    g = p["gen"]
    if g == "chunked":
        return ours.gen_chunked_offload_trace(p["layers"], p["offload"], p["iterations"], p["layer_bytes"],
                                              chunk_bytes=p["chunk"], seed=p["seed"])
    if g == "opt":
        return ours.gen_opt_offload_trace(p["model"], p["offload"], p["iterations"], chunk_bytes=p["chunk"],
                                          seed=p["seed"], quant_bits=p.get("quant_bits", 16))
    if g == "adversarial":
        base = ours.gen_kvswap_trace(p["requests"], p["policy"], kv_block_bytes=p["kv"], parallel_size=4, seed=0)
        return ours.gen_adversarial_trace(base, p["rate"], seed=p["seed"])
    if g == "random":
        return random_trace(p["seed"])
    raise ValueError(g)


def random_trace(seed: int):
    rng = random.Random(seed)
    kind = rng.choice(["offload", "kvswap", "adversarial", "activation"])
    if kind == "offload":
        layers = rng.randrange(3, 9)
        offload = sorted(rng.sample(range(1, layers + 1), rng.randrange(1, layers + 1)))
        return ours.gen_offload_trace(layers, offload, rng.randrange(2, 4),
                                      layer_bytes=rng.choice([4096, 65536, 98309, 1 << 20]), seed=seed)
    if kind == "activation":
        return ours.gen_activation_trace(rng.randrange(3, 9), rng.choice([4099, 49155, 1 << 20]), 2, seed=seed)
    base = ours.gen_kvswap_trace(rng.randrange(4, 12), rng.choice(["lifo", "fifo"]),
                                 kv_block_bytes=rng.choice([4096, 28672, 229_376]),
                                 parallel_size=rng.randrange(2, 5), seed=seed)
    if kind == "kvswap":
        return base
    return ours.gen_adversarial_trace(base, rng.choice([0.1, 0.25, 0.5]), seed=seed)


def run_reference(trace, system: str, chunk: int | None = None):
    """simulator._Replay's engine build + dispatch (simulator.py:253-284,
    404-426); `chunk` also sets PredictorConfig/EngineConfig.chunk_bytes
    (the simulator hard-codes PredictorConfig())."""
    rt = to_reference(trace)
    kind = {"specpipe": rsim.SystemKind.SPECPIPE, "synccc": rsim.SystemKind.SYNCCC}[system]
    if chunk is None:
        rp = rsim._Replay(rt, rsim.SimConfig(system=kind, record_stream=True))
        eng = rp.engine
        run = rp.run
    else:
        header = rt.header
        memory = rmem.HostMemory()
        cpu, gpu = rch.new_channel(seed=0)
        pred = rpred.Predictor(header.profile, rpred.PredictorConfig(chunk_bytes=chunk))
        spec_on = system == "specpipe"
        eng = reng.Engine(memory, cpu, gpu, pred,
                          reng.EngineConfig(chunk_bytes=chunk, speculate=spec_on, defer_swap_decrypt=spec_on,
                                            record_stream=True))
        blocks = {}
        for spec in header.blocks:
            if spec.resident == "cpu":
                b = memory.alloc(spec.kind, spec.nbytes, rmem.prng_fill(spec.content_seed))
                if isinstance(spec.kind, (rmem.ModelLayer, rmem.KvCache)):
                    pred.observe_swap_out(b.id)
            else:
                b = memory.alloc(spec.kind, spec.nbytes)
                eng.seed_device(b.id, rmem.prng_fill(spec.content_seed)(spec.nbytes))
            blocks[spec.id] = (b, rpred.classify(spec.nbytes, header.profile, pred.config))

        def run():
            io = 0
            for ev in rt.events:
                if isinstance(ev, rwl.SwapInRequest):
                    b, cls = blocks[ev.block]
                    eng.copy_h2d(reng.CopyRequest("h2d", b.base, b.len, cls, block_id=b.id))
                elif isinstance(ev, rwl.SwapOut):
                    b, cls = blocks[ev.block]
                    eng.copy_d2h(reng.CopyRequest("d2h", b.base, b.len, cls, block_id=b.id))
                elif isinstance(ev, rwl.SmallIoEvent):
                    eng.small_io(ev.direction, ev.size, rsim._small_io_payload(0, io, ev.size))
                    io += 1
                elif isinstance(ev, rwl.SyncEvent):
                    eng.sync()
                elif isinstance(ev, rwl.AppWriteEvent):
                    b, _ = blocks[ev.block]
                    eng.app_write(b.id, ev.offset, rsim._app_write_payload(ev.data_seed, ev.size))
            eng.finish()
    try:
        run()
        err = None
    except Exception as exc:  # defect C2 reproduces as EngineError
        err = f"{type(exc).__name__}: {exc}"
    return eng, err, rt


def schedule_record(name: str, p: dict, system: str, payloads_real: bool, chunk: int | None = None) -> dict:
    tr = make_trace(p)
    stub(crypto=True, payloads=not payloads_real)
    eng, err, _ = run_reference(tr, system, chunk)
    D = rch.Direction
    sched = {"sent_h2d": [list(x) for x in eng.cpu.channel.sent_log(D.HOST_TO_DEVICE)],
             "sent_d2h": [list(x) for x in eng.cpu.channel.sent_log(D.DEVICE_TO_HOST)],
             "actions": [action_tuple(a) for a in eng.actions]}
    rec = {"name": name, "params": p, "system": system, "chunk": chunk,
           "trace_sha256": hashlib.sha256("\n".join(ours.trace_to_lines(tr)).encode()).hexdigest(),
           "n_events": len(tr.events), "error": err, "report": eng.report(),
           "decision_log": eng.predictor.decision_log, "n_actions": len(sched["actions"]),
           "n_sent_h2d": len(sched["sent_h2d"]), "schedule_sha256": sha(sched),
           "delivered_sha256": None, "d2h_stream_sha256": None}
    if payloads_real:
        rec["delivered_sha256"] = sha([list(d) for d in eng.delivered])
        rec["d2h_stream_sha256"] = sha([list(d) for d in eng.d2h_stream])
        rec["n_delivered"] = len(eng.delivered)
    return rec


def schedules() -> list:
    out = []
    # config 1 at its real size: 8 x 64 MiB layers (2 x 32 MiB blocks), 3 iterations
    c1 = {"gen": "chunked", "layers": 8, "offload": list(range(1, 9)), "iterations": 3, "layer_bytes": 64 * MIB,
          "chunk": 32 * MIB, "seed": 0}
    for system in ("specpipe", "synccc"):
        out.append(schedule_record("config1_64mib", c1, system, payloads_real=True))
    # the bench's OPT-66B offload trace (61 x 32 MiB blocks per layer, 8 iterations)
    o66 = {"gen": "opt", "model": "opt-66b", "offload": [1, 2], "iterations": 8, "chunk": 32 * MIB, "seed": 0}
    for system in ("specpipe", "synccc"):
        out.append(schedule_record("opt66b_bench", o66, system, payloads_real=False))
    # OPT-175B, fp16 and the paper's 4-bit
    for bits in (16, 4):
        p = {"gen": "opt", "model": "opt-175b", "offload": [1, 2], "iterations": 2, "chunk": 32 * MIB, "seed": 0,
             "quant_bits": bits}
        out.append(schedule_record(f"opt175b_{bits}bit", p, "specpipe", payloads_real=False))
    # chunk-sweep points with the chunk set on predictor and engine (layers of
    # more than 64 chunks trip defect C2 in the reference)
    for mib in (1, 4, 16):
        p = {"gen": "opt", "model": "opt-66b", "offload": [1, 2], "iterations": 2, "chunk": mib * MIB, "seed": 0}
        out.append(schedule_record(f"opt66b_{mib}mib", p, "specpipe", payloads_real=False, chunk=mib * MIB))
    # SPEC criterion 5's population: 180 adversarial OPT-30B-shaped KV traces (scaled blocks)
    for policy in ("lifo", "fifo"):
        for rate in (0.1, 0.25, 0.5):
            for seed in range(30):
                p = {"gen": "adversarial", "policy": policy, "rate": rate, "seed": seed, "requests": 12,
                     "kv": 28 * 1024}
                out.append(schedule_record(f"adv_{policy}_{rate}_{seed}", p, "specpipe", payloads_real=True))
    for seed in range(12):
        out.append(schedule_record(f"random_{seed}", {"gen": "random", "seed": seed}, "specpipe",
                                   payloads_real=True))
    return out


def predictor_histories() -> list:
    out = []
    prof = rpred.ModelProfile("m", 1000, 10)
    for seed in range(40):
        rng = random.Random(seed)
        p = rpred.Predictor(prof)
        on_gpu = set(range(1, 13))
        ops, expect = [], []
        for _ in range(rng.randrange(30, 160)):
            r = rng.random()
            if r < 0.45 and on_gpu:
                b = rng.choice(sorted(on_gpu))
                on_gpu.discard(b)
                p.observe_swap_out(b)
                ops.append(["out", b])
            elif r < 0.85 and p.outstanding:
                outs = sorted(p.outstanding)
                batch = rng.sample(outs, rng.randrange(1, min(3, len(outs)) + 1))
                p.observe_swap_in(batch)
                on_gpu.update(batch)
                ops.append(["in", batch])
            else:
                p.observe_sync()
                ops.append(["sync"])
            h = p.recognize()
            preds = []
            for depth in (1, 2, 3):
                iv = rng.randrange(100)
                preds.append([iv, depth, [[[q.block, q.predicted_iv, q.leeway] for q in b]
                                          for b in p.predict_batches(iv, 8, depth)]])
            expect.append({"outstanding": sorted(p.outstanding),
                           "hypothesis": [h.kind.value, h.confidence, [list(c) for c in h.cycle], h.phase],
                           "predict": preds})
        out.append({"seed": seed, "ops": ops, "expect": expect, "decision_log": p.decision_log,
                    "in_batches": [list(b) for b in p.history.in_batches],
                    "events": [[e[0], sorted(e[1]) if e[0] == "in" else (e[1] if e[0] == "out" else None)]
                               for e in p.history.events],
                    "classify": {str(s): rpred.classify(s, prof).value for s in (1, 10, 1000, 999, 8192, 1 << 20)}})
    return out


def app_scenario() -> dict:
    """Speculate a FIFO pattern, then application writes over speculated and
    swapped-out ranges and reads of ranges with pending deferred decrypts."""
    stub(crypto=True, payloads=False)
    mem = rmem.HostMemory()
    cpu, gpu = rch.new_channel(seed=1)
    prof = rpred.ModelProfile("m", 4096, 64)
    pred = rpred.Predictor(prof)
    eng = reng.Engine(mem, cpu, gpu, pred, reng.EngineConfig(leeway=0))
    blocks = [mem.alloc(rmem.ModelLayer(i), 4096) for i in range(4)]
    for b in blocks:
        pred.observe_swap_out(b.id)
    W = rpred.TransferClass.MODEL_WEIGHTS
    verdicts, reads = [], []
    for it in range(3):
        for b in blocks:
            verdicts.append(eng.copy_h2d(reng.CopyRequest("h2d", b.base, b.len, W, block_id=b.id)).verdict)
            eng.sync()
            eng.copy_d2h(reng.CopyRequest("d2h", b.base, b.len, W, block_id=b.id))
            if it == 1:
                eng.app_write(blocks[b.id % 4].id, 7, b"\x01\x02\x03")
                reads.append(eng.app_read(b.id, 0, 16).hex())
    eng.sync()
    eng.finish()
    return {"verdicts": [v.value if v else None for v in verdicts], "reads": reads,
            "actions": [action_tuple(a) for a in eng.actions], "report": eng.report(),
            "decision_log": pred.decision_log}


def validator_records() -> dict:
    p = {"gen": "adversarial", "policy": "lifo", "rate": 0.25, "seed": 8, "requests": 12, "kv": 28 * 1024}
    stub(crypto=True, payloads=False)
    eng, err, _ = run_reference(make_trace(p), "specpipe")
    recs = [[r.id, r.base, r.len, r.iv, r.iv_span, r.state.value, r.block_id]
            for r in eng.validator.records.values()]
    return {"params": p, "error": err, "records": recs, "counters": dict(eng.validator.counters)}


def main() -> None:
    out = {"generator": "tests/golden/gen_schedule_golden.py (reference specpipe 0.1.0, crypto seams = identity)",
           "schedules": schedules(), "predictor": predictor_histories(), "app_scenario": app_scenario(),
           "validator": validator_records()}
    for r in out["schedules"]:
        if not r["name"].startswith("adv_"):
            print(f"{r['name']:22} {r['system']:9} events={r['n_events']:6} actions={r['n_actions']:6} "
                  f"nops={r['report']['nops']:5} err={r['error']}")
    with open(os.path.join(HERE, "schedules.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()

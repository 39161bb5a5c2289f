"""Trace replay through the B200 engine — the driver half of the reference's
simulator (`_Replay._build_engine` simulator.py:253-284 and
`_dispatch_engine` simulator.py:404-426) without its CPU cost model: here the
time is real (CUDA events / wall clock on the GPU box).

Systems (simulator.py SystemKind):
  specpipe — speculation on, deferred swap decrypts (the product path);
  synccc   — every transfer sealed/opened on the fly, synchronous decrypts;
  nocc     — no crypto at all: plain pinned-memory cudaMemcpyAsync swaps on
             the same streams (the "unencrypted swap" the north star compares
             against).
"""
from __future__ import annotations

import time
from dataclasses import dataclass

from .channel import new_channel
from .engine import CopyRequest, Engine, EngineConfig
from .memory import HostMemory, KvCache, ModelLayer
from .predictor import Predictor, PredictorConfig, classify
from .prng import app_write_payload, prng_fill, random_bytes, small_io_payload
from .workload import AppWriteEvent, ComputeEvent, SmallIoEvent, SwapInRequest, SwapOut, SyncEvent, Trace


@dataclass(frozen=True)
class ReplayConfig:
    system: str = "specpipe"
    workers: int = 2
    window: int = 64
    leeway: int = 8
    depth: int = 1
    seed: int = 0
    record_stream: bool = False
    plane: str = "gpu"
    chunk_bytes: int = 32 * 1024 * 1024
    predictor_chunk_bytes: int | None = None  # default: PredictorConfig() as the reference driver
    # "seeded": block payloads = prng_fill(content_seed), bit-exact with the
    # reference (parity runs); "fast": device-generated random bytes copied to
    # the pinned blocks (benchmarks: AES-CTR cost is data-independent, and
    # seeding 4 GB at CPU speed would dominate setup time)
    fill: str = "seeded"
    reference_compat: bool = True
    window_aware: bool | None = None  # EngineConfig.window_aware (None: on iff reference_compat is off)
    # the engine is libsppipe (engine.Engine); the whole trace is dispatched
    # in one sp_pipe_replay call unless `native_dispatch` is "python" (one
    # Engine call per event, the reference driver's shape)
    engine: str = "native"
    native_dispatch: str = "replay"
    reserve_bytes: int = 0
    record_history: int = 0  # EngineConfig.record_history (0: keep every validator record)
    # replay the trace's ComputeEvents as model work on the GPU (the
    # reference simulator charges them to the GPU timeline,
    # simulator.py:431-434); off: swaps only
    compute: bool = False
    crypto_sms: int = 0  # EngineConfig.crypto_sms: SM budget of the crypto launches (0: all)


@dataclass
class ReplayResult:
    engine: Engine | None
    wall_s: float
    swap_bytes: int
    payload_bytes: int
    error: str | None = None
    # native engine on the GPU: time until every observable result was final
    # (finish without draining encrypt-ahead of records discarded at finish);
    # wall_s additionally waits for that discarded work (the conservative number)
    observable_s: float | None = None

    @property
    def swap_gbs(self) -> float:
        return self.swap_bytes / self.wall_s / 1e9 if self.wall_s > 0 else 0.0

    @property
    def observable_gbs(self) -> float:
        t = self.observable_s if self.observable_s else self.wall_s
        return self.swap_bytes / t / 1e9 if t > 0 else 0.0


def prepare_memory(trace: Trace, config: ReplayConfig) -> HostMemory:
    """Host blocks of `trace` (ids = header order), allocated and filled once;
    reusable by several replays (see HostMemory.reset_runtime_state)."""
    memory = HostMemory()
    for spec in trace.header.blocks:
        if spec.resident == "cpu":
            memory.alloc(spec.kind, spec.nbytes, _fill_for(spec, config))
        else:
            memory.alloc(spec.kind, spec.nbytes)
    return memory


def build_engine(trace: Trace, config: ReplayConfig, memory: HostMemory | None = None):
    """Engine + block table exactly as simulator.py:253-284 builds them
    (optionally over pre-built host blocks from `prepare_memory`)."""
    header = trace.header
    reuse = memory is not None
    if reuse:
        memory.reset_runtime_state()
    else:
        memory = HostMemory()
    cpu, gpu = new_channel(seed=config.seed)
    pconf = PredictorConfig() if config.predictor_chunk_bytes is None else \
        PredictorConfig(chunk_bytes=config.predictor_chunk_bytes)
    if config.engine != "native":
        raise ValueError("the only engine is libsppipe (engine='native')")
    spec_on = config.system == "specpipe"
    econf = EngineConfig(
        window=config.window, leeway=config.leeway, depth=config.depth, workers=config.workers,
        chunk_bytes=config.chunk_bytes, speculate=spec_on, defer_swap_decrypt=spec_on,
        record_stream=config.record_stream, plane=config.plane, reference_compat=config.reference_compat,
        window_aware=config.window_aware, record_history=config.record_history, crypto_sms=config.crypto_sms)
    predictor = Predictor(header.profile, pconf)
    engine = Engine(memory, cpu, gpu, predictor, econf, reserve_bytes=config.reserve_bytes)
    blocks = {}
    for spec in header.blocks:
        if spec.resident == "cpu":
            block = memory.block(spec.id) if reuse else memory.alloc(spec.kind, spec.nbytes, _fill_for(spec, config))
            if isinstance(spec.kind, (ModelLayer, KvCache)):
                predictor.observe_swap_out(block.id)
        else:
            block = memory.block(spec.id) if reuse else memory.alloc(spec.kind, spec.nbytes)
            if config.plane == "gpu":
                dev = _device_bytes(spec.nbytes)
                if config.fill == "fast":
                    _fast_random(dev, spec.content_seed)
                else:
                    import torch

                    dev.copy_(torch.from_numpy(random_bytes(spec.content_seed, spec.nbytes)))
                engine.seed_device(block.id, dev)
            else:
                engine.seed_device(block.id, _DryPayload(spec.nbytes))
        blocks[spec.id] = (block, classify(spec.nbytes, header.profile, pconf))
    return engine, blocks


class _DryPayload:
    """Device content of the dry plane: a size, no bytes."""

    def __init__(self, n: int) -> None:
        self.n = n

    def numel(self) -> int:
        return self.n


def _device_bytes(n: int):
    import torch

    return torch.empty(n, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))


def _drain(engine, config: ReplayConfig) -> None:
    """Issue and finish all device work queued so far (clock boundaries)."""
    if config.plane != "gpu":
        return
    engine.flush(wait=True)


_EV_CODES = {"h2d": 2, "d2h": 3}


def encode_events(trace: Trace, blocks: dict, config: ReplayConfig, start: int = 0, stop: int | None = None):
    """Trace events -> sp_event tuples + payload bytes (small I/O and app
    writes, generated exactly as the per-event driver does)."""
    from .engine import _CLASS

    events, payload = [], bytearray()
    io_index = sum(1 for e in trace.events[:start] if isinstance(e, SmallIoEvent))
    for ev in trace.events[start:stop]:
        if isinstance(ev, SwapInRequest):
            block, cls = blocks[ev.block]
            events.append((0, _CLASS[cls], block.id, block.base, block.len, 0))
        elif isinstance(ev, SwapOut):
            block, cls = blocks[ev.block]
            events.append((1, _CLASS[cls], block.id, block.base, block.len, 0))
        elif isinstance(ev, SmallIoEvent):
            events.append((_EV_CODES[ev.direction], 2, 0, 0, ev.size, len(payload)))
            payload += small_io_payload(config.seed, io_index, ev.size)
            io_index += 1
        elif isinstance(ev, SyncEvent):
            events.append((4, 0, 0, 0, 0, 0))
        elif isinstance(ev, AppWriteEvent):
            block, _ = blocks[ev.block]
            events.append((5, 0, block.id, ev.offset, ev.size, len(payload)))
            payload += app_write_payload(ev.data_seed, ev.size)
        elif isinstance(ev, ComputeEvent) and config.compute:
            events.append((6, 0, 0, 0, ev.duration, 0))
    return events, bytes(payload)


def _fast_random(dev_tensor, seed: int) -> None:
    import torch

    g = torch.Generator(device=dev_tensor.device)
    g.manual_seed(seed)
    dev_tensor.copy_(torch.randint(0, 256, dev_tensor.shape, dtype=torch.uint8, device=dev_tensor.device,
                                   generator=g))


class _FastFill:
    """Host block filler: random bytes made on the GPU, copied to pinned memory."""

    def __init__(self, seed: int) -> None:
        self.seed = seed

    def fill_into(self, out) -> None:
        import torch

        dev = torch.empty(out.shape[0], dtype=torch.uint8, device="cuda")
        _fast_random(dev, self.seed)
        torch.from_numpy(out).copy_(dev)


def _fill_for(spec, config: ReplayConfig):
    if config.plane == "dry":
        return None  # the dry plane never reads payload bytes
    if config.fill == "fast":
        return _FastFill(spec.content_seed)
    return prng_fill(spec.content_seed)


def _swap_bytes_from(trace: Trace, start: int) -> int:
    size = {b.id: b.nbytes for b in trace.header.blocks}
    return sum(size[e.block] for e in trace.events[start:] if isinstance(e, (SwapOut, SwapInRequest)))


def run_engine(trace: Trace, config: ReplayConfig = ReplayConfig(), catch: bool = False,
               measure_from: int = 0, memory: HostMemory | None = None) -> ReplayResult:
    """Replay `trace`; with `catch`, an engine exception (e.g. the reference's
    defect C2 EngineError) is returned in `error` with the engine state at
    the point of failure, as the parity harness needs.  With `measure_from`,
    the clock starts (after draining the GPU) at that event index and
    `swap_bytes` counts only the swaps from there on (warm-up excluded)."""
    engine, blocks = build_engine(trace, config, memory)
    _drain(engine, config)
    mark = {"t0": time.perf_counter()}

    def at_mark() -> None:
        _drain(engine, config)
        mark["t0"] = time.perf_counter()

    segments = None
    observable = None
    if config.native_dispatch == "replay":
        # trace -> sp_event arrays before the clock starts (trace loading, not engine work)
        cut = measure_from if measure_from else 0
        segments = [engine.encode(*encode_events(trace, blocks, config, 0, cut))] if cut else []
        segments.append(engine.encode(*encode_events(trace, blocks, config, cut)))
        mark["t0"] = time.perf_counter()
    try:
        if segments is not None:
            for i, seg in enumerate(segments):
                if i:
                    at_mark()
                engine.replay_encoded(seg)
            if config.plane == "gpu":
                engine.finish(drain_discarded=False)
                observable = time.perf_counter() - mark["t0"]
                engine.flush(wait=True)  # ... then the discarded encrypt-ahead drains too
            else:
                engine.finish()
        else:
            _dispatch_all(engine, blocks, trace, config, measure_from, at_mark)
    except Exception as exc:
        if not catch:
            raise
        return ReplayResult(engine, time.perf_counter() - mark["t0"], trace.swap_bytes(), trace.payload_bytes(),
                            f"{type(exc).__name__}: {exc}")
    wall = time.perf_counter() - mark["t0"]
    return ReplayResult(engine, wall, _swap_bytes_from(trace, measure_from), trace.payload_bytes(),
                        observable_s=observable if segments is not None and config.plane == "gpu" else None)


def _dispatch_all(engine: Engine, blocks: dict, trace: Trace, config: ReplayConfig, measure_from: int = 0,
                  at_mark=None) -> None:
    io_index = 0
    for k, ev in enumerate(trace.events):
        if k == measure_from and k and at_mark is not None:
            at_mark()
        if isinstance(ev, SwapInRequest):
            block, cls = blocks[ev.block]
            engine.copy_h2d(CopyRequest("h2d", block.base, block.len, cls, block_id=block.id, submit_time=ev.t))
        elif isinstance(ev, SwapOut):
            block, cls = blocks[ev.block]
            engine.copy_d2h(CopyRequest("d2h", block.base, block.len, cls, block_id=block.id, submit_time=ev.t))
        elif isinstance(ev, SmallIoEvent):
            engine.small_io(ev.direction, ev.size, small_io_payload(config.seed, io_index, ev.size))
            io_index += 1
        elif isinstance(ev, SyncEvent):
            engine.sync()
        elif isinstance(ev, AppWriteEvent):
            block, _ = blocks[ev.block]
            engine.app_write(block.id, ev.offset, app_write_payload(ev.data_seed, ev.size))
        elif isinstance(ev, ComputeEvent):
            if config.compute:
                engine.compute(ev.duration)
    engine.finish()


def run_plain_native(trace: Trace, config: ReplayConfig = ReplayConfig(), memory: HostMemory | None = None,
                     measure_from: int = 0) -> ReplayResult:
    """NoCc through libsppipe (sp_pipe_plain_replay): the same swaps as plain
    pinned cudaMemcpyAsync from C++, on the pipe's copy streams — the
    unencrypted baseline with the same (native) dispatch cost as the
    encrypted native engine."""
    from dataclasses import replace

    cfg = replace(config, engine="native", plane="gpu")
    engine, blocks = build_engine(trace, cfg, memory)
    pre = engine.encode(*encode_events(trace, blocks, cfg, 0, measure_from)) if measure_from else None
    seg = engine.encode(*encode_events(trace, blocks, cfg, measure_from))
    _drain(engine, cfg)
    if pre is not None:
        engine.plain_replay_encoded(pre)
    t0 = time.perf_counter()
    engine.plain_replay_encoded(seg)
    wall = time.perf_counter() - t0
    # the engine only carries the plain run's device state (compute_stats);
    # its control plane saw no events
    return ReplayResult(engine, wall, _swap_bytes_from(trace, measure_from), trace.payload_bytes())


def main(argv: list[str] | None = None) -> int:
    """Replay reference-format JSONL traces (workload.py:188-260 schema v1)
    on the B200: one JSON line per (trace, system) with measured swap GB/s,
    the plain-copy baseline and the engine's report counters — the
    measured counterpart of the reference's `specpipe sim` (cli.py:119-183)."""
    import argparse
    import json

    from .workload import load_trace

    ap = argparse.ArgumentParser(prog="python -m paper_2411_03357_b200.replay")
    ap.add_argument("trace", nargs="+", help="JSONL trace file(s) in the reference schema")
    ap.add_argument("--system", action="append", choices=["specpipe", "synccc", "nocc"],
                    help="systems to run (default: all three)")
    ap.add_argument("--plane", choices=["gpu", "dry"], default="gpu")
    ap.add_argument("--dispatch", choices=["replay", "python"], default="replay",
                    help="one sp_pipe_replay call per trace, or one Engine call per event")
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--leeway", type=int, default=8)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3, help="timed runs per system (best reported)")
    ap.add_argument("--fix-c2", action="store_true", help="reference_compat=False (SURVEY App. C defect C2 fixed)")
    args = ap.parse_args(argv)
    systems = args.system or ["specpipe", "synccc", "nocc"]
    for path in args.trace:
        trace = load_trace(path)
        for system in systems:
            cfg = ReplayConfig(system="specpipe" if system == "nocc" else system,
                               plane=args.plane, window=args.window, leeway=args.leeway, depth=args.depth,
                               seed=args.seed, record_stream=False, fill="fast" if args.plane == "gpu" else "seeded",
                               reference_compat=not args.fix_c2, native_dispatch=args.dispatch)
            memory = prepare_memory(trace, cfg)
            row = {"trace": str(path), "system": system, "engine": "native", "plane": args.plane,
                   "swap_bytes": trace.swap_bytes(), "events": len(trace.events)}
            if system == "nocc":
                if args.plane != "gpu":
                    row["error"] = "nocc replays need --plane gpu"
                else:
                    runs = [run_plain_native(trace, cfg, memory=memory) for _ in range(args.reps + 1)][1:]
                    row["swap_gbs"] = round(max(r.swap_gbs for r in runs), 3)
                print(json.dumps(row), flush=True)
                continue
            res = None
            best = 0.0
            for _ in range(args.reps + (1 if args.plane == "gpu" else 0)):
                res = run_engine(trace, cfg, catch=True, memory=memory)
                if res.error:
                    break
                best = max(best, res.swap_gbs)
            rep = res.engine.report()
            row.update({"error": res.error, "swap_gbs": round(best, 3) if args.plane == "gpu" else None,
                        "hit": rep["hit"], "iv_ahead": rep["iv_ahead"], "miss": rep["miss"], "nops": rep["nops"],
                        "relinquishes": rep["relinquishes"] + rep["replans"],
                        "sequence_hit_rate": rep["sequence_hit_rate"], "data_msgs": rep["data_msgs"]})
            print(json.dumps(row), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""The speculative pipeline on libsppipe.so: the reference's `Engine` and
`Predictor` API (/root/reference/pkg/src/specpipe/engine.py:171-624,
predictor.py:316-375) over the native control plane and B200 data plane of
include/sppipe.h.

`NativePredictor` and `NativeEngine` take and return the same Python objects
as `predictor.Predictor` and `engine.Engine` (CopyRequest/CopyHandle, Action,
Prediction, PatternHypothesis, report() dict, decision_log, sent logs), so
the parity harness and the replay driver run unchanged on either.  Every
decision, counter and error comes from C++; Python only marshals.  There is
no Python fallback: without libsppipe.so construction raises
NativeUnavailable.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import random
import weakref
from dataclasses import dataclass
from typing import Iterable

from . import _native
from ._native import (SpAction, SpDecision, SpDelivery, SpEvent, SpPipeConfig, SpPrediction, SpPredConfig,
                      SpRecord, SpSent)
from .channel import Direction
from .engine import Action, ActionKind, CopyRequest, EngineConfig, EngineError, HandleState
from .gcm import GcmAuthError
from .memory import BoundsError, GuardOverlapError, HostMemory, KvCache, ModelLayer
from .predictor import (DEFAULT_CONFIG, AmbiguousProfile, ModelProfile, PatternHypothesis, PatternKind, Prediction,
                        PredictorConfig, TransferClass, UnknownBlock)
from .validator import OverlapError, RecordState, StateError, VerdictKind

_CLASS = {TransferClass.MODEL_WEIGHTS: 0, TransferClass.KV_CACHE: 1, TransferClass.SMALL_IO: 2}
_CLASS_BACK = {v: k for k, v in _CLASS.items()}
_PATTERN = [PatternKind.REPETITIVE, PatternKind.LIFO, PatternKind.FIFO, PatternKind.UNKNOWN]
_VERDICT = [VerdictKind.HIT, VerdictKind.IV_AHEAD, VerdictKind.IV_BEHIND, VerdictKind.STALE, VerdictKind.MISS, None]
_ACTION = [ActionKind.SPEC_ENCRYPT, ActionKind.H2D_DATA, ActionKind.NOP, ActionKind.D2H_DATA,
           ActionKind.RESOLVE_DECRYPT, ActionKind.RELINQUISH, ActionKind.SYNC_POINT]
_ERRORS = {
    _native.SP_EINVAL: ValueError, _native.SP_EAUTH: GcmAuthError, _native.SP_EENGINE: EngineError,
    _native.SP_EOVERLAP: OverlapError, _native.SP_ESTATE: StateError, _native.SP_EUNKNOWN_BLOCK: UnknownBlock,
    _native.SP_EBOUNDS: BoundsError, _native.SP_EGUARD: GuardOverlapError, _native.SP_EAMBIGUOUS: AmbiguousProfile,
    _native.SP_EKEY: KeyError,
}


def _check(rc: int) -> None:
    if rc == _native.SP_OK:
        return
    raise _ERRORS.get(rc, RuntimeError)(_native.pipe_error())


def _block_kind(kind) -> int:
    if isinstance(kind, ModelLayer):
        return 0
    if isinstance(kind, KvCache):
        return 1
    return 2


class NativePredictor:
    """predictor.Predictor on sp_pred_* (decision for decision)."""

    def __init__(self, profile: ModelProfile | None = None, config: PredictorConfig = DEFAULT_CONFIG) -> None:
        self._lib = _native.load_sppipe()
        self.profile = profile
        self.config = config
        c = SpPredConfig(config.small_io_threshold, config.swap_min, config.chunk_bytes, config.warmup_matches,
                         config.history_cap, profile.layer_param_bytes if profile else 0,
                         profile.kv_block_bytes if profile else 0)
        h = ctypes.c_void_p()
        _check(self._lib.sp_pred_create(ctypes.byref(c), ctypes.byref(h)))
        self._h = h

    def __del__(self) -> None:  # pragma: no cover - interpreter teardown
        try:
            if self._h:
                self._lib.sp_pred_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def classify(self, size: int) -> TransferClass:
        if self.profile is None:
            raise ValueError("no model profile configured")
        out = ctypes.c_int32()
        _check(self._lib.sp_pred_classify(self._h, size, ctypes.byref(out)))
        return _CLASS_BACK[out.value]

    def observe_swap_out(self, block: int) -> None:
        _check(self._lib.sp_pred_observe_out(self._h, block))

    def observe_swap_in(self, blocks: Iterable[int]) -> None:
        b = list(blocks)
        arr = (ctypes.c_int64 * max(1, len(b)))(*b)
        _check(self._lib.sp_pred_observe_in(self._h, arr, len(b)))

    def observe_sync(self) -> None:
        _check(self._lib.sp_pred_observe_sync(self._h))

    @property
    def outstanding(self) -> frozenset:
        n = ctypes.c_int64()
        _check(self._lib.sp_pred_outstanding(self._h, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_int64 * max(1, n.value))()
        _check(self._lib.sp_pred_outstanding(self._h, arr, n.value, ctypes.byref(n)))
        return frozenset(arr[:n.value])

    def recognize(self) -> PatternHypothesis:
        kind, conf, phase, clen = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.sp_pred_recognize(self._h, ctypes.byref(kind), ctypes.byref(conf), ctypes.byref(phase),
                                           ctypes.byref(clen)))
        k = _PATTERN[kind.value]
        if k is PatternKind.UNKNOWN:
            return PatternHypothesis(k)
        cycle = []
        for i in range(clen.value):
            n = ctypes.c_int32()
            _check(self._lib.sp_pred_cycle_entry(self._h, i, None, 0, ctypes.byref(n)))
            arr = (ctypes.c_int64 * max(1, n.value))()
            _check(self._lib.sp_pred_cycle_entry(self._h, i, arr, n.value, ctypes.byref(n)))
            cycle.append(tuple(arr[:n.value]))
        return PatternHypothesis(k, conf.value, tuple(cycle), phase.value)

    def predict_batches(self, current_iv: int, leeway: int, depth: int = 1) -> list[list[Prediction]]:
        n = ctypes.c_int32()
        cap = 256
        while True:
            arr = (SpPrediction * cap)()
            _check(self._lib.sp_pred_predict_batches(self._h, current_iv, leeway, depth, arr, cap, ctypes.byref(n)))
            if n.value <= cap:
                break
            cap = n.value
        out: list[list[Prediction]] = []
        for p in arr[:n.value]:
            while len(out) <= p.batch:
                out.append([])
            out[p.batch].append(Prediction(block=p.block, predicted_iv=p.predicted_iv, leeway=p.leeway))
        return out

    def predict_next(self, current_iv: int, leeway: int, depth: int = 1) -> list[Prediction]:
        return [p for b in self.predict_batches(current_iv, leeway, depth) for p in b]

    @property
    def decision_log(self) -> list[dict]:
        out = []
        d = SpDecision()
        for i in range(self._lib.sp_pred_decision_count(self._h)):
            _check(self._lib.sp_pred_decision(self._h, i, ctypes.byref(d)))
            out.append({"event": "lock" if d.event == 0 else "drop", "pattern": _PATTERN[d.pattern].value,
                        "confidence": d.confidence, "after_batches": d.after_batches})
        return out


class _Handle:
    """engine.CopyHandle whose state lives in the pipe."""

    def __init__(self, engine: "NativeEngine", seq: int, verdict: VerdictKind | None) -> None:
        self._engine = engine
        self.seq = seq
        self.verdict = verdict

    @property
    def done(self) -> bool:
        d = ctypes.c_int32()
        self._engine._lib.sp_pipe_handle_done(self._engine._h, self.seq, ctypes.byref(d))
        return bool(d.value)

    @property
    def state(self) -> HandleState:
        return HandleState.DONE if self.done else HandleState.PENDING


@dataclass(frozen=True)
class RecordView:
    """A validator record as the pipe holds it (validator.CiphertextRecord
    without the device payloads)."""

    id: int
    base: int
    len: int
    iv: int
    iv_span: int
    state: RecordState
    block_id: int | None

    @property
    def last_iv(self) -> int:
        return self.iv + self.iv_span - 1


class _ValidatorView:
    """Read-only view of the native validator (validator.Validator's
    queries: records, pending_records, pending_count)."""

    _STATES = (RecordState.PENDING, RecordState.COMMITTED, RecordState.INVALIDATED)

    def __init__(self, engine: "NativeEngine") -> None:
        self._engine = engine

    def _get(self, rid: int) -> RecordView:
        e = self._engine
        r = SpRecord()
        _check(e._lib.sp_pipe_record(e._h, rid, ctypes.byref(r)))
        return RecordView(r.id, r.base, r.len, r.iv, r.span, self._STATES[r.state],
                          None if r.block_id == -(1 << 63) else r.block_id)

    @property
    def records(self) -> dict:
        n = self._engine._lib.sp_pipe_record_count(self._engine._h)
        return {i: self._get(i) for i in range(1, n + 1)}

    def pending_records(self) -> list:
        return [r for r in self.records.values() if r.state is RecordState.PENDING]

    def pending_count(self) -> int:
        return len(self.pending_records())


class _Channel:
    def __init__(self, engine: "NativeEngine") -> None:
        self._engine = engine

    def sent_log(self, direction: Direction) -> list:
        e = self._engine
        d = direction.value
        n = e._lib.sp_pipe_sent_count(e._h, d)
        arr = (SpSent * max(1, n))()
        got = ctypes.c_int64()
        _check(e._lib.sp_pipe_sent_log(e._h, d, 0, arr, n, ctypes.byref(got)))
        return [(s.iv, bool(s.nop), s.size) for s in arr[:got.value]]


class _Endpoint:
    """Counters of one channel endpoint (channel.ChannelEndpoint view)."""

    def __init__(self, engine: "NativeEngine", send_dir: Direction, key) -> None:
        self._engine = engine
        self._send = send_dir.value
        self._recv = 1 - send_dir.value
        self.key = key
        self.channel = _Channel(engine)

    @property
    def send_iv(self) -> int:
        return int(self._engine._lib.sp_pipe_send_iv(self._engine._h, self._send))

    @property
    def recv_iv(self) -> int:
        return int(self._engine._lib.sp_pipe_recv_iv(self._engine._h, self._recv))


class NativeEngine:
    """engine.Engine on sp_pipe_* (same methods, arguments and errors)."""

    def __init__(self, memory: HostMemory, cpu, gpu, predictor: NativePredictor, config: EngineConfig | None = None,
                 reserve_bytes: int = 0) -> None:
        if not isinstance(predictor, NativePredictor):
            raise TypeError("NativeEngine needs a NativePredictor")
        self._lib = _native.load_sppipe()
        self.memory = memory
        self.predictor = predictor
        self.config = config or EngineConfig()
        c = self.config
        cfg = SpPipeConfig()
        cfg.window, cfg.leeway, cfg.depth, cfg.workers = c.window, c.leeway, c.depth, c.workers
        cfg.chunk_bytes, cfg.nop_bytes, cfg.ring_slots = c.chunk_bytes, c.nop_bytes, c.ring_slots
        cfg.speculate, cfg.defer_swap_decrypt, cfg.record_stream = c.speculate, c.defer_swap_decrypt, c.record_stream
        cfg.strict_auth, cfg.reference_compat = c.strict_auth, c.reference_compat
        cfg.window_aware = 1 if c.window_aware_on else 0
        cfg.dry = c.plane == "dry"
        cfg.hw_guards = bool(getattr(memory, "hw_guards", False))
        cfg.initial_h2d_iv, cfg.initial_d2h_iv = cpu.send_iv, gpu.send_iv
        # queued compute bytes that trigger a flush (SPPIPE_BATCH_MB overrides, for sweeps)
        cfg.batch_bytes = int(float(os.environ.get("SPPIPE_BATCH_MB", "64")) * (1 << 20))
        cfg.reserve_bytes = reserve_bytes
        h = ctypes.c_void_p()
        _check(self._lib.sp_pipe_create(ctypes.byref(cfg), bytes(cpu.key.key_bytes), predictor._h, ctypes.byref(h)))
        self._h = h
        # views hold a weak reference: no cycle, so the pipe (and its device
        # memory) is released as soon as the last user drops the engine
        me = weakref.proxy(self)
        self.cpu = _Endpoint(me, Direction.HOST_TO_DEVICE, cpu.key)
        self.gpu = _Endpoint(me, Direction.DEVICE_TO_HOST, gpu.key)
        self.validator = _ValidatorView(me)
        self._registered = 0
        self._rng = random.Random(0xC0DE)
        self._actions: list[Action] = []
        self._delivered: list = []
        self._d2h: list = []
        self._sync_blocks()

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.sp_pipe_destroy(self._h)
            self._h = None

    def __del__(self) -> None:  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- host blocks ------------------------------------------------------------------
    def _sync_blocks(self) -> None:
        """Register host blocks allocated since the last call (ids are dense)."""
        n = len(self.memory._blocks)
        if n == self._registered:
            return
        for b in list(self.memory.blocks())[self._registered:]:
            _check(self._lib.sp_pipe_register_block(self._h, b.id, b.base, b.len, _block_kind(b.kind),
                                                    b.data.ctypes.data))
        self._registered = n

    def seed_device(self, block_id: int, data) -> None:
        self._sync_blocks()
        if hasattr(data, "data_ptr"):
            n = data.numel() * data.element_size()
            _check(self._lib.sp_pipe_seed_device(self._h, block_id, data.data_ptr(), n, 1 if data.is_cuda else 0))
        elif hasattr(data, "numel"):  # dry payload: sizes only
            _check(self._lib.sp_pipe_seed_device(self._h, block_id, None, data.numel(), 1))
        else:
            buf = bytes(data)
            _check(self._lib.sp_pipe_seed_device(self._h, block_id, buf, len(buf), 0))

    # -- the Engine API ----------------------------------------------------------------
    def copy_h2d(self, req: CopyRequest) -> _Handle:
        if req.direction != "h2d":
            raise ValueError("copy_h2d takes a host-to-device request")
        self._sync_blocks()
        seq, verdict = ctypes.c_uint64(), ctypes.c_int32()
        block = -(1 << 63) if req.block_id is None else req.block_id
        _check(self._lib.sp_pipe_submit_h2d(self._h, req.base, req.len, _CLASS[req.transfer_class], block,
                                            ctypes.byref(seq), ctypes.byref(verdict)))
        return _Handle(self, seq.value, _VERDICT[verdict.value])

    def copy_d2h(self, req: CopyRequest) -> _Handle:
        if req.direction != "d2h":
            raise ValueError("copy_d2h takes a device-to-host request")
        self._sync_blocks()
        seq = ctypes.c_uint64()
        _check(self._lib.sp_pipe_submit_d2h(self._h, req.base, req.len, _CLASS[req.transfer_class], req.block_id,
                                            ctypes.byref(seq)))
        return _Handle(self, seq.value, None)

    def small_io(self, direction: str, size: int, payload: bytes | None = None) -> None:
        if direction not in ("h2d", "d2h"):
            raise ValueError(f"unknown direction {direction!r}")
        if payload is None:
            payload = self._rng.randbytes(size)  # engine.py:401, one generator per engine
        _check(self._lib.sp_pipe_small_io(self._h, 0 if direction == "h2d" else 1, bytes(payload), size))

    def sync(self) -> None:
        _check(self._lib.sp_pipe_sync(self._h))

    def speculate_tick(self) -> None:
        _check(self._lib.sp_pipe_speculate(self._h))

    def relinquish(self) -> int:
        n = ctypes.c_int64()
        _check(self._lib.sp_pipe_relinquish(self._h, ctypes.byref(n)))
        return n.value

    def drain_decrypts(self) -> None:
        _check(self._lib.sp_pipe_drain_decrypts(self._h))

    def finish(self, drain_discarded: bool = True) -> None:
        """engine.finish (engine.py:583-607).  drain_discarded=False returns
        once every observable result is final, leaving encrypt-ahead work of
        records discarded here to drain in the background (see
        sp_pipe_finish_observable)."""
        if drain_discarded or not hasattr(self._lib, "sp_pipe_finish_observable"):  # (older A/B builds)
            _check(self._lib.sp_pipe_finish(self._h))
        else:
            _check(self._lib.sp_pipe_finish_observable(self._h))

    def test_corrupt_in_flight(self, direction: Direction, index: int, byte_index: int = 0, bit: int = 0) -> None:
        """hook_corrupt_in_flight (channel.py:263-273): flip one bit of an
        in-flight (sent, not yet received) message."""
        _check(self._lib.sp_pipe_test_corrupt(self._h, direction.value, index, byte_index, 1 << bit))

    def flush(self, wait: bool = False) -> None:
        """Issue queued launches now (and with `wait`, drain the device)."""
        _check(self._lib.sp_pipe_flush(self._h, 1 if wait else 0))

    def app_write(self, block_id: int, offset: int, data: bytes) -> None:
        self._sync_blocks()
        buf = bytes(data)
        _check(self._lib.sp_pipe_app_write(self._h, block_id, offset, buf, len(buf), None))

    def app_read(self, block_id: int, offset: int, length: int) -> bytes:
        self._sync_blocks()
        out = ctypes.create_string_buffer(max(1, length))
        _check(self._lib.sp_pipe_app_read(self._h, block_id, offset, length, out))
        return out.raw[:length]

    # -- whole traces in one native call ------------------------------------------------
    @staticmethod
    def encode(events, payloads: bytes = b"") -> tuple:
        """events: sequence of (kind, cls, block, base, len, payload_offset)
        tuples (SP_EV_* kinds) -> an sp_event array ready for replay_encoded."""
        import numpy as np

        dt = np.dtype({"names": ["kind", "cls", "block", "base", "len", "payload"],
                       "formats": [np.int32, np.int32, np.int64, np.uint64, np.uint64, np.uint64],
                       "offsets": [f[1].offset for f in [(n, getattr(SpEvent, n)) for n, _ in SpEvent._fields_]],
                       "itemsize": ctypes.sizeof(SpEvent)})
        arr = np.array(events, dtype=dt) if events else np.zeros(0, dtype=dt)
        return arr, bytes(payloads)

    def replay_encoded(self, encoded: tuple) -> int:
        """Dispatch a whole encoded trace segment in one sp_pipe_replay call;
        returns the number of events dispatched."""
        arr, payloads = encoded
        self._sync_blocks()
        done = ctypes.c_uint64()
        rc = self._lib.sp_pipe_replay(self._h, arr.ctypes.data_as(ctypes.POINTER(SpEvent)), len(arr),
                                      payloads or None, ctypes.byref(done))
        _check(rc)
        return done.value

    def plain_replay_encoded(self, encoded: tuple) -> None:
        """The same trace segment as plain copies (no crypto, no control
        plane): the unencrypted-swap baseline on the same streams."""
        arr, payloads = encoded
        self._sync_blocks()
        _check(self._lib.sp_pipe_plain_replay(self._h, arr.ctypes.data_as(ctypes.POINTER(SpEvent)), len(arr),
                                              payloads or None))

    def replay_events(self, events, payloads: bytes = b"") -> int:
        return self.replay_encoded(self.encode(events, payloads))

    # -- reporting -------------------------------------------------------------------------
    def report(self) -> dict:
        n = ctypes.c_int32()
        arr = (ctypes.c_int64 * 64)()
        _check(self._lib.sp_pipe_report(self._h, arr, 64, ctypes.byref(n)))
        names = [self._lib.sp_pipe_counter_name(i).decode() for i in range(n.value)]
        vals = dict(zip(names, arr[:n.value]))
        out = {k: vals[k] for k in names[:30]}
        if vals["otf_burned_present"]:
            out["otf_burned_records"] = vals["otf_burned_records"]
        seq_batches = out["seq_batches"]
        out["sequence_hit_rate"] = out["seq_hits"] / seq_batches if seq_batches else 0.0
        out["ring_violations"] = vals["ring_violations"]
        out["ring_high_water"] = vals["ring_high_water"]
        out["send_iv"] = vals["send_iv"]
        out["gpu_send_iv"] = vals["gpu_send_iv"]
        return out

    @property
    def counters(self) -> dict:
        return {k: v for k, v in self.report().items() if isinstance(v, int)}

    def sequence_hit_rate(self) -> float:
        return self.report()["sequence_hit_rate"]

    @property
    def actions(self) -> list[Action]:
        total = self._lib.sp_pipe_action_count(self._h)
        have = len(self._actions)
        if total > have:
            arr = (SpAction * (total - have))()
            got = ctypes.c_int64()
            _check(self._lib.sp_pipe_actions(self._h, have, arr, total - have, ctypes.byref(got)))
            for a in arr[:got.value]:
                self._actions.append(Action(
                    _ACTION[a.kind], iv=a.iv, nbytes=a.nbytes,
                    record_id=None if a.record_id < 0 else a.record_id,
                    task_id=None if a.task_id < 0 else a.task_id,
                    committed=bool(a.flags & 1), otf=bool(a.flags & 2), count=a.count,
                    seq=None if a.seq < 0 else a.seq))
        return self._actions

    def _recorded(self, which: int, cache: list, with_addr: bool) -> list:
        total = self._lib.sp_pipe_delivered_count(self._h, which)
        d = SpDelivery()
        for i in range(len(cache), total):
            buf = ctypes.create_string_buffer(1)
            _check(self._lib.sp_pipe_delivered(self._h, which, i, ctypes.byref(d), None))
            digest = None
            if self.config.plane != "dry":
                buf = ctypes.create_string_buffer(max(1, d.size))
                _check(self._lib.sp_pipe_delivered(self._h, which, i, ctypes.byref(d), buf))
                digest = hashlib.sha256(buf.raw[:d.size]).hexdigest()
            cache.append((d.seq, d.addr, d.size, digest) if with_addr else (d.seq, d.size, digest))
        return cache

    @property
    def delivered(self) -> list:
        return self._recorded(0, self._delivered, True)

    @property
    def d2h_stream(self) -> list:
        return self._recorded(1, self._d2h, False)

    def plane_stats(self) -> dict:
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self._lib.sp_pipe_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        r, u, k = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self._lib.sp_pipe_pool_stats(self._h, ctypes.byref(r), ctypes.byref(u), ctypes.byref(k))
        return {"bytes_h2d": a.value, "bytes_d2h": b.value, "launches": c.value, "pool_reserved": r.value,
                "pool_used": u.value, "cached": k.value}

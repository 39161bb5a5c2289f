"""B200 data plane of the speculative pipeline: where the engine's seals,
opens and PCIe copies actually run.

Mapping of the reference's in-process model onto one GPU:

* host blocks (`memory.HostMemory`) are page-locked host arrays;
  `engine.device_mem` holds real HBM buffers;
* every seal/open of BOTH channel endpoints runs in the libspgcm kernels on
  the compute stream, batched per engine step (chunk runs, NOP pads and
  drains are one launch each);
* swap-in data (spec encrypt-ahead and on-the-fly) crosses PCIe on the H2D
  copy stream into an HBM staging slot and is sealed in place at its counter;
  swap-out plaintext returns on the D2H copy stream once the host endpoint's
  (deferred) open lands.  Cross-stream order uses CUDA events only: the host
  thread never waits except where the reference's semantics expose bytes to
  the host (digests, `app_read`, `finish`).

`DryPlane` runs the same engine with no bytes at all (sizes and counters
only) — the schedule the reference's simulator prices, usable without a GPU.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field
from typing import Any

from . import gcm as _gcm
from .channel import DeviceCiphertext

TAG = 16
NVTX = os.environ.get("SPGCM_NVTX", "0") == "1"  # NVTX ranges per plane operation (nsys/ncu timelines)


def _nvtx(name):
    """Decorator: wrap a plane method in an NVTX range when SPGCM_NVTX=1."""
    def deco(fn):
        if not NVTX:
            return fn

        def wrapped(self, *a, **kw):
            import torch

            torch.cuda.nvtx.range_push(name)
            try:
                return fn(self, *a, **kw)
            finally:
                torch.cuda.nvtx.range_pop()

        wrapped.__name__ = fn.__name__
        wrapped.__doc__ = fn.__doc__
        return wrapped

    return deco


def open_message_sync(key: bytes, direction: int, iv: int, msg: DeviceCiphertext):
    """Blocking open of one device message (channel.decrypt_at on device data)."""
    import torch

    ctx = _gcm.context_for(key)
    out = torch.empty(msg.declared_len, dtype=torch.uint8, device=msg.payload.device)
    st = torch.zeros(1, dtype=torch.int32, device=msg.payload.device)
    ctx.open_batch([(direction, iv, msg.payload, out, msg.auth_tag, msg.declared_len)], st)
    if int(st.item()) != 0:
        raise _gcm.GcmAuthError(f"tag mismatch at counter {iv}")
    return out


_STREAMS: dict = {}


def device_streams(device, n: int) -> tuple:
    """The device's long-lived data-plane streams (created once per process).

    Engines come and go (one per replay), but staging buffers are cached by
    the CUDA caching allocator per stream: fresh streams per engine would
    turn every staging allocation of a new engine into a cudaMalloc
    (2-5 ms per 32 MiB chunk on the B200 box, measured), so all planes on a
    device share one stream set.  Sharing only adds ordering between planes."""
    import torch

    key = (torch.device(device).index, n)
    s = _STREAMS.get(key)
    if s is None:
        with torch.cuda.device(torch.device(device)):
            s = tuple(torch.cuda.Stream(torch.device(device)) for _ in range(n))
        _STREAMS[key] = s
    return s


class GpuPlane:
    """Streams, staging and batched launches for one engine on one GPU.

    Compute-stream work (on-the-fly and token/NOP seals, swap-out seals, every
    open) is queued in issue order and flushed as one launch per run of
    same-kind operations: at `flush()` (the engine calls it at the end of
    every sync), before any host access, or when BATCH_BYTES of payload is
    pending.  Small host payloads (tokens, NOP pads) are staged in a byte
    arena that crosses PCIe in one copy per flush.  Speculative seals run on
    their own stream as soon as their H2D copy lands (SpecBatch); host
    landings of swap-outs run on the landing / D2H streams after the flush
    that seals them."""

    kind = "gpu"
    ARENA_BYTES = 1 << 20

    def __init__(self, key: bytes, device: int | None = None) -> None:
        import torch

        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        with torch.cuda.device(self.device):
            self.ctx = _gcm.context_for(key)
            self.s_comp, self.s_spec, self.s_h2d, self.s_d2h, self.s_land = device_streams(self.device, 5)
        self._host_ready: dict[int, Any] = {}  # block id -> event after last D2H into it
        self._h2d_done: dict[int, Any] = {}    # block id -> event after last H2D from it
        self._ops: list = []                   # ("wait", ev) | ("seal", item) | ("open", item)
        self._ops_bytes = 0
        self._window = torch.cuda.Event()      # recorded after the flush of the current window
        self._arena_host = bytearray()
        self._arena_dev = None
        self._arena_off = 0
        self._landings: list = []              # (block, jobs, direction) for the next flush
        self._landing_blocks: set = set()
        self._status = torch.zeros(1 << 16, dtype=torch.int32, device=self.device)
        self._status_used = 0
        self.bytes_h2d = 0
        self.bytes_d2h = 0
        self.launches = 0

    # -- helpers -------------------------------------------------------------------
    def _empty(self, n: int):
        with self.torch.cuda.stream(self.s_comp):
            return self.torch.empty(n, dtype=self.torch.uint8, device=self.device)

    def _status_slots(self, n: int):
        if self._status_used + n > self._status.numel():
            self.check_auth()
        s = self._status[self._status_used:self._status_used + n]
        self._status_used += n
        return s

    def _queue(self, kind: str, item, nbytes: int = 0) -> None:
        self._ops.append((kind, item))
        self._ops_bytes += nbytes
        if self._ops_bytes >= BATCH_BYTES:
            self.flush()

    def _wait_for(self, ev) -> None:
        """Order the compute queue after `ev` unless it belongs to the
        current window (queue order already covers that)."""
        if ev is not None and ev is not self._window:
            self._ops.append(("wait", ev))

    def _arena_views(self, n: int):
        """Payload + tag views of n bytes in the current small-payload arena."""
        need = ((n + 15) & ~15) + TAG
        if self._arena_dev is None or self._arena_off + need > self._arena_dev.numel():
            if self._arena_off:
                self.flush()
            self._arena_dev = self._empty(max(self.ARENA_BYTES, need))
            self._arena_off = 0
            self._arena_host = bytearray()
        o = self._arena_off
        self._arena_off += need
        return self._arena_dev[o:o + n], self._arena_dev[o + need - TAG:o + need], o

    def check_auth(self) -> None:
        """Raise GcmAuthError if any open since the last check failed."""
        self.flush()
        if self._status_used:
            self.s_comp.synchronize()
            self.s_land.synchronize()
            self.s_d2h.synchronize()
            bad = int(self._status[:self._status_used].abs().sum().item())
            self._status[:self._status_used].zero_()
            self._status_used = 0
            if bad:
                raise _gcm.GcmAuthError("authentication failed on the device")

    # -- flush ---------------------------------------------------------------------
    @_nvtx("spgcm.flush")
    def flush(self) -> None:
        torch = self.torch
        if self._arena_host:
            staged = torch.empty(len(self._arena_host), dtype=torch.uint8, pin_memory=True)
            staged.numpy()[:] = memoryview(self._arena_host).cast("B")
            with torch.cuda.stream(self.s_comp):
                self._arena_dev[:len(self._arena_host)].copy_(staged, non_blocking=True)
            # later payloads of this arena must start past the staged bytes
            self._arena_host = bytearray()
            self._arena_dev = None
            self._arena_off = 0
        if self._ops:
            ops, self._ops, self._ops_bytes = self._ops, [], 0
            i = 0
            while i < len(ops):
                kind = ops[i][0]
                if kind == "wait":
                    self.s_comp.wait_event(ops[i][1])
                    i += 1
                    continue
                j = i
                while j < len(ops) and ops[j][0] == kind:
                    j += 1
                items = [op[1] for op in ops[i:j]]
                if kind == "seal":
                    self.ctx.seal_batch(items, self.s_comp)
                else:
                    self.ctx.open_batch(items, self._status_slots(len(items)), self.s_comp)
                self.launches += 1
                i = j
            self._window.record(self.s_comp)
            self._window = torch.cuda.Event()
        if self._landings:
            self._flush_landings()

    flush_d2h = flush  # historical name (SpecBatch, engine)

    def _flush_landings(self) -> None:
        torch = self.torch
        landings, self._landings = self._landings, []
        self._landing_blocks = set()
        waited = set()
        total = 0
        for _, jobs, _ in landings:
            for m, _, _ in jobs:
                total += m.declared_len
                if m.ready is not None and id(m.ready) not in waited:
                    self.s_land.wait_event(m.ready)
                    waited.add(id(m.ready))
        with torch.cuda.stream(self.s_land):
            buf = torch.empty(total, dtype=torch.uint8, device=self.device)
        items, places, off = [], [], 0
        for block, jobs, direction in landings:
            for msg, iv, boff in jobs:
                view = buf[off:off + msg.declared_len]
                items.append((direction, iv, msg.payload, view, msg.auth_tag, msg.declared_len))
                places.append((block, view, boff, msg.declared_len))
                off += msg.declared_len
                msg.payload.record_stream(self.s_land)
        self.ctx.open_batch(items, self._status_slots(len(items)), self.s_land)
        self.launches += 1
        opened = torch.cuda.Event()
        opened.record(self.s_land)
        self.s_d2h.wait_event(opened)
        with torch.cuda.stream(self.s_d2h):
            last = None
            for block, view, boff, n in places:
                if block is not last:
                    pend = self._h2d_done.get(block.id)
                    if pend is not None:
                        self.s_d2h.wait_event(pend)
                    last = block
                torch.from_numpy(block.data[boff:boff + n]).copy_(view, non_blocking=True)
            buf.record_stream(self.s_d2h)
            ev = torch.cuda.Event()
            ev.record(self.s_d2h)
        for block, _, _ in landings:
            self._host_ready[block.id] = ev
        self.bytes_d2h += total

    def _before_host_read_of(self, block_id: int) -> None:
        if block_id in self._landing_blocks:
            self.flush()

    # -- seals ---------------------------------------------------------------------
    @_nvtx("spgcm.seal_host_chunks")
    def seal_host_chunks(self, block, inner: int, spans: list, direction: int, iv0: int,
                         speculative: bool = False) -> list:
        """H2D the plaintext of `block` [inner + off, +n) for each span (copy
        stream, now) and seal chunk i at iv0 + i in place.  Speculative seals
        launch on their own stream (SpecBatch); on-the-fly seals join the
        compute queue behind the copy's event."""
        if speculative:
            batch = SpecBatch(self)
            msgs = batch.add(block, inner, spans, direction, iv0)
            batch.launch()
            return msgs
        torch = self.torch
        self._before_host_read_of(block.id)
        total = sum(n for _, n in spans)
        first = spans[0][0]
        ev = self._host_ready.get(block.id)
        if ev is not None:
            self.s_h2d.wait_event(ev)
        src = torch.from_numpy(block.data[inner + first: inner + first + total])
        with torch.cuda.stream(self.s_h2d):
            buf = torch.empty(total + TAG * len(spans), dtype=torch.uint8, device=self.device)
            buf[:total].copy_(src if block.pinned is not None else src.pin_memory(), non_blocking=True)
            buf.record_stream(self.s_comp)
            buf.record_stream(self.s_land)
            done = torch.cuda.Event()
            done.record(self.s_h2d)
        self._h2d_done[block.id] = done
        self.bytes_h2d += total
        self._ops.append(("wait", done))
        msgs = []
        for i, (off, n) in enumerate(spans):
            view = buf[off - first: off - first + n]
            tag = buf[total + TAG * i: total + TAG * (i + 1)]
            self._queue("seal", (direction, iv0 + i, view, view, tag, n), n)
            msgs.append(DeviceCiphertext(view, tag, n, ready=self._window))
        return msgs

    def spec_batch(self) -> "SpecBatch":
        return SpecBatch(self)

    @_nvtx("spgcm.seal_device_chunks")
    def seal_device_chunks(self, src, spans: list, direction: int, iv0: int) -> list:
        """Seal device plaintext `src` chunk-wise into fresh staging (queued:
        one sealing launch covers a whole KV eviction)."""
        total = sum(n for _, n in spans)
        first = spans[0][0]
        buf = self._empty(total + TAG * len(spans))
        buf.record_stream(self.s_land)
        msgs = []
        for i, (off, n) in enumerate(spans):
            view = buf[off - first: off - first + n]
            tag = buf[total + TAG * i: total + TAG * (i + 1)]
            msgs.append(DeviceCiphertext(view, tag, n, ready=self._window))
            self._queue("seal", (direction, iv0 + i, src[off:off + n], view, tag, n), n)
        return msgs

    @_nvtx("spgcm.seal_small")
    def seal_bytes_device(self, payloads: list, direction: int, iv0: int, nop: bool = False) -> list:
        """Seal small host payloads (NOP pads, token I/O): staged in the byte
        arena, sealed by the next flush's launch."""
        msgs = []
        for i, p in enumerate(payloads):
            n = len(p)
            view, tag, o = self._arena_views(n)
            host = self._arena_host
            if len(host) < o:
                host.extend(bytes(o - len(host)))
            host[o:o + n] = p
            msg = DeviceCiphertext(view, tag, n, nop=nop, ready=self._window)
            self._queue("seal", (direction, iv0 + i, view, view, tag, n), n)
            msgs.append(msg)
        return msgs

    # -- opens ---------------------------------------------------------------------
    @_nvtx("spgcm.open_into")
    def open_into(self, jobs: list, direction: int) -> None:
        """jobs: (msg, iv, dst view or None), queued in order; NOPs open into
        scratch so their tags are still verified."""
        for msg, iv, dst in jobs:
            self._wait_for(msg.ready)
            if dst is None:
                dst = self._empty(msg.declared_len)
            self._queue("open", (direction, iv, msg.payload, dst, msg.auth_tag, msg.declared_len), msg.declared_len)

    def land_on_host(self, block, jobs: list, direction: int) -> None:
        """Host endpoint open of D2H messages, then the plaintext lands in
        `block` (jobs: (msg, iv, offset_in_block)).  Issued by the next flush
        (after the seals it depends on), on the landing / D2H streams, so
        landings overlap swap-ins and never wait on the compute stream's
        later commits."""
        self._landings.append((block, jobs, direction))
        self._landing_blocks.add(block.id)
        self._ops_bytes += sum(m.declared_len for m, _, _ in jobs)
        if self._ops_bytes >= BATCH_BYTES:
            self.flush()

    def host_sync(self, block_id: int | None = None) -> None:
        """Wait until D2H landings are visible to the host."""
        self.flush()
        if block_id is None:
            self.s_d2h.synchronize()
            return
        ev = self._host_ready.get(block_id)
        if ev is not None:
            ev.synchronize()

    def before_host_write(self, block_id: int) -> None:
        """The host is about to mutate `block_id`: in-flight copies that
        read or write it must be finished first."""
        self.flush()
        for table in (self._h2d_done, self._host_ready):
            ev = table.get(block_id)
            if ev is not None:
                ev.synchronize()

    def new_device_buffer(self, n: int):
        return self._empty(n)

    def device_from_host(self, data: bytes):
        t = self.torch.frombuffer(bytearray(data), dtype=self.torch.uint8)
        with self.torch.cuda.stream(self.s_comp):
            return t.to(self.device, non_blocking=False)

    def to_host_bytes(self, view) -> bytes:
        self.flush()
        self.s_comp.synchronize()
        return view.cpu().numpy().tobytes()

    def digests(self, views: list) -> list:
        self.flush()
        self.s_comp.synchronize()
        self.s_land.synchronize()
        return [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in views]

    def finish(self) -> None:
        self.flush()
        self.s_comp.synchronize()
        self.s_spec.synchronize()
        self.s_land.synchronize()
        self.s_h2d.synchronize()
        self.s_d2h.synchronize()
        self.check_auth()


BATCH_BYTES = 64 * 1024 * 1024  # flush a batched launch once it covers this much payload


class SpecBatch:
    """Encrypt-ahead work of one engine entry point: one H2D copy per block
    as tasks are added; sealing launches on the speculation stream cover up
    to BATCH_BYTES each (small KV blocks share one launch, big weight chunks
    start sealing while later chunks are still crossing PCIe).  Messages of a
    sub-batch share its `ready` event, recorded before any consumer waits."""

    def __init__(self, plane: "GpuPlane") -> None:
        self.plane = plane
        self.items: list = []
        self.bytes = 0
        self.ready = plane.torch.cuda.Event()
        self.last_copy = None

    def add(self, block, inner: int, spans: list, direction: int, iv0: int) -> list:
        p, torch = self.plane, self.plane.torch
        p._before_host_read_of(block.id)  # a pending landing into this block must be issued first
        total = sum(n for _, n in spans)
        first = spans[0][0]
        ev = p._host_ready.get(block.id)
        if ev is not None:
            p.s_h2d.wait_event(ev)
        src = torch.from_numpy(block.data[inner + first: inner + first + total])
        with torch.cuda.stream(p.s_h2d):
            buf = torch.empty(total + TAG * len(spans), dtype=torch.uint8, device=p.device)
            buf[:total].copy_(src if block.pinned is not None else src.pin_memory(), non_blocking=True)
            buf.record_stream(p.s_comp)
            buf.record_stream(p.s_spec)
            done = torch.cuda.Event()
            done.record(p.s_h2d)
        p._h2d_done[block.id] = done
        p.bytes_h2d += total
        self.last_copy = done
        msgs = []
        for i, (off, n) in enumerate(spans):
            view = buf[off - first: off - first + n]
            tag = buf[total + TAG * i: total + TAG * (i + 1)]
            self.items.append((direction, iv0 + i, view, view, tag, n))
            msgs.append(DeviceCiphertext(view, tag, n, ready=self.ready))
        self.bytes += total
        if self.bytes >= BATCH_BYTES:
            self.launch()
        return msgs

    def launch(self) -> None:
        if not self.items:
            return
        p = self.plane
        p.s_spec.wait_event(self.last_copy)
        p.ctx.seal_batch(self.items, p.s_spec)
        p.launches += 1
        self.ready.record(p.s_spec)
        self.items, self.bytes = [], 0
        self.ready = p.torch.cuda.Event()


class _DrySpecBatch:
    def __init__(self, plane) -> None:
        self.plane = plane

    def add(self, block, inner, spans, direction, iv0):
        return self.plane.seal_host_chunks(block, inner, spans, direction, iv0, speculative=True)

    def launch(self) -> None:
        pass


@dataclass(eq=False)
class _DryPayload:
    n: int

    def numel(self) -> int:
        return self.n

    def __getitem__(self, sl: slice) -> "_DryPayload":
        return _DryPayload(len(range(*sl.indices(self.n))))


class DryPlane:
    """No bytes, no GPU: messages carry only their sizes.  Used for schedule
    planning and for control-plane tests in CPU-only environments."""

    kind = "dry"

    def __init__(self, key: bytes | None = None) -> None:
        self.bytes_h2d = 0
        self.bytes_d2h = 0
        self.launches = 0

    def _msgs(self, sizes, nop=False):
        return [DeviceCiphertext(_DryPayload(n), None, n, nop=nop) for n in sizes]

    def seal_host_chunks(self, block, inner, spans, direction, iv0, speculative=False):
        self.bytes_h2d += sum(n for _, n in spans)
        return self._msgs([n for _, n in spans])

    def spec_batch(self):
        return _DrySpecBatch(self)

    def flush(self):
        pass

    flush_d2h = flush

    def seal_device_chunks(self, src, spans, direction, iv0):
        return self._msgs([n for _, n in spans])

    def seal_bytes_device(self, payloads, direction, iv0, nop=False):
        return self._msgs([len(p) for p in payloads], nop=nop)

    def open_into(self, jobs, direction):
        pass

    def land_on_host(self, block, jobs, direction):
        self.bytes_d2h += sum(m.declared_len for m, _, _ in jobs)

    def host_sync(self, block_id=None):
        pass

    def before_host_write(self, block_id):
        pass

    def check_auth(self):
        pass

    def new_device_buffer(self, n):
        return _DryPayload(n)

    def device_from_host(self, data):
        return _DryPayload(len(data))

    def to_host_bytes(self, view):
        raise RuntimeError("the dry plane holds no bytes")

    def digests(self, views):
        return [None] * len(views)

    def finish(self):
        pass

"""A B200 cost model for the reference simulator.

The reference's CostModel (simulator.py:57-113) prices confidential
transfers as CPU work: on-the-fly AES-GCM blocks the submitting thread at
5.8 GB/s per worker, then the ciphertext crosses PCIe.  On the B200 data
plane neither is true: both endpoints' crypto runs in k_gcm on
the GPU, overlapped with the copies, and the host only issues.  Refitting
the constants cannot express that (profiles/r1_sim_calibrated.json: the
refit predicted SyncCc at 0.52 of NoCc where the B200 measures 0.99), so
this tool keeps the reference's own replay loop, engine, predictor and
action stream (simulator.py:202-475) and replaces only the costing of each
action (`_consume_actions`, simulator.py:316-372) with the B200 plane's
timelines:

  * host: every action costs `issue_us` of control-plane + driver time on
    the application thread (measured per event, tools/host_prof_replay.py);
  * PCIe: two lanes at the plain pinned-copy rate (the plaintext crosses;
    the channel's crypto is on the device);
  * GPU crypto: `crypto_gbs` per pass plus a share of the `launch_us`
    latency per batch of messages (k_gcm: bench.py's kernel line and the
    small-launch table), started when its inputs are ready (the summed
    crypto time is reported: far below the makespan, so no queueing is
    modelled); a swap moves two passes (seal + open);
  * SPEC_ENCRYPT = the staging H2D copy + the seal (the wire is paid ahead);
    its committed H2D_DATA costs only the receiver's open;
  * on-the-fly H2D_DATA = wire, then seal + open;  D2H_DATA = seal + open,
    then wire; deferred decrypts are ready when the D2H copy lands;
  * SYNC_POINT waits for the batch's wires and opens, as in the reference;
    RESOLVE_DECRYPT is not a host wait (the open ran on the GPU): it holds
    back the later H2D copies (one in-order stream) until that landing;
  * a swap-out's landing never blocks the host; token D2H does.

NoCc keeps the reference's own plain costing.  Parameters come from
measured B200 numbers (see PARAMS); predictions go next to the bench's
measured ratios.  Build-container tool: imports the reference from
/root/reference; nothing here is on the product path.

    python tools/sim_b200.py profiles/r2_sim_b200.json
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

NS = 1_000_000_000

# Measured on one B200 (profiles/, r2): k_gcm per pass on batched messages
# (bench.py value, seal and open each), small-launch device latency (bench.py
# small_messages, 4 x 224 KiB), sustained pinned copies of 32 MiB / 224 KiB
# (profiles/r2_copy_probe.txt: copy engine 52.6 GB/s, k_xfer 49-51 GB/s),
# control-plane + issue cost per trace event (tools/host_prof_replay.py).
PARAMS = {
    "crypto_gbs": 480.0,
    "launch_us": 9.0,
    "msgs_per_launch": 8,
    "pcie_gbs": 52.0,
    "issue_us": 1.4,
}


def b200_replay_class():
    from specpipe import simulator as sim
    from specpipe.engine import ActionKind

    class B200Replay(sim._Replay):
        """The reference replay with the B200 plane's action costs."""

        def __init__(self, trace, config, params):
            self.p = params
            self.gpu_crypto = 0       # last crypto completion
            self.gpu_crypto_busy = 0  # summed crypto time (a capacity check: << makespan)
            self.h2d_floor = 0  # host bytes a later H2D copy reads land first (stream order, not a host wait)
            self._small_io = False
            super().__init__(trace, config)

        def _dispatch_engine(self, ev) -> None:
            # token D2H is the only transfer whose bytes the application
            # waits for; a swap-out's landing never blocks the host here
            self._small_io = isinstance(ev, sim.SmallIoEvent)
            super()._dispatch_engine(ev)

        def _ns(self, us: float) -> int:
            return int(round(us * 1000))

        def _wire(self, nbytes: int) -> int:
            return int(round(nbytes * NS / (self.p["pcie_gbs"] * 1e9)))

        def _crypto(self, nbytes: int, passes: int, start: int) -> int:
            # one pass per endpoint; a message's share of its launch latency.
            # A launch runs when its inputs are ready: the GPU's crypto
            # capacity (~480 GB/s per pass against ~50 GB/s per PCIe lane)
            # is far from saturated, so a job is not queued behind later-
            # starting ones (a single FIFO timeline would let encrypt-ahead
            # waiting on its wire hold back independent swap-out seals).
            dur = int(round(passes * nbytes * NS / (self.p["crypto_gbs"] * 1e9)))
            dur += self._ns(self.p["launch_us"] / self.p["msgs_per_launch"])
            self.gpu_crypto_busy += dur
            done = start + dur
            self.gpu_crypto = max(self.gpu_crypto, done)
            return done

        def _consume_actions(self) -> None:
            assert self.engine is not None
            issue = self._ns(self.p["issue_us"])
            for action in self.engine.actions[self._consumed:]:
                kind = action.kind
                if kind is ActionKind.SPEC_ENCRYPT:
                    # staging H2D copy of the predicted bytes, then the seal
                    self.pcie_h2d = max(self.pcie_h2d, self.t_app, self.h2d_floor) + self._wire(action.nbytes)
                    self.ready[action.record_id] = self._crypto(action.nbytes, 1, self.pcie_h2d)
                elif kind is ActionKind.H2D_DATA:
                    self.t_app += issue
                    if action.committed:
                        # ciphertext already on the device: the receiver's open
                        done = self._crypto(action.nbytes, 1, max(self.t_app, self.ready.get(action.record_id, 0)))
                    else:
                        self.pcie_h2d = max(self.pcie_h2d, self.t_app, self.h2d_floor) + self._wire(action.nbytes)
                        done = self._crypto(action.nbytes, 2, self.pcie_h2d)
                    self.batch_wires.append(done)
                elif kind is ActionKind.NOP:
                    self.t_app += issue
                    self.batch_wires.append(self._crypto(action.nbytes, 2, self.t_app))
                elif kind is ActionKind.D2H_DATA:
                    self.t_app += issue
                    sealed = self._crypto(action.nbytes, 2, self.t_app)
                    self.pcie_d2h = max(self.pcie_d2h, sealed) + self._wire(action.nbytes)
                    self.batch_wires.append(self.pcie_d2h)
                    if action.task_id is not None:
                        self.dec_ready[action.task_id] = self.pcie_d2h
                        self.dec_tail = max(self.dec_tail, self.pcie_d2h)
                    elif self._small_io:
                        self.t_app = max(self.t_app, self.pcie_d2h)
                    else:
                        self.dec_tail = max(self.dec_tail, self.pcie_d2h)
                elif kind is ActionKind.RESOLVE_DECRYPT:
                    # the host endpoint's open already ran on the GPU; the
                    # swap-in that re-reads the block waits for the landing on
                    # the (in-order) H2D stream, the host thread does not
                    if action.task_id in self.dec_ready:
                        self.h2d_floor = max(self.h2d_floor, self.dec_ready.pop(action.task_id))
                elif kind is ActionKind.SYNC_POINT:
                    self.t_app = max(self.t_app, self.gpu_free, *self.batch_wires) \
                        if self.batch_wires else max(self.t_app, self.gpu_free)
                    self.batch_wires.clear()
                self._log(action)
            self._consumed = len(self.engine.actions)

    return B200Replay


def stub_crypto() -> None:
    """Timing-only runs: the reference engine's AES-GCM seam (encrypt_at /
    decrypt_at, channel.py:85-115; engine.py:34) replaced by a tagged
    identity, so a 2 GB layer replays in seconds.  Decisions, counters and
    actions do not depend on the ciphertext bytes."""
    from specpipe import channel, engine

    def enc(key, iv, plaintext, direction=channel.Direction.HOST_TO_DEVICE):
        if len(plaintext) < 1:
            raise ValueError("plaintext must be at least 1 byte")
        tag = (direction.value.to_bytes(4, "big") + iv.to_bytes(8, "big") + b"stub")[:16]
        return channel.CiphertextMsg(payload=bytes(plaintext), auth_tag=tag, declared_len=len(plaintext))

    def dec(key, iv, msg, direction=channel.Direction.HOST_TO_DEVICE):
        tag = (direction.value.to_bytes(4, "big") + iv.to_bytes(8, "big") + b"stub")[:16]
        if msg.auth_tag != tag:
            raise channel.AuthError(f"authentication failed at counter {iv}")
        return msg.payload

    channel.encrypt_at = enc
    channel.decrypt_at = dec
    engine.encrypt_at = enc


def predict(trace_obj, params: dict, systems=("nocc", "synccc", "specpipe")) -> dict:
    from specpipe import simulator as sim

    cost = sim.CostModel(pcie_bw_plain=params["pcie_gbs"] * 1e9, pcie_bw_cc=params["pcie_gbs"] * 1e9,
                         fixed_overhead_plain=params["issue_us"] * 1e-6,
                         fixed_overhead_cc=params["issue_us"] * 1e-6)
    B200Replay = b200_replay_class()
    out = {}
    for system in systems:
        t = time.time()
        cfg = sim.SimConfig(system=sim.SystemKind(system), workers=1, cost=cost)
        rp = sim._Replay(trace_obj, cfg) if system == "nocc" else B200Replay(trace_obj, cfg, params)
        res = rp.run()
        m = res.metrics
        out[system] = {"throughput_gbs": round(m.throughput_bytes_per_s / 1e9, 3),
                       "makespan_ms": round(m.makespan_ns / 1e6, 3), "hit_rate": m.hit_rate,
                       "nops": m.nop_count, "sim_wall_s": round(time.time() - t, 1),
                       "timelines_ms": {k: round(getattr(rp, k, 0) / 1e6, 3) for k in
                                        ("t_app", "gpu_free", "pcie_h2d", "pcie_d2h", "dec_tail", "gpu_crypto", "gpu_crypto_busy")}}
        print(system, out[system], flush=True)
    for system in systems:
        if system != "nocc":
            out[f"{system}_vs_nocc"] = round(out[system]["throughput_gbs"] / out["nocc"]["throughput_gbs"], 4)
    return out


def main(out_path: str) -> None:
    from specpipe import workload as ref_workload

    from paper_2411_03357_b200 import workload

    def ref_trace(tr):
        # the replay here (like sp_pipe_replay) runs events back to back:
        # arrival times are dropped so the reference measures the same thing
        import dataclasses

        rt = ref_workload.parse_trace_lines(list(workload.trace_to_lines(tr)))
        evs = [dataclasses.replace(e, t=0) if hasattr(e, "t") else e for e in rt.events]
        return dataclasses.replace(rt, events=evs)

    stub_crypto()
    report = {"params": PARAMS, "model": __doc__.split("\n\n")[1]}
    # the bench's OPT-66B shape (61 x 32 MiB chunks per layer, the model's
    # compute per layer), 2 iterations so the pure-Python simulator (real
    # AES in the reference engine) finishes in minutes
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2)
    report["opt66b_2iter"] = predict(ref_trace(tr), PARAMS)
    kv = workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0)
    report["kv_opt30b"] = predict(ref_trace(kv), PARAMS)
    json.dump(report, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in report.items() if k != "model"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sim_b200.json")

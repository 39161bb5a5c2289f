"""Host-side profile of one native replay (config-5 OPT-66B trace at a given
block size): run under tools/native/sampler.c (LD_PRELOAD) so only the
replay window is sampled.

    SAMPLER_OUT=gpurun_out/samples LD_PRELOAD=lib/libsampler.so \\
        python tools/host_prof_replay.py 65536 specpipe|synccc|plain [gpu|dry] [reps]
"""
from __future__ import annotations

import ctypes
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # as bench.py: no idle BLAS pool spinning
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import (ReplayConfig, build_engine, encode_events,  # noqa: E402
                                          prepare_memory)


def sampler():
    for name in os.environ.get("LD_PRELOAD", "").split(":"):
        if "sampler" in name:
            lib = ctypes.CDLL(name)
            lib.sampler_start()
            if os.environ.get("SAMPLER_WALL_US"):  # wall-clock samples of this (the control) thread only
                lib.sampler_start_thread(int(os.environ["SAMPLER_WALL_US"]))
            lib.sampler_enable(0)
            return lib
    return None


def main() -> None:
    kv = sys.argv[1] == "kv"  # the bench's OPT-30B KV-swap trace (config 3) instead of config 5
    blk, system = (229_376 if kv else int(sys.argv[1])), sys.argv[2]
    plane = sys.argv[3] if len(sys.argv) > 3 else "gpu"
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    S = sampler()
    if kv:
        tr = workload.gen_adversarial_trace(
            workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
        cfg = ReplayConfig(system="specpipe" if system == "plain" else system, plane=plane, record_stream=False,
                           fill="fast", engine="native", reference_compat=False)
    else:
        tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=blk)
        cfg = ReplayConfig(system="specpipe" if system == "plain" else system, plane=plane, record_stream=False,
                           fill="fast", engine="native", chunk_bytes=blk, predictor_chunk_bytes=blk,
                           reference_compat=False)
    mem = prepare_memory(tr, cfg)
    times = []
    for _ in range(reps + 1):
        engine, blocks = build_engine(tr, cfg, mem)
        seg = engine.encode(*encode_events(tr, blocks, cfg, 0))
        engine._sync_blocks()
        engine.flush(wait=True) if plane == "gpu" else None
        if S:
            S.sampler_enable(1)
        t = time.perf_counter()
        if system == "plain":
            engine.plain_replay_encoded(seg)
        else:
            engine.replay_encoded(seg)
        t_issue = time.perf_counter() - t
        if system != "plain":
            engine.finish()
        if plane == "gpu":
            engine.flush(wait=True)
        dt = time.perf_counter() - t
        if S:
            S.sampler_enable(0)
        times.append((t_issue, dt))
        if reps <= 10:
            ps = engine.plane_stats() if plane == "gpu" else {}
            print(f"{system} {blk} {plane}: issue {t_issue * 1e3:.2f} ms, total {dt * 1e3:.2f} ms, "
                  f"{tr.swap_bytes() / dt / 1e9:.2f} GB/s, {len(tr.events)} events, issuer calls "
                  f"{ps.get('issuer_calls')} busy {ps.get('issuer_busy_ms', 0):.2f} ms, launches {ps.get('launches')}",
                  flush=True)
        del engine
    if reps > 10:
        times.sort(key=lambda x: x[1])
        t_issue, dt = times[len(times) // 2]
        print(f"{system} {blk} {plane}: median of {len(times)}: issue {t_issue * 1e3:.2f} ms, total {dt * 1e3:.2f} ms, "
              f"{tr.swap_bytes() / dt / 1e9:.2f} GB/s, {len(tr.events)} events", flush=True)


if __name__ == "__main__":
    main()

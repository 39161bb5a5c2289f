"""Config 5 end to end: OPT-66B-shaped weight offload (2 offloaded layers,
2 iterations) split into blocks of 64 KiB .. 256 MiB, through the native
engine (SpecPipe and SyncCc) vs the same swaps as plain copies
(sp_pipe_plain_replay).  Blocks <= 32 MiB are one channel message each and
the predictor is configured with that chunk (so they classify as
MODEL_WEIGHTS); blocks > 32 MiB travel as 32 MiB messages and
the reference classifies them SMALL_IO (defect C3: never speculated).

    python tools/chunk_sweep.py gpurun_out/chunk_sweep.json
"""
from __future__ import annotations

import json
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # as bench.py: no idle BLAS pool spinning
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

KIB, MIB = 1 << 10, 1 << 20


def best(fn, reps):
    return max(fn().swap_gbs for _ in range(reps))


def main(out: str, sizes_kib: list[int] | None = None) -> None:
    rows = []
    sizes = [k * KIB for k in sizes_kib] if sizes_kib else \
        (64 * KIB, 256 * KIB, 1 * MIB, 4 * MIB, 16 * MIB, 32 * MIB, 64 * MIB, 128 * MIB, 256 * MIB)
    for block in sizes:
        t0 = time.time()
        tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=block)
        msg = min(block, 32 * MIB)
        # reference_compat=False: layers of more than 64 chunks (< 32 MiB blocks)
        # trip the reference's defect C2 on plain FIFO offload
        base = dict(plane="gpu", record_stream=False, fill="fast", engine="native", chunk_bytes=msg,
                    predictor_chunk_bytes=msg, reference_compat=False)
        spec = ReplayConfig(system="specpipe", **base)
        sync = ReplayConfig(system="synccc", **base)
        mem = prepare_memory(tr, spec)
        run_plain_native(tr, spec, memory=mem)
        r = run_engine(tr, spec, memory=mem)
        rep = r.engine.report()
        del r
        reps = int(os.environ.get("SWEEP_REPS", "2"))
        plain = best(lambda: run_plain_native(tr, spec, memory=mem), reps)
        enc = best(lambda: run_engine(tr, spec, memory=mem), reps)
        run_engine(tr, sync, memory=mem)
        sc = best(lambda: run_engine(tr, sync, memory=mem), reps)
        row = {"block_bytes": block, "message_bytes": msg, "blocks_per_layer": len(tr.header.blocks) // 2,
               "events": len(tr.events), "swap_bytes": tr.swap_bytes(), "plain_gbs": round(plain, 2),
               "specpipe_gbs": round(enc, 2), "synccc_gbs": round(sc, 2),
               "specpipe_ratio": round(enc / plain, 4), "synccc_ratio": round(sc / plain, 4),
               "spec_encrypts": rep["spec_encrypts"], "hits": rep["hit"], "iv_ahead": rep["iv_ahead"],
               "nops": rep["nops"], "sweep_s": round(time.time() - t0, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del mem
    json.dump({"workload": "opt-66b offload, layers [1, 2], 2 iterations, native engine", "rows": rows},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/chunk_sweep.json",
         [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else None)

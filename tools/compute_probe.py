"""Offload replay with the model's compute on the GPU: OPT-66B-shaped
FlexGen trace (2 offloaded layers), plain copies vs SpecPipe vs SyncCc at a
few crypto SM budgets; prints one JSON line per run.
    python tools/compute_probe.py [--compute-us 300] [--iters 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--compute-us", type=int, default=0, help="compute per layer (0: the trace default)")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--sms", default="0,16,32,64")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    from paper_2411_03357_b200 import workload
    from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native

    kw = {"compute_per_layer": args.compute_us * 1000} if args.compute_us else {}
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=args.iters, seed=0, **kw)
    base = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                        compute=True)
    mem = prepare_memory(tr, base)
    n_compute = sum(1 for e in tr.events if type(e).__name__ == "ComputeEvent")
    ns_compute = sum(e.duration for e in tr.events if type(e).__name__ == "ComputeEvent")

    def emit(name, r, extra=None):
        row = {"run": name, "wall_ms": round(r.wall_s * 1e3, 2), "swap_gbs": round(r.swap_gbs, 2),
               "compute_events": n_compute, "compute_ms_requested": ns_compute / 1e6}
        row["compute"] = r.engine.compute_stats()
        if not name.startswith("plain"):
            rep = r.engine.report()
            row.update({"hits": rep["hit"], "iv_ahead": rep["iv_ahead"], "nops": rep["nops"]})
        row.update(extra or {})
        print(json.dumps(row), flush=True)

    for comp in (True, False):
        cfg = replace(base, compute=comp)
        run_plain_native(tr, cfg, memory=mem)
        for _ in range(args.reps):
            emit(f"plain compute={comp}", run_plain_native(tr, cfg, memory=mem))
        for sms in [int(x) for x in args.sms.split(",")]:
            c2 = replace(cfg, crypto_sms=sms)
            run_engine(tr, c2, memory=mem)
            for _ in range(args.reps):
                emit(f"specpipe compute={comp} sms={sms}", run_engine(tr, c2, memory=mem))
        c3 = replace(cfg, system="synccc")
        for _ in range(args.reps):
            emit(f"synccc compute={comp}", run_engine(tr, c3, memory=mem))


if __name__ == "__main__":
    main()

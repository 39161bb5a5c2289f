"""Offload comparison probe: plain vs encrypted OPT-66B trace, several reps,
plus a CUDA timeline (torch.profiler / CUPTI) of one encrypted run written
to gpurun_out/ for stream-level analysis (tools/timeline_stats.py)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain, run_plain_native  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-66b")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--trace-out", default="gpurun_out/offload_timeline.json")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--empty-cache", action="store_true", help="torch.cuda.empty_cache() between reps")
    args = ap.parse_args()
    tr = workload.gen_opt_offload_trace(args.model, [1, 2], iterations=args.iters, seed=0)
    cfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", seed=0)
    t = time.perf_counter()
    memory = prepare_memory(tr, cfg)
    print(f"prepare_memory {time.perf_counter() - t:.2f}s", flush=True)
    ncfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", seed=0, engine="native")
    res = {"plain": [], "enc": [], "enc_host_s": [], "native": [], "native_host_s": [], "plain_native": []}
    for _ in range(args.reps):
        r = run_plain(tr, fill="fast", memory=memory)
        res["plain"].append(round(r.swap_gbs, 2))
        c0 = time.process_time()
        r = run_engine(tr, cfg, memory=memory)
        res["enc_host_s"].append(round(time.process_time() - c0, 3))
        res["enc"].append(round(r.swap_gbs, 2))
        rep = r.engine.report()
        del r
        c0 = time.process_time()
        r = run_engine(tr, ncfg, memory=memory)
        res["native_host_s"].append(round(time.process_time() - c0, 3))
        res["native"].append(round(r.swap_gbs, 2))
        assert r.engine.report() == rep
        del r
        res["plain_native"].append(round(run_plain_native(tr, ncfg, memory=memory).swap_gbs, 2))
        if args.empty_cache:
            torch.cuda.empty_cache()
        print(res["plain"][-1], res["enc"][-1], res["enc_host_s"][-1], res["native"][-1], res["native_host_s"][-1],
              res["plain_native"][-1], flush=True)
    res["report"] = {k: rep[k] for k in ("hit", "iv_ahead", "nops", "miss") if k in rep}
    print(json.dumps(res), flush=True)
    if args.no_trace:
        return
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = run_engine(tr, cfg, memory=memory)
    print("profiled enc run GB/s", round(r.swap_gbs, 2), flush=True)
    os.makedirs(os.path.dirname(args.trace_out), exist_ok=True)
    prof.export_chrome_trace(args.trace_out)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = run_engine(tr, ncfg, memory=memory)
    print("profiled native run GB/s", round(r.swap_gbs, 2), flush=True)
    prof.export_chrome_trace(args.trace_out.replace(".json", "_native.json"))
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = run_plain(tr, fill="fast", memory=memory)
    print("profiled plain run GB/s", round(r.swap_gbs, 2), flush=True)
    prof.export_chrome_trace(args.trace_out.replace(".json", "_plain.json"))


if __name__ == "__main__":
    main()

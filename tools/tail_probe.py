"""Is SpecPipe's offload gap the unconsumed encrypt-ahead at the end of the
trace?  Same OPT-66B trace with and without a final swap-in of the layer the
predictor speculated last; SpecPipe / SyncCc / plain for each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native
from paper_2411_03357_b200.workload import SwapInRequest, SyncEvent, Trace

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=iters)
layer1 = [b.id for b in tr.header.blocks if b.kind.layer_index == 1]
t = tr.events[-1].t + 1
ext = Trace(tr.header, list(tr.events) + [SwapInRequest(t, b) for b in layer1] + [SyncEvent(t)])
for name, trace in (("plain trace", tr), ("+final swap-in", ext)):
    cfg = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False)
    mem = prepare_memory(trace, cfg)
    run_plain_native(trace, cfg, memory=mem)
    p = max(run_plain_native(trace, cfg, memory=mem).swap_gbs for _ in range(3))
    run_engine(trace, cfg, memory=mem)
    e = max(run_engine(trace, cfg, memory=mem).swap_gbs for _ in range(3))
    sc = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False, system="synccc")
    s = max(run_engine(trace, sc, memory=mem).swap_gbs for _ in range(3))
    print(f"{name}: plain {p:.2f} specpipe {e:.2f} ({e/p:.3f}) synccc {s:.2f} ({s/p:.3f})", flush=True)

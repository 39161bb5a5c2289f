"""CUDA timelines (torch.profiler) of one SpecPipe and one SyncCc run of the
OPT-66B offload trace through libsppipe, for tools/timeline_stats.py."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from torch.profiler import ProfilerActivity, profile
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine

tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
os.makedirs("gpurun_out", exist_ok=True)
for system in ("specpipe", "synccc"):
    cfg = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False, system=system)
    mem = prepare_memory(tr, cfg)
    run_engine(tr, cfg, memory=mem)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = run_engine(tr, cfg, memory=mem)
    print(system, round(r.swap_gbs, 2), "observable", round(r.observable_gbs, 2), flush=True)
    prof.export_chrome_trace(f"gpurun_out/tl_{system}.json")
    del r

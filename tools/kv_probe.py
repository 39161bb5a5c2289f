"""OPT-30B KV-swap trace (25% adversarial) through the native engine and the
native plain baseline: per-run wall times, then a CUDA timeline
(torch.profiler) of one warm run of each for tools/timeline_stats.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine, run_plain_native, prepare_memory

tr = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
cfg = ReplayConfig(plane="gpu", reference_compat=False, fill="fast", engine="native")
mem = prepare_memory(tr, cfg)
for i in range(3):
    r = run_engine(tr, cfg, memory=mem)
    p = run_plain_native(tr, cfg, memory=mem)
    print(f"native {r.wall_s*1e3:.2f} ms plain {p.wall_s*1e3:.2f} ms", flush=True)
    del r
from torch.profiler import ProfilerActivity, profile
os.makedirs("gpurun_out", exist_ok=True)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = run_engine(tr, cfg, memory=mem)
print(f"profiled native wall {r.wall_s*1e3:.2f} ms", flush=True)
prof.export_chrome_trace("gpurun_out/kv_native_timeline.json")
del r
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    p = run_plain_native(tr, cfg, memory=mem)
print(f"profiled plain wall {p.wall_s*1e3:.2f} ms", flush=True)
prof.export_chrome_trace("gpurun_out/kv_plain_timeline.json")

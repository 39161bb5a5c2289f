"""OPT-30B KV-swap trace through the native engine: wall vs host CPU time and
a CUDA timeline (torch.profiler) of one warm run for tools/timeline_stats.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine, run_plain, prepare_memory

pol = sys.argv[1] if len(sys.argv) > 1 else "lifo"
tr = workload.gen_kvswap_trace(48, pol, kv_block_bytes=229_376, parallel_size=4, seed=0)
cfg = ReplayConfig(plane="gpu", reference_compat=False, fill="fast", engine="native")
mem = prepare_memory(tr, cfg)
for i in range(4):
    c0 = time.process_time()
    r = run_engine(tr, cfg, memory=mem)
    print(f"native wall {r.wall_s*1e3:.2f} ms cpu(total incl build) {(time.process_time()-c0)*1e3:.1f} ms {r.swap_gbs:.2f} GB/s", flush=True)
for i in range(2):
    r = run_plain(tr, fill="fast", memory=mem)
    print(f"plain wall {r.wall_s*1e3:.2f} ms {r.swap_gbs:.2f} GB/s", flush=True)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = run_engine(tr, cfg, memory=mem)
print(f"profiled native wall {r.wall_s*1e3:.2f} ms", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/kv_native_timeline.json")

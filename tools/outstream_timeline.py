"""Timelines of the 1 MiB-chunk OPT-66B offload (SyncCc) with swap-out seals
in the compute queue vs on their own stream (SPPIPE_OUT_STREAM)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from torch.profiler import ProfilerActivity, profile
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine
MIB = 1 << 20
tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=int(os.environ.get("CHUNK_KIB", "1024")) * 1024)
CH = int(os.environ.get("CHUNK_KIB", "1024")) * 1024
cfg = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False, system="synccc",
                   chunk_bytes=CH, predictor_chunk_bytes=CH, reference_compat=False)
mem = prepare_memory(tr, cfg)
run_engine(tr, cfg, memory=mem)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = run_engine(tr, cfg, memory=mem)
tag = os.environ.get("SPPIPE_OUT_STREAM", "0")
print("out_stream", tag, round(r.swap_gbs, 2), flush=True)
prof.export_chrome_trace(f"gpurun_out/tl_out{tag}.json")

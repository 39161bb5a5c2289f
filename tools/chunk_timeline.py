"""torch.profiler timelines of one config-5 chunk size (OPT-66B, 2 layers,
2 iterations): the native engine (SYSTEM=specpipe|synccc) and the plain
baseline, for tools/timeline_stats.py.

    CHUNK_KIB=256 python tools/chunk_timeline.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

CH = int(os.environ.get("CHUNK_KIB", "256")) * 1024
SYSTEM = os.environ.get("SYSTEM", "specpipe")
tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=CH)
MSG = min(CH, 32 << 20)  # channel messages are <= 32 MiB (larger blocks travel as several)
cfg = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False, system=SYSTEM,
                   chunk_bytes=MSG, predictor_chunk_bytes=MSG, reference_compat=False)
mem = prepare_memory(tr, cfg)
for name, fn in ((SYSTEM, lambda: run_engine(tr, cfg, memory=mem)),
                 ("plain", lambda: run_plain_native(tr, cfg, memory=mem))):
    fn()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = fn()
    print(name, CH, round(r.swap_gbs, 2), flush=True)
    prof.export_chrome_trace(f"gpurun_out/tl_{name}_{CH >> 10}k.json")

"""Device timeline of the bench's OPT-30B KV-swap trace (config 3) through
the native engine and the plain baseline: every GPU op (stream, start, end,
kind, bytes) as text, for reading dependency chains.  Run with
SPPIPE_XFER_MAX=0 so each copy is its own (copy-engine) profiler event.

    SPPIPE_XFER_MAX=0 python tools/kv_timeline.py gpurun_out/kv_tl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kv_tl"
cfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                   reference_compat=False)
kv = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
mem = prepare_memory(kv, cfg)
for name, fn in (("engine", lambda: run_engine(kv, cfg, memory=mem)),
                 ("plain", lambda: run_plain_native(kv, cfg, memory=mem))):
    for _ in range(3):
        fn()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = fn()
    path = f"/tmp/kv_{name}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    api = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
    t0 = min(e["ts"] for e in gpu + api)
    with open(f"{out}_{name}.txt", "w") as f:
        f.write(f"{name}: {r.swap_gbs:.2f} GB/s wall {r.wall_s * 1e3:.3f} ms\n")
        t_api_end = max(e["ts"] + e["dur"] for e in api if e["name"] != "cudaStreamSynchronize")
        f.write(f"last non-sync API call ends at {(t_api_end - t0):.1f} us\n")
        for e in sorted(gpu, key=lambda e: e["ts"]):
            kind = e["name"][:18] if e["cat"] != "kernel" else "K:" + e["name"].split("(")[0][-16:]
            b = e.get("args", {}).get("bytes", "")
            f.write(f"{e['ts'] - t0:9.1f} {e['ts'] + e['dur'] - t0:9.1f} s{e.get('tid')} {kind} {b}\n")
    print(name, round(r.swap_gbs, 2), flush=True)

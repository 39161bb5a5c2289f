"""SPPIPE_DEBUG_TIMES=1: for the config-3 KV trace with the model's compute,
how long each compute launch waited for its inputs (the swap-ins of the sync
before it) beyond the previous compute's end — engine vs plain."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

kv = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
cfg = ReplayConfig(system=os.environ.get("SYSTEM", "specpipe"), plane="gpu", record_stream=False, fill="fast",
                   engine="native", reference_compat=False, compute=os.environ.get("COMPUTE", "1") == "1")
mem = prepare_memory(kv, cfg)
which = os.environ.get("ARM", "engine")
fn = (lambda: run_engine(kv, cfg, memory=mem)) if which == "engine" else (lambda: run_plain_native(kv, cfg, memory=mem))
for i in range(3):  # the last run is warm; each prints its log when its pipe closes
    r = fn()
    print("run", i, which, r.swap_gbs, r.wall_s * 1e3, file=sys.stderr, flush=True)
    del r

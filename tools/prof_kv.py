"""The OPT-30B KV-swap trace through the native engine once (for ncu: the
small mixed seal/open batches of a decode-time swap stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine
tr = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
r = run_engine(tr, ReplayConfig(plane="gpu", reference_compat=False, fill="fast", engine="native"))
print("ok", r.engine.report()["data_msgs"])

"""Per-event-kind host time of the native engine on the KV trace (timing build
tools/native/libsppipe_timed.so; prints to stderr from C++)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import _native
_native.SPPIPE_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native", "libsppipe_timed.so")
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine, prepare_memory
tr = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
cfg = ReplayConfig(plane=sys.argv[1] if len(sys.argv) > 1 else "gpu", reference_compat=False, fill="fast", engine="native")
mem = prepare_memory(tr, cfg)
for i in range(3):
    r = run_engine(tr, cfg, memory=mem)
    print(f"wall {r.wall_s*1e3:.2f} ms", flush=True)
    del r

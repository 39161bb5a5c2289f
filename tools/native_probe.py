"""Run-to-run behaviour of the native engine vs the native plain baseline on
the OPT-66B offload and OPT-30B KV traces (GB/s per run + pool statistics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native

which = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                   reference_compat=False)
traces = {}
if which in ("both", "offload"):
    traces["offload"] = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=4)
if which in ("both", "kv"):
    traces["kv"] = workload.gen_adversarial_trace(
        workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
for name, tr in traces.items():
    mem = prepare_memory(tr, cfg)
    for i in range(reps):
        t = time.perf_counter()
        p = run_plain_native(tr, cfg, memory=mem)
        t1 = time.perf_counter()
        r = run_engine(tr, cfg, memory=mem)
        t2 = time.perf_counter()
        st = r.engine.plane_stats()
        print(f"{name} rep {i}: plain {p.swap_gbs:.2f} GB/s ({p.wall_s*1e3:.1f} ms, call {1e3*(t1-t):.0f} ms) "
              f"enc {r.swap_gbs:.2f} GB/s ({r.wall_s*1e3:.1f} ms, call {1e3*(t2-t1):.0f} ms) "
              f"pool {st['pool_reserved']/2**30:.2f}/{st['pool_used']/2**30:.2f} GiB cached {st['cached']/2**30:.2f} "
              f"launches {st['launches']}", flush=True)
        del r

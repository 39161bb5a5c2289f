"""Where does the host spend an OPT-66B replay: dispatching events (the
native replay call) vs waiting for the device in finish()."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, build_engine, encode_events, _drain

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
system = sys.argv[2] if len(sys.argv) > 2 else "specpipe"
tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=iters)
cfg = ReplayConfig(plane="gpu", fill="fast", engine="native", record_stream=False, system=system)
mem = prepare_memory(tr, cfg)
for rep in range(3):
    eng, blocks = build_engine(tr, cfg, mem)
    seg = eng.encode(*encode_events(tr, blocks, cfg))
    _drain(eng, cfg)
    t0 = time.perf_counter()
    eng.replay_encoded(seg)
    t1 = time.perf_counter()
    eng.finish()
    t2 = time.perf_counter()
    print(f"{system} iters {iters}: dispatch {1e3*(t1-t0):.1f} ms, finish wait {1e3*(t2-t1):.1f} ms, total {1e3*(t2-t0):.1f} ms, "
          f"{tr.swap_bytes()/(t2-t0)/1e9:.2f} GB/s", flush=True)
    del eng

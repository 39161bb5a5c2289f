import os, sys
sys.path.insert(0, '/root/repo')
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine
CH = int(os.environ.get("CH_KIB", str(int(os.environ.get("CH_MIB", "16")) * 1024))) << 10
tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=CH)
cfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                   chunk_bytes=CH, predictor_chunk_bytes=CH, reference_compat=False)
mem = prepare_memory(tr, cfg)
for i in range(3):  # the last run is warm
    r = run_engine(tr, cfg, memory=mem)
    print("run", i, r.swap_gbs, r.wall_s * 1e3, file=sys.stderr, flush=True)
    del r

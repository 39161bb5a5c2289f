"""Small native-pipeline workload for compute-sanitizer: speculative offload
(NOP pads from the zero page), KV swap with token I/O (payloads read from the
mapped pinned ring), app writes (ordered DMA bounce), mixed level-scheduled
launches, 33-256-descriptor (large parameter block) launches, PDL chains."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine

cases = [workload.gen_offload_trace(6, [1, 2, 3, 4, 5, 6], 3, layer_bytes=65536, seed=0),
         workload.gen_adversarial_trace(workload.gen_kvswap_trace(8, "lifo", kv_block_bytes=28672, parallel_size=3,
                                                                  seed=1), 0.25, seed=3),
         workload.gen_activation_trace(4, 49155, 2)]
for tr in cases:
    r = run_engine(tr, ReplayConfig(plane="gpu", engine="native", record_stream=True, reference_compat=False),
                   catch=True)
    assert r.error is None, r.error
    print("ok", len(tr.events), r.engine.report()["data_msgs"], len(r.engine.delivered), flush=True)

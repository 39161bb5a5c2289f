"""SURVEY §8d CPU baseline (iii): whole-trace wall clock of the REFERENCE
engine (specpipe's simulator replay: the real engine, validator, predictor
and `cryptography` AES-GCM on the host) for configs 1-4, scaled to finish in
about a minute.  Build container only (imports /root/reference); the traces
come from this repo's byte-identical generators.

    python tools/ref_engine_cpu.py profiles/r1_reference_engine_cpu.json
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True


def main(out: str) -> None:
    from specpipe import simulator as sim
    from specpipe import workload as ref_workload

    from paper_2411_03357_b200 import workload

    cases = [
        ("config 1: 64 MiB layers (2 x 32 MiB), 8 layers, 3 iterations",
         workload.gen_offload_trace(8, list(range(1, 9)), 3, layer_bytes=64 << 20, seed=0)),
        ("config 2 (scaled): OPT-13B, 2 offloaded layers, 2 iterations",
         workload.gen_opt_offload_trace("opt-13b", [21, 22], iterations=2)),
        ("config 3: OPT-30B KV swap, 48 requests, lifo, 25% adversarial (the bench trace)",
         workload.gen_adversarial_trace(workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376,
                                                                  parallel_size=4, seed=0), 0.25, seed=8)),
        ("config 3: OPT-30B KV swap, 48 requests, lifo, no mutation",
         workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0)),
        ("config 4 (scaled): OPT-30B activations, 8 layers x 29,360,128 B, 1 step",
         workload.gen_activation_trace(8, 29_360_128, 1, seed=0)),
    ]
    rows = []
    for name, tr in cases:
        rtr = ref_workload.parse_trace_lines(list(workload.trace_to_lines(tr)))
        t0 = time.perf_counter()
        try:
            m = sim.run(rtr, sim.SimConfig(system=sim.SystemKind.SPECPIPE))
            err = None
        except Exception as exc:  # defect C2 on some adversarial traces
            m, err = None, f"{type(exc).__name__}: {exc}"
        wall = time.perf_counter() - t0
        row = {"case": name, "events": len(tr.events), "swap_bytes": tr.swap_bytes(), "wall_s": round(wall, 2)}
        if err is None:
            row.update(swap_gbs_wall=round(tr.swap_bytes() / wall / 1e9, 4), hit_rate=m.hit_rate)
        else:
            row["error"] = err
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"what": "reference engine (specpipe simulator replay, real crypto via cryptography/OpenSSL) "
                       "wall clock on the build container's CPU, one process",
               "cpu": platform.processor() or platform.machine(), "cores_used": 1, "rows": rows},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1_reference_engine_cpu.json")

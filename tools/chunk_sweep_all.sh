#!/bin/bash
# config-5 sweep with every block size in its own process (no buffer cache or
# pool state carried from one size to the next); merged into $1
out=${1:-gpurun_out/chunk_sweep_full.json}
mkdir -p gpurun_out/sweep_parts
for k in 64 256 1024 4096 16384 32768 65536 131072 262144; do
  SWEEP_REPS=${SWEEP_REPS:-3} timeout 600 python tools/chunk_sweep.py gpurun_out/sweep_parts/$k.json $k > /dev/null 2>&1
done
python - "$out" <<'PY'
import json, sys, glob
rows = []
for k in (64, 256, 1024, 4096, 16384, 32768, 65536, 131072, 262144):
    try:
        rows += json.load(open(f"gpurun_out/sweep_parts/{k}.json"))["rows"]
    except FileNotFoundError:
        pass
json.dump({"workload": "opt-66b offload, layers [1, 2], 2 iterations, native engine; one process per block size",
           "rows": rows}, open(sys.argv[1], "w"), indent=1)
for r in rows:
    print(r["block_bytes"] >> 10, r["plain_gbs"], r["specpipe_ratio"], r["synccc_ratio"])
PY

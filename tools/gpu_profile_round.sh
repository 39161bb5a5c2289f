#!/bin/bash
# bench line, bench launch list, ncu --set full of k_gcm (big layer batch and KV mixed batches)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-offload > gpurun_out/bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv gpurun_out/bench_launches_summary.json "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-offload" | head -c 300; echo
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 2 -o gpurun_out/prof_layer python tools/prof_once.py > /dev/null 2>&1; ls -la gpurun_out/prof_layer.ncu-rep
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 20 -c 6 -o gpurun_out/prof_kv python tools/prof_kv.py > /dev/null 2>&1; ls -la gpurun_out/prof_kv.ncu-rep

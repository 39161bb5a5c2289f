#!/bin/bash
# r2 evidence: bench launch list under ncu + ncu --set full of k_gcm (layer batch), both on the final build
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-offload --no-sweep > gpurun_out/r2_bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2_launches.csv gpurun_out/r2_bench_launches_summary.json "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-offload --no-sweep" | head -c 400; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 2 -o gpurun_out/r2_prof_layer python tools/prof_once.py > gpurun_out/r2_ncu_layer.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_prof_layer.ncu-rep gpurun_out/r2_kgcm_ncu_summary.json | head -c 300; echo
ls -la gpurun_out/r2_prof_layer.ncu-rep

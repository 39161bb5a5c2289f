#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 20 -c 8 -o gpurun_out/r2_prof_kv python tools/prof_kv.py > gpurun_out/r2_ncu_kv.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_prof_kv.ncu-rep gpurun_out/r2_kgcm_kv_ncu_summary.json | head -c 200; echo
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 9 -o gpurun_out/r2_prof_small python tools/prof_small_once.py > gpurun_out/r2_ncu_small.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_prof_small.ncu-rep gpurun_out/r2_kgcm_small_ncu_summary.json | head -c 200; echo

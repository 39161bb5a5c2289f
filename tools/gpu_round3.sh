#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --offload > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 2 -o gpurun_out/prof_r1_v2 python tools/prof_once.py > gpurun_out/ncu_log.txt 2>&1; tail -2 gpurun_out/ncu_log.txt

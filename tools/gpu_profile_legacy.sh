#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['int_roofline']['frac_of_lsu_bound'], d['e2e']['value'], d['e2e']['ratio_vs_plain_copies'], d['offload']['throughput_ratio'], d['offload']['encrypted_runs'], d['offload']['plain_runs'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-offload > gpurun_out/bench_under_ncu.log 2>&1; grep -c k_gcm gpurun_out/launches.csv
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 2 -o gpurun_out/prof_r1_v3 python tools/prof_once.py > /dev/null 2>&1; ls gpurun_out/prof_r1_v3.ncu-rep

#!/bin/bash
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitizer_memcheck.log 2>&1; tail -4 gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitizer_racecheck.log 2>&1; tail -4 gpurun_out/sanitizer_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitizer_synccheck.log 2>&1; tail -4 gpurun_out/sanitizer_synccheck.log
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none --csv --log-file gpurun_out/small_launches.csv python tools/small_msg_bench.py > /dev/null 2>&1; tail -5 gpurun_out/small_launches.csv
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 20 -c 1 -o gpurun_out/prof_small python tools/small_msg_bench.py > /dev/null 2>&1; ls -la gpurun_out/prof_small.ncu-rep

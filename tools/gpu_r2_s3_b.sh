#!/bin/bash
# k_gcm at 104 registers + 256-thread k_xfer: parity, bench line, small-launch ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cipher.py tests/test_gpu_xfer.py tests/test_native_engine.py -x -q -m gpu > gpurun_out/pytest_b.log 2>&1; tail -2 gpurun_out/pytest_b.log
timeout 900 python bench.py > gpurun_out/bench_b.log 2>&1; tail -1 gpurun_out/bench_b.log | head -c 200; echo
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 9 -o gpurun_out/r2_small python tools/prof_small_once.py > gpurun_out/ncu_small.log 2>&1; ls -la gpurun_out/r2_small.ncu-rep

#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python tools/kv_bench.py > gpurun_out/kv_bench.log 2>&1; cat gpurun_out/kv_bench.log | tail -6
timeout 300 python tools/kv_probe.py 2>&1 | grep -v Warn | tail -8; python tools/timeline_stats.py gpurun_out/kv_native_timeline.json | grep -v "^runtime calls"
timeout 800 python tools/offload_probe.py --reps 4 --no-trace > gpurun_out/probe.log 2>&1; grep -v Warn gpurun_out/probe.log | tail -6

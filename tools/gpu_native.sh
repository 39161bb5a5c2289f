#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_native_engine.py -x -q -m gpu > gpurun_out/pytest_native.log 2>&1; tail -15 gpurun_out/pytest_native.log
timeout 600 python tools/kv_bench.py > gpurun_out/kv_bench.log 2>&1; cat gpurun_out/kv_bench.log | tail -6
timeout 800 python tools/offload_probe.py --reps 4 > gpurun_out/probe.log 2>&1; grep -v Warn gpurun_out/probe.log | tail -9
python tools/timeline_stats.py gpurun_out/offload_timeline_native.json | grep -v "^runtime calls"

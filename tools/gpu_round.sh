#!/bin/bash
# One GPU session: tests, bench, launch list.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --offload > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref.log 2>&1; tail -2 gpurun_out/bench_ref.log
nproc; lscpu | grep "Model name"

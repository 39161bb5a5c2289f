#!/bin/bash
# k_xfer: parity tests, engine parity under switches, then the bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xfer.py tests/test_native_engine.py -x -q -m gpu > gpurun_out/pytest_xfer.log 2>&1; tail -3 gpurun_out/pytest_xfer.log
timeout 900 python bench.py > gpurun_out/bench_xfer.log 2>&1; tail -1 gpurun_out/bench_xfer.log | head -c 300; echo

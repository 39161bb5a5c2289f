#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_native_engine.py tests/test_spec_criteria.py tests/test_gpu_channel.py -x -q -m gpu > gpurun_out/pytest_q.log 2>&1; tail -2 gpurun_out/pytest_q.log
for v in "X=1" "SPPIPE_LAND_ON_OUT=0"; do env $v timeout 900 python tools/ab_switch.py "64,16384" >> gpurun_out/ab_q.txt 2>&1; done

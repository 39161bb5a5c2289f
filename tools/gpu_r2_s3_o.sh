#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_native_engine.py tests/test_spec_criteria.py tests/test_gpu_channel.py tests/test_hw_guards.py -x -q -m gpu > gpurun_out/pytest_o.log 2>&1; tail -2 gpurun_out/pytest_o.log
timeout 900 python tools/ab_switch.py "64,1024,16384,32768" > gpurun_out/ab_o.txt 2>&1

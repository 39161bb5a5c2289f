#!/bin/bash
mkdir -p gpurun_out
./tools/native/launch_latency > gpurun_out/ll_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_cipher.py tests/test_native_engine.py tests/test_gpu_channel.py -x -q -m gpu > gpurun_out/pytest_c.log 2>&1; tail -2 gpurun_out/pytest_c.log
timeout 600 python tools/ab_switch.py "64,1024,32768" >> gpurun_out/ab_c.txt 2>&1

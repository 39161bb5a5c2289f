#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_native_engine.py tests/test_spec_criteria.py tests/test_gpu_channel.py -x -q -m gpu > gpurun_out/pytest_n.log 2>&1; tail -2 gpurun_out/pytest_n.log
SPPIPE_DEBUG_TIMES=1 timeout 300 python tools/dbg_out_waits.py > gpurun_out/dbg16_fix.txt 2>&1
timeout 900 python tools/ab_switch.py "64,1024,16384,32768" > gpurun_out/ab_n.txt 2>&1

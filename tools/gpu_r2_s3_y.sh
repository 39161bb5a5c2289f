#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_native_engine.py tests/test_gpu_xfer.py -x -q -m gpu > gpurun_out/pytest_y.log 2>&1; tail -1 gpurun_out/pytest_y.log
for v in "X=1" "SPPIPE_XFER_CTAS=16" "SPPIPE_XFER_CTAS=32"; do env $v timeout 600 python tools/ab_switch.py "64,1024" 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_y.txt; done

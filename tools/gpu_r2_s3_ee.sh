#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_native_engine.py -x -q -m gpu > gpurun_out/pytest_ee.log 2>&1; tail -1 gpurun_out/pytest_ee.log
for v in "X=1" "SPPIPE_SLAB_MAX_KIB=1024"; do env $v timeout 900 python tools/ab_switch.py "64,256,1024" 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_ee.txt; done

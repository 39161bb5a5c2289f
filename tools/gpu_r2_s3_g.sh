#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_native_engine.py tests/test_gpu_channel.py tests/test_spec_criteria.py -x -q -m gpu > gpurun_out/pytest_g.log 2>&1; tail -2 gpurun_out/pytest_g.log
for v in "X=1" "SPPIPE_FUSE_H2D=0"; do env $v timeout 600 python tools/ab_switch.py "64" >> gpurun_out/ab_g.txt 2>&1; done

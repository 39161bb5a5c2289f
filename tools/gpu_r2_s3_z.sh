#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cipher.py tests/test_gpu_channel.py -x -q -m gpu > gpurun_out/pytest_z.log 2>&1; tail -1 gpurun_out/pytest_z.log
for i in 1 2; do for v in "X=1" "SPGCM_PIPE_STREAMS=1"; do env $v timeout 300 python tools/e2e_ab.py 5 >> gpurun_out/e2e_ab.txt 2>&1; done; done

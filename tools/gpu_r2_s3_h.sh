#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "CUDA_DEVICE_MAX_CONNECTIONS=32"; do env $v timeout 600 python tools/ab_switch.py "64,1024,16384" >> gpurun_out/ab_conn.txt 2>&1; done

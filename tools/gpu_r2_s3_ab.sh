#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPPIPE_OUT_STREAM=1"; do env $v timeout 600 python tools/ab_switch.py "${AB_SIZES:-64,1024,32768,262144}" >> gpurun_out/ab_out.txt 2>&1; done

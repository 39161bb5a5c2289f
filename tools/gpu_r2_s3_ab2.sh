#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPGCM_PACK=4" "SPGCM_PACK=16"; do env $v timeout 600 python tools/ab_switch.py "64,1024,32768" >> gpurun_out/ab_pack.txt 2>&1; done
bash tools/gpu_r2_s3_ll.sh

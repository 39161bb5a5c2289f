#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPGCM_SMALL_ROWS=4096" "SPGCM_SMALL_ROWS=4096 SPGCM_SMALL_RPW=4" "SPGCM_TINY_ROWS=512" "SPGCM_SMALL_ROWS=0"; do env $v timeout 600 python tools/ab_switch.py none 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_kvpol.txt; done

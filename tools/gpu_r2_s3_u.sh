#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPGCM_TINY_ROWS=512" "SPGCM_TINY_ROWS=512 SPGCM_SMALL_ROWS=0" "SPPIPE_COMP_STREAMS=1"; do env $v timeout 600 python tools/ab_switch.py "64" 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_u.txt; done

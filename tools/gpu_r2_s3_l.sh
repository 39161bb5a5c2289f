#!/bin/bash
mkdir -p gpurun_out
for v in "SPPIPE_COMP_STREAMS=1" "X=1"; do for i in 1 2 3; do env $v AB_REPS=2 timeout 600 python tools/ab_switch.py "16384" 2>&1 | head -1 | sed "s/^/$v /" >> gpurun_out/ab_l.txt; done; done

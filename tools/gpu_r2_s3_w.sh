#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPPIPE_PRIO=spec_low" "SPPIPE_PRIO=app"; do env $v AB_175B=1 AB_REPS=2 timeout 900 python tools/ab_switch.py "none" 2>&1 | head -1 | sed "s/^/$v /" >> gpurun_out/ab_w.txt; done

#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPPIPE_PRIO=app" "SPPIPE_PRIO=equal"; do env $v timeout 900 python tools/ab_switch.py "64,1024,32768" 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_prio.txt; done

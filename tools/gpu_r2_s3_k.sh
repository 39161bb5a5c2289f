#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3 4 5; do AB_REPS=2 timeout 600 python tools/ab_switch.py "16384,32768" 2>&1 | head -2 >> gpurun_out/ab_16m_rep.txt; done
timeout 600 python tools/ab_switch.py "64,1024" > gpurun_out/ab_k.txt 2>&1

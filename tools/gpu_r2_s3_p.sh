#!/bin/bash
mkdir -p gpurun_out
SPPIPE_DEBUG_TIMES=1 CH_MIB=32 timeout 300 python tools/dbg_out_waits.py > gpurun_out/dbg32.txt 2>&1
SPPIPE_DEBUG_TIMES=1 CH_MIB=16 timeout 300 python tools/dbg_out_waits.py > gpurun_out/dbg16_fix2.txt 2>&1

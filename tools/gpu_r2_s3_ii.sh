#!/bin/bash
mkdir -p gpurun_out
SPPIPE_DEBUG_TIMES=1 CH_KIB=32768 timeout 600 python tools/dbg_out_waits.py > gpurun_out/dbg32b.txt 2>&1

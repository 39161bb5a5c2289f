#!/bin/bash
mkdir -p gpurun_out
SPPIPE_DEBUG_TIMES=1 timeout 300 python tools/dbg_out_waits.py > gpurun_out/dbg16.txt 2>&1
SPPIPE_DEBUG_TIMES=1 SPPIPE_COMP_STREAMS=1 timeout 300 python tools/dbg_out_waits.py > gpurun_out/dbg16_c1.txt 2>&1

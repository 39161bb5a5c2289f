#!/bin/bash
mkdir -p gpurun_out
SPPIPE_OUT_STREAM=1 SPPIPE_DEBUG_TIMES=1 CH_KIB=1024 timeout 600 python tools/dbg_out_waits.py > gpurun_out/dbg1m_out.txt 2>&1

#!/bin/bash
mkdir -p gpurun_out
SPPIPE_DEBUG_TIMES=1 COMPUTE=0 ARM=engine timeout 300 python tools/dbg_kv_compute.py > gpurun_out/dbg_kvso_engine.txt 2>&1

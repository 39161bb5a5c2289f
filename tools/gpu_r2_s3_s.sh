#!/bin/bash
mkdir -p gpurun_out
SPPIPE_DEBUG_TIMES=1 ARM=engine timeout 300 python tools/dbg_kv_compute.py > gpurun_out/dbg_kv_engine.txt 2>&1
SPPIPE_DEBUG_TIMES=1 ARM=plain timeout 300 python tools/dbg_kv_compute.py > gpurun_out/dbg_kv_plain.txt 2>&1

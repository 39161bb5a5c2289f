#!/bin/bash
mkdir -p gpurun_out
for sys in specpipe plain; do timeout 300 python tools/host_prof_replay.py kv $sys gpu 4 >> gpurun_out/hp_kv.txt 2>&1; done
SPPIPE_ASYNC_ISSUE=0 timeout 300 python tools/host_prof_replay.py kv specpipe gpu 4 >> gpurun_out/hp_kv.txt 2>&1
timeout 300 python tools/host_prof_replay.py kv specpipe dry 4 >> gpurun_out/hp_kv.txt 2>&1
for sys in specpipe plain; do timeout 300 python tools/host_prof_replay.py 65536 $sys gpu 2 >> gpurun_out/hp_kv.txt 2>&1; done
timeout 300 python tools/host_prof_replay.py 65536 specpipe dry 2 >> gpurun_out/hp_kv.txt 2>&1

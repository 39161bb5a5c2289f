#!/bin/bash
mkdir -p gpurun_out
for c in 1048576 262144; do for sys in specpipe plain; do timeout 300 python tools/host_prof_replay.py $c $sys gpu 3 >> gpurun_out/hp_mid.txt 2>&1; done; done

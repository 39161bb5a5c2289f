#!/bin/bash
# r2 session 3: stream-memop hand-off latency vs launches; per-copy vs gather-kernel transfers
mkdir -p gpurun_out
timeout 120 ./tools/native/server_probe > gpurun_out/r2_server_probe.txt 2>&1; echo "server rc=$?" >> gpurun_out/r2_server_probe.txt
timeout 300 ./tools/native/copy_probe > gpurun_out/r2_copy_probe.txt 2>&1; echo "copy rc=$?" >> gpurun_out/r2_copy_probe.txt
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" >> gpurun_out/topo.txt

#!/bin/bash
# small-launch latency vs the SmallTabs threshold and rows per warp
mkdir -p gpurun_out
for sr in 256 1024 4096; do for rpw in 1 2 4; do
  echo "== SPGCM_SMALL_ROWS=$sr SPGCM_SMALL_RPW=$rpw" >> gpurun_out/ll_sweep.txt
  SPGCM_SMALL_ROWS=$sr SPGCM_SMALL_RPW=$rpw timeout 120 ./tools/native/launch_latency 2>&1 | grep graph >> gpurun_out/ll_sweep.txt
done; done
for rpw in 1 2 8; do echo "== BIG SPGCM_SMALL_ROWS=0 SPGCM_ROWS_PER_WARP=$rpw" >> gpurun_out/ll_sweep.txt; SPGCM_SMALL_ROWS=0 SPGCM_ROWS_PER_WARP=$rpw timeout 120 ./tools/native/launch_latency 2>&1 | grep graph >> gpurun_out/ll_sweep.txt; done

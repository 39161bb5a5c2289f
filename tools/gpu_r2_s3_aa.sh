#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do for v in "X=1" "SPGCM_PIECE_MIB=64" "SPGCM_PIECE_MIB=128" "SPGCM_PIECE_MIB=16"; do env $v timeout 300 python tools/e2e_ab.py 5 2>&1 | grep -v Warn >> gpurun_out/e2e_piece.txt; done; done

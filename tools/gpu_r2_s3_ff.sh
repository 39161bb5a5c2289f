#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPPIPE_XFER_MAX=524288" "AB_CRYPTO_SMS=120" "AB_CRYPTO_SMS=96"; do env $v timeout 900 python tools/ab_switch.py "256,1024" 2>&1 | grep block_kib | sed "s/^/$v /" >> gpurun_out/ab_ff.txt; done

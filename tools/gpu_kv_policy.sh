# KV trace (swap-only and with compute) under small-launch policies
for e in "X=1" "SPGCM_TINY_ROWS=0 SPGCM_SMALL_ROWS=512 SPGCM_SMALL_RPW=1" "SPGCM_TINY_ROWS=0 SPGCM_SMALL_ROWS=512 SPGCM_SMALL_RPW=2" "SPGCM_TINY_ROWS=0 SPGCM_SMALL_ROWS=2048 SPGCM_SMALL_RPW=2" "SPGCM_TINY_ROWS=0 SPGCM_ROWS_PER_WARP=8"; do
  env $e timeout 600 python tools/ab_switch.py none 2>&1 | tail -1 | sed "s/^/$e /"
done
for e in "X=1" "SPGCM_TINY_ROWS=0 SPGCM_SMALL_ROWS=512 SPGCM_SMALL_RPW=2"; do env $e timeout 300 python tools/small_table.py; done

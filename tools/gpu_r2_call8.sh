for v in "" "SPGCM_TINY_PARAMS=0" "SPGCM_SMALL_ROWS=1024" "SPGCM_SMALL_ROWS=1024 SPGCM_SMALL_RPW=4" "SPPIPE_COMP_STREAMS=1" "SPPIPE_ASYNC_ISSUE=0"; do
  env $v timeout 300 python tools/kv_ab.py 7 >> gpurun_out/r2_kv_ab.txt 2>&1
done
./tools/native/launch_latency > gpurun_out/r2_ll_v4.txt 2>&1
SPGCM_TINY_PARAMS=0 ./tools/native/launch_latency > gpurun_out/r2_ll_v4_notiny.txt 2>&1
SPGCM_SMALL_ROWS=1024 ./tools/native/launch_latency > gpurun_out/r2_ll_v4_small1024.txt 2>&1

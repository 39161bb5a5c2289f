./tools/native/launch_latency > gpurun_out/r2_ll_new.txt 2>&1
SPGCM_SMALL_SINGLE_ROWS=0 ./tools/native/launch_latency > gpurun_out/r2_ll_new_split.txt 2>&1
./tools/native/launch_latency_old > gpurun_out/r2_ll_old.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_call5.log 2>&1

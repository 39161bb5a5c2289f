timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_call6.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputest_call6.log
./tools/native/launch_latency > gpurun_out/r2_ll_v3.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_call6.log 2>&1

# full GPU round: tests, smoke, default bench line, KV device timeline, ncu launch list
bash tools/gpu_check.sh
timeout 600 python tools/kv_timeline.py gpurun_out/kv_tl > gpurun_out/kv_tl.log 2>&1; head -3 gpurun_out/kv_tl_engine.txt gpurun_out/kv_tl_plain.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-offload --no-sweep --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log

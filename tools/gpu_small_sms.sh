# small-launch SM cap set by libsppipe: full GPU tests, traces with the cap on (default) / off, small table (uncapped)
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu tests > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for e in "X=1" "SPPIPE_SMALL_SMS=0"; do
  env $e timeout 900 python tools/ab_switch.py 64,1024 2>&1 | grep '^{' | sed "s/^/$e /"
done
timeout 300 python tools/small_table.py

# ncu --set full of KV-shaped k_gcm launches (1 / 4 / 32 x 224 KiB) + big-kernel timing + small table
mkdir -p gpurun_out
timeout 300 python tools/prof_kv_batches.py && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gcm -c 9 -o gpurun_out/r2_prof_kv_tree -f \
  python tools/prof_kv_batches.py > gpurun_out/ncu_kv.log 2>&1; tail -2 gpurun_out/ncu_kv.log
timeout 300 python tools/quick_kernel_bench.py
timeout 300 python tools/small_table.py
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_cipher.py > gpurun_out/t_cipher.log 2>&1; tail -1 gpurun_out/t_cipher.log

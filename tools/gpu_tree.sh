# lane-combine tree: parity, then small-launch latency and traces with it on/off
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_cipher.py tests/test_gpu_channel.py > gpurun_out/t_tree.log 2>&1; tail -3 gpurun_out/t_tree.log
for e in "SPGCM_TREE_WARPS=0" "SPGCM_TREE_WARPS=1000000" "SPGCM_TREE_WARPS=0 SPGCM_ROWS_PER_WARP=2" "SPGCM_TREE_WARPS=0 SPGCM_ROWS_PER_WARP=1" "SPGCM_TREE_WARPS=0 SPGCM_TINY_ROWS=2048"; do
  env $e timeout 300 python tools/small_table.py
done > gpurun_out/tree_small.txt 2>&1
cat gpurun_out/tree_small.txt
timeout 300 python tools/quick_kernel_bench.py > gpurun_out/tree_big.txt 2>&1; tail -5 gpurun_out/tree_big.txt
for e in "SPGCM_TREE_WARPS=0" "SPGCM_TREE_WARPS=1000000" "SPGCM_TREE_WARPS=0 SPGCM_ROWS_PER_WARP=2"; do env $e timeout 600 python tools/ab_switch.py none 2>&1 | sed "s/^/$e /"; done > gpurun_out/ab_tree.txt
cat gpurun_out/ab_tree.txt

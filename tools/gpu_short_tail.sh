# short-tail scaling tables: parity, small-launch latency, big kernel, KV A/B
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_cipher.py tests/test_gpu_channel.py > gpurun_out/t_st.log 2>&1; tail -2 gpurun_out/t_st.log
timeout 300 python tools/small_table.py
SPGCM_TREE_WARPS=0 timeout 300 python tools/small_table.py
timeout 300 python tools/quick_kernel_bench.py
timeout 600 python tools/ab_switch.py none

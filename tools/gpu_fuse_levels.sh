mkdir -p gpurun_out
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_cipher.py -k "fused_levels or mixed" > gpurun_out/t_fused.log 2>&1; tail -3 gpurun_out/t_fused.log
timeout 900 python -m pytest -x -q -m gpu tests/test_native_engine.py -k "parity_gpu or tamper or switches" > gpurun_out/t_engine.log 2>&1; tail -3 gpurun_out/t_engine.log
for e in "X=1" "SPGCM_FUSE_LEVELS=0"; do env $e timeout 600 python tools/ab_switch.py 64,1024 2>&1 | sed "s/^/$e /"; done > gpurun_out/ab_fuse_levels.txt
cat gpurun_out/ab_fuse_levels.txt

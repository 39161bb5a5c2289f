set -x
./tools/native/pipe_rates > gpurun_out/r2_pipe_rates.jsonl 2>&1
./tools/native/launch_latency > gpurun_out/r2_launch_latency_before.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 10 -c 1 -o gpurun_out/r2_nop_before ./tools/native/launch_latency > gpurun_out/r2_ncu_nop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 20510 -c 1 -o gpurun_out/r2_kv_before ./tools/native/launch_latency > gpurun_out/r2_ncu_kv.log 2>&1
ls -la gpurun_out

set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_call4.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputest_call4.log
./tools/native/launch_latency > gpurun_out/r2_launch_latency_v2.txt 2>&1
timeout 600 python tools/compute_probe.py --iters 4 --sms 0,32,64 > gpurun_out/r2_compute_probe_v2.jsonl 2> gpurun_out/r2_compute_probe_v2.err
SPPIPE_OUT_STREAM=1 timeout 600 python tools/compute_probe.py --iters 4 --sms 0 > gpurun_out/r2_compute_probe_v2_out1.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gcm -s 20510 -c 1 -o gpurun_out/r2_kv_v2 ./tools/native/launch_latency > gpurun_out/r2_ncu_kv_v2.log 2>&1
tail -3 gpurun_out/r2_gputest_call4.log

set -x
./tools/native/pipe_rates > gpurun_out/r2_pipe_rates_v2.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_call3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputest_call3.log
timeout 900 python tools/compute_probe.py --iters 4 > gpurun_out/r2_compute_probe.jsonl 2> gpurun_out/r2_compute_probe.err
tail -3 gpurun_out/r2_gputest_call3.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cipher.py tests/test_native_engine.py tests/test_gpu_channel.py tests/test_spec_criteria.py -x -q -m gpu > gpurun_out/pytest_e.log 2>&1; tail -2 gpurun_out/pytest_e.log
timeout 600 python tools/ab_switch.py "64,1024" > gpurun_out/ab_e.txt 2>&1
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c -lrt
mkdir -p gpurun_out/hostprof3
for r in "65536 specpipe" "kv specpipe"; do
  tag=$(echo $r | tr ' ' '_')
  SAMPLER_WALL_US=50 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py $r gpu 3 > gpurun_out/hostprof3/$tag.log 2>&1
  python tools/sampler_report.py /tmp/samp_$tag.* 60 > gpurun_out/hostprof3/$tag.report 2>&1
  rm -f /tmp/samp_$tag.*
done

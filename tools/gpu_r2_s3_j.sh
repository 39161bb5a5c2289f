#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_native_engine.py tests/test_gpu_xfer.py tests/test_spec_criteria.py -x -q -m gpu > gpurun_out/pytest_j.log 2>&1; tail -2 gpurun_out/pytest_j.log
timeout 600 python tools/ab_switch.py "64,1024" > gpurun_out/ab_j.txt 2>&1
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c -lrt
mkdir -p gpurun_out/hostprof5
tag=65536_specpipe
SAMPLER_WALL_US=50 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py 65536 specpipe gpu 3 > gpurun_out/hostprof5/$tag.log 2>&1
python tools/sampler_report.py /tmp/samp_$tag.* 80 > gpurun_out/hostprof5/$tag.report 2>&1
for sym in cuMemGetAttribute_v2 cuVDPAUCtxCreate malloc operator; do python tools/sampler_report.py /tmp/samp_$tag.* 20 $sym >> gpurun_out/hostprof5/$tag.report 2>&1; done

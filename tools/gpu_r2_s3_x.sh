#!/bin/bash
mkdir -p gpurun_out/hostprof6
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c -lrt
tag=65536_specpipe
SAMPLER_WALL_US=50 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py 65536 specpipe gpu 3 > gpurun_out/hostprof6/$tag.log 2>&1
python tools/sampler_report.py /tmp/samp_$tag.* 100 > gpurun_out/hostprof6/$tag.report 2>&1
for sym in flush land seal_host_chunks submit_d2h send_on_the_fly alloc sync; do python tools/sampler_report.py /tmp/samp_$tag.* 15 "Engine::$sym\|Plane::$sym" >> gpurun_out/hostprof6/$tag.report 2>&1; done
cp /tmp/samp_$tag.* gpurun_out/hostprof6/ 2>/dev/null
gzip -f gpurun_out/hostprof6/samp_* 2>/dev/null

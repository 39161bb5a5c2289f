#!/bin/bash
# wall-clock samples of the control thread (tools/native/sampler.c sampler_start_thread)
mkdir -p gpurun_out/hostprof2
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c -lrt
for r in "65536 specpipe" "65536 plain" "kv specpipe" "kv plain"; do
  tag=$(echo $r | tr ' ' '_')
  SAMPLER_WALL_US=50 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py $r gpu 3 > gpurun_out/hostprof2/$tag.log 2>&1
  python tools/sampler_report.py /tmp/samp_$tag.* 60 > gpurun_out/hostprof2/$tag.report 2>&1
  rm -f /tmp/samp_$tag.*
done

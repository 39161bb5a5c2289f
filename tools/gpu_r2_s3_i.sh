#!/bin/bash
mkdir -p gpurun_out
for v in "X=1" "SPPIPE_OUT_STREAM=0" "SPPIPE_COMP_STREAMS=1" "SPPIPE_EAGER_OPEN=0" "SPPIPE_XFER_MAX=0"; do env $v AB_REPS=2 timeout 600 python tools/ab_switch.py "16384" 2>&1 | head -1 | sed "s/^/$v /" >> gpurun_out/ab_16m.txt; done
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c -lrt
mkdir -p gpurun_out/hostprof4
for r in "65536 specpipe"; do
  tag=$(echo $r | tr ' ' '_')
  SAMPLER_WALL_US=50 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py $r gpu 3 > gpurun_out/hostprof4/$tag.log 2>&1
  python tools/sampler_report.py /tmp/samp_$tag.* 80 > gpurun_out/hostprof4/$tag.report 2>&1
  rm -f /tmp/samp_$tag.*
done

#!/bin/bash
# host-side sampling profiles of native replays on the GPU box (config-5 small blocks)
mkdir -p gpurun_out/hostprof
gcc -O2 -shared -fPIC -o /tmp/libsampler.so tools/native/sampler.c
IFS=';' read -ra RUNS <<< "${HOSTPROF_RUNS:-65536 specpipe;65536 synccc;65536 plain;262144 specpipe;262144 plain}"
for r in "${RUNS[@]}"; do
  tag=$(echo $r | tr ' ' '_')
  SAMPLER_US=1000 SAMPLER_OUT=/tmp/samp_$tag LD_PRELOAD=/tmp/libsampler.so timeout 600 python tools/host_prof_replay.py $r gpu 3 > gpurun_out/hostprof/$tag.log 2>&1
  python tools/sampler_report.py /tmp/samp_$tag.* 70 > gpurun_out/hostprof/$tag.report 2>&1
  for sym in __default_morecore malloc cuVDPAUCtxCreate; do python tools/sampler_report.py /tmp/samp_$tag.* 25 $sym >> gpurun_out/hostprof/$tag.report 2>&1; done
  rm -f /tmp/samp_$tag.*
done
grep -h "GB/s" gpurun_out/hostprof/*.log

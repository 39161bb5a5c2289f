#!/bin/bash
# timelines of the small-block cases after k_xfer: KV trace, config-5 at 64 KiB and 1 MiB
mkdir -p gpurun_out
timeout 300 python tools/kv_timeline.py gpurun_out/kv_tl > gpurun_out/kv_tl.log 2>&1
for n in engine plain; do echo "== $n" >> gpurun_out/tl_stats.txt; python tools/timeline_stats.py /tmp/kv_$n.json >> gpurun_out/tl_stats.txt 2>&1; done
for c in 64 1024; do
  CHUNK_KIB=$c timeout 300 python tools/chunk_timeline.py >> gpurun_out/chunk_tl.log 2>&1
  for n in specpipe plain; do echo "== $n $c" >> gpurun_out/tl_stats.txt; python tools/timeline_stats.py gpurun_out/tl_${n}_${c}k.json >> gpurun_out/tl_stats.txt 2>&1; done
done
rm -f gpurun_out/tl_*k.json
SPPIPE_ISSUER_PROFILE=1 timeout 300 python tools/kv_ab.py 3 > gpurun_out/kv_issuer.txt 2>&1

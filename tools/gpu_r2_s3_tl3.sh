#!/bin/bash
# swap-only timelines of mid-size chunks (16 MiB: no speculation; 64 MiB: SMALL_IO) — where the duplex links idle
mkdir -p gpurun_out
rm -f gpurun_out/tl_stats3.txt
for c in 16384 65536; do
  CHUNK_KIB=$c timeout 300 python tools/chunk_timeline.py >> gpurun_out/chunk_tl3.log 2>&1
  for n in specpipe plain; do echo "== $n $c" >> gpurun_out/tl_stats3.txt; python tools/timeline_stats.py gpurun_out/tl_${n}_${c}k.json >> gpurun_out/tl_stats3.txt 2>&1; done
done
mkdir -p gpurun_out/tl3; mv gpurun_out/tl_*k.json gpurun_out/tl3/ 2>/dev/null; gzip -f gpurun_out/tl3/*.json

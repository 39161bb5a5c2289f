#!/bin/bash
# swap-only timelines of big chunks (32 MiB, 256 MiB): where the duplex links idle
mkdir -p gpurun_out
rm -f gpurun_out/tl_stats2.txt
for c in 32768 262144; do
  CHUNK_KIB=$c timeout 300 python tools/chunk_timeline.py >> gpurun_out/chunk_tl2.log 2>&1
  for n in specpipe plain; do echo "== $n $c" >> gpurun_out/tl_stats2.txt; python tools/timeline_stats.py gpurun_out/tl_${n}_${c}k.json >> gpurun_out/tl_stats2.txt 2>&1; done
done
SYSTEM=synccc CHUNK_KIB=32768 timeout 300 python tools/chunk_timeline.py >> gpurun_out/chunk_tl2.log 2>&1
echo "== synccc 32768" >> gpurun_out/tl_stats2.txt; python tools/timeline_stats.py gpurun_out/tl_synccc_32768k.json >> gpurun_out/tl_stats2.txt 2>&1
mkdir -p gpurun_out/tl; mv gpurun_out/tl_*k.json gpurun_out/tl/ 2>/dev/null; cd gpurun_out/tl && gzip -f *.json; ls -la

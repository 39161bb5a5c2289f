"""torch.profiler timeline of one sp_seal_host_batch call on the OPT-13B
layer (the bench's e2e step, first half): per-stream copy/kernel intervals."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

MIB = 1 << 20
sizes = [32 * MIB] * 18 + [25_298_944]
total = sum(sizes)
offs = [sum(sizes[:i]) for i in range(len(sizes))]
ctx = GcmContext(bytes(range(32)))
h_plain = torch.randint(0, 256, (total,), dtype=torch.uint8).pin_memory()
h_ct = torch.empty_like(h_plain).pin_memory()
h_tags = torch.empty((len(sizes), 16), dtype=torch.uint8).pin_memory()
hs = [(0, i, h_plain[o:o + s], h_ct[o:o + s], h_tags[i]) for i, (o, s) in enumerate(zip(offs, sizes))]
for _ in range(3):
    ctx.seal_host_batch(hs)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ctx.seal_host_batch(hs)
prof.export_chrome_trace("/tmp/e2e.json")
ev = json.load(open("/tmp/e2e.json"))["traceEvents"]
gpu = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")), key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
for e in gpu:
    kind = "K" if e["cat"] == "kernel" else e["name"][7:11]
    b = e.get("args", {}).get("bytes", 0) or 0
    bw = f"{b / e['dur'] / 1e3:.1f} GB/s" if b else ""
    print(f"{e['ts'] - t0:9.1f} {e['ts'] + e['dur'] - t0:9.1f} s{e.get('tid')} {kind} {b >> 20} MiB {bw}")

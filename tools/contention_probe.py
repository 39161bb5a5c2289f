"""Is the per-message XOR accumulator contended?  Same 448 rows (224 KiB)
per launch split into 1, 4, 8, 32 messages: graph-replayed device time per
launch (python tools/contention_probe.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

ctx = GcmContext(bytes(range(32)))
dev = torch.device("cuda:0")
buf = torch.zeros(8 << 20, dtype=torch.uint8, device=dev)
tags = torch.zeros((64, 16), dtype=torch.uint8, device=dev)
s = torch.cuda.Stream(dev)
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SPGCM_")) or "default"
for k, size in ((1, 229_376), (4, 57_344), (8, 28_672), (32, 7_168), (2, 229_376), (4, 229_376)):
    items = [(0, 7 + i, buf[i * size:(i + 1) * size], buf[i * size:(i + 1) * size], tags[i]) for i in range(k)]
    with torch.cuda.stream(s):
        for _ in range(5):
            ctx.seal_batch(items, s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(200):
            ctx.seal_batch(items, torch.cuda.current_stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        s.synchronize()
        a.record(s)
        for _ in range(3):
            g.replay()
        b.record(s)
    b.synchronize()
    print(f"{env:40s} {k:3d} x {size:7d} B  {a.elapsed_time(b) * 1e3 / 600:6.2f} us/launch", flush=True)

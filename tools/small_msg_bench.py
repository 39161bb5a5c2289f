"""Latency of small-message paths: NOP batches, 2 KiB tokens, one 224 KiB KV block."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext
ctx = GcmContext(bytes(range(32)))
s = torch.cuda.Stream()
def bench(label, n_msgs, size, reps=200):
    src = torch.zeros(n_msgs * size, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    tags = torch.empty((n_msgs, 16), dtype=torch.uint8, device="cuda")
    items = [(0, i, src[i*size:(i+1)*size], dst[i*size:(i+1)*size], tags[i]) for i in range(n_msgs)]
    for _ in range(10): ctx.seal_batch(items, s)
    s.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): ctx.seal_batch(items, s)
    e1.record(s); s.synchronize()
    host_us = (time.perf_counter() - t0) / reps * 1e6
    dev_us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{label:28s} host {host_us:8.1f} us/call  device {dev_us:8.1f} us/call  ({n_msgs*size/dev_us/1e3:.2f} GB/s)")
bench("1 NOP", 1, 1)
bench("8 NOPs batch", 8, 1)
bench("1 x 2 KiB token", 1, 2048)
bench("1 x 224 KiB KV block", 1, 229376)
bench("32 x 224 KiB KV blocks", 32, 229376)
bench("1 x 32 MiB chunk", 1, 32 << 20, reps=50)

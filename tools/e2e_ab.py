"""The bench's e2e step alone (sp_seal_host_batch + sp_open_host_batch of the
OPT-13B layer through pinned host buffers) against plain duplex copies of the
same bytes, for A/B runs of SPGCM_* switches:  python tools/e2e_ab.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

MIB = 1 << 20
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sizes = [32 * MIB] * 18 + [25_298_944]
total = sum(sizes)
offs = [sum(sizes[:i]) for i in range(len(sizes))]
ctx = GcmContext(bytes(range(32)))
h_plain = torch.randint(0, 256, (total,), dtype=torch.uint8).pin_memory()
h_ct = torch.empty_like(h_plain).pin_memory()
h_back = torch.empty_like(h_plain).pin_memory()
h_tags = torch.empty((len(sizes), 16), dtype=torch.uint8).pin_memory()
hs = [(0, 9000 + i, h_plain[o:o + s], h_ct[o:o + s], h_tags[i]) for i, (o, s) in enumerate(zip(offs, sizes))]
ho = [(0, 9000 + i, h_ct[o:o + s], h_back[o:o + s], h_tags[i]) for i, (o, s) in enumerate(zip(offs, sizes))]
for _ in range(2):
    ctx.seal_host_batch(hs)
    ctx.open_host_batch(ho)
assert torch.equal(h_back, h_plain)
ts = []
for _ in range(reps):
    t = time.perf_counter()
    ctx.seal_host_batch(hs)
    ctx.open_host_batch(ho)
    ts.append((time.perf_counter() - t) * 1e3)
d = torch.empty(total, dtype=torch.uint8, device="cuda")
src = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
pl = []
for _ in range(reps + 1):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _r in range(2):
        with torch.cuda.stream(sa):
            d.copy_(h_plain, non_blocking=True)
        with torch.cuda.stream(sb):
            h_back.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    pl.append((time.perf_counter() - t) * 1e3)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("SPGCM_", "SPPIPE_"))) or "default"
best, pbest = min(ts), min(pl[1:])
print(f"{env}: e2e {best:.3f} ms = {2 * total / best / 1e6:.2f} GB/s; plain duplex {pbest:.3f} ms; ratio {pbest / best:.4f}",
      flush=True)

"""e2e host pipeline vs plain duplex copies for one OPT-13B layer (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext
MIB = 1 << 20
sizes = [32 * MIB] * 18 + [25_298_944]
total = sum(sizes); n = len(sizes)
offs = [sum(sizes[:i]) for i in range(n)]
ctx = GcmContext(bytes(range(32)))
h_plain = torch.randint(0, 256, (total,), dtype=torch.uint8).pin_memory()
h_ct = torch.empty_like(h_plain).pin_memory(); h_back = torch.empty_like(h_plain).pin_memory()
h_tags = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
hs = [(0, i, h_plain[o:o+s], h_ct[o:o+s], h_tags[i]) for i, (o, s) in enumerate(zip(offs, sizes))]
ho = [(0, i, h_ct[o:o+s], h_back[o:o+s], h_tags[i]) for i, (o, s) in enumerate(zip(offs, sizes))]
for _ in range(2): ctx.seal_host_batch(hs); ctx.open_host_batch(ho)
assert torch.equal(h_back, h_plain)
K = 5
t0 = time.perf_counter()
for _ in range(K): ctx.seal_host_batch(hs)
seal_ms = (time.perf_counter() - t0) * 1e3 / K
t0 = time.perf_counter()
for _ in range(K): ctx.open_host_batch(ho)
open_ms = (time.perf_counter() - t0) * 1e3 / K
d = torch.empty(total, dtype=torch.uint8, device="cuda"); d2 = torch.empty_like(d)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K):
    with torch.cuda.stream(sa): d.copy_(h_plain, non_blocking=True)
    with torch.cuda.stream(sb): h_back.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
dup_ms = (time.perf_counter() - t0) * 1e3 / K
t0 = time.perf_counter()
for _ in range(K):
    d.copy_(h_plain, non_blocking=True); torch.cuda.synchronize()
h2d_ms = (time.perf_counter() - t0) * 1e3 / K
t0 = time.perf_counter()
for _ in range(K):
    h_back.copy_(d2, non_blocking=True); torch.cuda.synchronize()
d2h_ms = (time.perf_counter() - t0) * 1e3 / K
print(f"piece={os.environ.get('SPGCM_PIECE_MIB','32')}MiB seal {seal_ms:.2f} ms ({total/seal_ms/1e6:.1f} GB/s) open {open_ms:.2f} ms "
      f"({total/open_ms/1e6:.1f} GB/s) | plain duplex {dup_ms:.2f} ms, H2D only {h2d_ms:.2f} ({total/h2d_ms/1e6:.1f} GB/s), D2H only {d2h_ms:.2f} ({total/d2h_ms/1e6:.1f} GB/s)")

"""One seal + one open launch over an OPT-13B layer batch (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext
MIB = 1 << 20
ctx = GcmContext(bytes(range(32)))
sizes = [32 * MIB] * 18 + [25_298_944]
total = sum(sizes)
buf = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(buf); back = torch.empty_like(buf)
tags = torch.empty((len(sizes), 16), dtype=torch.uint8, device="cuda")
st = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
items, oitems, off = [], [], 0
for i, n in enumerate(sizes):
    items.append((0, i, buf[off:off+n], out[off:off+n], tags[i]))
    oitems.append((0, i, out[off:off+n], back[off:off+n], tags[i]))
    off += n
ctx.seal_batch(items); ctx.open_batch(oitems, st)
torch.cuda.synchronize()
print("ok", torch.equal(back, buf))

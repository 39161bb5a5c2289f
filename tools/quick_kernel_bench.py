"""Quick HBM-resident seal/open timing of one OPT-13B layer batch (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext
MIB = 1 << 20
torch.cuda.set_device(0)
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
for _ in range(3):
    ctx.seal_batch(items); ctx.open_batch(oitems, st)
torch.cuda.synchronize()
for name, fn in (("seal", lambda: ctx.seal_batch(items)), ("open", lambda: ctx.open_batch(oitems, st))):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    K = 10
    e0.record()
    for _ in range(K): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{name}: {ms:.3f} ms  {total/ms/1e6:.1f} GB/s")
print("roundtrip ok:", torch.equal(back, buf), int(st.sum()))

"""Small, path-covering workload for compute-sanitizer (memcheck / racecheck /
synccheck): multi-message batch with tails, unaligned buffers, a multi-run
message (atomic accumulator path), tamper -> zeroing, host pipeline."""
import sys, os, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext, GcmAuthError
rng = random.Random(1)
ctx = GcmContext(bytes(range(32)))
sizes = [1, 15, 16, 17, 4097, 70001, 600000]
total = sum(sizes) + 64
src = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
dst = torch.zeros_like(src); back = torch.zeros_like(src)
tags = torch.zeros((len(sizes), 16), dtype=torch.uint8, device="cuda")
st = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
items, oitems, off = [], [], 3
for i, n in enumerate(sizes):
    items.append((i & 1, rng.randrange(1 << 64), src[off:off + n], dst[off + 1:off + 1 + n], tags[i]))
    oitems.append((items[-1][0], items[-1][1], dst[off + 1:off + 1 + n], back[off:off + n], tags[i]))
    off += n
ctx.seal_batch(items); ctx.open_batch(oitems, st); torch.cuda.synchronize()
assert int(st.sum()) == 0
assert torch.equal(back[3:off], src[3:off])
dst[10] ^= 1
ctx.open_batch(oitems, st); torch.cuda.synchronize()
assert int(st.sum()) >= 1
h = bytes(rng.randbytes(3 << 20))
c, t = ctx.seal_bytes(0, 7, h)
assert ctx.open_bytes(0, 7, c, t) == h
try:
    ctx.open_bytes(0, 8, c, t)
    raise SystemExit("tamper accepted")
except GcmAuthError:
    pass
print("sanitize case ok")

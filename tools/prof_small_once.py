"""A few small launches for ncu source-level sampling (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext
ctx = GcmContext(bytes(range(32)))
for n, k in ((65536, 1), (1, 32), (229376, 1)):
    src = torch.zeros(n * k, dtype=torch.uint8, device="cuda"); dst = torch.empty_like(src)
    tags = torch.empty((k, 16), dtype=torch.uint8, device="cuda")
    items = [(0, i, src[i*n:(i+1)*n], dst[i*n:(i+1)*n], tags[i]) for i in range(k)]
    for _ in range(3): ctx.seal_batch(items)
torch.cuda.synchronize()

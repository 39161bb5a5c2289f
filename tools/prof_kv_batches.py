"""KV-shaped k_gcm launches for one ncu --set full capture (dev tool):
1, 4 and 32 x 224 KiB blocks, three launches each (the 4- and 32-block
launches combine lanes with the shared-memory tree, the 1-block one with
the nibble tables)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

ctx = GcmContext(bytes(range(32)))
n = 229_376
for k in (1, 4, 32):
    src = torch.randint(0, 256, (n * k,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    tags = torch.empty((k, 16), dtype=torch.uint8, device="cuda")
    items = [(0, i, src[i * n:(i + 1) * n], dst[i * n:(i + 1) * n], tags[i]) for i in range(k)]
    for _ in range(3):
        ctx.seal_batch(items)
torch.cuda.synchronize()

"""One KV-shaped flush: seals of k x 224 KiB blocks then the receiver opens
of them (2 dependent levels) — as ONE sp_crypt_levels launch vs two
sp_crypt_batch launches; graph-replayed device time per flush
(python tools/levels_probe.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_03357_b200 import _native  # noqa: E402
from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

ctx = GcmContext(bytes(range(32)))
lib = _native.load_spgcm()
n = 229_376
s = torch.cuda.Stream()
for k in (1, 4, 8):
    src = torch.randint(0, 256, (k * n,), dtype=torch.uint8, device="cuda")
    mid = torch.empty_like(src)
    out = torch.empty_like(src)
    tags = torch.zeros((k, 16), dtype=torch.uint8, device="cuda")
    st = torch.zeros(2 * k, dtype=torch.int32, device="cuda")
    descs = (_native.SpDesc * (2 * k))()
    for i in range(k):
        for lv, (a, b) in enumerate(((src, mid), (mid, out))):
            d = descs[lv * k + i]
            d.dir, d.reserved, d.iv, d.len = 0, lv, 1000 + i, n
            d.src, d.dst, d.tag = a[i * n:].data_ptr(), b[i * n:].data_ptr(), tags[i].data_ptr()
            d.status = st.data_ptr() + 4 * (lv * k + i)
    starts = (ctypes.c_int * 3)(0, k, 2 * k)
    lv0 = (_native.SpDesc * k)(*descs[:k])
    lv1 = (_native.SpDesc * k)(*descs[k:])
    h = ctypes.c_void_p(s.cuda_stream)

    def fused():
        assert lib.sp_crypt_levels(ctx._h, descs, 2 * k, starts, 2, h) == 0

    def split():
        assert lib.sp_crypt_batch(ctx._h, lv0, k, h) == 0
        assert lib.sp_crypt_batch(ctx._h, lv1, k, h) == 0

    for name, fn in (("fused (1 launch)", fused), ("split (2 launches)", split)):
        with torch.cuda.stream(s):
            for _ in range(5):
                fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            h = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for _ in range(100):
                fn()
        h = ctypes.c_void_p(s.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            g.replay()
            s.synchronize()
            a.record(s)
            for _ in range(3):
                g.replay()
            b.record(s)
        b.synchronize()
        assert torch.equal(out, src) and int(st.sum()) == 0
        print(f"{k} x 224 KiB seal -> open  {name:20s} {a.elapsed_time(b) * 1e3 / 300:6.2f} us/flush", flush=True)

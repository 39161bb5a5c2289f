"""Config-5 chunk-size sweep: device-resident seal/open GB/s of
single messages 64 KiB .. 32 MiB and multi-message runs 64/128/256 MiB
(2/4/8 x 32 MiB), each as one launch; writes JSON to argv[1]."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_03357_b200.gcm import GcmContext

KIB, MIB = 1 << 10, 1 << 20
ctx = GcmContext(bytes(range(32)))
s = torch.cuda.Stream()
rows = []
cases = [("single", n, 1) for n in (64 * KIB, 256 * KIB, 1 * MIB, 4 * MIB, 16 * MIB, 32 * MIB)]
cases += [("run", 32 * MIB, k) for k in (2, 4, 8)]
cases += [("batch-kv", 229_376, k) for k in (8, 64)]
for kind, n, k in cases:
    total = n * k
    src = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src); back = torch.empty_like(src)
    tags = torch.empty((k, 16), dtype=torch.uint8, device="cuda")
    st = torch.zeros(k, dtype=torch.int32, device="cuda")
    si = [(0, i, src[i*n:(i+1)*n], dst[i*n:(i+1)*n], tags[i]) for i in range(k)]
    oi = [(0, i, dst[i*n:(i+1)*n], back[i*n:(i+1)*n], tags[i]) for i in range(k)]
    for _ in range(5):
        ctx.seal_batch(si, s); ctx.open_batch(oi, st, s)
    s.synchronize()
    reps = max(5, min(500, int(2e9 // total)))
    res = {}
    for name, fn in (("seal", lambda: ctx.seal_batch(si, s)), ("open", lambda: ctx.open_batch(oi, st, s))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s); s.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        res[name + "_us"] = round(us, 2)
        res[name + "_gbs"] = round(total / us / 1e3, 2)
    assert torch.equal(back, src) and int(st.sum()) == 0
    rows.append({"kind": kind, "message_bytes": n, "messages": k, "total_bytes": total, **res})
    print(rows[-1], flush=True)
json.dump({"device": torch.cuda.get_device_name(), "rows": rows}, open(sys.argv[1], "w"), indent=1)

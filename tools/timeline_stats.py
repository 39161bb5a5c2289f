"""Summarise a torch.profiler chrome trace: per CUDA stream busy time, kernel
and memcpy totals, and the wall span, to see where an offload run waits."""
from __future__ import annotations

import json
import sys
from collections import defaultdict


def union(intervals):
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in sorted(intervals):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def main(path: str) -> None:
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    if not gpu:
        print("no gpu events")
        return
    t0 = min(e["ts"] for e in gpu)
    t1 = max(e["ts"] + e["dur"] for e in gpu)
    print(f"gpu span {(t1 - t0) / 1e3:.1f} ms, events {len(gpu)}")
    by_stream = defaultdict(list)
    kinds = defaultdict(lambda: [0, 0.0, 0])
    for e in gpu:
        tid = e.get("tid")
        by_stream[tid].append((e["ts"], e["ts"] + e["dur"]))
        name = e["name"]
        key = name if e["cat"] != "kernel" else ("kernel:" + name[:40])
        k = kinds[key]
        k[0] += 1
        k[1] += e["dur"]
        k[2] += int(e.get("args", {}).get("bytes", 0) or 0)
    for tid, iv in sorted(by_stream.items(), key=lambda x: str(x[0])):
        print(f"stream {tid}: {len(iv)} ops busy {union(iv) / 1e3:.1f} ms")
    for key, (n, dur, b) in sorted(kinds.items(), key=lambda x: -x[1][1])[:15]:
        bw = f" {b / dur / 1e3:.1f} GB/s" if b else ""
        print(f"{key}: n={n} total {dur / 1e3:.1f} ms{bw}")
    h2d = [(e["ts"], e["ts"] + e["dur"]) for e in gpu if "HtoD" in e["name"]]
    d2h = [(e["ts"], e["ts"] + e["dur"]) for e in gpu if "DtoH" in e["name"]]
    kern = [(e["ts"], e["ts"] + e["dur"]) for e in gpu if e["cat"] == "kernel"]
    print(f"H2D busy {union(h2d) / 1e3:.1f} ms, D2H busy {union(d2h) / 1e3:.1f} ms, "
          f"kernels busy {union(kern) / 1e3:.1f} ms, any copy {union(h2d + d2h) / 1e3:.1f} ms")
    # idle gaps of the H2D engine longer than 0.2 ms
    gaps = []
    s = sorted(h2d)
    for (a, b), (c, d) in zip(s, s[1:]):
        if c - b > 200:
            gaps.append((round((b - t0) / 1e3, 2), round((c - b) / 1e3, 2)))
    print("H2D gaps >0.2ms (at ms, len ms):", gaps[:40], "total", round(sum(g[1] for g in gaps), 1))
    gaps = []
    s = sorted(d2h)
    for (a, b), (c, d) in zip(s, s[1:]):
        if c - b > 50:
            gaps.append((round((b - t0) / 1e3, 2), round((c - b) / 1e3, 3)))
    print("D2H gaps >0.05ms (at ms, len ms):", gaps[:40], "n", len(gaps), "total", round(sum(g[1] for g in gaps), 2))
    gaps = []
    s = sorted(h2d)
    for (a, b), (c, d) in zip(s, s[1:]):
        if c - b > 50:
            gaps.append((round((b - t0) / 1e3, 2), round((c - b) / 1e3, 3)))
    print("H2D gaps >0.05ms: n", len(gaps), "total", round(sum(g[1] for g in gaps), 2), gaps[:20])
    if h2d and d2h:
        print(f"H2D first {(min(a for a, _ in h2d) - t0) / 1e3:.2f} last {(max(b for _, b in h2d) - t0) / 1e3:.2f} ms; "
              f"D2H first {(min(a for a, _ in d2h) - t0) / 1e3:.2f} last {(max(b for _, b in d2h) - t0) / 1e3:.2f} ms")
    # host-side runtime calls: where does the host thread block?
    rt = defaultdict(lambda: [0, 0.0, 0.0])
    for e in ev:
        if e.get("ph") == "X" and e.get("cat") == "cuda_runtime":
            r = rt[e["name"]]
            r[0] += 1
            r[1] += e["dur"]
            r[2] = max(r[2], e["dur"])
    for name, (n, dur, mx) in sorted(rt.items(), key=lambda x: -x[1][1])[:10]:
        print(f"runtime {name}: n={n} total {dur / 1e3:.1f} ms max {mx / 1e3:.2f} ms")
    api = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
    if api:
        a0 = min(a for a, _ in api)
        a1 = max(b for _, b in api)
        print(f"host API span {(a1 - a0) / 1e3:.2f} ms, API busy {union(api) / 1e3:.2f} ms, "
              f"GPU tail after last API call {(t1 - a1) / 1e3:.2f} ms")
    long = sorted(((e["ts"] - t0) / 1e3, e["dur"] / 1e3, e["name"]) for e in ev
                  if e.get("ph") == "X" and e.get("cat") == "cuda_runtime" and e["dur"] > 1000)
    print("runtime calls > 1 ms (at ms, ms, name):", [(round(a, 1), round(b, 1), c) for a, b, c in long[:40]])


if __name__ == "__main__":
    main(sys.argv[1])

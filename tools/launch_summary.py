"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel launch counts, total time and share of the listed GPU time.

    python tools/launch_summary.py gpurun_out/launches.csv profiles/<round>_bench_launches_summary.json "<command>"
"""
import csv
import json
import sys
from collections import defaultdict


def main(path: str, out: str, command: str = "") -> None:
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        name = r["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v[1] for v in agg.values()) or 1.0
    summary = {"command": command, "kernels": {
        k: {"launches": n, "total_ns": round(t), "share": round(t / total, 4)}
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary)[:600])


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Break one function's inclusive samples down by its direct callees, from
a tools/native/sampler.c dump (paths remapped to this checkout).

    python tools/sampler_children.py samples.txt 'Plane::flush()' [top] [remap_from=remap_to]
"""
from __future__ import annotations

import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sampler_report import load, resolve  # noqa: E402


def main(path, target, top=25, remap=None):
    samples, maps = load(path)
    if remap:
        a, b = remap.split("=")
        maps = [(lo, hi, off, p.replace(a, b)) for lo, hi, off, p in maps]
    addrs = {x for s in samples for x in s if x}
    sym = resolve(addrs, maps)
    kids = collections.Counter()
    total = 0
    for s in samples:
        names = [sym[x] for x in s if x]
        for i, nm in enumerate(names):
            if target in nm:
                total += 1
                kids[names[i - 1] if i > 0 else "(self)"] += 1
                break
    print(f"{target}: {total} samples ({100 * total / max(1, len(samples)):.1f}% of {len(samples)})")
    for k, v in kids.most_common(top):
        print(f"{100 * v / max(1, total):6.1f}%  {k[:150]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25,
         sys.argv[4] if len(sys.argv) > 4 else None)

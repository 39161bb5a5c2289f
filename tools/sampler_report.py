"""Symbolise a tools/native/sampler.c dump: self and inclusive sample shares
per function (addr2line on the mapped ELF files).

    python tools/sampler_report.py /tmp/samples.txt [top] [callers-of-symbol]
"""
from __future__ import annotations

import collections
import subprocess
import sys


def load(path):
    lines = open(path).read().splitlines()
    n = int(lines[0].split()[1])
    samples = [[int(x, 16) for x in ln.split()] for ln in lines[1:1 + n]]
    maps = []
    for ln in lines[2 + n:]:
        parts = ln.split()
        if len(parts) < 6 or not parts[5].startswith("/"):
            continue
        lo, hi = (int(x, 16) for x in parts[0].split("-"))
        maps.append((lo, hi, int(parts[2], 16), parts[5]))
    return samples, maps


def resolve(addrs, maps):
    by_file = collections.defaultdict(set)
    where = {}
    for a in addrs:
        for lo, hi, off, path in maps:
            if lo <= a < hi:
                # file offset -> vaddr: PIE/.so segments map at (lo - off)
                rel = a - lo + off
                where[a] = (path, rel)
                by_file[path].add(rel)
                break
    names = {}
    for path, rels in by_file.items():
        rels = sorted(rels)
        try:
            out = subprocess.run(["addr2line", "-f", "-C", "-e", path] + [hex(r) for r in rels],
                                 capture_output=True, text=True, timeout=600).stdout.splitlines()
        except Exception:
            out = []
        for i, r in enumerate(rels):
            fn = out[2 * i] if 2 * i < len(out) else "?"
            if fn == "??":
                fn = "?"
            names[(path, r)] = f"{fn} [{path.rsplit('/', 1)[-1]}]"
    return {a: names.get(where[a], "?") if a in where else "?" for a in addrs}


def callers(samples, sym, target, top):
    """Which libsppipe frames sit above `target` (first non-libc/libstdc++ frame)."""
    c = collections.Counter()
    for s in samples:
        names = [sym[a] for a in s if a]
        for i, nm in enumerate(names):
            if target in nm:
                for up in names[i + 1:]:
                    if "libsppipe" in up or "libspgcm" in up:
                        c[up] += 1
                        break
                break
    print(f"--- callers of {target}")
    for k, v in c.most_common(top):
        print(f"{v:6d}  {k[:160]}")


def main(path, top=40, target=None):
    samples, maps = load(path)
    addrs = {a for s in samples for a in s if a}
    sym = resolve(addrs, maps)
    if target:
        callers(samples, sym, target, top)
        return
    self_c = collections.Counter(sym[s[0]] for s in samples if s[0])
    incl = collections.Counter()
    for s in samples:
        seen = set()
        for a in s:
            if a and sym[a] not in seen:
                seen.add(sym[a])
                incl[sym[a]] += 1
    n = len(samples)
    print(f"{n} samples")
    print("--- self")
    for k, v in self_c.most_common(top):
        print(f"{100 * v / n:6.2f}%  {k[:160]}")
    print("--- inclusive")
    for k, v in incl.most_common(top):
        print(f"{100 * v / n:6.2f}%  {k[:160]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else None)

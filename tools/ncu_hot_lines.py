#!/usr/bin/env python3
"""Hottest SASS lines (warp-stall samples) of a `--set full --import-source on`
capture, each with its CUDA source line: tools/ncu_hot_lines.py REPORT [kernel-regex] [N]."""
import csv
import subprocess
import sys


def main(path, kregex=None, top=40):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kregex:
        cmd += ["-k", f"regex:{kregex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader([l for l in out.splitlines() if l.startswith('"')]))
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr = rows[hi]
    src = hdr.index("Source")
    samp = next(i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All"))
    ex = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
    cuda_line = ""
    recs = []
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= samp:
            continue
        s = r[src].strip()
        try:
            v = float(r[samp] or 0)
        except ValueError:
            v = 0.0
        if not s.startswith(("/*", "@")) and not s[:1].isupper():
            cuda_line = s[:90]
            continue
        total += v
        recs.append((v, s[:70], cuda_line, r[ex] if ex is not None else ""))
    recs.sort(key=lambda x: -x[0])
    print(f"{path}: {total:.0f} samples")
    for v, s, c, e in recs[:top]:
        print(f"{v / max(total, 1):6.3f}  {s:70s} exec={e:>10s}  | {c}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, int(sys.argv[3]) if len(sys.argv) > 3 else 40)

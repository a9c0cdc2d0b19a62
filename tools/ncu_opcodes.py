#!/usr/bin/env python3
"""PC-sampling stall attribution by SASS opcode from an .ncu-rep (source page).

tools/ncu_opcodes.py REPORT [kernel-regex]  -- needs a `--set full` capture
(SourceCounters section).  Sums the warp-stall samples of every SASS line per
opcode (predicate and modifiers stripped) and prints the top opcodes with
their dominant stall reasons.
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def main(path, kregex=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
    if kregex:
        cmd += ["-k", f"regex:{kregex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr_i = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr = rows[hdr_i]
    src = hdr.index("Source")
    cols = [i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All")]
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") or h.startswith("Stall ")]
    tot = defaultdict(float)
    per = defaultdict(lambda: defaultdict(float))
    count = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= src or r[src] == "Source":
            continue
        s = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip())
        op = s.split(" ")[0].split(".")[0] if s else "?"
        if not op or not op[0].isalpha():
            continue
        count[op] += 1
        for c in cols:
            try:
                tot[op] += float(r[c] or 0)
            except ValueError:
                pass
        for c in reasons:
            try:
                per[op][hdr[c]] += float(r[c] or 0)
            except ValueError:
                pass
    total = sum(tot.values()) or 1.0
    print(f"PC-sampling stall attribution by SASS opcode: {path}  (total samples {total:.0f})")
    for op, v in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
        top = sorted(per[op].items(), key=lambda kv: -kv[1])[:4]
        rs = " ".join(f"{k}={x:.0f}" for k, x in top if x > 0)
        print(f"  {op:8s} lines={count[op]:4d} samples={v:7.0f} ({100 * v / total:5.1f}%)  {rs}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)

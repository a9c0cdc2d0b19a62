#!/usr/bin/env python3
"""Dynamic SASS opcode histogram (warp-level instructions executed per
output element) from an `ncu --page source --csv --print-source sass` dump.
tools/ncu_dyn_hist.py SRC.csv N_ELEMENTS"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
n = float(sys.argv[2])
hdr = rows[1]
si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
c = Counter()
for r in rows[2:]:
    s = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip())
    op = s.split(" ")[0]
    op = ".".join(op.split(".")[:2]) if op.startswith(("IMAD", "ISETP")) else op.split(".")[0]
    c[op] += float(r[ei] or 0)
tot = sum(c.values())
print(f"{sys.argv[1]}: {tot * 32 / n:.2f} thread-instructions per element")
for op, v in c.most_common(25):
    print(f"  {op:16s} {v * 32 / n:6.2f}")

#!/usr/bin/env python3
"""Per-source-line stall samples and executed instructions of one kernel:
joins an `ncu --page source --csv --print-source sass` dump (gzip ok) with
`nvdisasm -g -c` line info of the same cubin by instruction offset.
tools/sass_line_profile.py NCU_SASS.csv[.gz] NVDISASM.txt KERNEL_SUBSTRING [TOP]"""
import csv
import gzip
import re
import sys
from collections import defaultdict


def main(csv_path, dis_path, kname, top=40):
    op = gzip.open if csv_path.endswith(".gz") else open
    rows = list(csv.reader(op(csv_path, "rt")))
    hdr = rows[1]
    ai, si = hdr.index("Address"), hdr.index("Source")
    sa, ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    recs = [(int(r[ai], 16), float(r[sa] or 0), float(r[ex] or 0)) for r in rows[2:] if len(r) > ex]
    base = recs[0][0]
    lines, cur, infn = {}, None, False
    for ln in open(dis_path):
        if ln.startswith("//---") and ".text." in ln:
            infn = kname in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            lines[int(m.group(1), 16)] = cur
    agg_s, agg_e = defaultdict(float), defaultdict(float)
    for a, s, e in recs:
        key = lines.get(a - base)
        agg_s[key] += s
        agg_e[key] += e
    ts, te = sum(agg_s.values()), sum(agg_e.values())
    src = {}
    for k in agg_s:
        if k and k[0].endswith(".cu"):
            try:
                src[k] = open(f"paper_2109_01329_b200/csrc/{k[0]}").read().splitlines()[k[1] - 1].strip()[:80]
            except (OSError, IndexError):
                src[k] = ""
    print(f"{len(recs)} instructions, {ts:.0f} samples, {te:.0f} executed")
    for k in sorted(agg_s, key=lambda k: -agg_s[k])[:top]:
        print(f"{agg_s[k] / ts:6.3f} samp {agg_e[k] / te:6.3f} exec  {k}  {src.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)

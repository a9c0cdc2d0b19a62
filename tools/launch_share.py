#!/usr/bin/env python3
"""Per-kernel share of an ncu `--metrics gpu__time_duration.sum --csv` launch list:
tools/launch_share.py LAUNCHES.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    tot, cnt = defaultdict(float), defaultdict(int)
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"][:90]
                tot[k] += float(d["Metric Value"].replace(",", ""))
                cnt[k] += 1
    T = sum(tot.values()) or 1.0
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
        print(f"{v / T:6.3f} share  {cnt[k]:6d} launches  {v / cnt[k] / 1e3:10.1f} us avg  {k}")


if __name__ == "__main__":
    main(sys.argv[1])

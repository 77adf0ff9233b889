#!/usr/bin/env python
"""Per-kernel share of device time from an ncu launch list
(--metrics gpu__time_duration.sum --csv).  Usage: launch_shares.py launches.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    tot[name] += v
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.3f} {100 * v / all_ms:6.1f}%")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {all_ms:10.3f}")

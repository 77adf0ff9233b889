#!/usr/bin/env python
"""Per-phase breakdown of one kernel from an ncu source page (SASS only):
the SASS is cut at every BAR.SYNC / BAR.RED (the phase barriers of the
sweep), and each segment reports its share of warp-stall samples, executed
instructions, FP64-pipe instructions and its top stall reasons.

    ncu -i REP --page source --csv --print-source sass --launch-skip S \
        --launch-count 1 > sass.csv
    python tools/sass_phases.py sass.csv
"""
import collections
import csv
import re
import sys

FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
    segs = []
    cur = None

    def new(label):
        return {"label": label, "samples": 0, "inst": 0, "fp64": 0, "lds": 0, "sts": 0,
                "ops": collections.Counter(), "stall": collections.Counter(), "n": 0}

    cur = new("start")
    seen = set()
    for r in rows:
        if not r or not r[0].startswith("0x") or r[0] in seen:
            continue
        seen.add(r[0])
        sass = r[ix["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", sass).split(" ")[0]
        base = op.split(".")[0]
        try:
            smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            ie = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        cur["samples"] += smp
        cur["inst"] += ie
        cur["n"] += 1
        cur["ops"][base] += ie
        if base in FP64:
            cur["fp64"] += ie
        for s in stalls:
            try:
                cur["stall"][s[6:]] += int(r[ix[s]] or 0)
            except ValueError:
                pass
        if base in ("BAR", "BAR.SYNC") or op.startswith("BAR."):
            segs.append(cur)
            cur = new(f"after {op} @{r[0][-5:]}")
    segs.append(cur)
    ts = sum(s["samples"] for s in segs) or 1
    ti = sum(s["inst"] for s in segs) or 1
    tf = sum(s["fp64"] for s in segs) or 1
    print(f"{'segment':28s} {'sass':>5s} {'samp%':>6s} {'inst%':>6s} {'fp64%':>6s} "
          f"{'fp64/inst':>9s}  top stalls (share of the segment's samples)")
    for s in segs:
        if s["inst"] == 0 and s["samples"] == 0:
            continue
        top = ", ".join(f"{k} {100 * v / max(s['samples'], 1):.0f}%"
                        for k, v in s["stall"].most_common(4))
        print(f"{s['label'][:28]:28s} {s['n']:5d} {100 * s['samples'] / ts:6.1f} "
              f"{100 * s['inst'] / ti:6.1f} {100 * s['fp64'] / tf:6.1f} "
              f"{s['fp64'] / max(s['inst'], 1):9.2f}  {top}")
    tot = collections.Counter()
    for s in segs:
        tot.update(s["ops"])
    print("opcodes:", ", ".join(f"{k} {100 * v / ti:.1f}%" for k, v in tot.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1])

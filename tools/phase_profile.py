"""Attribute warp-stall samples and executed instructions of the sweep
kernel to its phases (P0..P9), by SASS address ranges.

    ncu -i REP --page source --csv --print-source cuda,sass \
        --launch-skip S --launch-count 1 > cs.csv
    python tools/phase_profile.py cs.csv
"""
import collections
import csv
import sys

# a code line that opens each phase of sweep.cuh (comment lines carry no SASS)
MARKS = [("P0 load", "qv[f] = __ldg(A.src[f] + off)"),
         ("P1 slopes", "SA[v * T + ci] = limited_slope(pv[-SS]"),
         ("P3 trace", "const bool flat = q >= nn - 2"),
         ("P4 solve", "const SmemVec ql"),
         ("P7 lagrange", "const double dxp = dx0 + dt"),
         ("P7b cslopes", "SA[v * T + ci] = limited_slope(cv[-SS]"),
         ("P8 slivers", "const double delta = CF[ci] * dt;"),
         ("P9 remap", "const double dxe = __ldg(A.dx + q);")]


def main(path):
    rows = list(csv.reader(open(path)))
    src = {}  # (file, line) -> text
    cur = None
    line_of_addr = {}
    last = None
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0].isdigit():
            last = (cur, int(r[0]))
            src[last] = r[1]
        if len(r) > 7 and r[2].startswith("0x"):
            try:
                line_of_addr[int(r[2], 16)] = (last, int(r[4]), int(r[7]), r[3])
            except ValueError:
                pass
    mark_lines = {}
    for (f, ln), text in src.items():
        if f == "sweep.cuh":
            for name, tag in MARKS:
                if tag in text:
                    mark_lines[ln] = name
    addrs = sorted(line_of_addr)
    order = sorted(mark_lines)
    # an instruction belongs to the phase of the last sweep.cuh line issued
    # before it in address order (inlined helpers inherit it)
    phase = "prologue"
    agg = collections.defaultdict(lambda: [0, 0])
    for a in addrs:
        (f, ln), smp, ie, _ = line_of_addr[a]
        if f == "sweep.cuh":
            cands = [m for m in order if m <= ln]
            phase = mark_lines[cands[-1]] if cands else "prologue"
        agg[phase][0] += smp
        agg[phase][1] += ie
    ts = sum(v[0] for v in agg.values())
    ti = sum(v[1] for v in agg.values())
    for k, v in agg.items():
        print(f"{k:14s} samples {100*v[0]/ts:5.1f}%  instructions {100*v[1]/ti:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])

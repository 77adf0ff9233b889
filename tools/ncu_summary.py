#!/usr/bin/env python
"""Summarise an ncu report (--set full) of the sweep/sources kernels:
duration, DRAM bytes, FP64 pipe utilisation, occupancy, stall mix and the
SASS opcode mix.  Usage: python tools/ncu_summary.py report.ncu-rep [--json out]"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
           "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__block_size", "launch__grid_size",
           "smsp__warps_eligible.avg.per_cycle_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "launch__shared_mem_per_block_dynamic"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                d[m] = r[hdr.index(m)]
        st = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.03:
                    st[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1]))
        out.append(d)
    return out


def opcode_mix(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                           "--print-source", "sass"))))
    mixes, cur, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = collections.Counter()
            mixes.append((r[1], cur))
            continue
        if r and r[0] == "Address":
            hdr = {n: i for i, n in enumerate(r)}
            continue
        if cur is not None and hdr and len(r) == len(hdr):
            src = r[hdr["Source"]].strip().split()
            if not src:
                continue
            op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
            cur[op.split(".")[0]] += int(r[hdr["Instructions Executed"]] or 0)
    return mixes


if __name__ == "__main__":
    rep = sys.argv[1]
    res = raw(rep)
    mixes = opcode_mix(rep)
    for i, d in enumerate(res):
        print(d["kernel"][:90])
        for k, v in d.items():
            if k not in ("kernel", "stalls_per_issue"):
                print(f"   {k:62s} {v}")
        print("   stalls/issue:", {k: round(v, 2) for k, v in d["stalls_per_issue"].items()})
        if i < len(mixes):
            tot = sum(mixes[i][1].values()) or 1
            top = mixes[i][1].most_common(14)
            d["opcode_mix_pct"] = {k: round(100.0 * v / tot, 1) for k, v in top}
            print("   opcodes %:", d["opcode_mix_pct"])
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

#!/usr/bin/env python
"""Benchmark: MHD cell-updates/s of the PPMLR time step on B200.

One "step" is one Harness::advance (CFL dt, the three directional PPMLR
sweeps in XYZ/ZYX order, dipole sources, frozen core) over the whole
synthetic grid.  Default workload: C4 of BASELINE.json, the
weak-scaling blast wave, 512^3 cells per GPU (x-slab per rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config blast512]
                  [--precision strict|fast] [--impl ours|reference]

For N>1 launch one rank per GPU with torch.distributed.run (NCCL); the
halo exchange and the dt min-reduction go through torch.distributed.

Prints ONE JSON line (rank 0).  value = whole-job cell-updates/s timed with
CUDA events on the block's stream (max over ranks); e2e = the same metric
through the public API with host buffers (initial state uploaded from pinned
host memory, dt read back every step, final interior downloaded), timed by
wall clock around synchronised regions.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MHD cell-updates/sec (3 sweeps) at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "cell-updates/s"
HBM_FALLBACK_GBS = 6650.0
# Algorithmic work per cell-update.
ALG = {
    "blast": dict(F=2500.0, B=512.0, F_sweep=(2500.0 - 279.0 - 78.0) / 3.0, B_sweep=128.0),
    "orszag_tang": dict(F=3330.0, B=512.0, F_sweep=1163.0, B_sweep=128.0),
    "magnetosphere": dict(F=3910.0, B=608.0, F_sweep=1163.0, B_sweep=152.0),
    "briowu": dict(F=2500.0, B=512.0, F_sweep=714.0, B_sweep=128.0),
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def workload(name, gpus):
    """(physics kind, config dict) of a bench workload, computed here without
    importing the product package, so that the reference arm (which must not
    load the product's native library) prints the same `config` as ours."""
    g = max(int(gpus), 1)
    if name.startswith("blast"):
        n = 512 if name == "blast512" else int(name[5:])
        kind, wl, grid = "blast", f"blast_{n}^3x{g}", [n * g, n, n]
    elif name == "ot512":
        kind, wl, grid = "orszag_tang", "orszag_tang", [512, 512, 4]
    elif name == "mag160":
        kind, wl, grid = "magnetosphere", "magnetosphere_160x150x150", [160, 150, 150]
    elif name == "mag1024":
        kind, wl, grid = "magnetosphere", "magnetosphere_1024x768x768", [1024, 768, 768]
    elif name == "briowu":
        kind, wl, grid = "briowu", "briowu", [256, 4, 4]
    else:
        raise SystemExit(f"unknown config {name}")
    cells = grid[0] * grid[1] * grid[2]
    return kind, {"workload": wl, "grid": grid, "cells_per_gpu": cells // g,
                  "partition": f"x-slab ({g},1,1)",
                  "l2": "inputs (2 state buffers of 8 FP64 planes) >> 126 MB L2 at the "
                        "headline sizes; no flush needed" if cells >= 1 << 24 else
                        "state fits L2 partly: correctness config, not a headline"}


def make_config(name, gpus):
    from paper_1607_02214_b200 import configs
    if name == "blast512":
        return configs.blast(n=512, gpus=gpus), "blast"
    if name.startswith("blast"):
        return configs.blast(n=int(name[5:]), gpus=gpus), "blast"
    if name == "ot512":
        return configs.orszag_tang(n=512), "orszag_tang"
    if name == "mag160":
        return configs.magnetosphere(), "magnetosphere"
    if name == "mag1024":
        return configs.magnetosphere(nx=1024, nyz=768, d=0.05, partition=(gpus, 1, 1)), \
            "magnetosphere"
    if name == "briowu":
        return configs.brio_wu(), "briowu"
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.dev = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # nvidia-smi can take longer to start than a short timed region lasts
        # (C3: 10 steps = 18 ms): wait for its first row so the region is
        # always bracketed by samples
        t0 = time.time()
        while self.proc and self._rows() < 1 and time.time() - t0 < 5.0:
            time.sleep(0.05)
        self.n0 = self._rows()
        return self

    def _rows(self):
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except Exception:
            return 0

    def __exit__(self, *exc):
        t0 = time.time()
        while self.proc and self._rows() <= self.n0 and time.time() - t0 < 0.5:
            time.sleep(0.02)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for ln in open(self.path):
                p = [x.strip() for x in ln.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        under = sorted(sm)[len(sm) // 4:] or sm  # drop the idle head of the samples
        return {"sm_mhz": float(np.median(under)) if under else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def fp64_peak_tflops(device=0):
    import ctypes
    from paper_1607_02214_b200 import _native as N
    out = ctypes.c_double()
    N.check(N.lib.ppmlr_gpu_fp64_peak(device, ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------ CPU baseline

def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# The bounded CPU sample of each workload: (specs, harness kwargs, ic, steps
# per thread, whether the rate is extrapolated to the workload's size).  The
# step count is FIXED per workload, so every CPU leg (our line's
# cpu_baseline and the --impl reference arm) times the same sample.
def _cpu_sample(name):
    if name.startswith("blast"):
        n = 64
        return ([(-0.5, 0.5, -0.5, 0.5, 1.0 / n, n, 1.05)] * 3, dict(boundary=0),
                (3, (10.0, 0.1, 0.1)), 24,
                "64^3 blast unit block (the C4 IC/physics at 1/512 of the cells)", True)
    if name in ("mag160", "mag1024"):
        return ([(-100.0, 30.0, -10.0, 10.0, 0.4, 160, 1.05),
                 (-100.0, 100.0, -10.0, 10.0, 0.4, 150, 1.05),
                 (-100.0, 100.0, -10.0, 10.0, 0.4, 150, 1.05)],
                dict(boundary=2, with_dipole=True), (-1, ()), 1,
                "C3 160x150x150 magnetosphere (stretched grid, dipole, frozen core)",
                name == "mag1024")
    if name == "ot512":
        tp = 2.0 * np.pi
        return ([(0.0, tp, 0.0, tp, tp / 512, 512, 1.05)] * 2
                + [(0.0, tp * 4 / 512, 0.0, tp * 4 / 512, tp / 512, 4, 1.05)],
                dict(boundary=1), (2, (5.0 / 3.0,)), 2, "C2 Orszag-Tang 512x512x4", False)
    if name == "briowu":
        d = 1.0 / 256
        return ([(0.0, 1.0, 0.0, 1.0, d, 256, 1.05), (0.0, 4 * d, 0.0, 4 * d, d, 4, 1.05),
                 (0.0, 4 * d, 0.0, 4 * d, d, 4, 1.05)],
                dict(boundary=0, gamma=2.0), (1, ()), 200, "C1 Brio-Wu 256x4x4", False)
    raise SystemExit(f"unknown config {name}")


def cpu_baseline(name, threads=None):
    """The reference's own CPU implementation (oracle/_ref, built from the
    unmodified sources) on a bounded sample of workload `name`, one
    independent harness per host thread, a fixed number of steps each (one
    untimed step first).  Falls back to the C restatement ("port") when the
    reference build is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    threads = threads or os.cpu_count() or 1
    specs, kw, ic, steps, sample, extrapolated = _cpu_sample(name)
    if not po.have_ref():
        return cpu_baseline_port(name, threads)
    po.ref_bench(specs, ic[0], ic[1], 1, 1, **kw)  # warm-up (page-in, caches)
    r1, s1 = po.ref_bench(specs, ic[0], ic[1], 1, 1, **kw)
    rate, secs = po.ref_bench(specs, ic[0], ic[1], threads, steps, **kw)
    how = ("per-cell rate EXTRAPOLATED to the workload's size (the reference is serial "
           "per block; cell-updates/s of the sample)" if extrapolated else
           "the workload itself, fewer steps")
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "extrapolated": extrapolated,
            "sample": f"{sample}: one independent harness per thread, {steps} steps x "
                      f"{threads} threads in {secs:.1f} s; {how} (oracle/_ref: unmodified "
                      f"reference sources, g++ -O3)",
            "single_core": {"value": r1, "unit": UNIT, "sample": "1 step, 1 thread"},
            "cpu_model": _cpu_model()}


def cpu_baseline_port(name, threads, seconds_target=10.0):
    """Fallback without oracle/_ref: the C restatement on a 48^3 blast.  (It
    takes the IC from the product's host planning; never used when the
    reference build exists, as it does on the GPU box.)"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_1607_02214_b200 import configs, host_block_state
    cfg = configs.blast(n=48)
    st = host_block_state(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic)
    o = po.opts()
    c = po.consts()
    cells = 48 ** 3

    def one(k, out):
        blk = po.OracleBlock([48] * 3, 4, st["centers"], st["spacings"], [[1, 1]] * 3,
                             st["fields"].copy())
        t0 = time.perf_counter()
        for s in range(k):
            blk.advance(o, c, s)
        out.append(time.perf_counter() - t0)

    tmp = []
    one(1, tmp)
    steps = max(1, int(seconds_target / max(tmp[0], 1e-3) / 2))
    res = []
    ths = [threading.Thread(target=one, args=(steps, res)) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    secs = max(res)
    return {"value": cells * steps * threads / secs, "unit": UNIT, "cores": threads,
            "kind": "port", "sample": f"48^3 blast, {steps} steps x {threads} threads "
                                      "(C restatement oracle/ppmlr_oracle.c)"}


# ------------------------------------------------------------ our arm

def bench_single(args):
    import torch
    import paper_1607_02214_b200 as P
    cfg, kind = make_config(args.config, 1)
    _, wl_cfg = workload(args.config, 1)
    assert wl_cfg["workload"] == cfg.name and wl_cfg["cells_per_gpu"] == cfg.cells, wl_cfg
    cfg.options.precision = args.precision
    alg = ALG[kind]
    cells = cfg.cells
    torch.cuda.init()
    peak_fp64 = fp64_peak_tflops(0)
    hbm, hbm_src = measured_peaks()

    h = P.Harness(cfg.specs, cfg.partition, cfg.options)
    if cfg.ic[0] == "magnetosphere":
        h.init_magnetosphere()
    else:
        h.init_with(*cfg.ic)
    blk = h.block(0)
    stream = torch.cuda.ExternalStream(blk.stream())
    h.run(args.warmup)
    blk.synchronize()

    # ---- timed region: K steps, per-sweep CUDA events inside the library
    blk.timing(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        h.run(args.steps)
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    sweep_ms, kernels, sweep_launches = blk.timing(False)
    value = cells * args.steps / (ms * 1e-3)

    # ---- dominant kernel roofline (the directional sweep)
    avg_sweep_s = sweep_ms * 1e-3 / max(sweep_launches, 1)
    sweep_bytes = cells * alg["B_sweep"]
    sweep_flops = cells * alg["F_sweep"]
    frac_hbm = (sweep_bytes / avg_sweep_s) / (hbm * 1e9)
    frac_fp64 = (sweep_flops / avg_sweep_s) / (peak_fp64 * 1e12)
    bound = "fp64" if frac_fp64 >= frac_hbm else "hbm"
    traffic = None  # dram__bytes_read+write per sweep launch, from an ncu --set full capture
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    if os.path.exists(prof):
        try:
            rec = json.load(open(prof)).get(kind, {})
            if "bytes_per_cell" in rec:
                traffic = rec["bytes_per_cell"] * cells
        except Exception:
            traffic = None
    roofline = {
        "bound": bound,
        "achieved": (sweep_flops / avg_sweep_s / 1e12) if bound == "fp64"
        else (sweep_bytes / avg_sweep_s / 1e9),
        "peak": peak_fp64 if bound == "fp64" else hbm,
        "unit": "TFLOP/s" if bound == "fp64" else "GB/s",
        "frac": frac_fp64 if bound == "fp64" else frac_hbm,
        "traffic": traffic,
        "kernel": "sweep_kernel (x/y/z)",
        "per_launch": {"cells": cells, "alg_bytes": sweep_bytes, "alg_flops": sweep_flops,
                       "avg_ms": avg_sweep_s * 1e3, "launches": sweep_launches},
        "frac_hbm": frac_hbm, "frac_fp64": frac_fp64,
        "peak_fp64_tflops_measured": peak_fp64, "peak_hbm_gbs": hbm,
        "peak_hbm_source": hbm_src,
        "sweep_share_of_step": sweep_ms / ms,
        # whole step against BASELINE.md §3's roofline formula
        "step_frac": value / min(hbm * 1e9 / alg["B"], peak_fp64 * 1e12 / alg["F"]),
    }

    # ---- end to end through the public API with host buffers
    e2e = bench_e2e(h, cfg, args, cells) if not args.no_e2e else None
    h.close()
    del h

    # ---- the other precision mode on the same workload (timing only)
    other = None
    if not args.no_secondary:
        prec2 = "strict" if args.precision == "fast" else "fast"
        cfg2, _ = make_config(args.config, 1)
        cfg2.options.precision = prec2
        h2 = P.Harness(cfg2.specs, cfg2.partition, cfg2.options)
        if cfg2.ic[0] == "magnetosphere":
            h2.init_magnetosphere()
        else:
            h2.init_with(*cfg2.ic)
        st2 = torch.cuda.ExternalStream(h2.block(0).stream())
        h2.run(args.warmup)
        h2.block(0).synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(st2)
        h2.run(args.steps)
        f1.record(st2)
        f1.synchronize()
        ms2 = f0.elapsed_time(f1)
        other = {"precision": prec2, "value": cells * args.steps / (ms2 * 1e-3),
                 "ms_per_step": ms2 / args.steps,
                 "note": "strict = bit-identical to the reference CPU build; fast = "
                         "reciprocal-multiply divisions + FMA, rel. L1 <= 1e-11 / Linf <= 1e-9"}
        h2.close()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "precision": args.precision,
        "data": "synthetic (deterministic IC, no RNG)",
        "config": wl_cfg,
        "clocks": clk.summary(), "e2e": e2e, "gpu_launches": int(kernels),
        "roofline": roofline, "other_precision": other,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)


def bench_e2e(h, cfg, args, cells):
    """K x Harness.advance() (dt read back each step) bracketed by the upload
    of the initial state from pinned host memory and the download of the
    final interior into pinned host memory."""
    import torch
    import paper_1607_02214_b200 as P
    # the initial state (and the dipole, which travels with it) evaluated
    # straight into pinned host buffers: no second host copy (C5 is 39 GB)
    g = cfg.options.ghost
    nx, ny, nz = (int(s.cells) for s in cfg.specs)
    shape = (nz + 2 * g, ny + 2 * g, nx + 2 * g)
    host_in = torch.empty(shape + (8,), dtype=torch.float64, pin_memory=True).numpy()
    host_bd = None
    if cfg.options.with_dipole:
        host_bd = torch.empty(shape + (3,), dtype=torch.float64, pin_memory=True).numpy()
    st = P.host_block_state(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic, fields_out=host_in,
                            bd_out=host_bd)
    host_out = torch.empty((nz, ny, nx, 8), dtype=torch.float64, pin_memory=True).numpy()
    blk = h.block(0)
    k = args.steps
    # one untimed pass through the same calls (first-touch costs of the
    # transfer paths), then the timed one
    blk.upload(host_in, host_bd, st["frozen_idx"], st["frozen_states"])
    h.advance()
    blk.download_interior(out=host_out)
    torch.cuda.synchronize()
    # wall clock is exposed to host jitter (a 45 ms C3 pass moved by 20 ms
    # between runs): passes shorter than 1 s are repeated, up to 10 or 2 s
    # in all, and the best is kept
    best, spent = None, 0.0
    for n in range(10):
        t0 = time.perf_counter()
        blk.upload(host_in, host_bd, st["frozen_idx"], st["frozen_states"])
        for _ in range(k):
            h.advance()
        blk.download_interior(out=host_out)
        t1 = time.perf_counter()
        best = t1 - t0 if best is None else min(best, t1 - t0)
        spent += t1 - t0
        if t1 - t0 >= 1.0 or (n >= 2 and spent >= 2.0):
            break
    h2d = host_in.nbytes + (host_bd.nbytes if host_bd is not None else 0)
    d2h = host_out.nbytes + 8 * k
    return {"value": cells * k / best, "unit": UNIT,
            "h2d_bytes_per_step": h2d / k, "d2h_bytes_per_step": d2h / k,
            "how": f"upload(pinned) + {k} x advance() + download_interior(pinned), wall "
                   "clock, after one untimed pass; passes under 1 s repeated (up to 10, "
                   "2 s in all) and the best kept"}


def bench_reference(args):
    """The reference arm: the reference's own CPU implementation
    (oracle/_ref, the unmodified sources) on the host cores, timed on the
    same fixed sample as our line's cpu_baseline.  It never imports the
    product package (no product native library is loaded here)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _, wl_cfg = workload(args.config, args.gpus)
    cb = cpu_baseline(args.config)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic IC, no RNG)", "config": wl_cfg,
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="blast512")
    ap.add_argument("--precision", default="fast", choices=["strict", "fast"])
    ap.add_argument("--force-dist", action="store_true",
                    help="run the torch.distributed (NCCL) driver even on one rank")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the timing of the other precision mode")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return bench_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.force_dist:
        from paper_1607_02214_b200 import dist
        return dist.bench_distributed(args, METRIC, UNIT, ALG, make_config, ClockSampler,
                                      fp64_peak_tflops, measured_peaks, cpu_baseline,
                                      workload)
    return bench_single(args)


if __name__ == "__main__":
    main()

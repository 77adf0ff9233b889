"""Golden digests of the BASELINE.json configurations, from the REFERENCE.

Runs the unmodified reference (oracle/_ref/libppmlr_ref.so, built by
oracle/Makefile from /root/reference) on the benchmark configurations at
their stated step counts and stores, per run: every step's dt, the simulated
time, the sha256 of the final interior (z, y, x, 8 float64, the layout of
``Harness.gather_interior``) and its per-field L1 sums.  The GPU strict build
must reproduce each sha (tests/test_gpu_baseline.py); the fast build is then
checked against the strict one on the device at the same size.

    python tests/golden/make_golden_baseline.py [name ...]   # -> baseline_runs.json

Runs in parallel, one process per case (the reference is single-threaded):
C2 (512x512x4, 100 steps) is ~7 CPU-minutes, C3 (160x150x150, 30 steps) ~5.

Cases (BASELINE.json configs; /root/reference/proj/src/
harness.cpp:59-92 is the stepped function):
  c1_briowu_256x4x4_220      C1 Brio-Wu shock tube, gamma = 2, outflow
  c2_orszag_tang_512x512x4_100  C2 Orszag-Tang vortex, periodic
  c3_magnetosphere_160x150x150_30  C3 dipole magnetosphere, stretched grid
  blast_64_10, blast_128_6   C4 physics on grids whose every axis takes the
                             compile-time sweep tile (n % 64 == 0)
  dipole_64_6                C5 physics (dipole, frozen core, magnetosphere
                             boundary) with y and z multiples of 64
"""
from __future__ import annotations

import hashlib
import json
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
OUT = os.path.join(HERE, "baseline_runs.json")


def _uni(lo, hi, n):
    return (lo, hi, lo, hi, (hi - lo) / n, n, 1.05)


def _tp(n):
    return 2.0 * math.pi * n / 512


# name: (specs, harness kwargs, ic, steps); ic = ("mag",) or (kind, params)
CASES = {
    "c1_briowu_256x4x4_220": (
        [(0.0, 1.0, 0.0, 1.0, 1 / 256, 256, 1.05),
         (0.0, 4 / 256, 0.0, 4 / 256, 1 / 256, 4, 1.05),
         (0.0, 4 / 256, 0.0, 4 / 256, 1 / 256, 4, 1.05)],
        dict(gamma=2.0, boundary=0), (1, ()), 220),
    "c2_orszag_tang_512x512x4_100": (
        [_uni(0.0, 2 * math.pi, 512), _uni(0.0, 2 * math.pi, 512),
         (0.0, _tp(4), 0.0, _tp(4), 2 * math.pi / 512, 4, 1.05)],
        dict(boundary=1), (2, (5.0 / 3.0,)), 100),
    "c3_magnetosphere_160x150x150_30": (
        [(-100.0, 30.0, -10.0, 10.0, 0.4, 160, 1.05),
         (-100.0, 100.0, -10.0, 10.0, 0.4, 150, 1.05),
         (-100.0, 100.0, -10.0, 10.0, 0.4, 150, 1.05)],
        dict(boundary=2, with_dipole=True), ("mag",), 30),
    "blast_64_10": ([_uni(-0.5, 0.5, 64)] * 3, dict(boundary=0), (3, (10.0, 0.1, 0.1)), 10),
    "blast_128_6": ([_uni(-0.5, 0.5, 128)] * 3, dict(boundary=0), (3, (10.0, 0.1, 0.1)), 6),
    "dipole_64_6": (
        [(-48.0, 28.8, -48.0, 28.8, 1.2, 64, 1.05),
         (-38.4, 38.4, -38.4, 38.4, 1.2, 64, 1.05),
         (-38.4, 38.4, -38.4, 38.4, 1.2, 64, 1.05)],
        dict(boundary=2, with_dipole=True), ("mag",), 6),
}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def run_case(name):
    import pyoracle as po
    specs, kw, ic, steps = CASES[name]
    t0 = time.time()
    h = po.RefHarness(specs, (1, 1, 1), **kw)
    if ic[0] == "mag":
        h.init_magnetosphere()
    else:
        h.init_ic(*ic)
    dts = [h.advance() for _ in range(steps)]
    fin = h.gather()
    return name, {
        "specs": [list(s) for s in specs], "options": kw,
        "ic": list(ic[:1]) + ([list(ic[1])] if len(ic) > 1 else []),
        "steps": steps, "dts": [float(d).hex() for d in dts], "time": float(h.time()).hex(),
        "final_sha": digest(fin), "final_l1": np.abs(fin).sum(axis=(0, 1, 2)).tolist(),
        "cpu_seconds": round(time.time() - t0, 1)}


def main(names):
    import pyoracle as po
    if not po.have_ref():
        raise SystemExit("oracle/_ref/libppmlr_ref.so missing: make -C oracle")
    old = json.load(open(OUT)) if os.path.exists(OUT) else {}
    with mp.get_context("spawn").Pool(min(len(names), os.cpu_count() or 1)) as pool:
        for name, rec in pool.imap_unordered(run_case, names):
            old[name] = rec
            print(name, rec["final_sha"][:16], rec["cpu_seconds"], "s", flush=True)
            with open(OUT, "w") as f:
                json.dump(old, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))

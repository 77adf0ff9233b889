"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference sources (compiled by oracle/Makefile into
oracle/_ref/libppmlr_ref.so; needs /root/reference at build time) and stores
small known-answer fixtures:

* axes.npz      build_axis edges for the benchmark/default axis specs
* layouts.json  layout() of the reference partition shapes + error texts
* strips.npz    sweep_1d on seeded random strips (dir 0/1/2, bd on/off),
                inputs and outputs, plus strips that must throw
* runs.npz      whole Harness runs on small grids of every benchmark
                physics (Brio-Wu, Orszag-Tang, magnetosphere w/ dipole +
                frozen core, blast, partition_ic): initial ghost-inclusive
                state, geometry, bd, frozen list, per-step dt, final interior

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import pyoracle as po  # noqa: E402


def uni(lo, hi, n):
    return (lo, hi, lo, hi, (hi - lo) / n, n, 1.05)


from tests_golden_specs import AXES, BAD_AXES  # noqa: E402


def gen_axes():
    out = {}
    for k, s in AXES.items():
        e, c, sp = po.ref_build_axis(s)
        out[k + "/spec"] = np.array(s, dtype=np.float64)
        out[k + "/edges"] = e
        out[k + "/centers"] = c
        out[k + "/spacings"] = sp
    errs = {}
    for k, s in BAD_AXES.items():
        try:
            po.ref_build_axis(s)
            errs[k] = None
        except po.OracleError as ex:
            errs[k] = [ex.kind, ex.msg]
    np.savez_compressed(os.path.join(HERE, "axes.npz"), **out)
    return errs


def gen_layouts(axis_errors):
    default = [AXES["default_x"], AXES["default_yz"], AXES["default_yz"]]
    c3 = [AXES["c3_x"], AXES["default_yz"], AXES["default_yz"]]
    c5 = [AXES["c5_x"], AXES["c5_yz"], AXES["c5_yz"]]
    parts = {"default": (default, [(1, 1, 1), (3, 1, 1), (3, 3, 3), (4, 3, 3), (6, 3, 3),
                                   (4, 5, 5), (6, 5, 5), (2, 1, 1), (8, 1, 1), (2, 3, 3),
                                   (1, 2, 1), (5, 1, 1), (0, 1, 1)]),
             "c3": (c3, [(1, 1, 1), (2, 1, 1), (4, 1, 1), (8, 1, 1), (8, 3, 3)]),
             "c5": (c5, [(2, 1, 1), (4, 1, 1), (8, 1, 1)])}
    res = {"axis_errors": axis_errors, "layouts": []}
    for gname, (specs, plist) in parts.items():
        for p in plist:
            entry = {"grid": gname, "partition": list(p)}
            try:
                blocks, iono = po.ref_layout(specs, *p)
                entry["blocks"] = blocks.tolist()
                entry["ionosphere_rank"] = iono
            except po.OracleError as ex:
                entry["error"] = [ex.kind, ex.msg]
            res["layouts"].append(entry)
    with open(os.path.join(HERE, "layouts.json"), "w") as f:
        json.dump(res, f, indent=1)


def gen_strips():
    rng = np.random.default_rng(20161018)
    c = po.consts()
    out = {}
    k = 0
    for case in range(18):
        n = [8, 16, 33, 5, 1, 40][case % 6]
        g = 4
        nn = n + 2 * g
        st = np.zeros((nn, 8))
        st[:, 0] = rng.uniform(0.5, 2, nn)
        st[:, 7] = rng.uniform(0.5, 2, nn)
        st[:, 1:4] = rng.uniform(-0.5, 0.5, (nn, 3))
        st[:, 4:7] = rng.uniform(-1, 1, (nn, 3))
        if case % 5 == 0:  # quiescent stretch: u* = 0 at some edges
            st[: nn // 2, 1:4] = 0.0
            st[: nn // 2, 4:8] = st[0, 4:8]
            st[: nn // 2, 0] = st[0, 0]
        bd = rng.uniform(-1, 1, (nn, 3)) if case % 2 else None
        dx = rng.uniform(0.5, 1.5, nn) if case % 3 else np.full(nn, 0.25)
        d = case % 3
        dt = 0.4 * po.orc_strip_max_dt(st, bd, dx, n, g, d, c)
        res = st.copy()
        po.ref_sweep_1d(res, bd, dx, n, g, dt, d)
        pre = f"s{k}/"
        out[pre + "in"] = st
        out[pre + "out"] = res
        out[pre + "bd"] = bd if bd is not None else np.zeros(0)
        out[pre + "dx"] = dx
        out[pre + "meta"] = np.array([n, g, d, dt])
        k += 1
    out["count"] = np.array(k)
    # failing strips: crossing interfaces, negative density
    errs = []
    nn = 24
    st = np.zeros((nn, 8))
    st[:, 0] = 1.0
    st[:, 7] = 0.01
    st[:, 1] = np.where(np.arange(nn) < nn // 2, 5.0, -5.0)
    dx = np.full(nn, 0.1)
    for d in range(3):
        s2 = st.copy()
        if d != 0:
            s2[:, 1 + d], s2[:, 1] = st[:, 1], 0.0
        try:
            po.ref_sweep_1d(s2, None, dx, nn - 8, 4, 0.1, d)
            errs.append(None)
        except po.OracleError as ex:
            errs.append([ex.kind, ex.msg])
        out[f"e{d}/in"] = s2 if d else st
    out["errors"] = np.array(json.dumps(errs))
    np.savez_compressed(os.path.join(HERE, "strips.npz"), **out)


RUNS = {
    # name: (specs, kwargs, ic, steps, partition)
    "briowu": ([(0.0, 48 / 256, 0.0, 48 / 256, 1 / 256, 48, 1.05),
                (0.0, 4 / 256, 0.0, 4 / 256, 1 / 256, 4, 1.05),
                (0.0, 4 / 256, 0.0, 4 / 256, 1 / 256, 4, 1.05)],
               dict(gamma=2.0), (1, ()), 12, (1, 1, 1)),
    "orszag_tang": ([uni(0, 2 * math.pi, 16), uni(0, 2 * math.pi, 16),
                     (0.0, 2 * math.pi * 4 / 16, 0.0, 2 * math.pi * 4 / 16, 2 * math.pi / 16, 4,
                      1.05)],
                    dict(boundary=1), (2, (5.0 / 3.0,)), 6, (1, 1, 1)),
    "magnetosphere": ([(-12.0, 6.0, -12.0, 6.0, 1.5, 12, 1.05),
                       (-10.5, 10.5, -10.5, 10.5, 1.5, 14, 1.05),
                       (-7.5, 7.5, -7.5, 7.5, 1.5, 10, 1.05)],
                      dict(boundary=2, with_dipole=True), ("mag",), 4, (1, 1, 1)),
    "magnetosphere_stretched": ([(-100.0, 30.0, -10.0, 10.0, 5.0, 20, 1.05),
                                 (-100.0, 100.0, -10.0, 10.0, 5.0, 27, 1.05),
                                 (-100.0, 100.0, -10.0, 10.0, 5.0, 27, 1.05)],
                                dict(boundary=2, with_dipole=True, cfl=0.4), ("mag",), 3,
                                (1, 1, 1)),
    "blast": ([uni(-0.5, 0.5, 12)] * 3, dict(), (3, (10.0, 0.1, 0.25)), 5, (1, 1, 1)),
    "partition_ic": ([uni(-1.0, 1.0, 12)] * 3, dict(), (4, ()), 4, (1, 1, 1)),
}


def digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


BIG = 40_000  # doubles; larger arrays are stored as sha256 digests only


def gen_runs():
    out = {}
    for name, (specs, kw, ic, steps, part) in RUNS.items():
        h = po.RefHarness(specs, part, **kw)
        if ic[0] == "mag":
            h.init_magnetosphere()
        else:
            h.init_ic(*ic)
        pre = name + "/"
        out[pre + "specs"] = np.array(specs, dtype=np.float64)
        init = h.fields(0)
        out[pre + "init_sha"] = np.array(digest(init))
        if init.size <= BIG:
            out[pre + "init"] = init
        cen, spa = zip(*[h.axis(0, a) for a in range(3)])
        for a in range(3):
            out[pre + f"centers{a}"] = cen[a]
            out[pre + f"spacings{a}"] = spa[a]
        if kw.get("with_dipole"):
            bd = h.bd(0)
            out[pre + "bd_sha"] = np.array(digest(bd))
            if bd.size <= BIG:
                out[pre + "bd"] = bd
        fi, fs = h.frozen(0)
        out[pre + "frozen_idx"] = fi
        out[pre + "frozen_states"] = fs
        dts = [h.advance() for _ in range(steps)]
        out[pre + "dts"] = np.array(dts)
        fin = h.gather()
        out[pre + "final_sha"] = np.array(digest(fin))
        out[pre + "final_l1"] = np.abs(fin).sum(axis=(0, 1, 2))
        if fin.size <= BIG:
            out[pre + "final"] = fin
        out[pre + "time"] = np.array(h.time())
        opts = dict(cfl=0.5, boundary=0, with_sources=True, gamma=5.0 / 3.0)
        opts.update({k: v for k, v in kw.items() if k in opts})
        out[pre + "opts"] = np.array(json.dumps({**opts, "ic": list(ic[:1]) + [list(ic[1])]
                                                 if len(ic) > 1 else list(ic),
                                                 "with_dipole": bool(kw.get("with_dipole")),
                                                 "steps": steps}))
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)


if __name__ == "__main__":
    errs = gen_axes()
    gen_layouts(errs)
    gen_strips()
    gen_runs()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))

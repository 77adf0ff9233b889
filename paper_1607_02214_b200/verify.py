"""``ppmlr verify`` on the GPU path: the physics suites of the reference's
src/verify.cpp (sod, briowu, convergence, conservation, partition) with every
time step computed by the device kernels — ``strip_max_dt`` and
``sweep_strips`` for the 1-D suites (run_strip, verify.cpp:42-52), the GPU
``Harness`` for the 3-D ones.

The reference solutions the 1-D metrics are measured against are restated
here from the reference's own oracles: Toro's exact Riemann solver
(src/oracles/exact_riemann.cpp) and the first-order HLL MHD tube at 8000
cells (src/oracles/hll_mhd.cpp), in the reference's operation order.
Thresholds and metrics are the reference's.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import (IC_GAUSSIAN, IC_PARTITION, OUTFLOW, PERIODIC, AxisSpec, Harness,
                  HarnessOptions, UnphysicalState, build_axis, strip_max_dt, sweep_strips)

GHOST = 4


@dataclass
class CheckResult:
    """verify.hpp:8-13."""
    name: str
    metric: float
    threshold: float
    passed: bool


def _seqsum(a):
    """Left-to-right sum (the reference's `+=` loops)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    return float(np.add.accumulate(a)[-1]) if a.size else 0.0


# ----------------------------------------------------------- 1-D strips

def make_strip(n, dx):
    """verify.cpp:18-25: n interior cells, 4 ghosts, zero states."""
    return np.zeros((n + 2 * GHOST, 8)), np.full(n + 2 * GHOST, dx)


def _fill(states, n, periodic):
    """fill_outflow / fill_periodic (verify.cpp:27-39)."""
    g = GHOST
    for k in range(g):
        if periodic:
            states[k] = states[k + n]
            states[g + n + k] = states[g + k]
        else:
            states[k] = states[g]
            states[g + n + k] = states[g + n - 1]


class GpuStrips:
    """The 1-D engine of the suites: strip_max_dt and sweep_1d on the GPU."""

    def __init__(self, precision="strict", device=0):
        self.precision, self.device = precision, device

    def max_dt(self, states, dx, n, gamma):
        return strip_max_dt(states, None, dx, n, GHOST, 0, gamma, 1.0, self.device)

    def sweep(self, states, dx, n, dt, gamma):
        states[:] = sweep_strips(states, None, dx, n, GHOST, dt, 0, gamma, 1.0, 0.0,
                                 self.precision, self.device)[0]


def run_strip(states, dx, n, t_end, cfl, gamma, periodic, engine):
    """run_strip (verify.cpp:42-52)."""
    t = 0.0
    while t < t_end:
        _fill(states, n, periodic)
        dt = cfl * engine.max_dt(states, dx, n, gamma)
        if t + dt >= t_end:
            dt = t_end - t
        engine.sweep(states, dx, n, dt, gamma)
        t += dt
        if dt <= 0.0:
            raise UnphysicalState("verify: time step collapsed to zero")
    return states


class ExactRiemann:
    """Toro's exact Riemann solver (exact_riemann.cpp), states (rho, u, p)."""

    def __init__(self, left, right, gamma):
        self.l, self.r, self.g = left, right, gamma
        self.al = math.sqrt(gamma * left[2] / left[0])
        self.ar = math.sqrt(gamma * right[2] / right[0])
        if 2.0 * (self.al + self.ar) / (gamma - 1.0) <= right[1] - left[1]:
            raise RuntimeError("exact Riemann: vacuum is generated")
        ex = (gamma - 1.0) / (2.0 * gamma)
        p = math.pow((self.al + self.ar - 0.5 * (gamma - 1.0) * (right[1] - left[1])) /
                     (self.al / math.pow(left[2], ex) + self.ar / math.pow(right[2], ex)),
                     1.0 / ex)
        p = max(p, 1e-14)
        for _ in range(200):
            fl, dl = self._wave(p, left, self.al)
            fr, dr = self._wave(p, right, self.ar)
            f = fl + fr + (right[1] - left[1])
            nxt = p - f / (dl + dr)
            if nxt <= 0.0:
                nxt = 0.5 * p
            if abs(nxt - p) <= 1e-14 * p:
                p = nxt
                break
            p = nxt
        self.pstar = p
        self.ustar = 0.5 * (left[1] + right[1]) + 0.5 * (
            self._wave(p, right, self.ar)[0] - self._wave(p, left, self.al)[0])

    def _wave(self, p, s, a):
        g = self.g
        if p > s[2]:
            A = 2.0 / ((g + 1.0) * s[0])
            B = (g - 1.0) / (g + 1.0) * s[2]
            root = math.sqrt(A / (p + B))
            return (p - s[2]) * root, root * (1.0 - 0.5 * (p - s[2]) / (B + p))
        pr = p / s[2]
        ex = (g - 1.0) / (2.0 * g)
        d = math.pow(pr, -(g + 1.0) / (2.0 * g)) / (s[0] * a)
        return 2.0 * a / (g - 1.0) * (math.pow(pr, ex) - 1.0), d

    def sample(self, xi):
        g = self.g
        gm, gp = g - 1.0, g + 1.0
        l, r, al, ar, ps, us = self.l, self.r, self.al, self.ar, self.pstar, self.ustar
        if xi <= us:
            if ps > l[2]:
                sl = l[1] - al * math.sqrt(gp / (2.0 * g) * ps / l[2] + gm / (2.0 * g))
                if xi <= sl:
                    return l
                return (l[0] * (ps / l[2] + gm / gp) / (gm / gp * ps / l[2] + 1.0), us, ps)
            astar = al * math.pow(ps / l[2], gm / (2.0 * g))
            if xi <= l[1] - al:
                return l
            if xi >= us - astar:
                return (l[0] * math.pow(ps / l[2], 1.0 / g), us, ps)
            u = 2.0 / gp * (al + gm / 2.0 * l[1] + xi)
            a = 2.0 / gp * (al + gm / 2.0 * (l[1] - xi))
            return (l[0] * math.pow(a / al, 2.0 / gm), u, l[2] * math.pow(a / al, 2.0 * g / gm))
        if ps > r[2]:
            sr = r[1] + ar * math.sqrt(gp / (2.0 * g) * ps / r[2] + gm / (2.0 * g))
            if xi >= sr:
                return r
            return (r[0] * (ps / r[2] + gm / gp) / (gm / gp * ps / r[2] + 1.0), us, ps)
        astar = ar * math.pow(ps / r[2], gm / (2.0 * g))
        if xi >= r[1] + ar:
            return r
        if xi <= us + astar:
            return (r[0] * math.pow(ps / r[2], 1.0 / g), us, ps)
        u = 2.0 / gp * (-ar + gm / 2.0 * r[1] + xi)
        a = 2.0 / gp * (ar - gm / 2.0 * (r[1] - xi))
        return (r[0] * math.pow(a / ar, 2.0 / gm), u, r[2] * math.pow(a / ar, 2.0 * g / gm))


def hll_solve(left, right, bx, gamma, t_end, cells, cfl=0.8, x0=0.0, x1=1.0, x_split=0.5):
    """First-order HLL MHD tube with outflow ends (hll_mhd.cpp:69-119);
    states (rho, u, v, w, by, bz, p); returns the final (cells, 7) states."""
    dx = (x1 - x0) / cells
    x = x0 + (np.arange(cells) + 0.5) * dx

    def to_cons(s):
        rho, u, v, w, by, bz, p = (s[..., q] for q in range(7))
        ke = 0.5 * rho * (u * u + v * v + w * w)
        me = 0.5 * (bx * bx + by * by + bz * bz)
        return np.stack([rho, rho * u, rho * v, rho * w, by, bz,
                         p / (gamma - 1.0) + ke + me], -1)

    def to_prim(U):
        rho = U[..., 0]
        if np.any(rho <= 0.0):
            raise RuntimeError("hll reference: negative density")
        u, v, w = U[..., 1] / rho, U[..., 2] / rho, U[..., 3] / rho
        by, bz = U[..., 4], U[..., 5]
        ke = 0.5 * rho * (u * u + v * v + w * w)
        me = 0.5 * (bx * bx + by * by + bz * bz)
        p = (gamma - 1.0) * (U[..., 6] - ke - me)
        if np.any(p <= 0.0):
            raise RuntimeError("hll reference: negative pressure")
        return np.stack([rho, u, v, w, by, bz, p], -1)

    def fast_x(s):
        rho, p = s[..., 0], s[..., 6]
        a2 = gamma * s[..., 6] / rho
        b2 = (bx * bx + s[..., 4] * s[..., 4] + s[..., 5] * s[..., 5]) / rho
        disc = np.sqrt(np.where((a2 + b2) * (a2 + b2) - 4.0 * a2 * bx * bx / rho < 0.0, 0.0,
                                (a2 + b2) * (a2 + b2) - 4.0 * a2 * bx * bx / rho))
        del p
        return np.sqrt(0.5 * (a2 + b2 + disc))

    def flux(s):
        rho, u, v, w, by, bz, p = (s[..., q] for q in range(7))
        pt = p + 0.5 * (bx * bx + by * by + bz * bz)
        e = to_cons(s)[..., 6]
        udotb = u * bx + v * by + w * bz
        return np.stack([rho * u, rho * u * u + pt - bx * bx, rho * u * v - bx * by,
                         rho * u * w - bx * bz, by * u - bx * v, bz * u - bx * w,
                         (e + pt) * u - bx * udotb], -1)

    U = to_cons(np.where((x < x_split)[:, None], np.asarray(left, float)[None],
                         np.asarray(right, float)[None]))
    il = np.maximum(np.arange(cells + 1) - 1, 0)
    ir = np.minimum(np.arange(cells + 1), cells - 1)
    t = 0.0
    while t < t_end:
        prim = to_prim(U)
        smax = float(np.max(np.abs(prim[:, 1]) + fast_x(prim)))
        dt = min(cfl * dx / smax, t_end - t)
        L, R = prim[il], prim[ir]
        cl, cr = fast_x(L), fast_x(R)
        sl = np.minimum(L[:, 1] - cl, R[:, 1] - cr)
        sr = np.maximum(L[:, 1] + cl, R[:, 1] + cr)
        fl, fr = flux(L), flux(R)
        ul, ur = U[il], U[ir]
        hll = (sr[:, None] * fl - sl[:, None] * fr + (sl * sr)[:, None] * (ur - ul)) / \
            (sr - sl)[:, None]
        f = np.where((sl >= 0.0)[:, None], fl, np.where((sr <= 0.0)[:, None], fr, hll))
        U = U - dt / dx * (f[1:] - f[:-1])
        t += dt
    return to_prim(U)


def sod_check(engine):
    """verify.cpp:54-77."""
    n, t_end, gamma = 512, 0.2, 5.0 / 3.0
    dx = 1.0 / n
    s, d = make_strip(n, dx)
    x = (np.arange(n) + 0.5) * dx
    s[GHOST:GHOST + n, 0] = np.where(x < 0.5, 1.0, 0.125)
    s[GHOST:GHOST + n, 7] = np.where(x < 0.5, 1.0, 0.1)
    run_strip(s, d, n, t_end, 0.5, gamma, False, engine)
    ref = ExactRiemann((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), gamma)
    err = [abs(s[GHOST + i, 0] - ref.sample((x[i] - 0.5) / t_end)[0]) for i in range(n)]
    l1 = _seqsum(err) / n
    return CheckResult("sod.l1_rho", l1, 0.01, l1 < 0.01)


def briowu_check(engine):
    """verify.cpp:79-112 (gamma 2, HLL reference at 8000 cells)."""
    n, nref, t_end, gamma = 800, 8000, 0.1, 2.0
    s, d = make_strip(n, 1.0 / n)
    x = (np.arange(n) + 0.5) / n
    left = x < 0.5
    s[GHOST:GHOST + n, 0] = np.where(left, 1.0, 0.125)
    s[GHOST:GHOST + n, 7] = np.where(left, 1.0, 0.1)
    s[GHOST:GHOST + n, 4] = 0.75
    s[GHOST:GHOST + n, 5] = np.where(left, 1.0, -1.0)
    run_strip(s, d, n, t_end, 0.5, gamma, False, engine)
    ref = hll_solve((1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1.0), (0.125, 0.0, 0.0, 0.0, -1.0, 0.0, 0.1),
                    0.75, gamma, t_end, nref)
    per = nref // n
    avg = np.array([_seqsum(ref[i * per:(i + 1) * per, 0]) / per for i in range(n)])
    l1 = _seqsum(np.abs(s[GHOST:GHOST + n, 0] - avg)) / n
    return CheckResult("briowu.l1_rho", l1, 0.03, l1 < 0.03)


def _advection_profile(x):
    return 1.0 + 0.25 * math.tanh(2.0 * math.sin(2.0 * 3.14159265358979323846 * x))


def advection_error(n, engine):
    """verify.cpp:122-140: one period of a smooth profile at u = 1."""
    dx = 1.0 / n
    s, d = make_strip(n, dx)
    x = [(i + 0.5) * dx for i in range(n)]
    s[GHOST:GHOST + n, 0] = [_advection_profile(xi) for xi in x]
    s[GHOST:GHOST + n, 1] = 1.0
    s[GHOST:GHOST + n, 7] = 1.0
    run_strip(s, d, n, 1.0, 0.5, 5.0 / 3.0, True, engine)
    err = [abs(s[GHOST + i, 0] - _advection_profile(x[i])) for i in range(n)]
    return _seqsum(err) / n


def convergence_check(engine):
    """verify.cpp:142-147."""
    e64, e128 = advection_error(64, engine), advection_error(128, engine)
    order = math.log2(e64 / e128)
    return CheckResult("advection.order_64_128", order, 2.5, order >= 2.5)


# --------------------------------------------------------------- 3-D suites

def _cube(n):
    return [AxisSpec(-1.0, 1.0, -1.0, 1.0, 2.0 / n, n, 1.05)] * 3


def conservation_check(precision="strict", device=0):
    """verify.cpp:166-195: periodic 32^3 gaussian pressure pulse, 50 steps,
    relative drift of total mass and energy."""
    specs = _cube(32)
    h = Harness(specs, (1, 1, 1), HarnessOptions(boundary=PERIODIC, with_sources=False,
                                                 precision=precision, device=device))
    h.init_with(IC_GAUSSIAN, ())
    sp = [build_axis(s).spacings for s in specs]
    vol = (sp[0][None, None, :] * sp[1][None, :, None]) * sp[2][:, None, None]
    gm1 = 5.0 / 3.0 - 1.0

    def totals():
        f = h.gather_interior()
        rho, v, b, p = f[..., 0], f[..., 1:4], f[..., 4:7], f[..., 7]
        k2 = (v[..., 0] * v[..., 0] + v[..., 1] * v[..., 1]) + v[..., 2] * v[..., 2]
        m2 = (b[..., 0] * b[..., 0] + b[..., 1] * b[..., 1]) + b[..., 2] * b[..., 2]
        energy = (p / gm1 + (0.5 * rho) * k2) + m2 / (2.0 * 1.0)
        return _seqsum(rho * vol), _seqsum(energy * vol)

    m0, e0 = totals()
    h.run(50)
    m1, e1 = totals()
    drift = max(abs(m1 - m0) / m0, abs(e1 - e0) / e0)
    return CheckResult("conservation.rel_drift", drift, 1e-11, drift < 1e-11)


def partition_check(part, name, precision="strict", device=0):
    """verify.cpp:205-226: a split layout against (1,1,1), worst relative
    difference over every field of every cell."""
    specs = _cube(12)
    opts = HarnessOptions(boundary=OUTFLOW, with_sources=True, precision=precision,
                          device=device)
    ref, split = Harness(specs, (1, 1, 1), opts), Harness(specs, part, opts)
    for h in (ref, split):
        h.init_with(IC_PARTITION, ())
        h.run(10)
    a, b = ref.gather_interior(), split.gather_interior()
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    worst = float(np.max(np.abs(a - b) / scale))
    return CheckResult(f"partition.{name}", worst, 1e-13, worst < 1e-13)


def suite_names():
    """verify.cpp:230-232."""
    return ["sod", "briowu", "convergence", "conservation", "partition"]


def run_suite(name, precision="strict", device=0, engine=None):
    """verify.cpp:234-243.  `engine` replaces the GPU 1-D engine (tests)."""
    kw = dict(precision=precision, device=device)
    eng = engine or GpuStrips(precision, device)
    if name == "sod":
        return [sod_check(eng)]
    if name == "briowu":
        return [briowu_check(eng)]
    if name == "convergence":
        return [convergence_check(eng)]
    if name == "conservation":
        return [conservation_check(**kw)]
    if name == "partition":
        return [partition_check((2, 1, 1), "2x1x1", **kw), partition_check((2, 3, 3), "2x3x3", **kw)]
    from .api import InvalidSpec
    raise InvalidSpec(f"unknown verification suite: '{name}'")


def cmd_verify(suite="all", precision="strict", device=0, out=print):
    """tools/ppmlr_main.cpp:80-93: the table and the exit status."""
    names = suite_names() if suite == "all" else [suite]
    ok = True
    out(f"{'check':<28s} {'metric':>14s} {'threshold':>14s} result")
    for n in names:
        for r in run_suite(n, precision, device):
            out(f"{r.name:<28s} {r.metric:14.6e} {r.threshold:14.6e} "
                f"{'pass' if r.passed else 'FAIL'}")
            ok = ok and r.passed
    return 0 if ok else 1

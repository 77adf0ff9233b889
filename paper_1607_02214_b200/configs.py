"""The benchmark configurations of BASELINE.json.

Each config is a grid (three AxisSpecs), harness options and an initial
condition.  ``scaled(name, ...)`` gives reduced grids of the same physics for
parity tests (the CPU oracle must finish in seconds there).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from .api import (IC_BLAST, IC_BRIOWU, IC_ORSZAG_TANG, MAGNETOSPHERE, OUTFLOW, PERIODIC,
                  AxisSpec, HarnessOptions)


@dataclass
class Config:
    name: str
    specs: list
    options: HarnessOptions
    ic: tuple            # (kind, params) or ("magnetosphere",)
    partition: tuple = (1, 1, 1)
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def cells(self):
        n = 1
        for s in self.specs:
            n *= int(s.cells)
        return n


def brio_wu(nx=256, nt=4, **kw):
    """C1: Brio-Wu shock tube along x, gamma = 2, outflow."""
    d = 1.0 / 256
    specs = [AxisSpec(0.0, nx * d, 0.0, nx * d, d, nx, 1.05),
             AxisSpec(0.0, nt * d, 0.0, nt * d, d, nt, 1.05),
             AxisSpec(0.0, nt * d, 0.0, nt * d, d, nt, 1.05)]
    return Config("briowu", specs, HarnessOptions(boundary=OUTFLOW, gamma=2.0, **kw),
                  (IC_BRIOWU, ()))


def orszag_tang(n=512, nz=4, **kw):
    """C2: Orszag-Tang vortex, periodic, gamma = 5/3."""
    tp = 2.0 * math.pi
    specs = [AxisSpec(0.0, tp, 0.0, tp, tp / n, n, 1.05),
             AxisSpec(0.0, tp, 0.0, tp, tp / n, n, 1.05),
             AxisSpec(0.0, tp * nz / n, 0.0, tp * nz / n, tp / n, nz, 1.05)]
    return Config("orszag_tang", specs, HarnessOptions(boundary=PERIODIC, **kw),
                  (IC_ORSZAG_TANG, (5.0 / 3.0,)))


def magnetosphere(nx=160, nyz=150, d=0.4, partition=(1, 1, 1), **kw):
    """C3 (160x150x150, d=0.4) / C5 (1024x768x768, d=0.05): solar wind -
    magnetosphere dipole problem on the stretched grid."""
    specs = [AxisSpec(-100.0, 30.0, -10.0, 10.0, d, nx, 1.05),
             AxisSpec(-100.0, 100.0, -10.0, 10.0, d, nyz, 1.05),
             AxisSpec(-100.0, 100.0, -10.0, 10.0, d, nyz, 1.05)]
    return Config(f"magnetosphere_{nx}x{nyz}x{nyz}", specs,
                  HarnessOptions(boundary=MAGNETOSPHERE, with_dipole=True, **kw),
                  ("magnetosphere",), partition)


def magnetosphere_small(n=(64, 36, 36), dcell=1.2, **kw):
    """The survey's 64x36x36 uniform magnetosphere."""
    hx = (-48.0, 28.8)
    hy = (-21.6, 21.6)
    specs = [AxisSpec(hx[0], hx[1], hx[0], hx[1], dcell, n[0], 1.05),
             AxisSpec(hy[0], hy[1], hy[0], hy[1], dcell, n[1], 1.05),
             AxisSpec(hy[0], hy[1], hy[0], hy[1], dcell, n[2], 1.05)]
    return Config("magnetosphere_small", specs,
                  HarnessOptions(boundary=MAGNETOSPHERE, with_dipole=True, **kw),
                  ("magnetosphere",))


def blast(n=512, gpus=1, p_in=10.0, p_out=0.1, radius=0.1, **kw):
    """C4: weak-scaling blast wave, n^3 per GPU, one blast per unit block."""
    specs = [AxisSpec(-0.5, gpus - 0.5, -0.5, gpus - 0.5, 1.0 / n, n * gpus, 1.05),
             AxisSpec(-0.5, 0.5, -0.5, 0.5, 1.0 / n, n, 1.05),
             AxisSpec(-0.5, 0.5, -0.5, 0.5, 1.0 / n, n, 1.05)]
    return Config(f"blast_{n}^3x{gpus}", specs, HarnessOptions(boundary=OUTFLOW, **kw),
                  (IC_BLAST, (p_in, p_out, radius)), (gpus, 1, 1))


def init(h, cfg: Config):
    if cfg.ic[0] == "magnetosphere":
        h.init_magnetosphere()
    else:
        h.init_with(*cfg.ic)

"""``ppmlr report`` on the GPU path: tools/ppmlr_main.cpp:107-139 (cmd_report).

Desk-scale live runs of the reference's partition shapes (decomp.cpp:110-112,
reference_configs) on the 24 x 30 x 30 grid every shape divides evenly, each
with every block of the layout driven by the multi-block harness
(per-block streams, halo pulls, device-side global dt), and one CSV row per
shape with the reference's columns:

    nx,ny,nz,ranks,tde_units,bytes_per_step,mean_compute_s,mean_transfer_s,
    predicted_speedup

bytes_per_step is the TransferLedger total over the steps (the reference's
accounting); mean_compute_s / mean_transfer_s aggregate the per-rank step
timings (perfmodel.cpp aggregate) -- on the GPU every block's step is one
stream-ordered device step, so compute is its wall time and transfer 0
(the halo copies are peer loads inside it); predicted_speedup is the
reference's bandwidth model (perfmodel.cpp predict_speedup) at efficiency
0.732, restated here because it is host arithmetic, not the hot path.
"""
from __future__ import annotations

import time

import numpy as np

from .api import AxisSpec, Harness, HarnessOptions, build_axis, tde_units

REFERENCE_CONFIGS = [(3, 1, 1), (3, 3, 3), (4, 3, 3), (6, 3, 3), (4, 5, 5), (6, 5, 5)]
DEVICE_BW, HOST_BW = 250e9, 51.2e9       # perfmodel.hpp BandwidthSpec defaults
WORKLOAD_FLOOR_CELLS = 64 * 64 * 64       # perfmodel.hpp kWorkloadFloorCells


def total_ranks(c):
    """decomp.cpp:42-44 (the blocks plus the ionosphere rank)."""
    return c[0] * c[1] * c[2] + 1


def mas():
    """perfmodel.cpp:9-13"""
    return DEVICE_BW / HOST_BW


def predict_speedup(c, n, efficiency=0.732):
    """perfmodel.cpp:28-39"""
    if not (0.0 < efficiency <= 1.0):
        raise ValueError("efficiency must lie in (0, 1]")
    cells = (n[0] // c[0]) * (n[1] // c[1]) * (n[2] // c[2])
    util = min(1.0, cells / WORKLOAD_FLOOR_CELLS)
    return min(mas() * efficiency * util, mas())


def _ic(h):
    """The report's initial condition (ppmlr_main.cpp:121-128), evaluated on
    the host per block, ghost-inclusive."""
    out = []
    for r in range(h.block_count()):
        cen, _, _ = h.block_geometry(r)
        z, y, x = np.meshgrid(cen[2], cen[1], cen[0], indexing="ij")
        w = np.exp(-(x * x + y * y + z * z) / 8.0)
        f = np.zeros(z.shape + (8,))
        f[..., 0] = 1.0 + 0.3 * w
        f[..., 7] = 1.0 + 0.2 * w
        f[..., 4] = -y * 0.1
        f[..., 5] = x * 0.1
        f[..., 6] = 0.2 * 0.1
        out.append(f)
    return out


def cmd_report(steps=5, transport="direct", devices=None, out=print):
    ax = AxisSpec(-4.8, 4.8, -4.8, 4.8, 0.4, 24, 1.05)
    ay = AxisSpec(-6.0, 6.0, -6.0, 6.0, 0.4, 30, 1.05)
    specs = [ax, ay, ay]
    n = [build_axis(s).n for s in specs]
    out("nx,ny,nz,ranks,tde_units,bytes_per_step,mean_compute_s,mean_transfer_s,"
        "predicted_speedup")
    rows = []
    for c in REFERENCE_CONFIGS:
        opts = HarnessOptions(boundary="outflow", with_dipole=False, transport=transport)
        h = Harness(specs, c, opts, devices=devices)
        h.set_state(_ic(h))
        comp = []
        for _ in range(steps):
            t0 = time.perf_counter()
            h.advance()
            comp.append(time.perf_counter() - t0)
        nb = h.block_count()
        mean_compute = sum(comp) / len(comp)  # every rank records the step's time
        bytes_per_step = h.ledger()[0] // steps
        row = (c[0], c[1], c[2], total_ranks(c), tde_units(c), bytes_per_step, mean_compute,
               0.0, predict_speedup(c, n))
        out("%d,%d,%d,%d,%d,%d,%.3e,%.3e,%.4f" % row)
        rows.append(row)
        h.close()
        del nb
    return rows

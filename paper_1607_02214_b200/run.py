"""``ppmlr run`` on the GPU path: tools/ppmlr_main.cpp:56-78 (cmd_run).

Steps a configuration, writes ``snapshot_%06d.bin`` (PPLR v1) at the
cadence and after the last step, then ``ledger.csv`` and ``timing.csv``, and
prints the reference's summary line.  Snapshots are captured on the device
and drained to disk by a host thread while the next steps run.

timing.csv keeps the reference's columns (rank,step,compute_seconds,
transfer_seconds).  All blocks of a Harness share one GPU and one stream, so
compute_seconds is the wall time of the whole device step (it ends with the
dt read-back) for every rank, and transfer_seconds is 0: the halo copies are
device-to-device copies inside the step.
"""
from __future__ import annotations

import os
import time

from . import configs
from .api import Harness


def cmd_run(cfg: configs.Config, steps: int, cadence: int, out_dir: str, quiet=False):
    os.makedirs(out_dir, exist_ok=True)
    h = Harness(cfg.specs, cfg.partition, cfg.options)
    configs.init(h, cfg)
    timings = []
    for s in range(1, steps + 1):
        t0 = time.perf_counter()
        h.advance()
        dt_wall = time.perf_counter() - t0
        for r in range(h.block_count()):
            timings.append((r, s - 1, dt_wall, 0.0))
        if s % cadence == 0 or s == steps:
            h.write_snapshot(os.path.join(out_dir, f"snapshot_{s:06d}.bin"), wait=False)
    h.snapshot_wait()
    with open(os.path.join(out_dir, "ledger.csv"), "w") as f:
        f.write(h.ledger_csv())
    with open(os.path.join(out_dir, "timing.csv"), "w") as f:
        f.write("rank,step,compute_seconds,transfer_seconds\n")
        for r, st, c, t in timings:
            f.write(f"{r},{st},{c:.9e},{t:.9e}\n")
    b, m, _ = h.ledger()
    n = max(len(timings), 1)
    line = (f"steps={h.step_count()} time={h.time():.6e} bytes={b} messages={m} "
            f"mean_compute={sum(t[2] for t in timings) / n:.3e} "
            f"mean_transfer={sum(t[3] for t in timings) / n:.3e}")
    if not quiet:
        print(line)
    return h, line

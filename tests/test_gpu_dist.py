"""The distributed driver on the device with several ranks: DeviceRankBlock's
pack -> transport -> unpack, the boundary-first split launches (sweep_part /
end_step_part) that overlap each exchange with the interior work, and the
MIN all-reduce of dt.  Every rank runs on GPU 0 with gloo through pinned host
buffers (this pool gives one GPU; NCCL refuses two ranks on one device), so
the ranks' kernels never wait on each other.  The gathered state must equal
the in-process single-block harness bit for bit (strict), with and without
the overlap, for 2 and 4 x-slabs."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp, world, cfg, steps, overlap, precision="strict"):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(ROOT, "tests", "workers", "dist_gpu_worker.py"),
           "--out", str(tmp), "--cfg", cfg, "--steps", str(steps), "--overlap", str(overlap),
           "--precision", precision]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]


@pytest.mark.parametrize("world,cfg,overlap", [(2, "blast", 1), (2, "blast", 0),
                                               (4, "blast", 1), (4, "magnetosphere", 1)])
def test_device_ranks_match_single_block(gpu, tmp_path, world, cfg, overlap):
    from paper_1607_02214_b200 import configs
    steps = 6
    _run(tmp_path, world, cfg, steps, overlap)
    c = {"blast": lambda: configs.blast(n=24, gpus=world, radius=0.3),
         "magnetosphere": lambda: configs.magnetosphere_small()}[cfg]()
    h = gpu.Harness(c.specs, (1, 1, 1), c.options)
    configs.init(h, c)
    h.run(steps)
    want = h.gather_interior()
    from paper_1607_02214_b200.api import layout
    blocks, _ = layout(c.specs, (world, 1, 1))
    got = np.zeros_like(want)
    for b in blocks:
        part = np.load(tmp_path / f"rank{b.rank}.npy")
        got[:, :, b.lo[0]:b.lo[0] + b.n[0]] = part
    assert bits_equal(got, want)
    # every rank holds the same next global dt, the harness's next dt
    dts = {float(np.load(tmp_path / f"dt{b.rank}.npy")[0]) for b in blocks}
    assert len(dts) == 1
    assert dts.pop() == h.compute_global_dt()

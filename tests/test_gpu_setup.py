"""§8(f)-2 device-side setup: make_block's dipole field (stepper.cpp:63-69,
physics.cpp:14-21) and the built-in init_with ICs (harness.cpp:35-43) are
evaluated by a CUDA kernel (block.cu init_state_kernel).  They must equal
the host evaluation (host.cpp make_ic / dipole, itself pinned to the
reference by tests/golden) bit for bit; PPMLR_HOST_INIT=1 forces the host
path through the same API, so both are compared here on the same grids."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


def _build(gpu, specs, opts, ic, host):
    if host:
        os.environ["PPMLR_HOST_INIT"] = "1"
    try:
        h = gpu.Harness(specs, (1, 1, 1), opts)
        if ic is not None:
            h.init_with(*ic)
        b = h.block(0)
        state = b.download()
        bd = b.state_view(interior=False, dipole=True)
        bd = None if bd is None else np.stack([t.cpu().numpy() for t in bd], axis=-1)
    finally:
        os.environ.pop("PPMLR_HOST_INIT", None)
    h.close()
    return state, bd


def _cases():
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    tp = 2.0 * math.pi
    yield "default+dipole C3", configs.magnetosphere().specs, HarnessOptions(
        boundary=2, with_dipole=True), None
    yield "default+dipole C5-shaped", configs.magnetosphere(nx=256, nyz=192, d=0.2).specs, \
        HarnessOptions(boundary=2, with_dipole=True), None
    cube = [AxisSpec.uniform(-0.5, 0.5, 24)] * 3
    yield "blast", [AxisSpec(-0.5, 1.5, -0.5, 1.5, 1 / 20, 40, 1.05)] + cube[1:], \
        HarnessOptions(), (3, (10.0, 0.1, 0.1))
    yield "briowu", configs.brio_wu(nx=64).specs, HarnessOptions(gamma=2.0), (1, ())
    yield "orszag_tang", configs.orszag_tang(n=48).specs, HarnessOptions(boundary=1), \
        (2, (5.0 / 3.0,))
    yield "uniform", cube, HarnessOptions(), (0, (1.0, 0.1, -0.2, 0.3, 0.5, 0.6, 0.7, 2.0))
    yield "blast ghost 6", cube, HarnessOptions(ghost=6), (3, (10.0, 0.1, 0.2))
    yield "dipole stretched odd", [AxisSpec(-100.0, 30.0, -10.0, 10.0, 2.5, 41, 1.05),
                                   AxisSpec(-100.0, 100.0, -10.0, 10.0, 2.5, 40, 1.05),
                                   AxisSpec(-100.0, 100.0, -10.0, 10.0, 2.0, 48, 1.05)], \
        HarnessOptions(boundary=2, with_dipole=True), (3, (2.0, 1.0, 0.3))
    del tp


@pytest.mark.parametrize("case", list(range(8)))
def test_device_setup_equals_host(gpu, case):
    name, specs, opts, ic = list(_cases())[case]
    dev_state, dev_bd = _build(gpu, specs, opts, ic, host=False)
    host_state, host_bd = _build(gpu, specs, opts, ic, host=True)
    # the device holds kG = 4 ghost layers; download() maps them into the
    # caller's g-ghost layout, so compare the whole array
    assert bits_equal(dev_state, host_state), name
    if opts.with_dipole:
        assert dev_bd is not None and bits_equal(dev_bd, host_bd), name


def test_device_setup_matches_host_block_state(gpu):
    """The device-initialised state equals host_block_state (the host
    restatement used by the CPU tests) on the kG window."""
    from paper_1607_02214_b200 import configs
    c = configs.magnetosphere()
    h = gpu.Harness(c.specs, (1, 1, 1), c.options)
    h.init_with(3, (5.0, 0.5, 10.0))
    st = gpu.host_block_state(c.specs, (1, 1, 1), c.options, 0, (3, (5.0, 0.5, 10.0)))
    bd = np.stack([t.cpu().numpy() for t in h.block(0).state_view(interior=False, dipole=True)],
                  axis=-1)
    g = c.options.ghost
    sl = slice(g - 4, None if g == 4 else -(g - 4))
    want_bd = st["bd"][sl, sl, sl]
    assert bits_equal(bd[:, :, :want_bd.shape[2]], want_bd)
    # the interior (the magnetosphere boundary refills the sunward ghost
    # shell with the wind on upload, which host_block_state does not)
    ins = slice(g, -g)
    assert bits_equal(h.block(0).download()[ins, ins, ins], st["fields"][ins, ins, ins])
    h.close()

"""The knobs that reach the hot path (SURVEY.md §8(b) knob table) against
the live reference build, bit for bit in strict mode: pressure floor, ghost
width (results must not depend on it; only the ledger does), staged
transport, sources off, and the fast build on the same knobs within the
stated tolerance."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, rel_errors

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif("not __import__('pyoracle').have_ref()")]


def _blast_specs(n):
    return [(-0.5, 0.5, -0.5, 0.5, 1.0 / n, n, 1.05)] * 3


def _pair(gpu, oracle, specs, part, ic, steps, precision="strict", **kw):
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    ref = oracle.RefHarness(specs, part, **kw)
    ref.init_ic(*ic)
    opts = {k: v for k, v in kw.items() if k != "transport"}
    if "boundary" in opts:
        opts["boundary"] = {0: gpu.OUTFLOW, 1: gpu.PERIODIC, 2: gpu.MAGNETOSPHERE}[opts["boundary"]]
    h = gpu.Harness([AxisSpec(*s) for s in specs], part,
                    HarnessOptions(precision=precision,
                                   transport="staged" if kw.get("transport", 1) == 0
                                   else "direct", **opts))
    h.init_with(*ic)
    for _ in range(steps):
        ref.advance()
    h.run(steps)
    return h, ref


def test_pressure_floor_bitwise(gpu, oracle):
    """pressure_floor > 0 disables the Lagrangian checks and floors p
    (physics.cpp:40-55, ppm1d.cpp:184): a strong blast into near vacuum."""
    h, ref = _pair(gpu, oracle, _blast_specs(24), (1, 1, 1), (gpu.IC_BLAST, (100.0, 1e-4, 0.2)),
                   6, pressure_floor=1e-3)
    assert bits_equal(h.gather_interior(), ref.gather())
    assert h.time() == ref.time()


@pytest.mark.parametrize("ghost", [5, 6])
def test_ghost_width_changes_only_the_ledger(gpu, oracle, ghost):
    h, ref = _pair(gpu, oracle, _blast_specs(16), (2, 1, 1), (gpu.IC_SMOOTH, ()), 4,
                   ghost=ghost)
    assert bits_equal(h.gather_interior(), ref.gather())
    assert h.ledger() == ref.ledger()


def test_staged_transport_and_no_sources(gpu, oracle):
    h, ref = _pair(gpu, oracle, _blast_specs(16), (2, 1, 1), (gpu.IC_PARTITION, ()), 5,
                   transport=0, with_sources=False)
    assert bits_equal(h.gather_interior(), ref.gather())
    assert h.ledger() == ref.ledger()
    assert h.ledger_csv() == ref.ledger_csv()


def test_fast_build_on_the_floor_within_tolerance(gpu, oracle):
    h, ref = _pair(gpu, oracle, _blast_specs(24), (1, 1, 1), (gpu.IC_BLAST, (100.0, 1e-4, 0.2)),
                   6, precision="fast", pressure_floor=1e-3)
    l1, linf = rel_errors(h.gather_interior(), ref.gather())
    assert np.all(l1 <= 1e-11) and np.all(linf <= 1e-9), (l1, linf)


def test_gpu_sweep_strips_with_floor_bitwise(gpu, oracle):
    rng = np.random.default_rng(11)
    n, g = 40, 4
    st = np.zeros((3, n + 2 * g, 8))
    st[..., 0] = rng.uniform(0.5, 1.5, st.shape[:2])
    st[..., 1] = rng.uniform(-0.5, 0.5, st.shape[:2])
    st[..., 7] = rng.uniform(1e-6, 1e-4, st.shape[:2])
    dx = np.full(n + 2 * g, 1.0 / n)
    want = st.copy()
    for k in range(3):
        oracle.ref_sweep_1d(want[k], None, dx, n, g, 0.002, 0, pressure_floor=1e-3)
    got = gpu.sweep_strips(st.copy(), None, dx, n, g, 0.002, 0, pressure_floor=1e-3)
    assert bits_equal(got, want)


def test_cached_dt_is_dropped_when_the_state_changes(gpu):
    """run/advance leave the next dt on the device and skip the next
    standalone CFL pass; any upload must invalidate it."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    specs = [AxisSpec(*s) for s in _blast_specs(16)]
    a = gpu.Harness(specs, (1, 1, 1), HarnessOptions())
    a.init_with(gpu.IC_BLAST, (10.0, 0.1, 0.2))
    a.run(2)
    a.init_with(gpu.IC_SMOOTH, ())          # new state: the cached dt is stale
    dts = [a.advance() for _ in range(3)]
    b = gpu.Harness(specs, (1, 1, 1), HarnessOptions())
    b.init_with(gpu.IC_SMOOTH, ())
    want = [b.advance() for _ in range(3)]
    assert dts == want
    assert bits_equal(a.gather_interior(), b.gather_interior())
    c = gpu.Harness(specs, (1, 1, 1), HarnessOptions())
    c.init_with(gpu.IC_SMOOTH, ())
    c.run(3)                                 # one window: same dts, same state
    assert bits_equal(c.gather_interior(), want_state := b.gather_interior())
    assert c.time() == b.time()


@pytest.mark.parametrize("dims,boundary,ic", [
    ((17, 13, 11), 0, (3, (10.0, 0.1, 0.3))),   # odd sizes: partial tiles, OOB boxes
    ((67, 9, 130), 0, (4, ())),                 # one long axis (runtime tile), odd short ones
    ((36, 20, 12), 1, (4, ())),                 # periodic
    ((257, 6, 5), 0, (5, ())),                  # > 256 cells: the compile-time tile, partial tail
])
def test_odd_sizes_bitwise_vs_reference(gpu, oracle, dims, boundary, ic):
    specs = [(-1.0, 1.0, -1.0, 1.0, 2.0 / n, n, 1.05) for n in dims]
    h, ref = _pair(gpu, oracle, specs, (1, 1, 1), ic, 4, boundary=boundary)
    assert bits_equal(h.gather_interior(), ref.gather())
    assert h.time() == ref.time()


def test_odd_sizes_magnetosphere_partitioned(gpu, oracle):
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    specs = [(-48.0, 28.8, -48.0, 28.8, 1.2, 64, 1.05),
             (-22.8, 22.8, -22.8, 22.8, 1.2, 38, 1.05),
             (-20.4, 20.4, -20.4, 20.4, 1.2, 34, 1.05)]
    ref = oracle.RefHarness(specs, (2, 1, 1), boundary=2, with_dipole=True)
    ref.init_magnetosphere()
    h = gpu.Harness([AxisSpec(*s) for s in specs], (2, 1, 1),
                    HarnessOptions(boundary=gpu.MAGNETOSPHERE, with_dipole=True))
    h.init_magnetosphere()
    for _ in range(4):
        ref.advance()
    h.run(4)
    assert bits_equal(h.gather_interior(), ref.gather())


@pytest.mark.slow
@pytest.mark.parametrize("cfg,steps", [("ot512", 100), ("briowu", 220)])
def test_fast_build_long_runs_within_tolerance(gpu, cfg, steps):
    """BASELINE configs C2 (Orszag-Tang 512x512x4, L1 error vs the CPU
    reference after 100 steps) and C1 (Brio-Wu 256x4x4 to t~0.1, 220 steps):
    the fast build against the strict build, which is bit-identical to the
    reference."""
    from dataclasses import replace
    from paper_1607_02214_b200 import configs
    c = configs.orszag_tang(n=512) if cfg == "ot512" else configs.brio_wu()
    out = {}
    for prec in ("strict", "fast"):
        h = gpu.Harness(c.specs, c.partition, replace(c.options, precision=prec))
        configs.init(h, c)
        h.run(steps)
        out[prec] = h.gather_interior()
    l1, linf = rel_errors(out["fast"], out["strict"])
    print(cfg, "rel L1", l1.max(), "rel Linf", linf.max())
    assert np.all(l1 <= 1e-11) and np.all(linf <= 1e-9), (l1, linf)


def test_upload_with_a_new_frozen_core_recaptures_the_step(gpu):
    """The step graphs bake in the frozen-core slot map (pointers and
    bounding box); an upload that replaces the frozen set must drop them.
    A harness that already stepped, re-uploaded with a smaller frozen set,
    must match a fresh harness given the same upload, bit for bit."""
    from paper_1607_02214_b200 import configs
    cfg = configs.magnetosphere_small()
    st = gpu.host_block_state(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic)
    nf = len(st["frozen_idx"])
    assert nf > 8
    keep = slice(0, nf // 2)                 # a different frozen set and box
    out = []
    for warm in (True, False):
        h = gpu.Harness(cfg.specs, (1, 1, 1), cfg.options)
        configs.init(h, cfg)
        if warm:
            h.run(2)                         # step graphs captured
        h.block(0).upload(st["fields"], st["bd"], st["frozen_idx"][keep],
                          st["frozen_states"][keep])
        h.run(3)
        out.append(h.gather_interior())
    assert bits_equal(out[0], out[1])

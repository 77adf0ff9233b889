"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden vectors.  Strict mode must be bit-identical; fast mode
within the stated tolerance (per-field relative L1 <= 1e-11, Linf <= 1e-9
after N steps)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import bits_equal, digest, golden_case, rel_errors, run_names

pytestmark = pytest.mark.gpu

FAST_L1, FAST_LINF = 1e-11, 1e-9


# ------------------------------------------------------------ exact division

def test_exact_division_matches_ieee_divide(gpu):
    """The strict kernels' shared-reciprocal division (exact_div.cuh) is
    bit-identical to the compiler's `/` on 2^28 operand pairs including
    zeros, denormals, extremes, inf/nan bit patterns."""
    import ctypes
    from paper_1607_02214_b200 import _native as N
    bad = ctypes.c_longlong()
    ex = np.zeros(4)
    for seed in (1, 12345):
        N.check(N.lib.ppmlr_gpu_selftest_division(0, 1 << 27, seed, ctypes.byref(bad),
                                                  ex.ctypes.data_as(N._dp)))
        assert bad.value == 0, (bad.value, ex.tolist())


# ------------------------------------------------------------ sweep_1d

def test_sweep_strips_match_reference_golden(gpu, golden_strips):
    for k in range(int(golden_strips["count"])):
        pre = f"s{k}/"
        n, g, d, dt = golden_strips[pre + "meta"]
        bd = golden_strips[pre + "bd"]
        out = gpu.sweep_strips(golden_strips[pre + "in"].copy(), None if bd.size == 0 else bd,
                               golden_strips[pre + "dx"], int(n), int(g), float(dt), int(d))
        assert bits_equal(out[0], golden_strips[pre + "out"]), f"strip {k}"


def _random_batch(rng, ns, n, bd_on, quiet=False):
    nn = n + 8
    st = np.zeros((ns, nn, 8))
    st[..., 0] = rng.uniform(0.3, 2.5, (ns, nn))
    st[..., 7] = rng.uniform(0.1, 2.5, (ns, nn))
    st[..., 1:4] = rng.uniform(-0.6, 0.6, (ns, nn, 3))
    st[..., 4:7] = rng.uniform(-1.2, 1.2, (ns, nn, 3))
    if quiet:
        st[:, : nn // 2, 1:4] = 0.0
        st[:, : nn // 2, 4:] = st[:, :1, 4:]
        st[:, : nn // 2, 0] = st[:, :1, 0]
    bd = rng.uniform(-1, 1, (ns, nn, 3)) if bd_on else None
    dx = rng.uniform(0.4, 1.6, nn)
    return st, bd, dx


@pytest.mark.parametrize("direction", [0, 1, 2])
@pytest.mark.parametrize("bd_on", [False, True])
@pytest.mark.parametrize("n", [1, 7, 33, 150, 300])
def test_sweep_strips_bitwise_vs_oracle(gpu, oracle, direction, bd_on, n):
    rng = np.random.default_rng(1000 * n + 10 * direction + bd_on)
    ns = 37
    st, bd, dx = _random_batch(rng, ns, n, bd_on, quiet=(n % 2 == 1))
    c = oracle.consts()
    dt = min(oracle.orc_strip_max_dt(st[s], None if bd is None else bd[s], dx, n, 4, direction, c)
             for s in range(ns)) * 0.45
    wants, first_err = [], None
    for s in range(ns):
        want = st[s].copy()
        try:
            oracle.orc_sweep_1d(want, None if bd is None else bd[s].copy(), dx, n, 4, dt,
                                direction, c)
        except oracle.OracleError as e:
            first_err = first_err or e.msg
        wants.append(want)
    if first_err is not None:  # the GPU must fail the same way (first strip in order)
        with pytest.raises(gpu.Error) as ex:
            gpu.sweep_strips(st.copy(), bd, dx, n, 4, dt, direction)
        assert str(ex.value) == first_err
        return
    got = gpu.sweep_strips(st.copy(), bd, dx, n, 4, dt, direction)
    for s in range(ns):
        assert bits_equal(got[s], wants[s]), (s, np.abs(got[s] - wants[s]).max())


def test_sweep_strips_errors_match_reference(gpu, golden_strips):
    errs = json.loads(str(golden_strips["errors"]))
    for d in range(3):
        with pytest.raises(gpu.StepRejected) as ex:
            gpu.sweep_strips(golden_strips[f"e{d}/in"].copy(), None, np.full(24, 0.1), 16, 4, 0.1,
                             d)
        assert str(ex.value) == errs[d][1]


def test_sweep_strips_first_failing_strip_reported(gpu, oracle):
    """Several strips fail; the error names the first in loop order, as the
    reference's sweep would."""
    rng = np.random.default_rng(3)
    st, _, dx = _random_batch(rng, 12, 20, False)
    st[5, :, 1] = np.where(np.arange(28) < 14, 30.0, -30.0)   # collides
    st[9, :, 1] = np.where(np.arange(28) < 10, 30.0, -30.0)
    want = st[5].copy()
    with pytest.raises(oracle.OracleError) as e1:
        oracle.orc_sweep_1d(want, None, dx, 20, 4, 0.05, 0, oracle.consts())
    with pytest.raises(gpu.Error) as e2:
        gpu.sweep_strips(st.copy(), None, dx, 20, 4, 0.05, 0)
    assert str(e2.value) == e1.value.msg


@pytest.mark.parametrize("n", [16, 150])
def test_fast_sweep_within_tolerance(gpu, oracle, n):
    rng = np.random.default_rng(99 + n)
    st, bd, dx = _random_batch(rng, 24, n, True)
    c = oracle.consts()
    dt = 0.4 * min(oracle.orc_strip_max_dt(st[s], bd[s], dx, n, 4, 1, c) for s in range(24))
    got = gpu.sweep_strips(st.copy(), bd, dx, n, 4, dt, 1, precision="fast")
    want = st.copy()
    for s in range(24):
        oracle.orc_sweep_1d(want[s], bd[s].copy(), dx, n, 4, dt, 1, c)
    l1, linf = rel_errors(got[:, 4:4 + n], want[:, 4:4 + n])
    assert l1.max() <= FAST_L1 and linf.max() <= FAST_LINF, (l1.max(), linf.max())


# ------------------------------------------------------------ harness

def _harness(gpu, specs, opts, ic, partition=(1, 1, 1)):
    h = gpu.Harness(specs, partition, opts)
    if ic[0] == "magnetosphere":
        h.init_magnetosphere()
    else:
        h.init_with(*ic)
    return h


@pytest.mark.parametrize("name", run_names())
def test_harness_matches_reference_golden_runs(gpu, golden_runs, name):
    pre = name + "/"
    specs, opts, ic, steps = golden_case(golden_runs, name)
    h = _harness(gpu, specs, opts, ic)
    dts = [h.advance() for _ in range(steps)]
    assert bits_equal(np.array(dts), golden_runs[pre + "dts"])
    fin = h.gather_interior()
    assert digest(fin) == str(golden_runs[pre + "final_sha"]), name
    assert h.time() == float(golden_runs[pre + "time"])
    assert h.step_count() == steps


@pytest.mark.parametrize("name", ["blast", "magnetosphere", "orszag_tang"])
def test_run_graph_equals_stepwise_advance(gpu, golden_runs, name):
    specs, opts, ic, steps = golden_case(golden_runs, name)
    a = _harness(gpu, specs, opts, ic)
    b = _harness(gpu, specs, opts, ic)
    for _ in range(steps):
        a.advance()
    b.run(steps)
    assert bits_equal(a.gather_interior(), b.gather_interior())
    assert a.time() == b.time()


def _oracle_from_host(oracle, gpu, specs, opts, ic):
    st = gpu.host_block_state(specs, (1, 1, 1), opts, 0, ic)
    n = [len(c) - 8 for c in st["centers"]]
    return oracle.OracleBlock(n, 4, st["centers"], st["spacings"], [[1, 1]] * 3, st["fields"],
                              st["bd"], st["frozen_idx"], st["frozen_states"])


def _magnetosphere_bricks():
    # y, z on the compile-time tile (64) with x = 66: the persistent kernel's
    # y / z sweeps read B_d from the bricks, the last x group partial
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200.api import AxisSpec
    c = configs.magnetosphere_small()
    c.specs[:] = [AxisSpec(-48.0, -48.0 + 66 * 1.2, -48.0, -48.0 + 66 * 1.2, 1.2, 66, 1.05)] + [
        AxisSpec(-38.4, 38.4, -38.4, 38.4, 1.2, 64, 1.05)] * 2
    return c


@pytest.mark.parametrize("cfg,steps", [("briowu", 30), ("orszag_tang", 8), ("blast", 6),
                                       ("magnetosphere_small", 6), ("magnetosphere_bricks", 4)])
def test_harness_bitwise_vs_oracle(gpu, oracle, cfg, steps):
    from paper_1607_02214_b200 import configs
    c = {"briowu": lambda: configs.brio_wu(nx=128),
         "orszag_tang": lambda: configs.orszag_tang(n=64),
         "blast": lambda: configs.blast(n=32, radius=0.2),
         "magnetosphere_small": lambda: configs.magnetosphere_small(),
         "magnetosphere_bricks": _magnetosphere_bricks}[cfg]()
    h = _harness(gpu, c.specs, c.options, c.ic)
    ob = _oracle_from_host(oracle, gpu, c.specs, c.options, c.ic)
    o = oracle.opts(boundary=c.options.boundary, cfl=c.options.cfl,
                    with_sources=c.options.with_sources)
    k = oracle.consts(gamma=c.options.gamma)
    for s in range(steps):
        assert h.advance() == ob.advance(o, k, s), s
    assert bits_equal(h.gather_interior(), ob.interior())


def test_partition_invariance_bitwise(gpu):
    """verify.cpp:205-226 (criterion 8) at 0 ulp, plus the magnetosphere
    physics with x-slabs and a 3-D split."""
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    cube = [AxisSpec.uniform(-1.0, 1.0, 12)] * 3
    for part in [(2, 1, 1), (2, 3, 3)]:
        ref = _harness(gpu, cube, HarnessOptions(), (gpu.IC_PARTITION, ()))
        spl = _harness(gpu, cube, HarnessOptions(), (gpu.IC_PARTITION, ()), part)
        ref.run(10)
        spl.run(10)
        assert bits_equal(ref.gather_interior(), spl.gather_interior()), part
    m = configs.magnetosphere_small()
    ref = _harness(gpu, m.specs, m.options, m.ic)
    ref.run(8)
    want = ref.gather_interior()
    for part in [(2, 1, 1), (4, 1, 1), (8, 1, 1), (2, 3, 3)]:
        spl = _harness(gpu, m.specs, m.options, m.ic, part)
        spl.run(8)
        assert bits_equal(spl.gather_interior(), want), part


def test_ledger_matches_byte_model_and_transport_accounting(gpu):
    """acceptance.cpp criteria 2 and 4."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    cube = [AxisSpec.uniform(-2.4, 2.4, 12)] * 3
    for part in [(2, 1, 1), (2, 3, 3)]:
        h = _harness(gpu, cube, HarnessOptions(), (gpu.IC_SMOOTH, ()), part)
        h.run(3)
        assert h.ledger()[0] == 3 * 4 * gpu.exchanged_bytes(cube, part, 4, 64)
    events = []
    for transport in ("direct", "staged"):
        h = _harness(gpu, cube, HarnessOptions(transport=transport), (gpu.IC_SMOOTH, ()),
                     (3, 1, 1))
        h.advance()
        events.append(h.ledger()[2])
    assert events[1] - events[0] == 96


def test_frozen_core_bitwise_unchanged(gpu):
    from paper_1607_02214_b200 import configs
    m = configs.magnetosphere_small()
    h = _harness(gpu, m.specs, m.options, m.ic)
    idx, states = h.frozen()
    assert len(idx) > 0
    h.run(5)
    g = 4
    full = h.block(0).download()
    flat = full.reshape(-1, 8)
    assert bits_equal(flat[idx], states)


def test_periodic_needs_single_block(gpu):
    from paper_1607_02214_b200 import configs
    c = configs.orszag_tang(n=16)
    with pytest.raises(gpu.InvalidSpec):
        gpu.Harness(c.specs, (2, 1, 1), c.options)


def test_unphysical_state_raised_with_reference_message(gpu, oracle):
    """An oversized CFL number makes Lagrangian interfaces cross; the GPU
    raises the same exception type and message (axis, line, zone) as the
    restatement of the reference (stepper.cpp:270-276)."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    cube = [AxisSpec.uniform(-0.5, 0.5, 16)] * 3
    opts = HarnessOptions(cfl=2.5)
    ic = (gpu.IC_BLAST, (10.0, 0.1, 0.3))
    h = _harness(gpu, cube, opts, ic)
    ob = _oracle_from_host(oracle, gpu, cube, opts, ic)
    o = oracle.opts(cfl=2.5)
    k = oracle.consts()
    err_o = err_g = None
    for s in range(20):
        try:
            ob.advance(o, k, s)
        except oracle.OracleError as e:
            err_o = (s, e.msg)
            break
    for s in range(20):
        try:
            h.advance()
        except gpu.Error as e:
            err_g = (s, str(e))
            break
    assert err_o is not None
    assert err_g == err_o


# ------------------------------------------------------------ full size

@pytest.mark.slow
def test_c3_magnetosphere_full_size_bitwise(gpu, oracle):
    """C3 160x150x150 (stretched grid, dipole, frozen core): 2 steps vs the
    restatement of the reference (~20 s of CPU)."""
    from paper_1607_02214_b200 import configs
    c = configs.magnetosphere()
    h = _harness(gpu, c.specs, c.options, c.ic)
    ob = _oracle_from_host(oracle, gpu, c.specs, c.options, c.ic)
    o = oracle.opts(boundary=2, cfl=c.options.cfl)
    k = oracle.consts()
    for s in range(2):
        assert h.advance() == ob.advance(o, k, s)
    assert bits_equal(h.gather_interior(), ob.interior())


@pytest.mark.slow
def test_conservation_periodic_at_scale(gpu):
    """Criterion 7 (verify.cpp:163-193) at 256^3: mass and total energy of a
    periodic box are conserved to 1e-11 relative after 10 steps."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    n = 256
    specs = [AxisSpec.uniform(-1.0, 1.0, n)] * 3
    h = _harness(gpu, specs, HarnessOptions(boundary=gpu.PERIODIC, with_sources=False),
                 (gpu.IC_GAUSSIAN, ()))

    def totals():
        f = h.gather_interior()
        rho, v, b, p = f[..., 0], f[..., 1:4], f[..., 4:7], f[..., 7]
        e = p / (5.0 / 3.0 - 1.0) + 0.5 * rho * (v * v).sum(-1) + 0.5 * (b * b).sum(-1)
        vol = (2.0 / n) ** 3
        return rho.sum() * vol, e.sum() * vol

    m0, e0 = totals()
    h.run(10)
    m1, e1 = totals()
    assert max(abs(m1 - m0) / m0, abs(e1 - e0) / e0) < 1e-11


# ------------------------------------------------------------ fast mode

@pytest.mark.parametrize("cfg,steps", [("blast", 12), ("orszag_tang", 12),
                                       ("magnetosphere_small", 8), ("briowu", 40)])
def test_fast_mode_within_tolerance_of_strict(gpu, cfg, steps):
    """The tolerance gate of the fast build: after N
    full steps, per-field relative L1 <= 1e-11 and Linf <= 1e-9 against the
    bit-exact strict path (itself pinned to the reference)."""
    from paper_1607_02214_b200 import configs
    mk = {"briowu": lambda **kw: configs.brio_wu(nx=128, **kw),
          "orszag_tang": lambda **kw: configs.orszag_tang(n=64, **kw),
          "blast": lambda **kw: configs.blast(n=32, radius=0.2, **kw),
          "magnetosphere_small": lambda **kw: configs.magnetosphere_small(**kw)}[cfg]
    res = {}
    for prec in ("strict", "fast"):
        c = mk(precision=prec)
        h = _harness(gpu, c.specs, c.options, c.ic)
        h.run(steps)
        res[prec] = h.gather_interior()
    a, b = res["fast"].reshape(-1, 8), res["strict"].reshape(-1, 8)
    n = a.shape[0]
    d = np.abs(a - b)
    l1 = d.sum(0) / np.maximum(np.abs(b).sum(0), n * 1e-12)
    linf = d.max(0) / np.maximum(np.abs(b).max(0), 1e-12)
    assert l1.max() <= FAST_L1 and linf.max() <= FAST_LINF, (l1.max(), linf.max())


def test_pack_unpack_slabs_in_reference_order(gpu):
    """Device halo slabs equal the reference HaloSlab payload order
    (exchange.cpp:30-51: t2 -> t1 -> layer -> 8 scalars) and unpack lands
    them in the receiver's opposite ghost shell (exchange.cpp:53-82)."""
    import ctypes
    import torch
    from paper_1607_02214_b200 import _native as N
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    specs = [AxisSpec.uniform(-1, 1, 10), AxisSpec.uniform(-1, 1, 6), AxisSpec.uniform(-1, 1, 8)]
    h = _harness(gpu, specs, HarnessOptions(), (gpu.IC_PARTITION, ()))
    blk = h.block(0)
    full = blk.download()  # (S2, S1, S0, 8), ghost 4
    g, n = 4, (10, 6, 8)
    for face in range(6):
        a = face // 2
        for layers in (1, 4):
            buf = torch.zeros(n[(a + 1) % 3] * n[(a + 2) % 3] * layers * 8, dtype=torch.float64,
                              device="cuda")
            N.check(N.lib.ppmlr_gpu_block_pack_face(blk.h, face, layers,
                                                    ctypes.c_void_p(buf.data_ptr())))
            N.check(N.lib.ppmlr_gpu_block_synchronize(blk.h))
            lo = g if face % 2 == 0 else g + n[a] - layers
            sl = [slice(g, g + n[2]), slice(g, g + n[1]), slice(g, g + n[0])]
            sl[2 - a] = slice(lo, lo + layers)
            order = {0: (0, 1, 2, 3), 1: (2, 0, 1, 3), 2: (1, 2, 0, 3)}[a]
            want = np.ascontiguousarray(np.transpose(full[tuple(sl)], order)).reshape(-1)
            assert bits_equal(buf.cpu().numpy(), want), (face, layers)
            # unpack into the opposite face's ghost shell
            N.check(N.lib.ppmlr_gpu_block_unpack_face(blk.h, face ^ 1, layers,
                                                      ctypes.c_void_p(buf.data_ptr())))
            N.check(N.lib.ppmlr_gpu_block_synchronize(blk.h))
            after = blk.download()
            lo2 = g + n[a] if (face ^ 1) % 2 == 1 else g - layers
            sl2 = list(sl)
            sl2[2 - a] = slice(lo2, lo2 + layers)
            assert bits_equal(after[tuple(sl2)], full[tuple(sl)]), (face, layers)


def test_distributed_driver_single_rank_nccl(gpu):
    """dist.py on the device with a world-size-1 NCCL group: the block's dt
    slot is all-reduced in place through torch (via __cuda_array_interface__),
    kernels run on torch's stream, and the result equals the in-process
    harness bit for bit.  (Multi-rank exchanges are covered by the gloo test
    tests/test_dist_cpu.py; this pool exposes one GPU.)"""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200 import dist as pdist
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = configs.magnetosphere_small()
        blk = pdist.DeviceRankBlock(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic, 0)
        ex = pdist.Exchanger(blk.info, blk.n, lambda n: torch.empty(n, dtype=torch.float64,
                                                                    device="cuda"))
        pdist.run_rank(blk, ex, 5, 0, cfg.options.cfl, cfg.options.with_sources)
        torch.cuda.synchronize()
        blk.check()
        got = blk.interior()
        blk.close()
    finally:
        dist.destroy_process_group()
    h = _harness(gpu, cfg.specs, cfg.options, cfg.ic)
    h.run(5)
    assert bits_equal(got, h.gather_interior())


@pytest.mark.parametrize("n", [16, 64])
def test_fast_mode_raises_the_reference_failure(gpu, oracle, n):
    """The fast build detects the same unphysical step as the reference:
    same exception type at the same step (cfl 2.5 makes Lagrangian interfaces
    cross), on the runtime tile (16) and the persistent compile-time-tile
    kernel (64).  (The failing zone may differ within the tolerance of the
    fast arithmetic, so only the type and the step are compared.)"""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    cube = [AxisSpec.uniform(-0.5, 0.5, n)] * 3
    ic = (gpu.IC_BLAST, (10.0, 0.1, 0.3))
    ob = _oracle_from_host(oracle, gpu, cube, HarnessOptions(cfl=2.5), ic)
    o, k = oracle.opts(cfl=2.5), oracle.consts()
    err_o = None
    for s in range(20):
        try:
            ob.advance(o, k, s)
        except oracle.OracleError as e:
            err_o = (s, e.kind)
            break
    h = _harness(gpu, cube, HarnessOptions(cfl=2.5, precision="fast"), ic)
    err_g = None
    for s in range(20):
        try:
            h.advance()
        except gpu.Error as e:
            err_g = (s, type(e).__name__)
            break
    assert err_o is not None
    assert err_g is not None and err_g[0] == err_o[0]
    assert err_g[1] == {"StepRejected": "StepRejected", "UnphysicalState": "UnphysicalState"}[
        err_o[1]]

"""The CPU oracle (plain-C restatement, oracle/ppmlr_oracle.c) is pinned to
the reference: bit-for-bit against the golden vectors generated from the
reference build, and — where oracle/_ref exists — against the live reference
on fresh seeded inputs.  CPU only."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import bits_equal, digest, golden_case, run_names


def test_restatement_matches_golden_strips(oracle, golden_strips):
    c = oracle.consts()
    for k in range(int(golden_strips["count"])):
        pre = f"s{k}/"
        n, g, d, dt = golden_strips[pre + "meta"]
        st = golden_strips[pre + "in"].copy()
        bd = golden_strips[pre + "bd"]
        bd = None if bd.size == 0 else bd.copy()
        oracle.orc_sweep_1d(st, bd, golden_strips[pre + "dx"].copy(), int(n), int(g), float(dt),
                            int(d), c)
        assert bits_equal(st, golden_strips[pre + "out"]), f"strip {k}"


def test_restatement_error_strips(oracle, golden_strips):
    errs = json.loads(str(golden_strips["errors"]))
    c = oracle.consts()
    for d in range(3):
        st = golden_strips[f"e{d}/in"].copy()
        with pytest.raises(oracle.OracleError) as ex:
            oracle.orc_sweep_1d(st, None, np.full(24, 0.1), 16, 4, 0.1, d, c)
        assert [ex.value.kind, ex.value.msg] == errs[d]


def _oracle_block(oracle, runs, name, init=None):
    pre = name + "/"
    g = 4
    cen = [runs[pre + f"centers{a}"] for a in range(3)]
    spa = [runs[pre + f"spacings{a}"] for a in range(3)]
    n = [len(c) - 2 * g for c in cen]
    if init is None:
        init = runs[pre + "init"]
    bd = runs[pre + "bd"] if pre + "bd" in runs.files else None
    return oracle.OracleBlock(n, g, cen, spa, [[1, 1]] * 3, init.copy(), bd,
                              runs[pre + "frozen_idx"], runs[pre + "frozen_states"])


@pytest.mark.parametrize("name", run_names())
def test_restatement_matches_golden_runs(oracle, golden_runs, name):
    from paper_1607_02214_b200 import host_block_state
    pre = name + "/"
    specs, opts, ic, steps = golden_case(golden_runs, name)
    init = golden_runs[pre + "init"] if pre + "init" in golden_runs.files else None
    if init is None:  # large init stored by digest: regenerate on the host, pinned by sha
        st = host_block_state(specs, (1, 1, 1), opts, 0, ic)
        init = st["fields"]
        assert digest(init) == str(golden_runs[pre + "init_sha"])
        bd = st["bd"]
    else:
        bd = golden_runs[pre + "bd"] if pre + "bd" in golden_runs.files else None
    blk = _oracle_block(oracle, golden_runs, name, init)
    if bd is not None and blk.bd is None:
        blk.bd = np.ascontiguousarray(bd)
        blk._s.bd = blk.bd.ctypes.data_as(oracle._dp)
    o = oracle.opts(boundary=opts.boundary, cfl=opts.cfl, with_sources=opts.with_sources)
    c = oracle.consts(gamma=opts.gamma)
    dts = [blk.advance(o, c, s) for s in range(steps)]
    assert bits_equal(np.array(dts), golden_runs[pre + "dts"])
    fin = np.ascontiguousarray(blk.interior())
    assert digest(fin) == str(golden_runs[pre + "final_sha"])
    if pre + "final" in golden_runs.files:
        assert bits_equal(fin, golden_runs[pre + "final"])


@pytest.mark.skipif("not __import__('pyoracle').have_ref()")
def test_restatement_vs_live_reference_random_strips(oracle):
    rng = np.random.default_rng(7)
    c = oracle.consts()
    for trial in range(200):
        n = int(rng.integers(1, 48))
        nn = n + 8
        st = np.zeros((nn, 8))
        st[:, 0] = rng.uniform(0.2, 3, nn)
        st[:, 7] = rng.uniform(0.05, 3, nn)
        st[:, 1:4] = rng.uniform(-1.5, 1.5, (nn, 3))
        st[:, 4:7] = rng.uniform(-2, 2, (nn, 3))
        bd = rng.uniform(-2, 2, (nn, 3)) if trial % 2 else None
        dx = rng.uniform(0.3, 2.0, nn)
        d = trial % 3
        # a few oversized steps exercise the error paths
        fac = 3.0 if trial % 17 == 0 else 0.45
        dt = fac * oracle.orc_strip_max_dt(st, bd, dx, n, 4, d, c)
        a, b = st.copy(), st.copy()
        ea = eb = None
        try:
            oracle.ref_sweep_1d(a, bd, dx, n, 4, dt, d)
        except oracle.OracleError as e:
            ea = (e.kind, e.msg)
        try:
            oracle.orc_sweep_1d(b, bd, dx, n, 4, dt, d, c)
        except oracle.OracleError as e:
            eb = (e.kind, e.msg)
        assert ea == eb, trial
        if ea is None:
            assert bits_equal(a, b), trial


@pytest.mark.skipif("not __import__('pyoracle').have_ref()")
def test_restatement_vs_live_reference_pressure_floor(oracle):
    """pressure_floor > 0 disables the Lagrangian checks and floors p."""
    rng = np.random.default_rng(11)
    c = oracle.consts(pressure_floor=1e-3)
    for trial in range(40):
        n = 20
        nn = n + 8
        st = np.zeros((nn, 8))
        st[:, 0] = rng.uniform(0.5, 2, nn)
        st[:, 7] = rng.uniform(1e-4, 0.05, nn)
        st[:, 1:4] = rng.uniform(-2, 2, (nn, 3))
        st[:, 4:7] = rng.uniform(-1, 1, (nn, 3))
        dx = np.full(nn, 0.5)
        dt = 0.45 * oracle.orc_strip_max_dt(st, None, dx, n, 4, 0, c)
        a, b = st.copy(), st.copy()
        ea = eb = None
        try:
            oracle.ref_sweep_1d(a, None, dx, n, 4, dt, 0, pressure_floor=1e-3)
        except oracle.OracleError as e:
            ea = (e.kind, e.msg)
        try:
            oracle.orc_sweep_1d(b, None, dx, n, 4, dt, 0, c)
        except oracle.OracleError as e:
            eb = (e.kind, e.msg)
        assert ea == eb
        if ea is None:
            assert bits_equal(a, b)

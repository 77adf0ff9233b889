"""`ppmlr verify`: the reference's physics suites
(src/verify.cpp) with every step computed by the GPU kernels.  On CPU the
same suite code driven by the C oracle's sweep pins the restated reference
solutions (exact Riemann, HLL tube) and the metric arithmetic against the
reference's own run_suite; on the GPU the metrics must equal the
reference's (strict mode is bit-identical)."""
from __future__ import annotations

import pytest

needs_ref = pytest.mark.skipif("not __import__('pyoracle').have_ref()")


class OracleStrips:
    """The C restatement's sweep_1d / strip_max_dt as the 1-D engine."""

    def __init__(self, oracle):
        self.o = oracle

    def max_dt(self, states, dx, n, gamma):
        return self.o.orc_strip_max_dt(states, None, dx, n, 4, 0, self.o.consts(gamma))

    def sweep(self, states, dx, n, dt, gamma):
        self.o.orc_sweep_1d(states, None, dx, n, 4, dt, 0, self.o.consts(gamma))


@needs_ref
@pytest.mark.parametrize("suite", ["sod", "briowu", "convergence"])
def test_1d_suites_match_reference_metrics_on_cpu(oracle, suite):
    from paper_1607_02214_b200.verify import run_suite
    mine = run_suite(suite, engine=OracleStrips(oracle))
    ref = oracle.ref_run_suite(suite)
    assert [(r.metric, r.passed) for r in mine] == ref


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("suite", ["sod", "briowu", "convergence", "conservation",
                                   "partition"])
def test_gpu_suites_reproduce_reference_metrics(gpu, oracle, suite):
    from paper_1607_02214_b200.verify import run_suite
    mine = run_suite(suite)
    ref = oracle.ref_run_suite(suite)
    assert [(r.metric, r.passed) for r in mine] == ref
    assert all(r.passed for r in mine)


@pytest.mark.gpu
def test_gpu_strip_max_dt_bitwise_vs_oracle(gpu, oracle):
    import numpy as np
    rng = np.random.default_rng(7)
    n, g = 37, 4
    for direction in range(3):
        st = np.zeros((5, n + 2 * g, 8))
        st[..., 0] = rng.uniform(0.5, 2.0, st.shape[:2])
        st[..., 1:7] = rng.uniform(-1.0, 1.0, st.shape[:2] + (6,))
        st[..., 7] = rng.uniform(0.1, 1.0, st.shape[:2])
        bd = rng.uniform(-0.5, 0.5, st.shape[:2] + (3,))
        dx = rng.uniform(0.5, 1.5, n + 2 * g)
        want = min(oracle.orc_strip_max_dt(st[k].copy(), bd[k].copy(), dx, n, g, direction,
                                           oracle.consts()) for k in range(5))
        got = gpu.strip_max_dt(st, bd, dx, n, g, direction)
        assert np.float64(got).view(np.int64) == np.float64(want).view(np.int64)


@pytest.mark.gpu
def test_cli_verify_and_run(gpu, tmp_path, capsys):
    from paper_1607_02214_b200.__main__ import main
    assert main(["verify", "sod"]) == 0
    assert "sod.l1_rho" in capsys.readouterr().out
    assert main(["run", "--config", "mag_small", "--steps", "2", "--cadence", "1",
                 "--out", str(tmp_path)]) == 0
    assert (tmp_path / "snapshot_000002.bin").exists()
    assert main(["verify", "nosuch"]) == 1
    # report (ppmlr_main.cpp:107-139): the reference's CSV header and one
    # row per reference partition shape
    capsys.readouterr()
    assert main(["report", "--steps", "1"]) == 0
    lines = [ln for ln in capsys.readouterr().out.splitlines() if ln]
    assert lines[0] == ("nx,ny,nz,ranks,tde_units,bytes_per_step,mean_compute_s,"
                        "mean_transfer_s,predicted_speedup")
    assert [ln.split(",")[:3] for ln in lines[1:]] == [
        ["3", "1", "1"], ["3", "3", "3"], ["4", "3", "3"], ["6", "3", "3"], ["4", "5", "5"],
        ["6", "5", "5"]]

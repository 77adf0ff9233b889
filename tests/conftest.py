"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; everything else runs
on CPU.  The CPU checkers (oracle/) are test infrastructure only."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def rel_errors(a, b):
    """Per-field relative L1 and Linf of a vs reference b (fields last)."""
    a = a.reshape(-1, a.shape[-1])
    b = b.reshape(-1, b.shape[-1])
    d = np.abs(a - b)
    scale1 = np.maximum(np.abs(b).sum(axis=0), 1e-300)
    scaleinf = np.maximum(np.abs(b).max(axis=0), 1e-300)
    return d.sum(axis=0) / scale1, d.max(axis=0) / scaleinf


@pytest.fixture(scope="session")
def golden_runs():
    return np.load(os.path.join(GOLDEN, "runs.npz"))


@pytest.fixture(scope="session")
def golden_strips():
    return np.load(os.path.join(GOLDEN, "strips.npz"))


@pytest.fixture(scope="session")
def golden_axes():
    return np.load(os.path.join(GOLDEN, "axes.npz"))


@pytest.fixture(scope="session")
def golden_layouts():
    with open(os.path.join(GOLDEN, "layouts.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    return pyoracle


@pytest.fixture(scope="session")
def gpu():
    import paper_1607_02214_b200 as p
    if p.device_count() < 1:
        pytest.skip("no CUDA device visible")
    return p


def run_names():
    return ["briowu", "orszag_tang", "magnetosphere", "magnetosphere_stretched", "blast",
            "partition_ic"]


def golden_case(runs, name):
    """(specs, options kwargs, ic, steps) of a golden run, product types."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    meta = json.loads(str(runs[name + "/opts"]))
    specs = [AxisSpec(*map(float, s[:5]), int(s[5]), float(s[6])) for s in runs[name + "/specs"]]
    opts = HarnessOptions(cfl=meta["cfl"], boundary=meta["boundary"],
                          with_sources=meta["with_sources"], gamma=meta["gamma"],
                          with_dipole=meta["with_dipole"])
    ic = meta["ic"]
    if ic[0] == "mag":
        ic = ("magnetosphere",)
    else:
        ic = (int(ic[0]), tuple(ic[1]))
    return specs, opts, ic, int(meta["steps"])

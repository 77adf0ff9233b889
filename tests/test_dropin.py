"""The C++ drop-in: tests/dropin/gpu_harness.hpp binds
include/ppmlr_gpu.h behind the reference's own RunConfig / Harness API;
dropin_demo steps ppmlr::Harness (the reference build) and GpuHarness side
by side and requires every dt and the final interior to be bit-identical."""
from __future__ import annotations

import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dropin", "dropin_demo")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_demo not built")
@pytest.mark.parametrize("px,ndev", [(1, 1), (2, 1), (4, 1), (4, 4), (8, 3)])
def test_cpp_dropin_bit_identical(gpu, px, ndev):
    out = subprocess.run([BIN, "5", str(px), str(ndev)], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "drop-in OK" in out.stdout

"""Snapshot / gather path and the ledger CSV:
the PPLR files and ledger rows the GPU harness writes are byte-identical to
the reference's (src/snapshot.cpp:58-123, exchange.cpp:84-91,
tools/ppmlr_main.cpp:20-31), checked against the live reference."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits_equal

needs_ref = pytest.mark.skipif("not __import__('pyoracle').have_ref()")

# the survey's 64x36x36 magnetosphere
SPECS = [(-48.0, 28.8, -48.0, 28.8, 1.2, 64, 1.05),
         (-21.6, 21.6, -21.6, 21.6, 1.2, 36, 1.05),
         (-21.6, 21.6, -21.6, 21.6, 1.2, 36, 1.05)]


def _ref_run(oracle, steps, part=(1, 1, 1)):
    ref = oracle.RefHarness(SPECS, part, boundary=2, with_dipole=True)
    ref.init_magnetosphere()
    for _ in range(steps):
        ref.advance()
    return ref


@needs_ref
def test_reader_and_writer_match_reference_files(oracle, tmp_path):
    from paper_1607_02214_b200 import build_axis
    from paper_1607_02214_b200.api import AxisSpec
    from paper_1607_02214_b200.snapshot import read_snapshot, write_snapshot
    ref = _ref_run(oracle, 2)
    path = str(tmp_path / "ref.bin")
    ref.write_snapshot(path)
    snap = read_snapshot(path)
    assert snap.dims == (64, 36, 36) and snap.step == 2 and snap.ghost == 4
    assert snap.time == ref.time()
    assert bits_equal(snap.states(), ref.gather())
    for a in range(3):
        assert bits_equal(snap.edges[a], build_axis(AxisSpec(*SPECS[a])).edges)
    mine = str(tmp_path / "py.bin")
    write_snapshot(mine, snap)
    assert open(mine, "rb").read() == open(path, "rb").read()


@needs_ref
def test_reader_rejects_bad_files_like_reference(oracle, tmp_path):
    from paper_1607_02214_b200 import InvalidSpec
    from paper_1607_02214_b200.snapshot import read_snapshot
    ref = _ref_run(oracle, 0)
    path = str(tmp_path / "ref.bin")
    ref.write_snapshot(path)
    data = open(path, "rb").read()
    cases = {"magic": (b"XXXX" + data[4:], "snapshot: bad magic in"),
             "version": (data[:4] + (2).to_bytes(4, "little") + data[8:],
                         "snapshot: unsupported version 2"),
             "payload": (data[:-8], "snapshot: truncated field payload in")}
    for name, (blob, msg) in cases.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(blob)
        with pytest.raises(InvalidSpec, match=msg):
            read_snapshot(str(p))
    with pytest.raises(InvalidSpec, match="snapshot: cannot open"):
        read_snapshot(str(tmp_path / "absent.bin"))


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("part", [(1, 1, 1), (2, 1, 1), (2, 3, 3)])
def test_gpu_snapshot_and_ledger_bytes_equal_reference(gpu, oracle, tmp_path, part):
    """The file ppmlr run would write, and its ledger.csv, byte for byte."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    specs = [AxisSpec(*s) for s in SPECS]
    h = gpu.Harness(specs, part, HarnessOptions(boundary=gpu.MAGNETOSPHERE, with_dipole=True))
    h.init_magnetosphere()
    h.run(3)
    ref = _ref_run(oracle, 3, part)
    mine, theirs = str(tmp_path / "gpu.bin"), str(tmp_path / "ref.bin")
    h.write_snapshot(mine)
    ref.write_snapshot(theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    assert h.ledger_csv() == ref.ledger_csv()


@pytest.mark.gpu
@needs_ref
def test_async_snapshot_holds_the_captured_step(gpu, oracle, tmp_path):
    """write_snapshot(wait=False) captures on the device; stepping on while
    the host drains it does not change the file."""
    from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
    specs = [AxisSpec(*s) for s in SPECS]
    h = gpu.Harness(specs, (2, 1, 1), HarnessOptions(boundary=gpu.MAGNETOSPHERE,
                                                     with_dipole=True))
    h.init_magnetosphere()
    h.run(2)
    mine = str(tmp_path / "gpu.bin")
    h.write_snapshot(mine, wait=False)
    h.run(3)
    h.snapshot_wait()
    theirs = str(tmp_path / "ref.bin")
    _ref_run(oracle, 2, (2, 1, 1)).write_snapshot(theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    with pytest.raises(gpu.InvalidSpec, match="snapshot: cannot open for writing"):
        h.write_snapshot(str(tmp_path / "no" / "such" / "dir.bin"))


@pytest.mark.gpu
def test_cmd_run_writes_cadence_snapshots_ledger_and_timing(gpu, tmp_path):
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200.run import cmd_run
    from paper_1607_02214_b200.snapshot import read_snapshot
    cfg = configs.magnetosphere_small()
    out = str(tmp_path / "run")
    h, line = cmd_run(cfg, steps=5, cadence=2, out_dir=out, quiet=True)
    names = sorted(os.listdir(out))
    assert names == ["ledger.csv", "snapshot_000002.bin", "snapshot_000004.bin",
                     "snapshot_000005.bin", "timing.csv"]
    last = read_snapshot(os.path.join(out, "snapshot_000005.bin"))
    assert last.step == 5 and bits_equal(last.states(), h.gather_interior())
    assert len(open(os.path.join(out, "ledger.csv")).read().splitlines()) == 1 + 5 * 4
    assert len(open(os.path.join(out, "timing.csv")).read().splitlines()) == 1 + 5
    assert line.startswith("steps=5 time=")

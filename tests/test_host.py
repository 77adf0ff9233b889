"""Host-side pieces of the drop-in boundary, CPU only: the C-ABI library
loads and exports every symbol include/ppmlr_gpu.h declares; geometry,
decomposition, initial conditions and block geometry are bit-identical to
the reference (golden vectors from the reference build)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_1607_02214_b200 as P
from paper_1607_02214_b200 import _native
from paper_1607_02214_b200.api import AxisSpec, HarnessOptions
from conftest import bits_equal, digest, golden_case, run_names


def test_library_exports_every_header_symbol():
    names = _native.exported_symbols_from_header()
    assert len(names) > 40
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = {ln.split(".")[-2] for ln in out.stdout.splitlines() if ".cubin" in ln}
    assert archs == {"sm_100a"}, archs


def _spec(arr):
    return AxisSpec(*map(float, arr[:5]), int(arr[5]), float(arr[6]))


def test_build_axis_matches_reference(golden_axes):
    keys = sorted({k.split("/")[0] for k in golden_axes.files})
    for k in keys:
        ax = P.build_axis(_spec(golden_axes[k + "/spec"]))
        assert bits_equal(ax.edges, golden_axes[k + "/edges"]), k
        assert bits_equal(ax.centers, golden_axes[k + "/centers"]), k
        assert bits_equal(ax.spacings, golden_axes[k + "/spacings"]), k


def test_build_axis_errors_match_reference(golden_layouts):
    from tests_golden_specs import BAD_AXES
    for k, spec in BAD_AXES.items():
        want = golden_layouts["axis_errors"][k]
        with pytest.raises(P.InvalidSpec) as ex:
            P.build_axis(AxisSpec(*spec[:5], int(spec[5]), spec[6]))
        assert [type(ex.value).__name__, str(ex.value)] == want


def test_layout_matches_reference(golden_layouts):
    from tests_golden_specs import AXES
    grids = {"default": [AXES["default_x"], AXES["default_yz"], AXES["default_yz"]],
             "c3": [AXES["c3_x"], AXES["default_yz"], AXES["default_yz"]],
             "c5": [AXES["c5_x"], AXES["c5_yz"], AXES["c5_yz"]]}
    for e in golden_layouts["layouts"]:
        specs = [AxisSpec(*s[:5], int(s[5]), s[6]) for s in grids[e["grid"]]]
        part = tuple(e["partition"])
        if "error" in e:
            with pytest.raises(P.InvalidSpec) as ex:
                P.layout(specs, part)
            assert [type(ex.value).__name__, str(ex.value)] == e["error"], part
            continue
        blocks, iono = P.layout(specs, part)
        assert iono == e["ionosphere_rank"]
        got = [[b.rank, *b.coords, *b.lo, *b.n, *b.neighbor] for b in blocks]
        assert got == e["blocks"], part


def test_rank_counts_and_pair_model():
    """acceptance.cpp criteria 1-2 inputs: rank counts and tde_units."""
    want = {(3, 1, 1): 4, (3, 3, 3): 28, (4, 3, 3): 37, (6, 3, 3): 55, (4, 5, 5): 101,
            (6, 5, 5): 151}
    for part, ranks in want.items():
        assert part[0] * part[1] * part[2] + 1 == ranks
    for c in [(1, 1, 1), (3, 1, 1), (3, 3, 3), (4, 3, 3), (6, 5, 5)]:
        brute = sum((x + 1 < c[0]) + (y + 1 < c[1]) + (z + 1 < c[2])
                    for z in range(c[2]) for y in range(c[1]) for x in range(c[0]))
        assert P.tde_units(c) == brute


def test_exchanged_bytes_model():
    cube = [AxisSpec.uniform(-2.4, 2.4, 12)] * 3
    # (2,1,1): one x-face pair, 12*12 face cells, 4 layers, 64 B, both ways
    assert P.exchanged_bytes(cube, (2, 1, 1), 4, 64) == 1 * 144 * 4 * 64 * 2
    # (2,3,3): x pairs 9 * 16 cells; y pairs 2*2*3 of 6*4 ... evaluated in closed form
    want = 0
    cnt = (2, 3, 3)
    cells = (12, 12, 12)
    for a in range(3):
        b, c = (a + 1) % 3, (a + 2) % 3
        want += (cnt[a] - 1) * cnt[b] * cnt[c] * (cells[b] // cnt[b]) * (cells[c] // cnt[c]) * 4 * 64 * 2
    assert P.exchanged_bytes(cube, cnt, 4, 64) == want


@pytest.mark.parametrize("name", run_names())
def test_host_initial_state_matches_reference(golden_runs, name):
    """make_block geometry, dipole, init_magnetosphere / init_with and the
    frozen core exactly as the reference builds them."""
    pre = name + "/"
    specs, opts, ic, _ = golden_case(golden_runs, name)
    st = P.host_block_state(specs, (1, 1, 1), opts, 0, ic)
    assert digest(st["fields"]) == str(golden_runs[pre + "init_sha"])
    if pre + "init" in golden_runs.files:
        assert bits_equal(st["fields"], golden_runs[pre + "init"])
    if pre + "bd_sha" in golden_runs.files:
        assert digest(st["bd"]) == str(golden_runs[pre + "bd_sha"])
    assert np.array_equal(st["frozen_idx"], golden_runs[pre + "frozen_idx"])
    assert bits_equal(st["frozen_states"].reshape(-1, 8),
                      golden_runs[pre + "frozen_states"].reshape(-1, 8))
    for a in range(3):
        assert bits_equal(st["centers"][a], golden_runs[pre + f"centers{a}"])
        assert bits_equal(st["spacings"][a], golden_runs[pre + f"spacings{a}"])


@pytest.mark.skipif("not __import__('pyoracle').have_ref()")
def test_partitioned_block_geometry_matches_reference(oracle):
    """Per-rank ghost-extended geometry (local_axis) and ICs of a split
    layout, against the live reference harness."""
    specs = [(-48.0, 28.8, -48.0, 28.8, 1.2, 64, 1.05),
             (-21.6, 21.6, -21.6, 21.6, 1.2, 36, 1.05),
             (-21.6, 21.6, -21.6, 21.6, 1.2, 36, 1.05)]
    for part in [(2, 1, 1), (4, 1, 1), (2, 3, 3)]:
        ref = oracle.RefHarness(specs, part, boundary=2, with_dipole=True)
        ref.init_magnetosphere()
        aspecs = [AxisSpec(*s[:5], s[5], s[6]) for s in specs]
        opts = HarnessOptions(boundary=2, with_dipole=True)
        for r in range(ref.blocks()):
            st = P.host_block_state(aspecs, part, opts, r, ("magnetosphere",))
            for a in range(3):
                c, s = ref.axis(r, a)
                assert bits_equal(st["centers"][a], c)
                assert bits_equal(st["spacings"][a], s)
            assert bits_equal(st["fields"], ref.fields(r))
            assert bits_equal(st["bd"], ref.bd(r))
            fi, fs = ref.frozen(r)
            assert np.array_equal(st["frozen_idx"], fi)


def test_invalid_partition_reports_every_violation():
    specs = [AxisSpec(-100, 30, -10, 10, 0.4, 156), AxisSpec(-100, 100, -10, 10, 0.4, 150),
             AxisSpec(-100, 100, -10, 10, 0.4, 150)]
    with pytest.raises(P.InvalidSpec) as ex:
        P.layout(specs, (8, 2, 1))
    msg = str(ex.value)
    assert "ny = 2 is even" in msg and "x ranks 8 do not divide 156 cells" in msg

"""bench.py's reference arm (the reference's own CPU build on the host
cores) runs without a GPU; its JSON line carries the contract's keys."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif("not __import__('pyoracle').have_ref()")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl",
                          "reference", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["workload"] == "blast_512^3x1"
    assert line["cpu_baseline"]["extrapolated"] is True


@pytest.mark.skipif("not __import__('pyoracle').have_ref()")
def test_reference_arm_loads_no_product_code():
    """The reference arm must time the reference alone: the product package
    is never imported and its native library never mapped."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', "
            "'briowu']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_MOD', any(m.startswith('paper_1607_02214_b200') for m in sys.modules)); "
            "print('PRODUCT_SO', 'libppmlr_b200' in maps); print('REF_SO', 'libppmlr_ref' in maps)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "PRODUCT_MOD False" in out.stdout and "PRODUCT_SO False" in out.stdout
    assert "REF_SO True" in out.stdout


def test_workload_names_match_the_configs():
    """bench.workload() (import-free, used by both arms) names exactly the
    grid our arm runs."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    for name in ("blast512", "blast64", "ot512", "mag160", "mag1024", "briowu"):
        for g in (1, 2, 8):
            if name == "mag1024" and g == 1:
                continue
            cfg, kind = b.make_config(name, g)
            k2, wl = b.workload(name, g)
            assert k2 == kind and wl["workload"] == cfg.name, (name, g)
            if name.startswith("blast"):
                assert wl["grid"] == [int(s.cells) for s in cfg.specs]


def _run_json(cmd):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "clocks",
        "e2e", "gpu_launches", "roofline")


@pytest.mark.gpu
def test_bench_line_single_gpu(gpu):
    line = _run_json([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "blast64",
                      "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    for key in KEYS:
        assert key in line, key
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    r = line["roofline"]
    assert r["bound"] in ("fp64", "hbm") and 0 < r["frac"] < 1


@pytest.mark.gpu
def test_bench_line_distributed_single_rank(gpu):
    """The torchrun arm (one rank per GPU over NCCL) on the one visible GPU."""
    line = _run_json([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                      "--nproc-per-node", "1", "--master-addr", "127.0.0.1", "--master-port",
                      "29533", os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config",
                      "blast64", "--steps", "3", "--warmup", "3", "--force-dist"])
    for key in KEYS:
        assert key in line, key
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert 0 < line["roofline"]["frac"] < 1

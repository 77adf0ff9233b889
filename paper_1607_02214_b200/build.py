"""In-tree build of the native library (sm_100a) and of the CPU checkers.

``python paper_1607_02214_b200/build.py`` (or ``__graft_entry__.build()``; it must
not import the package, whose import requires the built library)
produces ``paper_1607_02214_b200/libppmlr_b200.so`` with nvcc for
``-gencode arch=compute_100a,code=sm_100a``.  The strict translation units
are compiled with ``--fmad=false`` (bit parity with the reference); the fast
sweep with FMA contraction.  Host C++ uses ``-ffp-contract=off`` because the
geometry tables it computes feed the bit-exact kernels.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libppmlr_b200.so")
OBJ = os.path.join(PKG, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

UNITS = [
    # (source, fmad, extra)
    ("block.cu", False, []),
    ("sweep_strict.cu", False, []),
    ("sweep_fast.cu", True, []),
    ("sources_strict.cu", False, []),
    ("sources_fast.cu", True, []),
]
HOST_UNITS = ["host.cpp"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "ppmlr_gpu.h"), __file__]


def build_native(force=False, verbose_ptxas=False, defines=(), out=OUT, objdir=OBJ):
    """Compile and link the native library; `defines` / `out` / `objdir`
    build tuning variants side by side (tools/variants.py)."""
    os.makedirs(objdir, exist_ok=True)
    deps = _deps()
    objs = []
    for src, fmad, extra in UNITS:
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, deps):
            cmd = [NVCC, "-std=c++17", *ARCH, "-O3", "-lineinfo",
                   f"--fmad={'true' if fmad else 'false'}",
                   "-Xcompiler", "-fPIC,-ffp-contract=off", "-c", os.path.join(CSRC, src),
                   "-o", o, *extra, *[f"-D{d}" for d in defines]]
            if verbose_ptxas:
                cmd += ["-Xptxas", "-v"]
            # tuning experiments (tools/variants.py): extra nvcc flags
            cmd += os.environ.get("PPMLR_NVCC_EXTRA", "").split()
            _run(cmd)
    for src in HOST_UNITS:
        o = os.path.join(objdir, src.replace(".cpp", ".o"))
        objs.append(o)
        if force or _stale(o, deps):
            cuda_inc = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
            _run(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off",
                  f"-I{cuda_inc}", "-c", os.path.join(CSRC, src), "-o", o])
    if force or _stale(out, objs):
        _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart"])
    return out


def build_oracle():
    """CPU checkers (test infrastructure): oracle/liboracle.so always,
    oracle/_ref/libppmlr_ref.so when /root/reference is present."""
    _run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "all"])
    # the C++ drop-in check (tests/dropin): the reference's RunConfig drives
    # ppmlr::Harness and the GPU binding side by side
    if os.path.exists(OUT):
        _run(["make", "-C", os.path.join(ROOT, "tests", "dropin"), "all"])


def build_all(force=False):
    build_native(force=force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

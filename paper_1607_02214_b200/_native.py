"""ctypes binding of ``libppmlr_b200.so`` (include/ppmlr_gpu.h).

There is no CPU fallback: if the native library is missing this module
raises at import time, and every entry point runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PPMLR_LIB selects a tuning variant built by tools/variants.py (same ABI).
LIB_PATH = os.environ.get("PPMLR_LIB") or os.path.join(_HERE, "libppmlr_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1607_02214_b200/build.py` "
        "(nvcc, sm_100a).  There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p


# ---------------------------------------------------------------- errors
# ppmlr::Error hierarchy (proj/include/ppmlr/errors.hpp:9-30)

class Error(RuntimeError):
    """Base of all solver errors."""


class InvalidSpec(Error):
    pass


class UnphysicalState(Error):
    pass


class StepRejected(Error):
    pass


class OutOfRange(Error):
    pass


class RuntimeFailure(Error):
    """CUDA / driver failure."""


_BY_CODE = {1: InvalidSpec, 2: UnphysicalState, 3: StepRejected, 4: OutOfRange,
            5: RuntimeFailure}


def last_error() -> str:
    return lib.ppmlr_gpu_last_error().decode(errors="replace")


def check(rc: int):
    if rc:
        raise _BY_CODE.get(rc, Error)(last_error())


# ---------------------------------------------------------------- structs

class AxisSpecC(C.Structure):
    _fields_ = [("min", C.c_double), ("max", C.c_double), ("uniform_lo", C.c_double),
                ("uniform_hi", C.c_double), ("d_uniform", C.c_double), ("cells", C.c_int),
                ("ratio", C.c_double)]


class BlockDesc(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("lo", C.c_int * 3), ("ghost", C.c_int),
                ("centers", _dp * 3), ("spacings", _dp * 3), ("physical", (C.c_int * 2) * 3),
                ("gamma", C.c_double), ("mu0", C.c_double), ("pressure_floor", C.c_double),
                ("boundary", C.c_int), ("wind_rho", C.c_double), ("wind_p", C.c_double),
                ("wind_v", C.c_double * 3), ("wind_imf", C.c_double * 3),
                ("with_dipole", C.c_int), ("precision", C.c_int), ("device", C.c_int)]


class OptionsC(C.Structure):
    _fields_ = [("cfl", C.c_double), ("ghost", C.c_int), ("boundary", C.c_int),
                ("transport", C.c_int), ("with_sources", C.c_int), ("with_dipole", C.c_int),
                ("wind_rho", C.c_double), ("wind_p", C.c_double),
                ("wind_v", C.c_double * 3), ("wind_imf", C.c_double * 3),
                ("mu0", C.c_double), ("gamma", C.c_double), ("pressure_floor", C.c_double),
                ("precision", C.c_int), ("device", C.c_int)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_BP = _vp  # opaque handles
_sig("ppmlr_gpu_last_error", C.c_char_p)
_sig("ppmlr_gpu_version", C.c_char_p)
_sig("ppmlr_build_axis", C.c_int, C.POINTER(AxisSpecC), _dp, _dp, _dp, C.c_int, _ip)
_sig("ppmlr_layout", C.c_int, C.POINTER(AxisSpecC), C.c_int, C.c_int, C.c_int, _ip, C.c_int,
     _ip, _ip)
_sig("ppmlr_host_block_state", C.c_int, C.POINTER(AxisSpecC), C.c_int, C.c_int, C.c_int,
     C.POINTER(OptionsC), C.c_int, C.c_int, _dp, _dp, _dp, _i64p, _dp, _i64p, _dp, _dp)
_sig("ppmlr_gpu_device_count", C.c_int)
_sig("ppmlr_gpu_fp64_peak", C.c_int, C.c_int, _dp)
_sig("ppmlr_gpu_selftest_division", C.c_int, C.c_int, C.c_longlong, C.c_ulonglong,
     C.POINTER(C.c_longlong), _dp)
_sig("ppmlr_tde_units", C.c_long, C.c_int, C.c_int, C.c_int)
_sig("ppmlr_exchanged_bytes", C.c_uint64, C.POINTER(AxisSpecC), C.c_int, C.c_int, C.c_int,
     C.c_int, C.c_int)
_sig("ppmlr_gpu_block_create", C.c_int, C.POINTER(BlockDesc), C.POINTER(_vp))
_sig("ppmlr_gpu_block_destroy", None, _BP)
_sig("ppmlr_gpu_block_upload", C.c_int, _BP, _dp, _dp, _i64p, _dp, C.c_int64)
_sig("ppmlr_gpu_block_download", C.c_int, _BP, _dp)
_sig("ppmlr_gpu_block_download_interior", C.c_int, _BP, _dp)
_sig("ppmlr_gpu_block_snapshot_capture", C.c_int, _BP)
_sig("ppmlr_gpu_block_snapshot_read", C.c_int, _BP, C.c_int, C.c_int, C.c_int, _dp, C.c_int64,
     C.c_int64)
_sig("ppmlr_gpu_block_compute_dt", C.c_int, _BP, C.c_double, _dp)
_sig("ppmlr_gpu_block_fill_boundaries", C.c_int, _BP, C.c_int, C.c_int)
_sig("ppmlr_gpu_block_sweep", C.c_int, _BP, C.c_int, C.c_double)
_sig("ppmlr_gpu_block_sources", C.c_int, _BP, C.c_double)
_sig("ppmlr_gpu_block_restore_frozen", C.c_int, _BP)
_sig("ppmlr_gpu_block_advance", C.c_int, _BP, C.c_double, C.c_int, C.c_long, _dp)
_sig("ppmlr_gpu_block_run", C.c_int, _BP, C.c_double, C.c_int, C.c_long, C.c_long, _dp)
_sig("ppmlr_gpu_block_pack_face", C.c_int, _BP, C.c_int, C.c_int, _vp)
_sig("ppmlr_gpu_block_unpack_face", C.c_int, _BP, C.c_int, C.c_int, _vp)
_sig("ppmlr_gpu_block_copy_face", C.c_int, _BP, C.c_int, _BP, C.c_int)
_sig("ppmlr_gpu_block_dt_slot", _vp, _BP)
_sig("ppmlr_gpu_block_local_dt_async", C.c_int, _BP, C.c_double)
_sig("ppmlr_gpu_block_begin", C.c_int, _BP, C.c_double, C.c_long)
_sig("ppmlr_gpu_block_sweep_async", C.c_int, _BP, C.c_int, C.c_int)
_sig("ppmlr_gpu_block_end_step", C.c_int, _BP, C.c_double, C.c_int)
_sig("ppmlr_gpu_block_sweep_part", C.c_int, _BP, C.c_int, C.c_int, C.c_int)
_sig("ppmlr_gpu_block_end_step_part", C.c_int, _BP, C.c_double, C.c_int, C.c_int)
_sig("ppmlr_gpu_block_time", C.c_int, _BP, _dp)
_sig("ppmlr_gpu_block_stream", _vp, _BP)
_sig("ppmlr_gpu_block_set_stream", C.c_int, _BP, _vp)
_sig("ppmlr_gpu_block_synchronize", C.c_int, _BP)
_sig("ppmlr_gpu_block_state_view", C.c_int, _BP, C.POINTER(C.c_void_p),
     C.POINTER(C.c_longlong), C.POINTER(C.c_int))
_sig("ppmlr_gpu_block_dipole_view", C.c_int, _BP, C.POINTER(C.c_void_p))
_sig("ppmlr_gpu_block_init_ic", C.c_int, _BP, C.c_int, C.POINTER(C.c_double))
_sig("ppmlr_gpu_block_check", C.c_int, _BP)
_sig("ppmlr_gpu_block_timing", C.c_int, _BP, C.c_int, _dp, _dp, C.POINTER(C.c_long))
_sig("ppmlr_gpu_sweep_strips", C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
     C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int)
_sig("ppmlr_gpu_harness_create", C.c_int, C.POINTER(AxisSpecC), C.c_int, C.c_int, C.c_int,
     C.POINTER(OptionsC), C.POINTER(_vp))
_sig("ppmlr_gpu_harness_create_on", C.c_int, C.POINTER(AxisSpecC), C.c_int, C.c_int, C.c_int,
     C.POINTER(OptionsC), C.POINTER(C.c_int), C.c_int, C.POINTER(_vp))
_sig("ppmlr_gpu_harness_destroy", None, _vp)
_sig("ppmlr_gpu_harness_init_magnetosphere", C.c_int, _vp, C.c_double, C.c_double,
     C.c_double, C.c_double)
_sig("ppmlr_gpu_harness_init_ic", C.c_int, _vp, C.c_int, _dp)
_sig("ppmlr_gpu_harness_set_state", C.c_int, _vp, _dp)
_sig("ppmlr_gpu_harness_compute_dt", C.c_int, _vp, _dp)
_sig("ppmlr_gpu_harness_advance", C.c_int, _vp, _dp)
_sig("ppmlr_gpu_harness_run", C.c_int, _vp, C.c_long)
_sig("ppmlr_gpu_harness_gather", C.c_int, _vp, _dp)
_sig("ppmlr_gpu_harness_step_count", C.c_long, _vp)
_sig("ppmlr_gpu_harness_time", C.c_double, _vp)
_sig("ppmlr_gpu_harness_block_count", C.c_int, _vp)
_sig("ppmlr_gpu_harness_block", _vp, _vp, C.c_int)
_sig("ppmlr_gpu_harness_ledger", None, _vp, C.POINTER(C.c_uint64), C.POINTER(C.c_long),
     C.POINTER(C.c_long))
_sig("ppmlr_gpu_harness_frozen", C.c_int64, _vp, C.c_int, _i64p, _dp)
_sig("ppmlr_gpu_strip_max_dt", C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
     C.c_double, C.c_double, C.c_int, _dp)
_sig("ppmlr_gpu_harness_ledger_entries", C.c_long, _vp, C.POINTER(C.c_long),
     C.POINTER(C.c_int), C.POINTER(C.c_long), C.POINTER(C.c_uint64), C.POINTER(C.c_long),
     C.c_long)
_sig("ppmlr_gpu_harness_snapshot_begin", C.c_int, _vp, C.c_char_p)
_sig("ppmlr_gpu_harness_snapshot_wait", C.c_int, _vp)
_sig("ppmlr_gpu_harness_snapshot", C.c_int, _vp, C.c_char_p)
_sig("ppmlr_gpu_harness_block_geometry", C.c_int, _vp, C.c_int, _ip, _ip, _dp, _dp, _dp)


def ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def exported_symbols_from_header(header_path=None):
    """Every function name declared in include/ppmlr_gpu.h."""
    import re
    header_path = header_path or os.path.join(os.path.dirname(_HERE), "include", "ppmlr_gpu.h")
    text = open(header_path).read()
    return sorted(set(re.findall(r"\b(ppmlr_[a-z0-9_]+)\s*\(", text)))

"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  It wraps

* ``oracle/liboracle.so``       — the plain-C restatement (``ppmlr_oracle.c``)
* ``oracle/_ref/libppmlr_ref.so`` — the reference itself, compiled from the
  unmodified sources in /root/reference by ``oracle/Makefile`` (absent on a
  machine where it was never built).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libppmlr_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)

CODES = {0: "ok", 1: "InvalidSpec", 2: "UnphysicalState", 3: "StepRejected",
         4: "OutOfRange", 5: "Error", 6: "exception"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{CODES.get(code, code)}: {msg}")
        self.code = code
        self.kind = CODES.get(code, str(code))
        self.msg = msg


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


# ---------------------------------------------------------------- restatement

class OrcConsts(C.Structure):
    _fields_ = [("gamma", C.c_double), ("mu0", C.c_double), ("pressure_floor", C.c_double)]


class OrcBlock(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("ghost", C.c_int),
                ("centers", _dp * 3), ("spacings", _dp * 3),
                ("physical", (C.c_int * 2) * 3),
                ("fields", _dp), ("bd", _dp),
                ("frozen_idx", _i64p), ("frozen_states", _dp), ("n_frozen", C.c_int64)]


class OrcOpts(C.Structure):
    _fields_ = [("boundary", C.c_int), ("wind_rho", C.c_double), ("wind_p", C.c_double),
                ("wind_v", C.c_double * 3), ("wind_imf", C.c_double * 3),
                ("cfl", C.c_double), ("with_sources", C.c_int)]


_orc = None


def orc():
    global _orc
    if _orc is None:
        lib = C.CDLL(ORACLE_SO)
        lib.orc_sweep_1d.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int,
                                     C.POINTER(OrcConsts), C.c_char_p, C.c_int]
        lib.orc_strip_max_dt.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(OrcConsts)]
        lib.orc_strip_max_dt.restype = C.c_double
        for name in ("orc_compute_dt",):
            getattr(lib, name).argtypes = [C.POINTER(OrcBlock), C.c_double,
                                           C.POINTER(OrcConsts), _dp, C.c_char_p, C.c_int]
        lib.orc_apply_boundaries.argtypes = [C.POINTER(OrcBlock), C.POINTER(OrcOpts),
                                             C.c_char_p, C.c_int]
        lib.orc_sweep_axis.argtypes = [C.POINTER(OrcBlock), C.c_int, C.c_double,
                                       C.POINTER(OrcConsts), C.c_char_p, C.c_int]
        lib.orc_apply_sources.argtypes = [C.POINTER(OrcBlock), C.c_double,
                                          C.POINTER(OrcConsts), C.c_char_p, C.c_int]
        lib.orc_restore_frozen.argtypes = [C.POINTER(OrcBlock)]
        lib.orc_advance.argtypes = [C.POINTER(OrcBlock), C.POINTER(OrcOpts),
                                    C.POINTER(OrcConsts), C.c_long, _dp, C.c_char_p, C.c_int]
        _orc = lib
    return _orc


def consts(gamma=5.0 / 3.0, mu0=1.0, pressure_floor=0.0):
    return OrcConsts(gamma, mu0, pressure_floor)


def orc_sweep_1d(states, bd, dx, n, ghost, dt, direction, c):
    """In-place sweep of one strip (states AoS (n+2g, 8))."""
    msg = C.create_string_buffer(512)
    rc = orc().orc_sweep_1d(_ptr(states), _ptr(bd), _ptr(dx), n, ghost, dt, direction,
                            C.byref(c), msg, 512)
    if rc:
        raise OracleError(rc, msg.value.decode())


def orc_strip_max_dt(states, bd, dx, n, ghost, direction, c):
    return orc().orc_strip_max_dt(_ptr(states), _ptr(bd), _ptr(dx), n, ghost, direction,
                                  C.byref(c))


class OracleBlock:
    """A whole-domain (or any) block held for the C restatement.

    ``fields`` (S2, S1, S0, 8) float64 AoS, ghost-inclusive, reference index
    order; ``bd`` (S2, S1, S0, 3) or None; geometry per axis ghost-inclusive.
    """

    def __init__(self, n, ghost, centers, spacings, physical, fields, bd=None,
                 frozen_idx=None, frozen_states=None):
        self.n = tuple(int(v) for v in n)
        self.ghost = int(ghost)
        self.centers = [np.ascontiguousarray(c, dtype=np.float64) for c in centers]
        self.spacings = [np.ascontiguousarray(s, dtype=np.float64) for s in spacings]
        self.physical = [[int(p) for p in side] for side in physical]
        self.fields = np.ascontiguousarray(fields, dtype=np.float64)
        self.bd = None if bd is None else np.ascontiguousarray(bd, dtype=np.float64)
        if frozen_idx is None or len(frozen_idx) == 0:
            self.frozen_idx = np.zeros(1, np.int64)
            self.frozen_states = np.zeros((1, 8))
            self.n_frozen = 0
        else:
            self.frozen_idx = np.ascontiguousarray(frozen_idx, dtype=np.int64)
            self.frozen_states = np.ascontiguousarray(frozen_states, dtype=np.float64)
            self.n_frozen = len(frozen_idx)
        self._s = OrcBlock()
        self._s.n[:] = self.n
        self._s.ghost = self.ghost
        for a in range(3):
            self._s.centers[a] = _ptr(self.centers[a])
            self._s.spacings[a] = _ptr(self.spacings[a])
            self._s.physical[a][0] = self.physical[a][0]
            self._s.physical[a][1] = self.physical[a][1]
        self._s.fields = _ptr(self.fields)
        self._s.bd = _ptr(self.bd)
        self._s.frozen_idx = _ptr(self.frozen_idx, _i64p)
        self._s.frozen_states = _ptr(self.frozen_states)
        self._s.n_frozen = self.n_frozen

    def _call(self, fn, *args):
        msg = C.create_string_buffer(512)
        rc = fn(C.byref(self._s), *args, msg, 512)
        if rc:
            raise OracleError(rc, msg.value.decode())

    def compute_dt(self, cfl, c):
        out = C.c_double()
        self._call(orc().orc_compute_dt, cfl, C.byref(c), C.byref(out))
        return out.value

    def apply_boundaries(self, o):
        self._call(orc().orc_apply_boundaries, C.byref(o))

    def sweep_axis(self, axis, dt, c):
        self._call(orc().orc_sweep_axis, axis, dt, C.byref(c))

    def apply_sources(self, dt, c):
        self._call(orc().orc_apply_sources, dt, C.byref(c))

    def restore_frozen(self):
        orc().orc_restore_frozen(C.byref(self._s))

    def advance(self, o, c, step):
        out = C.c_double()
        self._call(orc().orc_advance, C.byref(o), C.byref(c), step, C.byref(out))
        return out.value

    def interior(self):
        g = self.ghost
        nx, ny, nz = self.n
        return self.fields[g:g + nz, g:g + ny, g:g + nx, :]


def opts(boundary=0, wind_rho=1.0, wind_p=0.1, wind_v=(-1.0, 0.0, 0.0),
         wind_imf=(0.0, 0.0, 0.0), cfl=0.5, with_sources=True):
    o = OrcOpts()
    o.boundary = boundary
    o.wind_rho = wind_rho
    o.wind_p = wind_p
    o.wind_v[:] = wind_v
    o.wind_imf[:] = wind_imf
    o.cfl = cfl
    o.with_sources = int(with_sources)
    return o


# ---------------------------------------------------------------- reference

class RefAxisSpec(C.Structure):
    _fields_ = [("min", C.c_double), ("max", C.c_double), ("uniform_lo", C.c_double),
                ("uniform_hi", C.c_double), ("d_uniform", C.c_double), ("cells", C.c_int),
                ("ratio", C.c_double)]


class RefOptions(C.Structure):
    _fields_ = [("cfl", C.c_double), ("ghost", C.c_int), ("boundary", C.c_int),
                ("transport", C.c_int), ("with_sources", C.c_int), ("with_dipole", C.c_int),
                ("wind_rho", C.c_double), ("wind_p", C.c_double),
                ("wind_v", C.c_double * 3), ("wind_imf", C.c_double * 3),
                ("mu0", C.c_double), ("gamma", C.c_double), ("pressure_floor", C.c_double)]


_ref = None


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        vp = C.c_void_p
        lib.ref_build_axis.argtypes = [C.POINTER(RefAxisSpec), _dp, _dp, _dp, C.c_int, _ip,
                                       C.c_char_p, C.c_int]
        lib.ref_sweep_1d.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int,
                                     C.c_double, C.c_double, C.c_double, C.c_char_p, C.c_int]
        lib.ref_strip_max_dt.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int,
                                         C.c_double, C.c_double]
        lib.ref_strip_max_dt.restype = C.c_double
        lib.ref_layout.argtypes = [C.POINTER(RefAxisSpec), C.c_int, C.c_int, C.c_int, _ip,
                                   C.c_int, _ip, _ip, C.c_char_p, C.c_int]
        lib.ref_harness_create.argtypes = [C.POINTER(RefAxisSpec), C.c_int, C.c_int, C.c_int,
                                           C.POINTER(RefOptions), C.c_char_p, C.c_int]
        lib.ref_harness_create.restype = vp
        lib.ref_harness_destroy.argtypes = [vp]
        lib.ref_harness_block_count.argtypes = [vp]
        lib.ref_harness_block_dims.argtypes = [vp, C.c_int, _ip, _ip, _ip]
        lib.ref_harness_block_axis.argtypes = [vp, C.c_int, C.c_int, _dp, _dp]
        lib.ref_harness_get_fields.argtypes = [vp, C.c_int, _dp]
        lib.ref_harness_set_fields.argtypes = [vp, C.c_int, _dp]
        lib.ref_harness_get_bd.argtypes = [vp, C.c_int, _dp]
        lib.ref_harness_frozen_count.argtypes = [vp, C.c_int]
        lib.ref_harness_frozen_count.restype = C.c_int64
        lib.ref_harness_get_frozen.argtypes = [vp, C.c_int, _i64p, _dp]
        lib.ref_harness_init_magnetosphere.argtypes = [vp, C.c_double, C.c_double, C.c_double,
                                                       C.c_double, C.c_char_p, C.c_int]
        lib.ref_harness_init_ic.argtypes = [vp, C.c_int, _dp, C.c_char_p, C.c_int]
        lib.ref_harness_advance.argtypes = [vp, _dp, C.c_char_p, C.c_int]
        lib.ref_harness_compute_dt.argtypes = [vp, _dp, C.c_char_p, C.c_int]
        lib.ref_harness_gather.argtypes = [vp, _dp]
        lib.ref_harness_step.argtypes = [vp]
        lib.ref_harness_step.restype = C.c_long
        lib.ref_harness_time.argtypes = [vp]
        lib.ref_harness_time.restype = C.c_double
        lib.ref_harness_ledger_bytes.argtypes = [vp]
        lib.ref_harness_ledger_bytes.restype = C.c_uint64
        lib.ref_harness_ledger_messages.argtypes = [vp]
        lib.ref_harness_ledger_messages.restype = C.c_long
        lib.ref_harness_ledger_copy_events.argtypes = [vp]
        lib.ref_harness_ledger_copy_events.restype = C.c_long
        lib.ref_harness_ledger_entries.argtypes = [vp] + [C.c_void_p] * 5 + [C.c_long]
        lib.ref_harness_ledger_entries.restype = C.c_long
        lib.ref_harness_write_snapshot.argtypes = [vp, C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_run_suite.argtypes = [C.c_char_p, _dp, C.POINTER(C.c_int), C.c_int,
                                      C.c_char_p, C.c_int]
        lib.ref_bench.argtypes = [C.POINTER(RefAxisSpec), C.POINTER(RefOptions), C.c_int, _dp,
                                  C.c_int, C.c_int, _dp, _dp, C.c_char_p, C.c_int]
        _ref = lib
    return _ref


def ref_axis_specs(specs):
    arr = (RefAxisSpec * 3)()
    for a, s in enumerate(specs):
        arr[a] = RefAxisSpec(*[float(v) for v in s[:5]], int(s[5]), float(s[6]))
    return arr


def ref_options(cfl=0.5, ghost=4, boundary=0, transport=1, with_sources=True,
                with_dipole=False, wind_rho=1.0, wind_p=0.1, wind_v=(-1.0, 0.0, 0.0),
                wind_imf=(0.0, 0.0, 0.0), mu0=1.0, gamma=5.0 / 3.0, pressure_floor=0.0):
    o = RefOptions()
    o.cfl, o.ghost, o.boundary, o.transport = cfl, ghost, boundary, transport
    o.with_sources, o.with_dipole = int(with_sources), int(with_dipole)
    o.wind_rho, o.wind_p = wind_rho, wind_p
    o.wind_v[:] = wind_v
    o.wind_imf[:] = wind_imf
    o.mu0, o.gamma, o.pressure_floor = mu0, gamma, pressure_floor
    return o


def ref_build_axis(spec):
    cap = int(spec[5]) + 8
    e, c, s = np.zeros(cap + 1), np.zeros(cap), np.zeros(cap)
    n = C.c_int()
    msg = C.create_string_buffer(512)
    rc = ref().ref_build_axis(C.byref(ref_axis_specs([spec] * 3)[0]), _ptr(e), _ptr(c),
                              _ptr(s), cap, C.byref(n), msg, 512)
    if rc:
        raise OracleError(rc, msg.value.decode())
    k = n.value
    return e[:k + 1].copy(), c[:k].copy(), s[:k].copy()


def ref_sweep_1d(states, bd, dx, n, ghost, dt, direction, gamma=5.0 / 3.0, mu0=1.0,
                 pressure_floor=0.0):
    msg = C.create_string_buffer(512)
    rc = ref().ref_sweep_1d(_ptr(states), _ptr(bd), _ptr(dx), n, ghost, dt, direction, gamma,
                            mu0, pressure_floor, msg, 512)
    if rc:
        raise OracleError(rc, msg.value.decode())


def ref_layout(specs, px, py, pz):
    buf = np.zeros(16 * px * py * pz, dtype=np.int32)
    nb, iono = C.c_int(), C.c_int()
    msg = C.create_string_buffer(1024)
    rc = ref().ref_layout(ref_axis_specs(specs), px, py, pz, _ptr(buf, _ip), px * py * pz,
                          C.byref(nb), C.byref(iono), msg, 1024)
    if rc:
        raise OracleError(rc, msg.value.decode())
    return buf.reshape(-1, 16)[:nb.value].copy(), iono.value


class RefHarness:
    """The reference ppmlr::Harness (unmodified sources) behind the shim."""

    def __init__(self, specs, partition=(1, 1, 1), **kw):
        self.specs = specs
        self._o = ref_options(**kw)
        msg = C.create_string_buffer(1024)
        self.h = ref().ref_harness_create(ref_axis_specs(specs), *partition, C.byref(self._o),
                                          msg, 1024)
        if not self.h:
            raise OracleError(1, msg.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_harness_destroy(self.h)
            self.h = None

    def _chk(self, rc, msg):
        if rc:
            raise OracleError(rc, msg.value.decode())

    def blocks(self):
        return ref().ref_harness_block_count(self.h)

    def dims(self, r=0):
        n, lo, g = (C.c_int * 3)(), (C.c_int * 3)(), C.c_int()
        ref().ref_harness_block_dims(self.h, r, n, lo, C.byref(g))
        return tuple(n), tuple(lo), g.value

    def axis(self, r, a):
        n, lo, g = self.dims(r)
        span = n[a] + 2 * g
        c, s = np.zeros(span), np.zeros(span)
        ref().ref_harness_block_axis(self.h, r, a, _ptr(c), _ptr(s))
        return c, s

    def shape(self, r=0):
        n, _, g = self.dims(r)
        return (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g)

    def fields(self, r=0):
        out = np.zeros(self.shape(r) + (8,))
        ref().ref_harness_get_fields(self.h, r, _ptr(out))
        return out

    def set_fields(self, r, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert f.shape == self.shape(r) + (8,)
        ref().ref_harness_set_fields(self.h, r, _ptr(f))

    def bd(self, r=0):
        out = np.zeros(self.shape(r) + (3,))
        ref().ref_harness_get_bd(self.h, r, _ptr(out))
        return out

    def frozen(self, r=0):
        k = ref().ref_harness_frozen_count(self.h, r)
        idx, st = np.zeros(max(k, 1), np.int64), np.zeros((max(k, 1), 8))
        ref().ref_harness_get_frozen(self.h, r, _ptr(idx, _i64p), _ptr(st))
        return idx[:k].copy(), st[:k].copy()

    def init_magnetosphere(self, rho_core=1.0, p_core=0.1, falloff=3.0, r_ref=3.0):
        msg = C.create_string_buffer(512)
        self._chk(ref().ref_harness_init_magnetosphere(self.h, rho_core, p_core, falloff,
                                                       r_ref, msg, 512), msg)

    def init_ic(self, kind, params=()):
        p = np.zeros(8)
        p[:len(params)] = params
        msg = C.create_string_buffer(512)
        self._chk(ref().ref_harness_init_ic(self.h, kind, _ptr(p), msg, 512), msg)

    def advance(self):
        dt = C.c_double()
        msg = C.create_string_buffer(1024)
        self._chk(ref().ref_harness_advance(self.h, C.byref(dt), msg, 1024), msg)
        return dt.value

    def compute_dt(self):
        dt = C.c_double()
        msg = C.create_string_buffer(1024)
        self._chk(ref().ref_harness_compute_dt(self.h, C.byref(dt), msg, 1024), msg)
        return dt.value

    def gather(self):
        nx, ny, nz = (int(s[5]) for s in self.specs)
        out = np.zeros((nz, ny, nx, 8))
        ref().ref_harness_gather(self.h, _ptr(out))
        return out

    def step(self):
        return ref().ref_harness_step(self.h)

    def time(self):
        return ref().ref_harness_time(self.h)

    def ledger(self):
        return (ref().ref_harness_ledger_bytes(self.h), ref().ref_harness_ledger_messages(self.h),
                ref().ref_harness_ledger_copy_events(self.h))

    def ledger_csv(self):
        """TransferLedger::to_csv (exchange.cpp:84-91) of the reference's entries."""
        n = ref().ref_harness_ledger_entries(self.h, None, None, None, None, None, 0)
        st, tr, ms = (C.c_long * n)(), (C.c_int * n)(), (C.c_long * n)()
        by, ev = (C.c_uint64 * n)(), (C.c_long * n)()
        ref().ref_harness_ledger_entries(self.h, st, tr, ms, by, ev, n)
        rows = ["step,transport,messages,bytes,copy_events"]
        rows += [f"{st[i]},{'direct' if tr[i] else 'staged'},{ms[i]},{by[i]},{ev[i]}"
                 for i in range(n)]
        return "\n".join(rows) + "\n"

    def write_snapshot(self, path):
        err = C.create_string_buffer(512)
        self._chk(ref().ref_harness_write_snapshot(self.h, os.fsencode(path), err, 512), err)


def ref_run_suite(name):
    """The reference's verify suite `name`: [(metric, passed), ...]."""
    m, p = np.zeros(8), (C.c_int * 8)()
    err = C.create_string_buffer(512)
    n = ref().ref_run_suite(name.encode(), _ptr(m), p, 8, err, 512)
    if n < 0:
        raise OracleError(-n, err.value.decode())
    return [(float(m[i]), bool(p[i])) for i in range(n)]


def ref_bench(specs, ic_kind, ic_params, threads, steps, **kw):
    p = np.zeros(8)
    p[:len(ic_params)] = ic_params
    o = ref_options(**kw)
    rate, secs = C.c_double(), C.c_double()
    msg = C.create_string_buffer(1024)
    rc = ref().ref_bench(ref_axis_specs(specs), C.byref(o), ic_kind, _ptr(p), threads, steps,
                         C.byref(rate), C.byref(secs), msg, 1024)
    if rc:
        raise OracleError(rc, msg.value.decode())
    return rate.value, secs.value

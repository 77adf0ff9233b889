"""Python mirror of the reference's hot-path API over the C-ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/ppmlr/*.hpp) so tests read like its own:
``build_axis``, ``layout``, ``Harness`` (``advance``, ``run``,
``compute_global_dt``, ``gather_interior`` ...), ``sweep_strips`` (batched
``sweep_1d``).  All numerics run in libppmlr_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import (Error, InvalidSpec, OutOfRange, RuntimeFailure, StepRejected,  # noqa: F401
                      UnphysicalState, check, ptr)

OUTFLOW, PERIODIC, MAGNETOSPHERE = 0, 1, 2
STRICT, FAST = 0, 1
_PRECISION = {"strict": STRICT, "fast": FAST, STRICT: STRICT, FAST: FAST}
_BOUNDARY = {"outflow": OUTFLOW, "periodic": PERIODIC, "magnetosphere": MAGNETOSPHERE,
             OUTFLOW: OUTFLOW, PERIODIC: PERIODIC, MAGNETOSPHERE: MAGNETOSPHERE}

# Synthetic initial conditions (ppmlr_gpu_harness_init_ic kinds)
IC_UNIFORM, IC_BRIOWU, IC_ORSZAG_TANG, IC_BLAST, IC_PARTITION, IC_SMOOTH, IC_GAUSSIAN = range(7)


@dataclass(frozen=True)
class AxisSpec:
    """grid.hpp:9-17"""
    min: float
    max: float
    uniform_lo: float
    uniform_hi: float
    d_uniform: float
    cells: int
    ratio: float = 1.05

    @staticmethod
    def uniform(lo, hi, cells):
        return AxisSpec(lo, hi, lo, hi, (hi - lo) / cells, cells, 1.05)

    def c(self):
        return N.AxisSpecC(float(self.min), float(self.max), float(self.uniform_lo),
                           float(self.uniform_hi), float(self.d_uniform), int(self.cells),
                           float(self.ratio))


def _specs3(specs):
    arr = (N.AxisSpecC * 3)()
    for a, s in enumerate(specs):
        arr[a] = s.c()
    return arr


@dataclass
class Axis:
    edges: np.ndarray
    centers: np.ndarray
    spacings: np.ndarray

    @property
    def n(self):
        return len(self.spacings)


def build_axis(spec: AxisSpec) -> Axis:
    """grid.cpp:61-135 (native restatement, bit-identical)."""
    cap = int(spec.cells) + 8
    e, c, s = np.zeros(cap + 1), np.zeros(cap), np.zeros(cap)
    n = C.c_int()
    check(N.lib.ppmlr_build_axis(C.byref(spec.c()), ptr(e), ptr(c), ptr(s), cap, C.byref(n)))
    k = n.value
    return Axis(e[:k + 1].copy(), c[:k].copy(), s[:k].copy())


@dataclass
class BlockInfo:
    """decomp.hpp:23-29"""
    rank: int
    coords: tuple
    lo: tuple
    n: tuple
    neighbor: tuple


def layout(specs, partition):
    """decomp.cpp:46-86; returns (blocks, ionosphere_rank)."""
    px, py, pz = partition
    cap = max(1, px * py * pz)
    buf = np.zeros(16 * cap, dtype=np.int32)
    nb, iono = C.c_int(), C.c_int()
    check(N.lib.ppmlr_layout(_specs3(specs), px, py, pz, ptr(buf, C.POINTER(C.c_int)), cap,
                             C.byref(nb), C.byref(iono)))
    out = []
    for r in buf.reshape(-1, 16)[:nb.value]:
        out.append(BlockInfo(int(r[0]), tuple(int(v) for v in r[1:4]),
                             tuple(int(v) for v in r[4:7]), tuple(int(v) for v in r[7:10]),
                             tuple(int(v) for v in r[10:16])))
    return out, iono.value


def tde_units(partition):
    return int(N.lib.ppmlr_tde_units(*partition))


def exchanged_bytes(specs, partition, ghost=4, bytes_per_cell=64):
    return int(N.lib.ppmlr_exchanged_bytes(_specs3(specs), *partition, ghost, bytes_per_cell))


@dataclass
class SolarWindParams:
    """stepper.hpp:13-18"""
    rho_sw: float = 1.0
    p_sw: float = 0.1
    v_sw: tuple = (-1.0, 0.0, 0.0)
    imf: tuple = (0.0, 0.0, 0.0)


@dataclass
class HarnessOptions:
    """harness.hpp:34-43 plus the device knobs."""
    cfl: float = 0.5
    ghost: int = 4
    boundary: int = OUTFLOW
    transport: str = "direct"
    with_sources: bool = True
    with_dipole: bool = False
    wind: SolarWindParams = field(default_factory=SolarWindParams)
    gamma: float = 5.0 / 3.0
    mu0: float = 1.0
    pressure_floor: float = 0.0
    precision: str = "strict"
    device: int = 0

    def c(self):
        o = N.OptionsC()
        o.cfl = self.cfl
        o.ghost = self.ghost
        o.boundary = _BOUNDARY[self.boundary]
        o.transport = 0 if self.transport == "staged" else 1
        o.with_sources = int(self.with_sources)
        o.with_dipole = int(self.with_dipole)
        o.wind_rho = self.wind.rho_sw
        o.wind_p = self.wind.p_sw
        o.wind_v[:] = self.wind.v_sw
        o.wind_imf[:] = self.wind.imf
        o.mu0, o.gamma, o.pressure_floor = self.mu0, self.gamma, self.pressure_floor
        o.precision = _PRECISION[self.precision]
        o.device = self.device
        return o


class Block:
    """A device-resident BlockState (non-owning view when from a Harness)."""

    def __init__(self, handle, owner=None, shape=None, ghost=4, device=0):
        self.h = handle
        self.device = device
        self._owner = owner
        self.shape = shape  # interior (nx, ny, nz)
        self.ghost = ghost

    def check(self):
        check(N.lib.ppmlr_gpu_block_check(self.h))

    def sweep(self, axis, dt):
        check(N.lib.ppmlr_gpu_block_sweep(self.h, axis, dt))

    def fill_boundaries(self, axis_mask=7, layers=4):
        check(N.lib.ppmlr_gpu_block_fill_boundaries(self.h, axis_mask, layers))

    def apply_sources(self, dt):
        check(N.lib.ppmlr_gpu_block_sources(self.h, dt))

    def restore_frozen(self):
        check(N.lib.ppmlr_gpu_block_restore_frozen(self.h))

    def compute_dt(self, cfl):
        out = C.c_double()
        check(N.lib.ppmlr_gpu_block_compute_dt(self.h, cfl, C.byref(out)))
        return out.value

    def download_interior(self, out=None):
        nx, ny, nz = self.shape
        if out is None:
            out = np.zeros((nz, ny, nx, 8))
        assert out.flags.c_contiguous and out.dtype == np.float64 and out.size == nx * ny * nz * 8
        check(N.lib.ppmlr_gpu_block_download_interior(self.h, ptr(out)))
        return out

    def upload(self, fields, bd=None, frozen_idx=None, frozen_states=None):
        """Ghost-inclusive AoS state (reference layout) host -> device."""
        assert fields.flags.c_contiguous and fields.dtype == np.float64
        nf = 0 if frozen_idx is None else len(frozen_idx)
        fi = None if nf == 0 else np.ascontiguousarray(frozen_idx, dtype=np.int64)
        fs = None if nf == 0 else np.ascontiguousarray(frozen_states, dtype=np.float64)
        bdc = None if bd is None else np.ascontiguousarray(bd, dtype=np.float64)
        check(N.lib.ppmlr_gpu_block_upload(self.h, ptr(fields), ptr(bdc),
                                           ptr(fi, C.POINTER(C.c_int64)), ptr(fs), nf))

    def download(self):
        nx, ny, nz = self.shape
        g = self.ghost
        out = np.zeros((nz + 2 * g, ny + 2 * g, nx + 2 * g, 8))
        check(N.lib.ppmlr_gpu_block_download(self.h, ptr(out)))
        return out

    def timing(self, enable):
        """(sweep_ms, kernels_enqueued, sweep_launches) since the last call;
        then enables/disables per-sweep event timing (no-graph launches)."""
        sw, tot, n = C.c_double(), C.c_double(), C.c_long()
        check(N.lib.ppmlr_gpu_block_timing(self.h, int(enable), C.byref(sw), C.byref(tot),
                                           C.byref(n)))
        return sw.value, tot.value, n.value

    def stream(self):
        return N.lib.ppmlr_gpu_block_stream(self.h)

    def synchronize(self):
        check(N.lib.ppmlr_gpu_block_synchronize(self.h))

    def state_view(self, interior=True, dipole=False):
        """The device-resident state as 8 torch tensors (z, y, x) viewing the
        library's memory (no copy; valid until the next step or upload);
        dipole=True: the 3 B_d planes instead (None without a dipole) --
        read-only: the y/z sweeps read B_d from brick copies the library
        builds at upload, so B_d changes go through Block.upload."""
        import torch
        pl = (C.c_void_p * 8)()
        st = (C.c_longlong * 3)()
        dims = (C.c_int * 3)()
        g = N.lib.ppmlr_gpu_block_state_view(self.h, pl, st, dims)
        if dipole:
            bp = (C.c_void_p * 3)()
            if not N.lib.ppmlr_gpu_block_dipole_view(self.h, bp):
                return None
            pl = list(bp) + [None] * 5
        out = []
        for f in range(3 if dipole else 8):
            shape = (dims[2], dims[1], dims[0])
            t = torch.as_tensor(_CudaArray(pl[f], shape, (st[2] * 8, st[1] * 8, 8)),
                                device=f"cuda:{self.device}")
            out.append(t[g:-g, g:-g, g:-g] if interior else t)
        return out


class _CudaArray:
    def __init__(self, ptr, shape, strides):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "strides": tuple(strides),
                                         "data": (int(ptr), False), "version": 3}


class Harness:
    """harness.hpp:48-87 on the GPU.  Every block of the layout is resident on
    ``options.device`` or, with ``devices=[...]``, block r on
    ``devices[r % len(devices)]`` (one process driving several GPUs, peer
    access over NVLink).  A whole-domain (1,1,1) layout steps as one CUDA
    graph; multi-block layouts step on per-block streams ordered by events."""

    def __init__(self, specs, partition=(1, 1, 1), options: HarnessOptions | None = None,
                 devices=None):
        self.specs = list(specs)
        self.partition = tuple(partition)
        self.options = options or HarnessOptions()
        h = C.c_void_p()
        if devices is None:
            check(N.lib.ppmlr_gpu_harness_create(_specs3(self.specs), *self.partition,
                                                 C.byref(self.options.c()), C.byref(h)))
        else:
            devs = (C.c_int * len(devices))(*devices)
            check(N.lib.ppmlr_gpu_harness_create_on(_specs3(self.specs), *self.partition,
                                                    C.byref(self.options.c()), devs,
                                                    len(devices), C.byref(h)))
        self.devices = list(devices) if devices is not None else [self.options.device]
        self.h = h
        self.layout, self.ionosphere_rank = layout(self.specs, self.partition)

    def close(self):
        if getattr(self, "h", None):
            N.lib.ppmlr_gpu_harness_destroy(self.h)
            self.h = None

    def __del__(self):
        if getattr(N, "lib", None) is not None:  # not at interpreter teardown
            self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --- initial state -------------------------------------------------
    def init_magnetosphere(self, rho_core=1.0, p_core=0.1, falloff=3.0, r_ref=3.0):
        check(N.lib.ppmlr_gpu_harness_init_magnetosphere(self.h, rho_core, p_core, falloff,
                                                         r_ref))

    def init_with(self, kind, params=()):
        p = np.zeros(8)
        p[:len(params)] = params
        check(N.lib.ppmlr_gpu_harness_init_ic(self.h, kind, ptr(p)))

    def set_state(self, per_block_fields):
        flat = np.concatenate([np.ascontiguousarray(f, dtype=np.float64).ravel()
                               for f in per_block_fields])
        check(N.lib.ppmlr_gpu_harness_set_state(self.h, ptr(flat)))

    # --- stepping --------------------------------------------------------
    def compute_global_dt(self):
        out = C.c_double()
        check(N.lib.ppmlr_gpu_harness_compute_dt(self.h, C.byref(out)))
        return out.value

    def advance(self):
        out = C.c_double()
        check(N.lib.ppmlr_gpu_harness_advance(self.h, C.byref(out)))
        return out.value

    def run(self, steps):
        check(N.lib.ppmlr_gpu_harness_run(self.h, int(steps)))

    # --- observers -------------------------------------------------------
    def step_count(self):
        return int(N.lib.ppmlr_gpu_harness_step_count(self.h))

    def time(self):
        return float(N.lib.ppmlr_gpu_harness_time(self.h))

    def block_count(self):
        return int(N.lib.ppmlr_gpu_harness_block_count(self.h))

    def block(self, rank=0):
        info = self.layout[rank]
        return Block(N.lib.ppmlr_gpu_harness_block(self.h, rank), owner=self, shape=info.n,
                     ghost=self.options.ghost, device=self.devices[rank % len(self.devices)])

    def gather_interior(self):
        nx, ny, nz = (build_axis(s).n for s in self.specs)
        out = np.zeros((nz, ny, nx, 8))
        check(N.lib.ppmlr_gpu_harness_gather(self.h, ptr(out)))
        return out

    def ledger(self):
        b, m, e = C.c_uint64(), C.c_long(), C.c_long()
        N.lib.ppmlr_gpu_harness_ledger(self.h, C.byref(b), C.byref(m), C.byref(e))
        return int(b.value), int(m.value), int(e.value)

    def ledger_entries(self):
        """TransferLedger.entries (exchange.hpp:40-61): one row per
        exchange_step as (step, transport, messages, bytes, copy_events)."""
        n = N.lib.ppmlr_gpu_harness_ledger_entries(self.h, None, None, None, None, None, 0)
        st, tr, ms = (C.c_long * n)(), (C.c_int * n)(), (C.c_long * n)()
        by, ev = (C.c_uint64 * n)(), (C.c_long * n)()
        N.lib.ppmlr_gpu_harness_ledger_entries(self.h, st, tr, ms, by, ev, n)
        return [(int(st[i]), "direct" if tr[i] else "staged", int(ms[i]), int(by[i]),
                 int(ev[i])) for i in range(n)]

    def ledger_csv(self):
        """TransferLedger::to_csv (exchange.cpp:84-91)."""
        rows = ["step,transport,messages,bytes,copy_events"]
        rows += [",".join(str(x) for x in e) for e in self.ledger_entries()]
        return "\n".join(rows) + "\n"

    def write_snapshot(self, path, wait=True):
        """write_snapshot(path, make_snapshot(h)) (snapshot.cpp:58-85,
        ppmlr_main.cpp:20-31).  With wait=False the state is captured on the
        device and the file is written by a host thread while stepping goes
        on; snapshot_wait() (or the next snapshot) joins it."""
        p = os.fsencode(path)
        if wait:
            check(N.lib.ppmlr_gpu_harness_snapshot(self.h, p))
        else:
            check(N.lib.ppmlr_gpu_harness_snapshot_begin(self.h, p))

    def snapshot_wait(self):
        check(N.lib.ppmlr_gpu_harness_snapshot_wait(self.h))

    def frozen(self, rank=0):
        k = N.lib.ppmlr_gpu_harness_frozen(self.h, rank, None, None)
        idx, st = np.zeros(max(k, 1), np.int64), np.zeros((max(k, 1), 8))
        N.lib.ppmlr_gpu_harness_frozen(self.h, rank, ptr(idx, C.POINTER(C.c_int64)), ptr(st))
        return idx[:k].copy(), st[:k].copy()

    def block_geometry(self, rank=0):
        """(centers[3], spacings[3], bd or None) ghost-inclusive, as make_block."""
        info = self.layout[rank]
        g = self.options.ghost
        spans = [info.n[a] + 2 * g for a in range(3)]
        cat_c, cat_s = np.zeros(sum(spans)), np.zeros(sum(spans))
        bd = None
        if self.options.with_dipole:
            bd = np.zeros((spans[2], spans[1], spans[0], 3))
        n, lo = (C.c_int * 3)(), (C.c_int * 3)()
        check(N.lib.ppmlr_gpu_harness_block_geometry(self.h, rank, n, lo, ptr(cat_c),
                                                     ptr(cat_s), ptr(bd)))
        offs = np.cumsum([0] + spans)
        cen = [cat_c[offs[a]:offs[a + 1]] for a in range(3)]
        spc = [cat_s[offs[a]:offs[a + 1]] for a in range(3)]
        return cen, spc, bd


def host_block_state(specs, partition=(1, 1, 1), options: HarnessOptions | None = None,
                     rank=0, ic=("magnetosphere",), fields_out=None, bd_out=None):
    """Host-side (no GPU) initial state of block `rank` as the Harness builds
    and uploads it.  ic = ("magnetosphere", [rho_core, p_core, falloff, r_ref])
    or (kind, params).  Returns dict(fields, bd, frozen_idx, frozen_states,
    centers, spacings); arrays ghost-inclusive, reference index order.
    fields_out / bd_out: caller arrays (e.g. pinned) of those shapes to fill
    in place."""
    options = options or HarnessOptions()
    blocks, _ = layout(specs, partition)
    info = blocks[rank]
    g = options.ghost
    spans = [info.n[a] + 2 * g for a in range(3)]
    cells = spans[0] * spans[1] * spans[2]
    fields = fields_out if fields_out is not None else np.zeros((spans[2], spans[1], spans[0], 8))
    assert fields.shape == (spans[2], spans[1], spans[0], 8) and fields.dtype == np.float64
    bd = None
    if options.with_dipole:
        bd = bd_out if bd_out is not None else np.zeros((spans[2], spans[1], spans[0], 3))
    if ic[0] == "magnetosphere":
        kind = -1
        p = np.array(list(ic[1]) if len(ic) > 1 else [1.0, 0.1, 3.0, 3.0], dtype=np.float64)
    else:
        kind = int(ic[0])
        p = np.zeros(8)
        p[:len(ic[1])] = ic[1]
    # frozen cells (magnetosphere only): the core r < 3 fits a box of
    # 6 / d_uniform (+ margin) cells per axis
    cap = 1
    if kind < 0:
        cap = 1
        for a in range(3):
            cap *= min(spans[a], int(math.ceil(6.0 / float(specs[a].d_uniform))) + 6)
        cap = max(1, min(cells, cap))
    fidx = np.zeros(cap, np.int64)
    fst = np.zeros((cap, 8))
    nf = C.c_int64(cap if kind < 0 else 0)
    cat_c, cat_s = np.zeros(sum(spans)), np.zeros(sum(spans))
    check(N.lib.ppmlr_host_block_state(_specs3(specs), *partition, C.byref(options.c()), rank,
                                       kind, ptr(p), ptr(fields), ptr(bd),
                                       ptr(fidx, C.POINTER(C.c_int64)),
                                       ptr(fst) if kind < 0 else None, C.byref(nf),
                                       ptr(cat_c), ptr(cat_s)))
    offs = np.cumsum([0] + spans)
    k = nf.value
    return dict(fields=fields, bd=bd, frozen_idx=fidx[:k].copy(),
                frozen_states=fst[:k].copy() if kind < 0 else np.zeros((0, 8)),
                centers=[cat_c[offs[a]:offs[a + 1]] for a in range(3)],
                spacings=[cat_s[offs[a]:offs[a + 1]] for a in range(3)])


def host_block_geometry(specs, partition=(1, 1, 1), options: HarnessOptions | None = None,
                        rank=0):
    """Ghost-inclusive centres and spacings of block `rank` (make_block's
    local axes), without evaluating any state."""
    options = options or HarnessOptions()
    blocks, _ = layout(specs, partition)
    info = blocks[rank]
    g = options.ghost
    spans = [info.n[a] + 2 * g for a in range(3)]
    cat_c, cat_s = np.zeros(sum(spans)), np.zeros(sum(spans))
    p = np.zeros(8)
    check(N.lib.ppmlr_host_block_state(_specs3(specs), *partition, C.byref(options.c()), rank,
                                       0, ptr(p), None, None, None, None, None,
                                       ptr(cat_c), ptr(cat_s)))
    offs = np.cumsum([0] + spans)
    return ([cat_c[offs[a]:offs[a + 1]] for a in range(3)],
            [cat_s[offs[a]:offs[a + 1]] for a in range(3)])


def device_count():
    return int(N.lib.ppmlr_gpu_device_count())


def sweep_strips(states, bd, dx, n, ghost, dt, direction, gamma=5.0 / 3.0, mu0=1.0,
                 pressure_floor=0.0, precision="strict", device=0):
    """Batched sweep_1d (ppm1d.cpp:317-364) of independent strips, in place.

    states: (nstrips, n+2g, 8) float64; bd: (nstrips, n+2g, 3) or None;
    dx: (n+2g,).  Raises StepRejected / UnphysicalState like sweep_1d."""
    states = np.ascontiguousarray(states, dtype=np.float64)
    if states.ndim == 2:
        states = states[None]
    ns = states.shape[0]
    bdp = None
    if bd is not None:
        bd = np.ascontiguousarray(bd, dtype=np.float64).reshape(ns, n + 2 * ghost, 3)
        bdp = ptr(bd)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    check(N.lib.ppmlr_gpu_sweep_strips(ptr(states), bdp, ptr(dx), n, ghost, ns, direction, dt,
                                       gamma, mu0, pressure_floor, _PRECISION[precision],
                                       device))
    return states


def strip_max_dt(states, bd, dx, n, ghost, direction, gamma=5.0 / 3.0, mu0=1.0, device=0):
    """strip_max_dt (ppm1d.cpp:307-315) on the device: the min over the
    strips' interior cells of dx / (|v_dir| + c_f,dir), bit-identical."""
    states = np.ascontiguousarray(states, dtype=np.float64)
    if states.ndim == 2:
        states = states[None]
    ns = states.shape[0]
    bdp = None
    if bd is not None:
        bd = np.ascontiguousarray(bd, dtype=np.float64).reshape(ns, n + 2 * ghost, 3)
        bdp = ptr(bd)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    out = C.c_double()
    check(N.lib.ppmlr_gpu_strip_max_dt(ptr(states), bdp, ptr(dx), n, ghost, ns, direction,
                                       gamma, mu0, device, C.byref(out)))
    return out.value


def version():
    return N.lib.ppmlr_gpu_version().decode()


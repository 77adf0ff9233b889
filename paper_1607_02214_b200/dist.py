"""Multi-GPU driver: one process (rank) per GPU, one block per rank.

The reference's in-process harness (harness.cpp:59-92, exchange.cpp:93-149)
becomes a distributed step over torch.distributed (NCCL over NVLink on the
B200 box; gloo through pinned host buffers for the CPU tests and for several
ranks sharing one GPU):

  dt       <- all_reduce(MIN) of every rank's cfl*min   (compute_global_dt)
  for axis in XYZ / ZYX:
      halo of the `axis` faces, 4 layers                 (exchange_step)
      physical-face fill along `axis`                    (apply_boundaries)
      sweep                                              (sweep_axis)
  halo of all faces, 1 layer; fill; sources + frozen core; the next local
  cfl*min fused into the sources epilogue; all_reduce(MIN)

Only what the next kernel reads is exchanged (ghosts are
pure copies, so this is bit-identical to the reference's 4-layer,
all-face exchanges; the ledger keeps the reference's accounting).  Slabs
are packed in the reference's HaloSlab order.

Overlap.  Every exchange is started by the kernel that produces the state it
carries, split in two launches (block.cu split_*): part 1 updates only the
tiles holding the 4 boundary x cells of either side, the faces are packed
and sent (NCCL on a communication stream), and part 2 -- the interior, ~98%
of the work at 512^3 -- runs on the compute stream while the halo travels.
The x halo of a ZYX step's x sweep is produced by its y sweep, the one of an
XYZ step by the previous step's sources; the 1-layer halo of the sources by
the z sweep (XYZ) or the x sweep (ZYX).  The receiving rank unpacks right
before the consumer.  No host synchronisation inside a step on NCCL.

The step logic (``advance``) is written against a small block interface so
the same code runs with the CUDA block (``DeviceRankBlock``) and, in the CPU
tests, with an oracle-backed block over gloo.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time

import numpy as np

ORDER = ((0, 1, 2), (2, 1, 0))  # sweep_order (stepper.cpp:288-290)


class _CudaPtr:
    """__cuda_array_interface__ view of device memory owned by the library."""

    def __init__(self, ptr, n, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def face_cells(n, face):
    a = face // 2
    return n[(a + 1) % 3] * n[(a + 2) % 3]


class Exchanger:
    """Halo slabs between neighbour ranks with torch.distributed P2P.

    transport "nccl": device buffers; the send/recv run on a communication
    stream that waits for the pack only, so they overlap the interior work
    issued after ``start``; ``finish`` makes the compute stream wait and
    unpacks.  transport "host": host (pinned, when the block is on a GPU)
    buffers that the pack/unpack kernels write and read directly; ``start``
    packs, ``finish`` waits for the pack, exchanges over gloo on the host
    (while the GPU runs the interior) and unpacks."""

    def __init__(self, info, n, make_buffer, group=None, transport="nccl", timing=False):
        self.info = info
        self.n = n
        self.group = group
        self.transport = transport
        self.send = {}
        self.recv = {}
        for face in range(6):
            if info.neighbor[face] >= 0:
                cnt = face_cells(n, face) * 4 * 8
                self.send[face] = make_buffer(cnt)
                self.recv[face] = make_buffer(cnt)
        self.messages = 0
        self.bytes_moved = 0
        self.pending = None
        self.comm = None
        self.timing = timing
        self.halo_events = []  # (start, end) CUDA events around the NCCL ops
        if transport == "nccl":
            import torch
            self.comm = torch.cuda.Stream()

    def faces(self, faces):
        return tuple(f for f in faces if self.info.neighbor[f] >= 0)

    def _ops(self, faces, layers):
        import torch.distributed as dist
        ops = []
        for f in faces:
            cnt = face_cells(self.n, f) * layers * 8
            nb = self.info.neighbor[f]
            ops.append(dist.P2POp(dist.isend, self.send[f][:cnt], nb, self.group))
            ops.append(dist.P2POp(dist.irecv, self.recv[f][:cnt], nb, self.group))
            self.messages += 1
            self.bytes_moved += cnt * 8
        return ops

    def start(self, blk, faces, layers):
        """Pack `faces` (those with a neighbour) and put them on the wire."""
        import torch.distributed as dist
        faces = self.faces(faces)
        assert self.pending is None, "one halo exchange in flight at a time"
        if not faces:
            return
        for f in faces:
            blk.pack_face(f, layers, self.send[f])
        if self.transport == "nccl":
            import torch
            ev = torch.cuda.Event()
            ev.record()
            self.comm.wait_event(ev)
            with torch.cuda.stream(self.comm):
                e0 = e1 = None
                if self.timing:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                reqs = dist.batch_isend_irecv(self._ops(faces, layers))
                if self.timing:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record()
                    self.halo_events.append((e0, e1))
            self.pending = (faces, layers, reqs)
        else:
            ev = blk.record_event()
            self.pending = (faces, layers, ev)

    def finish(self, blk, faces, layers):
        """Complete the exchange of `faces` (starting it first if nobody
        did) and unpack into the ghost shells."""
        import torch.distributed as dist
        faces = self.faces(faces)
        if not faces:
            return
        if self.pending is None:
            self.start(blk, faces, layers)
        got, lay, h = self.pending
        assert got == faces and lay == layers, (got, faces, lay, layers)
        self.pending = None
        if self.transport == "nccl":
            for r in h:
                r.wait()  # the compute stream waits for the NCCL work
        else:
            if h is not None:
                h.synchronize()  # the pack kernels have written the host buffers
            for r in dist.batch_isend_irecv(self._ops(faces, layers)):
                r.wait()
        for f in faces:
            blk.unpack_face(f, layers, self.recv[f])

    def exchange(self, blk, faces, layers):
        self.finish(blk, faces, layers)

    def allreduce_min(self, t):
        import torch.distributed as dist
        if self.transport == "nccl" or t.device.type == "cpu":
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        else:  # gloo with a device tensor: through the host
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MIN, group=self.group)
            t.copy_(h)

    def halo_ms(self):
        """Summed NCCL halo time of the timed exchanges (comm stream events)."""
        tot = 0.0
        for e0, e1 in self.halo_events:
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot


def begin(blk, cfl, first_step, group=None, ex=None):
    import torch.distributed as dist
    blk.begin(cfl, first_step)
    if ex is not None:
        ex.allreduce_min(blk.dt_tensor())
    else:
        dist.all_reduce(blk.dt_tensor(), op=dist.ReduceOp.MIN, group=group)


def _produce(blk, ex, launch, faces, layers, overlap):
    """Run a producing kernel; when its output feeds a halo exchange, split
    it: boundary tiles, start the exchange, interior tiles."""
    faces = ex.faces(faces) if faces else ()
    if faces and overlap and getattr(blk, "splits", False):
        launch(1)
        ex.start(blk, faces, layers)
        launch(2)
    else:
        launch(0)
        if faces:
            ex.start(blk, faces, layers)


def advance(blk, ex, step, cfl, with_sources, group=None, overlap=True):
    """One distributed Harness::advance; the dt slot holds the global dt on
    entry and the next step's global dt on exit.  A halo exchange the
    previous step started (the x faces of this step's first sweep) is
    finished here."""
    blk.check_stream()
    order = ORDER[0 if step % 2 == 0 else 1]
    next_first_x = ORDER[0 if (step + 1) % 2 == 0 else 1][0] == 0
    for k, axis in enumerate(order):
        ex.finish(blk, (2 * axis, 2 * axis + 1), 4)
        blk.fill_boundaries(1 << axis, 4)
        if k < 2:
            nxt = order[k + 1]
            need = ((2 * nxt, 2 * nxt + 1), 4)
        elif with_sources:
            need = (tuple(range(6)), 1)
        else:  # the frozen-core restore still changes the state: exchange after it
            need = ((), 4)
        _produce(blk, ex, lambda part, a=axis, s=k: blk.sweep_part(a, s, part), need[0],
                 need[1], overlap)
    if with_sources:
        ex.finish(blk, range(6), 1)
        blk.fill_boundaries(7, 1)
        _produce(blk, ex, lambda part: blk.end_step_part(cfl, True, part),
                 (0, 1) if next_first_x else (), 4, overlap)
    else:
        blk.end_step(cfl, False)
        if next_first_x:
            ex.start(blk, (0, 1), 4)
    ex.allreduce_min(blk.dt_tensor())


class DeviceRankBlock:
    """This rank's block, resident on its GPU (libppmlr_b200)."""

    def __init__(self, specs, partition, options, rank, ic, device):
        import torch
        from . import _native as N
        from .api import (_BOUNDARY, _PRECISION, check, host_block_geometry, host_block_state,
                          layout)
        self.N = N
        self.check_rc = check
        blocks, _ = layout(specs, partition)
        self.info = blocks[rank]
        # built-in ICs are evaluated on the device (no host copy of the
        # block); init_magnetosphere is streamed from the host
        on_device = ic[0] != "magnetosphere" and 0 <= int(ic[0]) <= 3
        if on_device:
            cen, spc = host_block_geometry(specs, partition, options, rank)
            st = None
        else:
            st = host_block_state(specs, partition, options, rank, ic)
            cen, spc = st["centers"], st["spacings"]
        d = N.BlockDesc()
        g = options.ghost
        self._geom = [np.ascontiguousarray(x) for x in list(cen) + list(spc)]
        for a in range(3):
            d.n[a] = self.info.n[a]
            d.lo[a] = self.info.lo[a]
            d.centers[a] = self._geom[a].ctypes.data_as(C.POINTER(C.c_double))
            d.spacings[a] = self._geom[3 + a].ctypes.data_as(C.POINTER(C.c_double))
            d.physical[a][0] = int(self.info.neighbor[2 * a] < 0)
            d.physical[a][1] = int(self.info.neighbor[2 * a + 1] < 0)
        d.ghost = g
        d.gamma, d.mu0, d.pressure_floor = options.gamma, options.mu0, options.pressure_floor
        d.boundary = _BOUNDARY[options.boundary]
        d.wind_rho, d.wind_p = options.wind.rho_sw, options.wind.p_sw
        d.wind_v[:] = options.wind.v_sw
        d.wind_imf[:] = options.wind.imf
        d.with_dipole = int(options.with_dipole)
        d.precision = _PRECISION[options.precision]
        d.device = device
        h = C.c_void_p()
        check(N.lib.ppmlr_gpu_block_create(C.byref(d), C.byref(h)))
        self.h = h
        self.device = device
        self.stream = torch.cuda.current_stream(device)
        check(N.lib.ppmlr_gpu_block_set_stream(h, C.c_void_p(self.stream.cuda_stream)))
        if on_device:
            p = np.zeros(8)
            p[:len(ic[1])] = ic[1]
            check(N.lib.ppmlr_gpu_block_init_ic(h, int(ic[0]),
                                                p.ctypes.data_as(C.POINTER(C.c_double))))
        else:
            self.upload(st["fields"], st["bd"], st["frozen_idx"], st["frozen_states"])
        self._dt = torch.as_tensor(_CudaPtr(N.lib.ppmlr_gpu_block_dt_slot(h), 1),
                                   device=f"cuda:{device}")
        self.n = self.info.n

    def upload(self, fields, bd, frozen_idx, frozen_states):
        """ghost-inclusive reference-layout state host -> device."""
        fi = frozen_idx
        self.check_rc(self.N.lib.ppmlr_gpu_block_upload(
            self.h, fields.ctypes.data_as(C.POINTER(C.c_double)),
            None if bd is None else bd.ctypes.data_as(C.POINTER(C.c_double)),
            fi.ctypes.data_as(C.POINTER(C.c_int64)) if len(fi) else None,
            frozen_states.ctypes.data_as(C.POINTER(C.c_double)) if len(fi) else None,
            len(fi)))

    def close(self):
        if getattr(self, "h", None):
            self.N.lib.ppmlr_gpu_block_destroy(self.h)
            self.h = None

    def dt_tensor(self):
        return self._dt

    def begin(self, cfl, first_step):
        self.check_rc(self.N.lib.ppmlr_gpu_block_begin(self.h, cfl, first_step))

    def pack_face(self, face, layers, buf):
        self.check_rc(self.N.lib.ppmlr_gpu_block_pack_face(self.h, face, layers,
                                                           C.c_void_p(buf.data_ptr())))

    def unpack_face(self, face, layers, buf):
        self.check_rc(self.N.lib.ppmlr_gpu_block_unpack_face(self.h, face, layers,
                                                             C.c_void_p(buf.data_ptr())))

    def fill_boundaries(self, mask, layers):
        self.check_rc(self.N.lib.ppmlr_gpu_block_fill_boundaries(self.h, mask, layers))

    splits = True  # sweep_part / end_step_part: boundary-first split launches

    def sweep_async(self, axis, s):
        self.check_rc(self.N.lib.ppmlr_gpu_block_sweep_async(self.h, axis, s))

    def sweep_part(self, axis, s, part):
        self.check_rc(self.N.lib.ppmlr_gpu_block_sweep_part(self.h, axis, s, part))

    def end_step(self, cfl, with_sources):
        self.check_rc(self.N.lib.ppmlr_gpu_block_end_step(self.h, cfl, int(with_sources)))

    def end_step_part(self, cfl, with_sources, part):
        self.check_rc(self.N.lib.ppmlr_gpu_block_end_step_part(self.h, cfl, int(with_sources),
                                                               part))

    def record_event(self):
        import torch
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return ev

    def check_stream(self):
        """Kernels go to the block's stream and torch's NCCL calls order
        against torch's current stream: they must be the same."""
        import torch
        cur = torch.cuda.current_stream(self.device).cuda_stream
        assert cur == self.stream.cuda_stream, \
            "dist.advance must run under the stream the block was created on"

    def check(self):
        self.check_rc(self.N.lib.ppmlr_gpu_block_check(self.h))

    def timing(self, enable):
        sw, k, n = C.c_double(), C.c_double(), C.c_long()
        self.check_rc(self.N.lib.ppmlr_gpu_block_timing(self.h, int(enable), C.byref(sw),
                                                        C.byref(k), C.byref(n)))
        return sw.value, k.value, n.value

    def interior(self, out=None):
        nx, ny, nz = self.n
        if out is None:
            out = np.zeros((nz, ny, nx, 8))
        self.check_rc(self.N.lib.ppmlr_gpu_block_download_interior(
            self.h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out


def run_rank(blk, ex, steps, first_step, cfl, with_sources, group=None, dt_ready=False,
             overlap=True):
    if not dt_ready:
        begin(blk, cfl, first_step, group, ex)
    for s in range(steps):
        advance(blk, ex, first_step + s, cfl, with_sources, group, overlap)
    # an exchange started for a step that is not run: drop it (its halo is
    # re-sent by the next window's first consumer)
    if ex.pending is not None:
        faces, layers, _ = ex.pending
        ex.finish(blk, faces, layers)


def _traffic(kind, cells):
    """dram bytes of one sweep launch scaled from the committed ncu capture
    (profiles/ncu_sweep_traffic.json), or None."""
    prof = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "ncu_sweep_traffic.json")
    try:
        rec = json.load(open(prof)).get(kind, {})
        return rec["bytes_per_cell"] * cells if "bytes_per_cell" in rec else None
    except (OSError, ValueError):
        return None


def _e2e_distributed(blk, ex, cfg, rank, world, args, cfl, srcs, cells_rank, local, UNIT):
    """End to end per rank through the block API, max over ranks: the
    rank's initial state uploaded from pinned host memory, K distributed
    steps, the interior downloaded into pinned host memory (one untimed pass
    first)."""
    import torch
    import torch.distributed as dist
    from .api import host_block_state
    g = cfg.options.ghost
    shape = tuple(blk.n[2 - a] + 2 * g for a in range(3)) + (8,)
    fin = torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    bdin = None
    if cfg.options.with_dipole:
        bdin = torch.empty(shape[:3] + (3,), dtype=torch.float64, pin_memory=True).numpy()
    # the rank's initial state evaluated straight into the pinned buffers
    st = host_block_state(cfg.specs, cfg.partition, cfg.options, rank, cfg.ic, fields_out=fin,
                          bd_out=bdin)
    nx, ny, nz = blk.n
    fout = torch.empty((nz, ny, nx, 8), dtype=torch.float64, pin_memory=True).numpy()
    k = args.steps

    def one(steps):
        blk.upload(fin, st["bd"], st["frozen_idx"], st["frozen_states"])
        run_rank(blk, ex, steps, 0, cfl, srcs)
        blk.interior(out=fout)

    one(1)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    one(k)
    t1 = time.perf_counter()
    el = torch.tensor([t1 - t0], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    h2d = fin.nbytes + (st["bd"].nbytes if st["bd"] is not None else 0)
    return {"value": cells_rank * world * k / float(el.item()), "unit": UNIT,
            "h2d_bytes_per_step": world * h2d / k,
            "d2h_bytes_per_step": world * (fout.nbytes + 8 * k) / k,
            "how": f"per rank: upload(pinned) + {k} distributed steps + "
                   "download_interior(pinned), wall clock, max over ranks, after one untimed pass"}


def bench_distributed(args, METRIC, UNIT, ALG, make_config, ClockSampler, fp64_peak_tflops,
                      measured_peaks, cpu_baseline, workload):
    """bench.py's N-GPU arm: weak scaling, one 512^3 x-slab per rank."""
    import torch
    import torch.distributed as dist
    for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"),
                 ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29511")):
        os.environ.setdefault(k, v)  # allow a single-rank run outside torchrun
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, kind = make_config(args.config, world)
    cfg.options.precision = args.precision
    cfg.options.device = local
    alg = ALG[kind]
    blk = DeviceRankBlock(cfg.specs, cfg.partition, cfg.options, rank, cfg.ic, local)
    ex = Exchanger(blk.info, blk.n, lambda n: torch.empty(n, dtype=torch.float64,
                                                          device=f"cuda:{local}"))
    cells_rank = blk.n[0] * blk.n[1] * blk.n[2]
    cfl, srcs = cfg.options.cfl, cfg.options.with_sources
    run_rank(blk, ex, args.warmup, 0, cfl, srcs)
    torch.cuda.synchronize()
    blk.timing(True)
    ex.timing = True
    ex.halo_events.clear()
    m0, b0 = ex.messages, ex.bytes_moved
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        run_rank(blk, ex, args.steps, args.warmup, cfl, srcs, dt_ready=True)
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    blk.check()
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    sweep_ms, kernels, launches = blk.timing(False)
    halo_ms = torch.tensor([ex.halo_ms()], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(halo_ms, op=dist.ReduceOp.MAX)
    halo = {"messages_per_step": (ex.messages - m0) / args.steps,
            "bytes_per_step": (ex.bytes_moved - b0) / args.steps,
            "nccl_ms_per_step": float(halo_ms.item()) / args.steps,
            "overlap": "boundary-first split launches; NCCL on a comm stream"}
    if halo["nccl_ms_per_step"] > 0:
        gbs = halo["bytes_per_step"] / (halo["nccl_ms_per_step"] * 1e-3) / 1e9
        halo.update({"achieved_gbs": gbs, "nvlink_peer_peak_gbs": 770.0,
                     "frac_nvlink": gbs / 770.0,
                     "share_of_step": halo["nccl_ms_per_step"] / (ms / args.steps)})
    ex.timing = False
    e2e = _e2e_distributed(blk, ex, cfg, rank, world, args, cfl, srcs, cells_rank, local, UNIT)
    value = cells_rank * world * args.steps / (ms * 1e-3)
    if rank == 0:
        peak = fp64_peak_tflops(local)
        hbm, hbm_src = measured_peaks()
        # per sweep (a split sweep is two timed launches)
        avg = max(sweep_ms * 1e-3 / max(3 * args.steps, 1), 1e-12)
        fb = cells_rank * alg["B_sweep"] / avg / (hbm * 1e9)
        ff = cells_rank * alg["F_sweep"] / avg / (peak * 1e12)
        bound = "fp64" if ff >= fb else "hbm"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "precision": args.precision, "data": "synthetic (deterministic IC, no RNG)",
            "config": workload(args.config, world)[1],
            "clocks": clk.summary(), "gpu_launches": int(kernels),
            "halo": halo,
            "roofline": {"bound": bound,
                         "achieved": (cells_rank * alg["F_sweep"] / avg / 1e12) if bound == "fp64"
                         else cells_rank * alg["B_sweep"] / avg / 1e9,
                         "peak": peak if bound == "fp64" else hbm,
                         "unit": "TFLOP/s" if bound == "fp64" else "GB/s",
                         "frac": ff if bound == "fp64" else fb,
                         "traffic": _traffic(kind, cells_rank),
                         "frac_hbm": fb, "frac_fp64": ff, "peak_hbm_source": hbm_src},
            "e2e": e2e,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config)
        print(json.dumps(line), flush=True)
    blk.close()
    dist.destroy_process_group()

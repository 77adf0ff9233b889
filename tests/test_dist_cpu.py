"""The multi-GPU step schedule (paper_1607_02214_b200/dist.py) on CPU:
world_size 2 over gloo, each rank driving an oracle-backed block through the
same `begin` / `advance` code the NCCL path runs (halo slabs in the
reference's HaloSlab order, P2P send/recv, MIN all-reduce of dt).  The
gathered result must equal the single-block run bit for bit (the reference's
partition-invariance criterion, verify.cpp:205-226)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleRankBlock:
    """dist.py block interface over the C restatement (test infrastructure)."""

    def __init__(self, specs, partition, options, rank, ic):
        import torch
        import pyoracle as po
        from paper_1607_02214_b200 import host_block_state, layout
        self.po = po
        blocks, _ = layout(specs, partition)
        self.info = blocks[rank]
        self.n = self.info.n
        st = host_block_state(specs, partition, options, rank, ic)
        phys = [[int(self.info.neighbor[2 * a] < 0), int(self.info.neighbor[2 * a + 1] < 0)]
                for a in range(3)]
        self.blk = po.OracleBlock(self.n, 4, st["centers"], st["spacings"], phys, st["fields"],
                                  st["bd"], st["frozen_idx"], st["frozen_states"])
        self.o = po.opts(boundary=options.boundary, cfl=options.cfl,
                         with_sources=options.with_sources)
        self.c = po.consts(gamma=options.gamma)
        self._dt = torch.zeros(1, dtype=torch.float64)

    def dt_tensor(self):
        return self._dt

    def _local_dt(self, cfl):
        self._dt[0] = self.blk.compute_dt(cfl, self.c)

    def begin(self, cfl, first_step):
        self._local_dt(cfl)

    def _face_view(self, face, layers, ghost):
        g = 4
        a = face // 2
        na = self.n[a]
        f = self.blk.fields  # (S2, S1, S0, 8)
        if ghost:  # receiver's shell facing the sender (exchange.cpp:17-27)
            lo = g + na if face % 2 == 1 else g - layers
        else:      # sender's outermost interior layers
            lo = g if face % 2 == 0 else g + na - layers
        sl = [slice(g, g + self.n[2]), slice(g, g + self.n[1]), slice(g, g + self.n[0])]
        sl[2 - a] = slice(lo, lo + layers)
        return f, tuple(sl), a

    def pack_face(self, face, layers, buf):
        f, sl, a = self._face_view(face, layers, ghost=False)
        v = f[sl]  # (z, y, x, 8); slab order t2 -> t1 -> layer -> 8
        order = {0: (0, 1, 2, 3), 1: (2, 0, 1, 3), 2: (1, 2, 0, 3)}[a]
        flat = np.ascontiguousarray(np.transpose(v, order)).reshape(-1)
        buf[:flat.size] = __import__("torch").from_numpy(flat)

    def unpack_face(self, face, layers, buf):
        f, sl, a = self._face_view(face, layers, ghost=True)
        shape = f[sl].shape
        order = {0: (0, 1, 2, 3), 1: (2, 0, 1, 3), 2: (1, 2, 0, 3)}[a]
        tshape = tuple(shape[i] for i in order)
        inv = np.argsort(order)
        data = buf[:int(np.prod(shape))].numpy().reshape(tshape)
        f[sl] = np.transpose(data, inv)

    def fill_boundaries(self, mask, layers):
        self.blk.apply_boundaries(self.o)

    splits = False  # no boundary-first split launches: exchanges start after the kernel

    def sweep_async(self, axis, s):
        self.blk.sweep_axis(axis, float(self._dt[0]), self.c)

    def sweep_part(self, axis, s, part):
        assert part == 0
        self.sweep_async(axis, s)

    def end_step(self, cfl, with_sources):
        if with_sources:
            self.blk.apply_sources(float(self._dt[0]), self.c)
        self.blk.restore_frozen()
        self._local_dt(cfl)

    def end_step_part(self, cfl, with_sources, part):
        assert part == 0
        self.end_step(cfl, with_sources)

    def record_event(self):
        return None

    def check_stream(self):
        pass

    def interior(self):
        return np.ascontiguousarray(self.blk.interior())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, partition, steps, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from paper_1607_02214_b200 import configs, dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg(configs, cfg_name)
    blk = OracleRankBlock(cfg.specs, partition, cfg.options, rank, cfg.ic)
    ex = pdist.Exchanger(blk.info, blk.n, lambda n: torch.zeros(n, dtype=torch.float64),
                         transport="host")
    pdist.run_rank(blk, ex, steps, 0, cfg.options.cfl, cfg.options.with_sources)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), blk.interior())
    dist.barrier()
    dist.destroy_process_group()


def _cfg(configs, name):
    if name == "magnetosphere_small":
        return configs.magnetosphere_small(n=(32, 18, 18), dcell=2.4)
    if name == "blast":
        return configs.blast(n=16, gpus=2, radius=0.3)
    if name == "blast_nosources":
        return configs.blast(n=16, gpus=2, radius=0.3, with_sources=False)
    raise ValueError(name)


@pytest.mark.parametrize("cfg_name,partition,steps", [("blast", (2, 1, 1), 4),
                                                      ("blast_nosources", (2, 1, 1), 3),
                                                      ("magnetosphere_small", (2, 1, 1), 3)])
def test_distributed_schedule_matches_single_block(tmp_path, oracle, cfg_name, partition,
                                                   steps):
    import torch.multiprocessing as mp
    from paper_1607_02214_b200 import configs, host_block_state, layout
    world = partition[0] * partition[1] * partition[2]
    port = _free_port()
    mp.spawn(_worker, args=(world, port, cfg_name, partition, steps, str(tmp_path)),
             nprocs=world, join=True)
    cfg = _cfg(configs, cfg_name)
    st = host_block_state(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic)
    ob = oracle.OracleBlock([len(c) - 8 for c in st["centers"]], 4, st["centers"],
                            st["spacings"], [[1, 1]] * 3, st["fields"], st["bd"],
                            st["frozen_idx"], st["frozen_states"])
    o = oracle.opts(boundary=cfg.options.boundary, cfl=cfg.options.cfl,
                    with_sources=cfg.options.with_sources)
    c = oracle.consts(gamma=cfg.options.gamma)
    for s in range(steps):
        ob.advance(o, c, s)
    want = np.ascontiguousarray(ob.interior())
    blocks, _ = layout(cfg.specs, partition)
    got = np.zeros_like(want)
    for b in blocks:
        part = np.load(tmp_path / f"rank{b.rank}.npy")
        got[b.lo[2]:b.lo[2] + b.n[2], b.lo[1]:b.lo[1] + b.n[1], b.lo[0]:b.lo[0] + b.n[0]] = part
    assert np.array_equal(got.view(np.int64), want.view(np.int64))

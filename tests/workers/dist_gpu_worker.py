"""One rank of the distributed driver (paper_1607_02214_b200/dist.py) on the
device: a DeviceRankBlock on GPU 0 (every rank of this test shares it), its
halos through pinned host buffers over gloo (transport "host": the pack and
unpack kernels write / read the pinned buffers directly), the boundary-first
split launches overlapping the exchanges.  Launched by tests/test_gpu_dist.py
with torch.distributed.run; writes its interior to OUT/rank<r>.npy."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--cfg", default="blast")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--overlap", type=int, default=1)
    ap.add_argument("--precision", default="strict")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_1607_02214_b200 import configs
    from paper_1607_02214_b200 import dist as pdist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    cfg = {"blast": lambda: configs.blast(n=24, gpus=world, radius=0.3),
           "magnetosphere": lambda: configs.magnetosphere_small()}[a.cfg]()
    cfg.options.precision = a.precision
    part = (world, 1, 1)
    blk = pdist.DeviceRankBlock(cfg.specs, part, cfg.options, rank, cfg.ic, 0)
    ex = pdist.Exchanger(blk.info, blk.n,
                         lambda n: torch.zeros(n, dtype=torch.float64, pin_memory=True),
                         transport="host")
    pdist.run_rank(blk, ex, a.steps, 0, cfg.options.cfl, cfg.options.with_sources,
                   overlap=bool(a.overlap))
    torch.cuda.synchronize()
    blk.check()
    np.save(os.path.join(a.out, f"rank{rank}.npy"), blk.interior())
    dt = float(blk.dt_tensor().cpu()[0])
    np.save(os.path.join(a.out, f"dt{rank}.npy"), np.array([dt]))
    blk.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Break an e2e pass (bench.py bench_e2e) into upload / first advance /
the other advances / download:  python tools/e2e_probe.py briowu|mag160|blast512"""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_1607_02214_b200 as P  # noqa: E402
from paper_1607_02214_b200 import configs  # noqa: E402

name = sys.argv[1]
cfg = {"briowu": configs.brio_wu, "mag160": configs.magnetosphere,
       "blast512": lambda: configs.blast(n=512)}[name]()
cfg.options.precision = 'fast'
h = P.Harness(cfg.specs, cfg.partition, cfg.options)
configs.init(h, cfg)
g = cfg.options.ghost
nx, ny, nz = (int(s.cells) for s in cfg.specs)
shape = (nz + 2 * g, ny + 2 * g, nx + 2 * g)
host_in = torch.empty(shape + (8,), dtype=torch.float64, pin_memory=True).numpy()
host_bd = (torch.empty(shape + (3,), dtype=torch.float64, pin_memory=True).numpy()
           if cfg.options.with_dipole else None)
st = P.host_block_state(cfg.specs, (1, 1, 1), cfg.options, 0, cfg.ic, fields_out=host_in,
                        bd_out=host_bd)
host_out = torch.empty((nz, ny, nx, 8), dtype=torch.float64, pin_memory=True).numpy()
blk = h.block(0)
gb_in = (host_in.nbytes + (host_bd.nbytes if host_bd is not None else 0)) / 1e9
for rep in range(3):
    t0 = time.perf_counter()
    blk.upload(host_in, host_bd, st["frozen_idx"], st["frozen_states"])
    t1 = time.perf_counter()
    h.advance()
    t2 = time.perf_counter()
    for _ in range(19):
        h.advance()
    t3 = time.perf_counter()
    blk.download_interior(out=host_out)
    t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms ({gb_in/(t1-t0):.1f} GB/s)  first advance "
          f"{1e3*(t2-t1):.2f}  19 advances {1e3*(t3-t2):.1f}  download {1e3*(t4-t3):.1f} ms "
          f"({host_out.nbytes/1e9/(t4-t3):.1f} GB/s)")

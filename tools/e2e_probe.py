import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1607_02214_b200 as P
from paper_1607_02214_b200 import configs
cfg = configs.brio_wu() if sys.argv[1] == 'briowu' else configs.magnetosphere()
cfg.options.precision = 'fast'
h = P.Harness(cfg.specs, cfg.partition, cfg.options); configs.init(h, cfg)
st = P.host_block_state(cfg.specs, (1,1,1), cfg.options, 0, cfg.ic)
host_in = torch.empty(st["fields"].shape, dtype=torch.float64, pin_memory=True).numpy(); host_in[...] = st["fields"]
nx, ny, nz = (int(s.cells) for s in cfg.specs)
host_out = torch.empty((nz, ny, nx, 8), dtype=torch.float64, pin_memory=True).numpy()
blk = h.block(0)
for rep in range(3):
    t0 = time.perf_counter(); blk.upload(host_in, st["bd"], st["frozen_idx"], st["frozen_states"]); t1 = time.perf_counter()
    h.advance(); t2 = time.perf_counter()
    for _ in range(19): h.advance()
    t3 = time.perf_counter(); blk.download_interior(out=host_out); t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} first-advance {1e3*(t2-t1):.2f} 19 advances {1e3*(t3-t2):.2f} download {1e3*(t4-t3):.2f} ms")

"""Step a mid-size dipole magnetosphere (every axis on the compile-time
tile) for ncu: python tools/prof_mag.py [nx nyz steps precision]"""
import sys

sys.path.insert(0, ".")
from paper_1607_02214_b200 import api, configs  # noqa: E402

nx, nyz, steps = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 192, 4)))
prec = sys.argv[4] if len(sys.argv) > 4 else "fast"
c = configs.magnetosphere(nx=nx, nyz=nyz, d=0.2, precision=prec)
h = api.Harness(c.specs, c.partition, c.options)
configs.init(h, c)
h.run(steps)
print("time", h.time())
h.close()

"""Step a dipole magnetosphere for ncu captures of the sweeps.

    python tools/prof_mag.py [NX NY NZ [STEPS [PRECISION]]]

Axes of 512 cells and more take the C5 spacing (d = 0.05), shorter ones
d = 0.2 (both stretched grids validate), so e.g. 1024 768 192 has C5's
x-y planes (6.4 MB per field) at a quarter of its memory."""
import sys

sys.path.insert(0, ".")
from paper_1607_02214_b200 import api, configs  # noqa: E402

a = sys.argv[1:]
dims = [int(v) for v in a[:3]] if len(a) >= 3 else [256, 192, 192]
steps = int(a[3]) if len(a) > 3 else 4
prec = a[4] if len(a) > 4 else "fast"
base = configs.magnetosphere(nx=256, nyz=192, d=0.2, precision=prec)


def spec(s, n):
    d = 0.05 if n >= 512 else 0.2
    return api.AxisSpec(s.min, s.max, s.uniform_lo, s.uniform_hi, d, n, s.ratio)


specs = [spec(s, n) for s, n in zip(base.specs, dims)]
h = api.Harness(specs, base.partition, base.options)
h.init_magnetosphere()
h.run(steps)
print("time", h.time())
h.close()

"""Command line (tools/ppmlr_main.cpp): ``run`` and ``verify`` on the GPU.

    python -m paper_1607_02214_b200 run --config mag160 --steps 20 --cadence 10 --out out/
    python -m paper_1607_02214_b200 verify [all|sod|briowu|convergence|conservation|partition]
    python -m paper_1607_02214_b200 report [--steps 5] [--transport direct|staged]

Errors print one ``error: ...`` line and exit 1, like the reference CLI
(ppmlr_main.cpp:185-188).
"""
from __future__ import annotations

import argparse
import sys


def _config(name, precision, gpus=1):
    from . import configs
    table = {
        "briowu": lambda: configs.brio_wu(precision=precision),
        "ot512": lambda: configs.orszag_tang(precision=precision),
        "mag160": lambda: configs.magnetosphere(precision=precision),
        "mag1024": lambda: configs.magnetosphere(nx=1024, nyz=768, d=0.05, precision=precision),
        "mag_small": lambda: configs.magnetosphere_small(precision=precision),
        "blast512": lambda: configs.blast(n=512, precision=precision),
    }
    if name.startswith("blast") and name not in table:
        return configs.blast(n=int(name[5:]), precision=precision)
    if name not in table:
        raise SystemExit(f"error: unknown config {name}")
    return table[name]()


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1607_02214_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="step a configuration, write snapshots + ledger")
    r.add_argument("--config", default="mag_small")
    r.add_argument("--steps", type=int, default=10)
    r.add_argument("--cadence", type=int, default=5)
    r.add_argument("--out", default="out")
    r.add_argument("--precision", default="strict", choices=["strict", "fast"])
    v = sub.add_parser("verify", help="the reference's physics suites on the GPU")
    v.add_argument("suite", nargs="?", default="all")
    v.add_argument("--precision", default="strict", choices=["strict", "fast"])
    rp = sub.add_parser("report", help="live runs of the reference partition shapes (CSV)")
    rp.add_argument("--steps", type=int, default=5)
    rp.add_argument("--transport", default="direct", choices=["direct", "staged"])
    a = ap.parse_args(argv)
    from .api import Error
    try:
        if a.cmd == "report":
            from .report import cmd_report
            cmd_report(a.steps, a.transport)
            return 0
        if a.cmd == "run":
            from .run import cmd_run
            cmd_run(_config(a.config, a.precision), a.steps, a.cadence, a.out)
            return 0
        from .verify import cmd_verify
        return cmd_verify(a.suite, a.precision)
    except Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python3
"""Per-launch kernel times of real iterations of a config, grouped by kernel
kind and active-set size (TAFV_KLOG lines: kind, cells, faces, fringe, us),
to see what the small level phases cost per cell against the large ones.

    TAFV_KLOG=1 python tools/phase_klog.py --config 2 --iters 5 2> klog.txt
    python tools/klog_summary.py klog.txt
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1704_01144_b200 import Solver, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
cfg = configs.get(a.config)
mesh = cfg.mesh()
s = Solver(mesh, "euler")
s.set_state(cfg.initial_state(mesh))
opt = cfg.options()
s.reference_integrate(opt, a.warmup)
s.set_flag("kernel_timing", 1)
recs = s.reference_integrate(opt, a.iters)
kt = s.kernel_times()
print("levels", [r["level_cells"] for r in recs], file=sys.stderr)
print("ms per iteration", s.stats()["ms_total"] / a.iters, {k: round(v["ms"] / a.iters, 4) for k, v in kt.items()},
      file=sys.stderr)

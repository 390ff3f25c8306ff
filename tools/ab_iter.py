#!/usr/bin/env python3
"""A/B two library builds (TAFV_GPU_LIB) with one-iteration calls (robust to
record-layout changes between builds): cell-updates/s over K iterations
after W warm-up, device time from the library's own call timer.

    TAFV_GPU_LIB=ablibs/r1.so python tools/ab_iter.py --config 2 --steps 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1704_01144_b200 import Solver, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--mesh-cache", default="")
a = ap.parse_args()
cfg = configs.get(a.config)
mesh = cfg.mesh()
s = Solver(mesh, "euler")
s.set_state(cfg.initial_state(mesh))
opt = cfg.options()
for _ in range(a.warmup):
    s.reference_integrate(opt, 1)
ms = ce = 0.0
for _ in range(a.steps):
    r = s.reference_integrate(opt, 1)[0]
    ms += s.stats()["ms_total"]
    ce += sum(n << (r["theta"] - l) for l, n in enumerate(r["level_cells"]))
print(f"{os.environ.get('TAFV_GPU_LIB') or 'in-tree'} cfg {a.config}: {ce / ms * 1e3 / 1e6:.1f} Mupd/s "
      f"{ms / a.steps:.4f} ms/iter")

#!/usr/bin/env python3
"""Profiling driver: config N at full size, W warm-up iterations, then K
iterations bracketed by cudaProfilerStart/Stop, so that
    ncu --profile-from-start off ... python tools/prof_region.py --config 4
captures only the steady-state iterations (no mesh build, no capture).

    python tools/prof_region.py --config 4 --warmup 3 --iters 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402  (cudaProfilerStart/Stop only)

from paper_1704_01144_b200 import Solver, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--graph", type=int, default=1, help="0: direct launches (per-kernel ncu ids are stable)")
ap.add_argument("--flag", action="append", default=[], help="library knob name=value")
a = ap.parse_args()
cfg = configs.get(a.config)
mesh = cfg.mesh()
s = Solver(mesh, "euler")
s.set_state(cfg.initial_state(mesh))
del mesh
s.set_flag("use_graph", a.graph)
for fv in a.flag:
    k, v = fv.split("=")
    s.set_flag(k, int(v))
opt = cfg.options()
s.reference_integrate(opt, a.warmup)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
recs = s.reference_integrate(opt, a.iters)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("levels", [r["level_cells"] for r in recs], "theta", [r["theta"] for r in recs])

"""Device time and C_eff per iteration from config 2's initial state (what the
e2e batch runs: one iteration from W0 per input) vs later iterations."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1704_01144_b200 import Solver, configs
cfg = configs.get(2); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
s = Solver(mesh, "euler")
def ceff(r):
    return sum(n << (r["theta"] - l) for l, n in enumerate(r["level_cells"]))
for rep in range(3):
    s.set_state(w0)
    for it in range(8):
        r = s.reference_integrate(opt, 1)[-1]
        st = s.stats()
        print(rep, it, r["level_cells"], ceff(r), "ms", round(st["ms_total"], 4), "plan", round(st["ms_plan"], 4),
              "Mupd/s", round(ceff(r) / st["ms_total"] / 1e3, 1))

"""Per-launch device time of the hot kernels vs active-set size: config 2's
mesh and state with injected two-level maps (tau = 0 on a ball of growing
radius, tau = 1 elsewhere), kernel timing inside the sweep graphs (TAFV_KLOG
lines on stderr, summarised by tools/klog_summary.py)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1704_01144_b200 import Solver, configs
from paper_1704_01144_b200.configs import smooth_to_fixpoint
cfg = configs.get(2); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
s = Solver(mesh, "euler")
c = mesh["cen"]
r = np.sqrt(((c - 0.5) ** 2).sum(axis=1))
s.set_flag("kernel_timing", 1)
for frac in (0.0001, 0.001, 0.01, 0.03, 0.1, 0.3):
    rad = np.quantile(r, frac)
    tau = np.where(r <= rad, 0, 1).astype(np.int32)
    tau = smooth_to_fixpoint(mesh, tau)
    for _ in range(3):
        s.set_state(w0)
        s.inject_levels(tau, 1e-5, opt)
        s.run_iteration()
    print("frac", frac, "tau0 cells", int((tau == 0).sum()), file=sys.stderr)

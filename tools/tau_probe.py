import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1704_01144_b200 import Solver, configs
for cid in (2, 3):
    cfg = configs.get(cid); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
    s = Solver(mesh, "euler"); s.set_state(w0)
    prev = None; same = 0; nchg = []
    for it in range(30):
        s.plan_iteration(opt)
        tau = s.get_array("tau")
        if prev is not None:
            d = int((tau != prev).sum()); nchg.append(d); same += d == 0
        prev = tau
        s.run_iteration()
    print(cid, "iterations with unchanged tau:", same, "of", len(nchg), "changed cells per iteration:", nchg[:12])

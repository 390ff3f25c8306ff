"""Do concurrent PCIe copies slow the solver's kernels? Device time of K iterations
with and without H2D / D2H copies looping on side streams."""
import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1704_01144_b200 import Solver, configs
cfg = configs.get(2); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
s = Solver(mesh, "euler")
s.set_state(w0)
s.reference_integrate(opt, 5)
w, W, t0, it = s.get_state()
hb = torch.empty(5_000_000, dtype=torch.float64).pin_memory()
db = torch.empty(5_000_000, dtype=torch.float64, device="cuda")
def run(mode):
    s.set_state(w, W, t0, it)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    if mode:
        with torch.cuda.stream(side):
            for _ in range(60):
                if mode & 1: hb.copy_(db, non_blocking=True)
                if mode & 2: db.copy_(hb, non_blocking=True)
    s.reference_integrate(opt, 20)
    st = s.stats()
    torch.cuda.synchronize()
    return st["ms_total"]
for mode in (0, 1, 2, 3, 0, 1):
    print("mode", mode, "(1=D2H 2=H2D)", "device ms / 20 it", round(run(mode), 3))

"""Aggregate throughput of 1 vs 2 independent solver instances running
concurrently (one host thread and one library stream each): how much of the
small-phase / tail idle time another independent input can fill."""
import os, sys, threading, time
sys.path.insert(0, os.getcwd())
from paper_1704_01144_b200 import Solver, configs
cfg = configs.get(2); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
K = 30
def ceff(r):
    return sum(n << (r["theta"] - l) for l, n in enumerate(r["level_cells"]))
sol = [Solver(mesh, "euler") for _ in range(3)]
for s in sol:
    s.set_state(w0); s.reference_integrate(opt, 3)
def work(s, out):
    s.set_state(w0)
    s.reference_integrate(opt, 2)
    t = time.perf_counter()
    recs = s.reference_integrate(opt, K)
    out.append((time.perf_counter() - t, sum(ceff(r) for r in recs)))
for n in (1, 2, 3, 1, 2, 3):
    outs = [[] for _ in range(n)]
    th = [threading.Thread(target=work, args=(sol[i], outs[i])) for i in range(n)]
    t = time.perf_counter()
    for x in th: x.start()
    for x in th: x.join()
    wall = time.perf_counter() - t
    tot = sum(o[0][1] for o in outs)
    print(n, "instances: aggregate", round(tot / max(o[0][0] for o in outs) / 1e6, 1), "Mupd/s (wall incl. set_state", round(wall, 3), "s)")

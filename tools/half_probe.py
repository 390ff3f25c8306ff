import os, sys, threading, time, copy
sys.path.insert(0, os.getcwd())
from paper_1704_01144_b200 import Solver, configs
def ceff(r):
    return sum(n << (r["theta"] - l) for l, n in enumerate(r["level_cells"]))
full = configs.get(2)
half = copy.deepcopy(full); half.n = (100, 100, 50); half.name = "half"
K = 30
def make(cfg):
    m = cfg.mesh(); w0 = cfg.initial_state(m); s = Solver(m, "euler"); s.set_state(w0); s.reference_integrate(cfg.options(), 3)
    return s, w0, cfg.options()
def work(x, out):
    s, w0, opt = x
    s.set_state(w0); s.reference_integrate(opt, 2)
    t = time.perf_counter(); recs = s.reference_integrate(opt, K)
    out.append((time.perf_counter() - t, sum(ceff(r) for r in recs)))
F = make(full); H = [make(half) for _ in range(2)]
for rep in range(2):
    o = []; work(F, o); print("full alone", round(o[0][1] / o[0][0] / 1e6, 1))
    o = []; work(H[0], o); print("half alone", round(o[0][1] / o[0][0] / 1e6, 1))
    outs = [[], []]
    th = [threading.Thread(target=work, args=(H[i], outs[i])) for i in range(2)]
    for x in th: x.start()
    for x in th: x.join()
    print("2 halves concurrent", round(sum(x[0][1] for x in outs) / max(x[0][0] for x in outs) / 1e6, 1))

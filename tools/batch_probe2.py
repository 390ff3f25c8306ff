import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1704_01144_b200 import Solver, configs
cfg = configs.get(2); mesh = cfg.mesh(); w0 = cfg.initial_state(mesh); opt = cfg.options()
s = Solver(mesh, "euler")
W0 = np.ascontiguousarray(w0 * mesh["vol"][:, None])
ins = [torch.from_numpy(W0.copy()).pin_memory() for _ in range(2)]
outs = [torch.empty_like(ins[0]).pin_memory() for _ in range(2)]
s.run_batch([ins[0]], [outs[0]], opt, 1)
K = 20
for dl in (0, 1, 0, 1):
    s.set_flag("dl_stream", dl)
    t = time.perf_counter(); s.run_batch([ins[j % 2] for j in range(K)], [outs[j % 2] for j in range(K)], opt, 1)
    print("dl_stream", dl, "batch per step ms", (time.perf_counter() - t) / K * 1e3)
ref = outs[0].clone()
s.set_flag("dl_stream", 1)
s.run_batch([ins[0], ins[1]], [outs[0], outs[1]], opt, 1)
print("same result", torch.equal(ref, outs[0]), torch.equal(ref, outs[1]))
s.set_state(None, ins[0].numpy())
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(K):
    s.reference_integrate(opt, 1)
print("iterate(1) per step ms", (time.perf_counter() - t) / K * 1e3)
s.set_state(None, ins[0].numpy())
t = time.perf_counter()
for _ in range(K):
    s.set_state(None, ins[0].numpy()); s.reference_integrate(opt, 1)
print("set_state+iterate(1) from W0 per step ms", (time.perf_counter() - t) / K * 1e3)

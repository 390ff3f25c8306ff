"""Timing probe for tafv_gpu_run_batch: batch wall time vs compute-only and copy-only."""
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
K = 10
for _ in range(2):
    t = time.perf_counter(); s.run_batch([ins[j % 2] for j in range(K)], [outs[j % 2] for j in range(K)], opt, 1)
    print("batch per step ms", (time.perf_counter() - t) / K * 1e3)
s.set_state(None, ins[0].numpy())
t = time.perf_counter()
for _ in range(K):
    s.reference_integrate(opt, 1)
print("iterate(1) per step ms", (time.perf_counter() - t) / K * 1e3)
t = time.perf_counter()
s.reference_integrate(opt, K)
print("iterate(K) per step ms", (time.perf_counter() - t) / K * 1e3)
d = torch.empty_like(ins[0], device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(K):
    d.copy_(ins[0], non_blocking=True)
torch.cuda.synchronize(); print("H2D per copy ms", (time.perf_counter() - t) / K * 1e3)
t = time.perf_counter()
for _ in range(K):
    outs[0].copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("D2H per copy ms", (time.perf_counter() - t) / K * 1e3)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(K):
    with torch.cuda.stream(s1): d.copy_(ins[0], non_blocking=True)
    with torch.cuda.stream(s2): outs[1].copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("H2D||D2H per pair ms", (time.perf_counter() - t) / K * 1e3)

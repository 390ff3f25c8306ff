#!/usr/bin/env python3
"""Stage times of the stateful end-to-end path (tafv_gpu_iterate_host) on a
config: untraced ms per iteration for several link chunk sizes
(TAFV_E2E_CHUNK_MB), then one traced (serialised) run with per-stage times
(TAFV_E2E_TRACE=1: upload, load, plan + sweep, scatter, download) and an
unsynchronised timeline of the same stage boundaries (TAFV_E2E_TRACE=2).

    python tools/e2e_trace.py --config 4 --chunks 16,64,256
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1704_01144_b200 import Solver, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--chunks", default="64")
a = ap.parse_args()
cfg = configs.get(a.config)
mesh = cfg.mesh()
s = Solver(mesh, "euler")
s.set_state(cfg.initial_state(mesh))
del mesh
opt = cfg.options()
s.reference_integrate(opt, 2)
W = torch.from_numpy(np.ascontiguousarray(s.get_state()[1])).pin_memory()
for mb in a.chunks.split(","):
    os.environ["TAFV_E2E_CHUNK_MB"] = mb
    s.iterate_host(W, opt, 1)
    t = time.perf_counter()
    s.iterate_host(W, opt, a.steps)
    dt = (time.perf_counter() - t) / a.steps
    print(f"chunk {mb} MB: {dt * 1e3:.1f} ms/iteration (device {s.stats()['ms_total'] / a.steps:.1f})", flush=True)
os.environ["TAFV_E2E_TRACE"] = "1"  # serialised stage times
s.iterate_host(W, opt, a.steps)
os.environ["TAFV_E2E_TRACE"] = "2"  # unsynchronised timeline
s.iterate_host(W, opt, a.steps)

#!/usr/bin/env python3
"""Time the in-library repartition (tafv_gpu_repartition, DistDriver::
repartition exchange.cpp:595-609) at a config's full size: `--world`
loopback ranks (host threads) on one GPU, slab shards cut by cell count,
`--iters` iterations, then a repartition by level cost; prints one JSON line
with the per-rank repartition wall times, the shard sizes before / after and
the setup time.

    python tools/repartition_time.py --config 4 --world 2
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1704_01144_b200 import Solver, configs, shard  # noqa: E402
from paper_1704_01144_b200.api import Comm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
cfg = configs.get(a.config)
t = time.perf_counter()
mesh = cfg.mesh()
w0 = cfg.initial_state(mesh)
opt = cfg.options()
roc = shard.partition_slabs(mesh, a.world, axis=0)
comm = Comm.loopback(a.world)
solvers = [None] * a.world
res, errs = {}, []
t_mesh = time.perf_counter() - t


def body(r):
    try:
        t0 = time.perf_counter()
        s = Solver(mesh, "euler", shard=(roc, r, comm))
        s.set_state(w0)
        t1 = time.perf_counter()
        s.reference_integrate(opt, a.iters)
        before = int((roc == r).sum())
        t2 = time.perf_counter()
        new = s.repartition(None, axis=0)
        t3 = time.perf_counter()
        res[r] = {"create_s": round(t1 - t0, 2), "repartition_s": round(t3 - t2, 3),
                  "repartition_ms_lib": round(float(s.get_array("repartition_ms")[0]), 1),
                  "owned_before": before, "owned_after": int((new == r).sum())}
        s.reference_integrate(opt, 1)  # runs on the new shards
        s.close()
    except Exception as e:  # pragma: no cover
        errs.append(repr(e))


th = [threading.Thread(target=body, args=(r,)) for r in range(a.world)]
for x in th:
    x.start()
for x in th:
    x.join()
comm.close()
print(json.dumps({"config": a.config, "world": a.world, "cells": int(len(mesh["vol"])), "mesh_s": round(t_mesh, 1),
                  "ranks": res, "errors": errs}))

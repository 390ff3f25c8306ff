#!/usr/bin/env python3
"""Full-size parity evidence for the configs the default GPU suite runs only
scaled (4: 80M cells; 5: 16M cells at tau0 1 % / 10 % / 50 %): the GPU path
and the multi-threaded CPU oracle side by side from the same mesh and state,
for the config's stated iteration count. Per iteration: dt, theta, level
counts and every plan list (tau, face cadences, cells_of_level, faces_of_cadence,
fringe) bit-exact; after the last
iteration w and W bitwise. One JSON line per run (profiles/r1_full_parity.jsonl).

    python tools/full_parity.py 4 5 [--iters N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import OracleSolver  # noqa: E402  (checker only)
from paper_1704_01144_b200 import Solver, configs  # noqa: E402


def run(cfg, iters):
    t = time.perf_counter()
    mesh = cfg.mesh()
    w0 = cfg.initial_state(mesh)
    opt = cfg.options()
    g = Solver(mesh, "euler")
    g.set_state(w0)
    o = OracleSolver(mesh, "euler", threads=os.cpu_count() or 8)
    o.init_values(w0.reshape(-1))
    o.set_options(opt.theta_max, opt.cfl, opt.dt_cap)
    tau = cfg.levels(mesh) if cfg.synthetic_levels else None
    n = len(mesh["vol"])
    per_it = []
    for i in range(iters):
        if tau is not None:
            g.inject_levels(tau, -1.0, opt)
            gl = g.plan_lists()
            o.kernel("compute_dt_max", np.arange(n, dtype=np.int32), cfl=opt.cfl, dt_cap=opt.dt_cap)
            dt = float(np.min(o.get("dt_max") / (2.0 ** gl["tau"])))
            o.inject_plan(gl["tau"], dt)
        else:
            g.plan_iteration(opt)
            o.plan_iteration()
        gl, ol = g.plan_lists(), o.plan_lists()
        lists_equal = all(np.array_equal(np.asarray(gl[k]), np.asarray(ol[k])) for k in ("tau", "face_cadence"))
        for k in ("cells_of_level", "faces_of_cadence", "fringe"):
            lists_equal = lists_equal and len(gl[k]) == len(ol[k]) and all(
                np.array_equal(a, b) for a, b in zip(gl[k], ol[k]))
        rg = g.run_iteration()
        ro = o.run_iteration()
        per_it.append({"iteration": i, "dt_equal": rg["dt"] == ro["dt"], "theta": rg["theta"],
                       "levels_equal": rg["level_cells"] == ro["level_cells"], "plan_lists_equal": lists_equal,
                       "level_cells": rg["level_cells"]})
    wg, Wg, t0g, _ = g.get_state()
    return {
        "config": cfg.name, "cells": n, "faces": int(len(mesh["fa"])), "iterations": iters,
        "tau0_share": cfg.synthetic_levels,
        "w_bitwise": bool(np.array_equal(wg.reshape(-1), o.get("w"))),
        "W_bitwise": bool(np.array_equal(Wg.reshape(-1), o.get("W"))),
        "t_equal": t0g == o.time()[0],
        "all_iterations_match": all(x["dt_equal"] and x["levels_equal"] and x["plan_lists_equal"] for x in per_it),
        "per_iteration": per_it,
        "wall_s": round(time.perf_counter() - t, 1),
        "oracle_threads": os.cpu_count(),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--tau0", default="0.01,0.1,0.5")
    args = ap.parse_args()
    for cid in args.configs:
        base = configs.get(cid)
        shares = [float(x) for x in args.tau0.split(",")] if base.synthetic_levels is not None else [None]
        for f in shares:
            cfg = base
            if f is not None:
                import copy
                cfg = copy.deepcopy(base)
                cfg.synthetic_levels = f
            print(json.dumps(run(cfg, args.iters or cfg.iterations)), flush=True)


if __name__ == "__main__":
    main()

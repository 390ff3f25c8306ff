#!/usr/bin/env python3
"""Run BASELINE configs at full size on one GPU for their stated iteration
counts and report throughput, levels, the conservation ledger inputs and
physical sanity (min density / pressure).

    python tools/run_configs.py 1 2 3 4 5 [--iters N] [--tau0 0.01,0.1,0.5]

One JSON line per run (config 5 once per tau0 share)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1704_01144_b200 import Solver, configs  # noqa: E402


def c_eff(r):
    return sum(n << (r["theta"] - l) for l, n in enumerate(r["level_cells"]))


def run(cfg, iters, tau0=None):
    t = time.perf_counter()
    mesh = cfg.mesh()
    t_mesh = time.perf_counter() - t
    w0 = cfg.initial_state(mesh)
    t = time.perf_counter()
    s = Solver(mesh, "euler")
    t_up = time.perf_counter() - t
    s.set_state(w0)
    opt = cfg.options()
    recs = []
    t = time.perf_counter()
    ms = 0.0
    if cfg.synthetic_levels is not None:
        import copy
        c2 = copy.deepcopy(cfg)
        c2.synthetic_levels = tau0 if tau0 is not None else cfg.synthetic_levels
        tau = c2.levels(mesh)
        for _ in range(iters):
            s.inject_levels(tau, -1.0, opt)
            recs.append(s.run_iteration())
            ms += s.stats()["ms_sweep"]
    else:
        recs = s.reference_integrate(opt, iters)
        ms = s.stats()["ms_total"]
    wall = time.perf_counter() - t
    w, W, t0, it = s.get_state()
    rho = w[:, 0]
    p = 0.4 * (w[:, 4] - 0.5 * (w[:, 1] ** 2 + w[:, 2] ** 2 + w[:, 3] ** 2) / rho)
    ce = sum(c_eff(r) for r in recs)
    out = {
        "config": cfg.name, "cells": len(mesh["vol"]), "faces": len(mesh["fa"]), "iterations": iters,
        "tau0_share": tau0, "t_end": t0, "cell_updates": ce,
        "device_ms": round(ms, 3), "cell_updates_per_s": ce / (ms / 1e3) if ms else None,
        "wall_s": round(wall, 3), "mesh_gen_s": round(t_mesh, 2), "upload_s": round(t_up, 2),
        "levels_first": recs[0]["level_cells"], "levels_last": recs[-1]["level_cells"],
        "theta": [r["theta"] for r in recs][:3] + ["..."],
        "cost_ratio_first": recs[0]["cost_ratio"],
        "mass_first_last": [recs[0]["total_extensive"][0], recs[-1]["total_extensive"][0]],
        "energy_first_last": [recs[0]["total_extensive"][4], recs[-1]["total_extensive"][4]],
        "min_rho": float(rho.min()), "min_p": float(p.min()), "finite": bool(np.isfinite(w).all()),
    }
    print(json.dumps(out), flush=True)
    s.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--tau0", default="0.01,0.1,0.5")
    a = ap.parse_args()
    for cid in a.configs:
        cfg = configs.get(cid)
        n = a.iters or cfg.iterations
        if cfg.synthetic_levels is not None:
            for f in [float(x) for x in a.tau0.split(",")]:
                run(cfg, n, f)
        else:
            run(cfg, n)


if __name__ == "__main__":
    main()

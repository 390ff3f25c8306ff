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


def load_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"])
    except Exception:
        return 6650.0


FLAGS = []


def run(cfg, iters, tau0=None):
    """One warm-up iteration (graph capture; excluded), then `iters` timed
    iterations as plan_iteration + run_iteration (device time of both from
    the library's events) with the plan's C_eff / F_eff / R_eff for the
    BASELINE.md byte model B_iter = 1220 C_eff + 568 F_eff + 312 R_eff."""
    t = time.perf_counter()
    mesh = cfg.mesh()
    t_mesh = time.perf_counter() - t
    w0 = cfg.initial_state(mesh)
    t = time.perf_counter()
    s = Solver(mesh, "euler")
    for fv in FLAGS:
        k, v = fv.split("=")
        s.set_flag(k, int(v))
    t_up = time.perf_counter() - t
    s.set_state(w0)
    opt = cfg.options()
    tau = None
    if cfg.synthetic_levels is not None:
        import copy
        c2 = copy.deepcopy(cfg)
        c2.synthetic_levels = tau0 if tau0 is not None else cfg.synthetic_levels
        tau = c2.levels(mesh)

    def plan():
        return s.inject_levels(tau, -1.0, opt) if tau is not None else s.plan_iteration(opt)

    plan()
    s.run_iteration()  # warm-up: graph instantiation
    recs, ce, fe, re_ = [], 0, 0, 0
    ms = 0.0
    t = time.perf_counter()
    for _ in range(iters):
        info = plan()
        ms += s.stats()["ms_plan"]        # this plan's device time
        ce, fe, re_ = ce + info["c_eff"], fe + info["f_eff"], re_ + info["r_eff"]
        recs.append(s.run_iteration())
        ms += s.stats()["ms_sweep"]       # run_iteration resets the stats first
    wall = time.perf_counter() - t
    w, W, t0, it = s.get_state()
    rho = w[:, 0]
    p = 0.4 * (w[:, 4] - 0.5 * (w[:, 1] ** 2 + w[:, 2] ** 2 + w[:, 3] ** 2) / rho)
    b_iter = 1220 * ce + 568 * fe + 312 * re_
    out = {
        "config": cfg.name, "cells": len(mesh["vol"]), "faces": len(mesh["fa"]), "iterations": iters,
        "tau0_share": tau0, "t_end": t0, "cell_updates": ce,
        "device_ms": round(ms, 3), "cell_updates_per_s": ce / (ms / 1e3) if ms else None,
        "byte_model_GBps": round(b_iter / (ms / 1e3) / 1e9, 1) if ms else None,
        "byte_model_frac": round(b_iter / (ms / 1e3) / 1e9 / load_peak(), 3) if ms else None,
        "f_eff_over_c_eff": round(fe / ce, 3),
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
    ap.add_argument("--flag", action="append", default=[], help="library knob name=value (A/B)")
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

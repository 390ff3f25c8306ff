#!/usr/bin/env python3
"""Sizes of the brick K1's per-brick structures on a config (face entries and
halo rows per 128-cell Morton brick): how many bricks fit a given stage.

    python tools/brick_probe.py 3 4
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_01144_b200 import Solver, configs  # noqa: E402

for cid in [int(a) for a in sys.argv[1:]] or [3]:
    cfg = configs.get(cid)
    mesh = cfg.mesh()
    s = Solver(mesh, "euler")
    s.set_flag("k1_brick", 1)
    info = s.get_array("brick_info")
    c = s.get_array("brick_counts")
    e, h = np.where(c[:, 0] < 0, -c[:, 0] - 1, c[:, 0]), c[:, 1]
    print("config", cid, "cells", len(mesh["vol"]), "bricks", int(info[0]), "ragged", int(info[1]), flush=True)
    for name, v in (("face entries", e), ("halo rows", h)):
        q = np.percentile(v, [1, 10, 50, 90, 99, 100])
        print(" ", name, "mean %.1f" % v.mean(), "percentiles 1/10/50/90/99/100:", q.astype(int).tolist())
    pool = ((h * 40 + 31) // 32) * 32 + ((e + 1) // 2 * 2) * 56
    for cap in (40960, 41856, 45056, 49152):
        print("  fits a pool of %d B (halo <= 320): %.1f %%" % (cap, 100.0 * np.mean((pool <= cap) & (h <= 320))))
    s.close()
    del s, mesh

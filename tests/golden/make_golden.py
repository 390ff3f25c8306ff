"""Generate golden fixtures from the REAL reference library (oracle/_ref).

Run in the build container (where /root/reference exists and
`make -C oracle ref` has built oracle/_ref/libtafv_ref.so):

    python tests/golden/make_golden.py

Each fixture is one scenario taken from the reference's own tests
(proj/tests/test_numerics.cpp, test_levels.cpp): the reference mesh
(generate_mesh, mesh.cpp:302-317), the initial state, the options, the
state after `n` iterations of reference_integrate / run_iteration, the
records and the first iteration's plan lists. GPU tests and oracle tests
compare against these without needing /root/reference at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import RefSolver, ref_generate_mesh  # noqa: E402

SCENARIOS = [
    # name, mesh spec, model, a, init, options (theta_max, cfl, dt_cap), n, mode
    # test_numerics.cpp:405-432 two-cell two-level hand case (injected plan)
    ("kat_two_cell", dict(dim=1, nx=2, periodic_x=True), "advection", (1.0, 0.0),
     ("values", [2.0, 1.0]), (3, 0.9, 1.0), 1, ("inject", [0, 1], 0.1)),
    # test_numerics.cpp:435-452 1D three levels from a 4x refined band
    ("line8_band4", dict(dim=1, nx=8, periodic_x=True, regions=[((0.375, 0.0, 0.625, 1.0), 4)]),
     "advection", (1.0, 0.0), ("gauss", dict(center=(0.5, 0.0), sigma=0.12)), (3, 0.9, 1.0), 10, "integrate"),
    # test_numerics.cpp:454-470 2D torus, two levels
    ("torus8_block2", dict(dim=2, nx=8, ny=8, periodic_x=True, periodic_y=True,
                           regions=[((0.25, 0.25, 0.75, 0.75), 2)]),
     "advection", (1.0, 0.5), ("gauss", dict(sigma=0.15)), (3, 0.5, 1.0), 10, "integrate"),
    # test_numerics.cpp:472-487 nonlinear flux
    ("line16_burgers", dict(dim=1, nx=16, periodic_x=True, regions=[((0.25, 0.0, 0.75, 1.0), 2)]),
     "burgers", (1.0, 0.0), ("gauss", dict(base=0.5, center=(0.5, 0.0), sigma=0.1)), (3, 0.9, 1.0), 10,
     "integrate"),
    # test_numerics.cpp:490-525 theta=0 == plain Heun (uniform line)
    ("line16_heun", dict(dim=1, nx=16, periodic_x=True), "advection", (1.0, 0.0),
     ("gauss", dict(center=(0.5, 0.0), sigma=0.12)), (3, 0.9, 1.0), 20, "heun"),
    # test_numerics.cpp:527-552 periodic mirror after one iteration (a = (1, 0.7))
    ("torus8_mirror", dict(dim=2, nx=8, ny=8, periodic_x=True, periodic_y=True,
                           regions=[((0.25, 0.25, 0.75, 0.75), 2)]),
     "advection", (1.0, 0.7), ("gauss", dict(sigma=0.15)), (3, 0.9, 1.0), 1, "integrate"),
    # test_numerics.cpp:615-637 monotone Burgers shock, transmissive ends
    ("line64_shock", dict(dim=1, nx=64, periodic_x=False), "burgers", (1.0, 0.0),
     ("step", dict(x=0.4, left=2.0, right=0.0)), (3, 0.45, 0.005), 40, "integrate"),
    # larger: 64x64 torus with a 2x refined block, 2 levels, many items per level
    ("torus64_block2", dict(dim=2, nx=64, ny=64, periodic_x=True, periodic_y=True,
                            regions=[((0.25, 0.25, 0.75, 0.75), 2)]),
     "advection", (1.0, 0.7), ("gauss", dict(sigma=0.15)), (3, 0.5, 1.0), 5, "integrate"),
    ("torus64_burgers", dict(dim=2, nx=64, ny=64, periodic_x=True, periodic_y=True,
                             regions=[((0.125, 0.125, 0.5, 0.5), 4)]),
     "burgers", (1.0, 0.3), ("gauss", dict(base=0.5, sigma=0.1)), (3, 0.45, 1.0), 5, "integrate"),
    # non-periodic 2D with a 4x block: transmissive boundaries + 3 levels
    ("box32_block4", dict(dim=2, nx=32, ny=32, regions=[((0.25, 0.25, 0.5, 0.5), 4)]),
     "advection", (1.0, 0.5), ("gauss", dict(center=(0.4, 0.4), sigma=0.1)), (3, 0.5, 1.0), 6, "integrate"),
]


def build(name, spec, model, a, init, opts, n, mode):
    mesh, adj, mh = ref_generate_mesh(**spec)
    s = RefSolver(mh, model, a)
    s.set_options(*opts)
    kind, args = init
    if kind == "values":
        s.init_values(np.array(args, dtype=np.float64))
    elif kind == "gauss":
        s.init_gaussian(**args)
    elif kind == "step":
        w = np.where(mesh["cen"][:, 0] < args["x"], args["left"], args["right"])
        s.init_values(w)
    w0 = s.get("w").copy()
    out = dict(mesh_dim=mesh["dim"], **{"mesh_" + k: v for k, v in mesh.items() if k != "dim"})
    out.update(adj_off=adj["off"], adj_face=adj["face"], adj_nb=adj["nb"], adj_sign=adj["sign"],
               mesh_hash=np.uint64(adj["hash"]))
    out.update(model=np.array(model), a=np.array(a, dtype=np.float64), opts=np.array(opts, dtype=np.float64),
               n=np.int32(n), w0=w0)
    plan = None
    if isinstance(mode, tuple) and mode[0] == "inject":
        s.inject_plan(np.array(mode[1], dtype=np.int32), mode[2])
        plan = s.plan_lists()
        recs = [s.run_iteration()]
        out.update(inject_tau=np.array(mode[1], dtype=np.int32), inject_dt=np.float64(mode[2]))
    elif mode == "heun":
        recs = s.plain_heun(n)
    else:
        s.plan_iteration()
        plan = s.plan_lists()
        recs = [s.run_iteration()]
        recs += s.integrate(n - 1)
    out["w"] = s.get("w")
    out["W"] = s.get("W")
    t0, it = s.time()
    out["t0"] = np.float64(t0)
    out["iteration"] = np.int32(it)
    if mode == "integrate" and n == 1:
        for k in ("face_wL", "face_wR", "phi_pred", "int_substep", "int_window"):
            out["final_" + k] = s.get(k)
    out["rec_dt"] = np.array([r["dt"] for r in recs])
    out["rec_theta"] = np.array([r["theta"] for r in recs], dtype=np.int32)
    out["rec_total"] = np.array([r["total_extensive"][0] for r in recs])
    out["rec_cost_ratio"] = np.array([r["cost_ratio"] for r in recs])
    out["rec_level_cells"] = np.array([r["level_cells"] + [0] * (8 - len(r["level_cells"])) for r in recs],
                                      dtype=np.int64)
    if plan is not None:
        out["plan_tau"] = plan["tau"]
        out["plan_cadence"] = plan["face_cadence"]
        out["plan_theta"] = np.int32(plan["theta"])
        out["plan_dt"] = np.float64(plan["dt"])
        for l, v in enumerate(plan["cells_of_level"]):
            out[f"plan_cells_{l}"] = v
        for l, v in enumerate(plan["faces_of_cadence"]):
            out[f"plan_faces_{l}"] = v
        for l, v in enumerate(plan["fringe"]):
            out[f"plan_fringe_{l}"] = v
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    return out


def main():
    for sc in SCENARIOS:
        out = build(*sc)
        print(f"{sc[0]:18s} cells={len(out['mesh_vol']):6d} faces={len(out['mesh_fa']):6d} "
              f"n={int(out['n'])} theta={list(out['rec_theta'][:3])}")


if __name__ == "__main__":
    main()

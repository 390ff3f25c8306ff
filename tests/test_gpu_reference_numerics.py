"""The reference's own numerics tests (proj/tests/test_numerics.cpp),
restated on the CUDA path through the public API: the scalar models run the
same LTS machinery and kernels as the Euler path (kernels.cuh templates), so
these pin the GPU against the reference's stated properties, not only
against the oracle. 1D meshes are built here in the reference generator's
layout (mesh.cpp:302-317: interior faces left-to-right with normal +x, then
the right and left boundary faces; periodic ends linked as partners)."""
import math

import numpy as np
import pytest

from paper_1704_01144_b200 import Solver, SolverOptions

pytestmark = pytest.mark.gpu


def line_mesh(nx, periodic=False, band=None):
    """Unit line of nx cells; band = (x0, x1, k): cells inside [x0, x1]
    split into 2^k (the generator's refined regions)."""
    edges = [0.0]
    h = 1.0 / nx
    for i in range(nx):
        a, b = i * h, (i + 1) * h
        k = 0
        if band is not None and a >= band[0] - 1e-12 and b <= band[1] + 1e-12:
            k = band[2]
        m = 1 << k
        for j in range(1, m + 1):
            edges.append(a + (b - a) * j / m)
    x = np.asarray(edges)
    n = len(x) - 1
    vol = np.diff(x)
    cen = np.zeros((n, 3))
    cen[:, 0] = 0.5 * (x[:-1] + x[1:])
    fl = list(range(n - 1)) + [n - 1, 0]
    fr = list(range(1, n)) + [-1, -1]
    fn = np.zeros((n + 1, 3))
    fn[:, 0] = 1.0
    fn[n, 0] = -1.0
    fc = np.zeros((n + 1, 3))
    fc[: n - 1, 0] = x[1:-1]
    fc[n - 1, 0] = 1.0
    fc[n, 0] = 0.0
    fp = np.full(n + 1, -1)
    if periodic:
        fp[n - 1], fp[n] = n, n - 1
    return {"dim": 1, "vol": vol, "cen": cen, "chl": vol.copy(), "fl": np.asarray(fl, np.int32),
            "fr": np.asarray(fr, np.int32), "fp": fp.astype(np.int32), "fn": fn, "fa": np.ones(n + 1),
            "fc": fc}


def test_stable_step_bound(gpu):
    """test_numerics.cpp:81-103: advection, zero-speed cap, burgers, cap clip
    (dt_max of the plan on the device)."""
    unit, halves = line_mesh(1), line_mesh(2)

    def dt_max(mesh, model, a, w, cfl, cap):
        s = Solver(mesh, model, a=a)
        s.set_state(np.full(len(mesh["vol"]), w))
        s.plan_iteration(SolverOptions(theta_max=0, cfl=cfl, dt_cap=cap))
        return s.get_array("dt_max")[0]

    assert dt_max(unit, "advection", (2.0, 0.0), 0.0, 0.9, 10.0) == 0.45
    assert dt_max(unit, "burgers", (1.0, 0.0), 0.0, 0.9, 1.0) == 1.0  # zero speed: the cap
    assert dt_max(halves, "burgers", (1.0, 0.0), 3.0, 0.9, 10.0) == pytest.approx(0.15, rel=1e-15)
    assert dt_max(unit, "advection", (2.0, 0.0), 0.0, 0.9, 0.25) == 0.25  # the cap clips a bound


def test_advected_profile_converges_first_order(gpu):
    """test_numerics.cpp:576-613: a Gaussian advected across a periodic line
    with a 2x-refined band (two levels every iteration) converges at first
    order or better in L1 under refinement."""
    sigma, base, amp = 0.1, 1.0, 1.0

    def exact(x, t):
        d = x - 0.5 - t
        d = d - np.floor(d + 0.5)
        return base + amp * np.exp(-d * d / (2.0 * sigma * sigma))

    def l1(nx):
        mesh = line_mesh(nx, periodic=True, band=(0.25, 0.75, 1))
        x = mesh["cen"][:, 0]
        s = Solver(mesh, "advection", a=(1.0, 0.0))
        s.set_state(base + amp * np.exp(-((x - 0.5) ** 2) / (2.0 * sigma * sigma)))
        opt = SolverOptions(theta_max=3, cfl=0.9, dt_cap=1.0)
        t = 0.0
        while t < 0.25:
            r = s.reference_integrate(opt, 1)[0]
            assert r["theta"] == 1  # the refined band keeps two levels in play
            t = r["t_start"] + r["advance"]
        w, _, t0, _ = s.get_state()
        assert t0 == t
        return float(np.sum(np.abs(w.reshape(-1) - exact(x, t0)) * mesh["vol"]))

    e32, e64, e128 = l1(32), l1(64), l1(128)
    assert e64 < e32 and e128 < e64
    assert math.log2(e32 / e64) >= 1.0 and math.log2(e64 / e128) >= 1.0


def test_adaptive_iterations_conserve_on_periodic_line(gpu):
    """test_numerics.cpp:434-451: 1D periodic line, three levels from a 4x
    refined band, Gaussian advected: the total drifts by <= 1e-12 relative
    over 10 iterations (first iteration at theta 2)."""
    mesh = line_mesh(8, periodic=True, band=(0.375, 0.625, 2))
    x = mesh["cen"][:, 0]
    s = Solver(mesh, "advection", a=(1.0, 0.0))
    w0 = 1.0 + np.exp(-((x - 0.5) ** 2) / (2.0 * 0.12 * 0.12))
    s.set_state(w0)
    total0 = math.fsum(w0 * mesh["vol"])
    recs = s.reference_integrate(SolverOptions(theta_max=3, cfl=0.9, dt_cap=1.0), 10)
    assert recs[0]["theta"] == 2
    for r in recs:
        assert abs(r["total_extensive"][0] - total0) <= 1e-12 * abs(total0)


def test_nonlinear_shock_monotone(gpu):
    """test_numerics.cpp:615-637: a Burgers step on a transmissive line
    stays monotone decreasing with no new extrema after every iteration."""
    mesh = line_mesh(64)
    x = mesh["cen"][:, 0]
    s = Solver(mesh, "burgers", a=(1.0, 0.0))
    s.set_state(np.where(x < 0.4, 2.0, 0.0))
    opt = SolverOptions(theta_max=3, cfl=0.45, dt_cap=0.005)
    for _ in range(40):
        s.reference_integrate(opt, 1)
        w = s.get_state()[0].reshape(-1)
        assert (w >= -1e-12).all() and (w <= 2.0 + 1e-12).all()
        assert (np.diff(w) <= 1e-12).all()


def _golden_mesh(name):
    from conftest import load_golden
    return load_golden(name)["mesh"]


def test_uniform_field_has_bitwise_zero_gradient(gpu):
    """test_numerics.cpp:105-123 (uniform subcase): a uniform field on a
    refined 2D mesh (the reference generator's torus with a 2x block) has a
    bitwise-zero gradient and stays bitwise uniform through iterations."""
    mesh = _golden_mesh("torus8_block2")
    for model, a in (("advection", (1.0, 0.5)), ("burgers", (1.0, 0.0))):
        s = Solver(mesh, model, a=a)
        s.set_state(np.full(len(mesh["vol"]), 0.75))
        s.reference_integrate(SolverOptions(theta_max=3, cfl=0.9, dt_cap=1.0), 3)
        g = s.get_array("grad")
        assert not np.any(g), model
        w = s.get_state()[0].reshape(-1)
        assert (w == 0.75).all(), model


def test_iterations_end_synchronous_with_consistent_extensive_values(gpu):
    """test_numerics.cpp (iterations end synchronous): after every iteration
    w == W / V bitwise on every cell and the time advanced by 2^theta dt."""
    mesh = _golden_mesh("torus8_block2")
    c = mesh["cen"]
    s = Solver(mesh, "advection", a=(1.0, 0.5))
    s.set_state(1.0 + np.exp(-((c[:, 0] - 0.5) ** 2 + (c[:, 1] - 0.5) ** 2) / (2 * 0.15 ** 2)))
    t = 0.0
    for _ in range(5):
        r = s.reference_integrate(SolverOptions(theta_max=3, cfl=0.9, dt_cap=1.0), 1)[0]
        w, W, t0, _ = s.get_state()
        assert (w.reshape(-1) == W.reshape(-1) / mesh["vol"]).all()
        assert r["t_start"] == t and t0 == t + r["dt"] * (1 << r["theta"])
        t = t0


def _plan_levels(mesh, chl, theta_max):
    """(raw, smoothed) levels the device plan assigns (dt_max classification,
    then Jacobi smoothing) for cell stable steps proportional to `chl`
    (advection at unit speed)."""
    m = dict(mesh)
    m["chl"] = np.asarray(chl, dtype=np.float64)
    s = Solver(m, "advection", a=(1.0, 0.0))
    s.set_state(np.ones(len(m["vol"])))
    s.plan_iteration(SolverOptions(theta_max=theta_max, cfl=0.5, dt_cap=1e30))
    return list(s.get_array("raw_level")), list(s.plan_lists()["tau"])


def test_classification_and_smoothing_kats(gpu):
    """test_levels.cpp:36-66 on the device plan: raw levels floor(log2 of the
    dt ratio) clamped to theta_max (ratios 5 -> 2, 1 -> 0, 3 -> 1, 1024 -> 3),
    and Jacobi smoothing [0,3,3] -> [0,1,2] on a line, [0,3,3,3] ->
    [0,1,2,1] across the periodic wrap."""
    for ratio, level in ((5.0, 2), (1.0, 0), (3.0, 1), (1024.0, 3)):
        raw, _ = _plan_levels(line_mesh(2), [1.0, ratio], 3)
        assert raw == [0, level], ratio
    assert _plan_levels(line_mesh(3), [1.0, 8.0, 8.0], 3) == ([0, 3, 3], [0, 1, 2])
    assert _plan_levels(line_mesh(4, periodic=True), [1.0, 8.0, 8.0, 8.0], 3) == ([0, 3, 3, 3], [0, 1, 2, 1])
    assert _plan_levels(line_mesh(3), [1.0, 1.0, 1.0], 4) == ([0, 0, 0], [0, 0, 0])

"""Python view of the multi-GPU decomposition (C ABI in include/tafv_gpu.h:
tafv_partition_slabs, tafv_shard_describe; host code, no GPU needed)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def mesh_view(mesh):
    keep = {k: np.ascontiguousarray(mesh[k], dtype=np.float64 if k in ("vol", "cen", "chl", "fn", "fa", "fc")
                                    else np.int32) for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc")}
    mv = N.MeshView(int(mesh["dim"]), len(keep["vol"]), len(keep["fa"]),
                    *[_ptr(keep[k]) for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc")])
    return mv, keep


def partition_slabs(mesh, nranks, axis=0, weight=None):
    lib = N.lib()
    mv, keep = mesh_view(mesh)
    out = np.empty(len(mesh["vol"]), dtype=np.int32)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float64)
    if lib.tafv_partition_slabs(C.byref(mv), nranks, axis, _ptr(w), _ptr(out)) != 0:
        raise ValueError(lib.tafv_shard_last_error().decode())
    return out


def describe(mesh, rank_of_cell, rank, nranks):
    """Local cells (global ids, with ring class), faces and exchange lists."""
    lib = N.lib()
    mv, keep = mesh_view(mesh)
    roc = np.ascontiguousarray(rank_of_cell, dtype=np.int32)
    cnt = np.zeros(8, dtype=np.int32)
    rc = lib.tafv_shard_describe(C.byref(mv), _ptr(roc), rank, nranks, _ptr(cnt), *([None] * 7))
    if rc != 0:
        raise ValueError(lib.tafv_shard_last_error().decode())
    n_own, n_r1, n_r2, nf, nfo, npeer, st, rt = (int(x) for x in cnt)
    cells = np.empty(n_own + n_r1 + n_r2, dtype=np.int32)
    faces = np.empty(nf, dtype=np.int32)
    peers = np.empty(max(1, npeer), dtype=np.int32)
    sc = np.empty(max(1, npeer), dtype=np.int32)
    rcn = np.empty(max(1, npeer), dtype=np.int32)
    sf = np.empty(max(1, st), dtype=np.int32)
    rf = np.empty(max(1, rt), dtype=np.int32)
    lib.tafv_shard_describe(C.byref(mv), _ptr(roc), rank, nranks, None, _ptr(cells), _ptr(faces),
                            _ptr(peers), _ptr(sc), _ptr(rcn), _ptr(sf), _ptr(rf))
    send, recv, so, ro = {}, {}, 0, 0
    for i in range(npeer):
        send[int(peers[i])] = sf[so:so + sc[i]].copy()
        recv[int(peers[i])] = rf[ro:ro + rcn[i]].copy()
        so += int(sc[i])
        ro += int(rcn[i])
    # ring class per local cell: 0 owned, 1 face neighbour of an owned cell, 2 other
    owned = roc[cells] == rank
    g2l = np.full(len(roc), -1, dtype=np.int64)
    g2l[cells] = np.arange(len(cells))
    # resolved right (kernels.cpp:15-20): right cell, or the periodic partner's left
    gfr, gfp = mesh["fr"][faces], mesh["fp"][faces]
    rr = np.where(gfr >= 0, gfr, np.where(gfp >= 0, mesh["fl"][np.maximum(gfp, 0)], -1))
    fl = g2l[mesh["fl"][faces]]
    fr = np.where(rr >= 0, g2l[np.maximum(rr, 0)], -1)
    cls = np.where(owned, 0, 2).astype(np.int8)
    inner = fr >= 0
    a, b = fl[inner], fr[inner]
    cls[b[owned[a] & ~owned[b]]] = 1
    cls[a[owned[b] & ~owned[a]]] = 1
    assert (cls == 0).sum() == n_own and (cls == 1).sum() == n_r1 and (cls == 2).sum() == n_r2
    return {"cells": cells, "faces": faces, "n_own": n_own, "n_r1": n_r1, "n_r2": n_r2,
            "n_faces_touch_own": nfo, "send": send, "recv": recv, "cls": cls}


def local_mesh(mesh, sh):
    """Reference-layout mesh dict of a shard (local ids = ascending global)."""
    cells, faces = sh["cells"], sh["faces"]
    g2l = np.full(len(mesh["vol"]), -1, dtype=np.int32)
    g2l[cells] = np.arange(len(cells), dtype=np.int32)
    f2l = np.full(len(mesh["fl"]), -1, dtype=np.int32)
    f2l[faces] = np.arange(len(faces), dtype=np.int32)
    fr = mesh["fr"][faces]
    fp = mesh["fp"][faces]
    return {
        "dim": mesh["dim"], "vol": mesh["vol"][cells], "cen": mesh["cen"][cells], "chl": mesh["chl"][cells],
        "fl": g2l[mesh["fl"][faces]], "fr": np.where(fr >= 0, g2l[np.maximum(fr, 0)], -1).astype(np.int32),
        "fp": np.where(fp >= 0, f2l[np.maximum(fp, 0)], -1).astype(np.int32), "fn": mesh["fn"][faces],
        "fa": mesh["fa"][faces], "fc": mesh["fc"][faces],
    }


def level_cost_weights(tau, theta=None):
    """DistDriver::repartition weights 2^(theta - tau) (exchange.cpp:598-603)."""
    import numpy as _np
    tau = _np.asarray(tau)
    th = int(tau.max()) if theta is None else int(theta)
    return _np.ldexp(1.0, th - tau)


def smooth_levels(mesh, tau):
    """smooth_to_fixpoint (levels.cpp:33-51) on the host (tafv_level_smooth)."""
    lib = N.lib()
    mv, keep = mesh_view(mesh)
    t = np.ascontiguousarray(tau, dtype=np.int32).copy()
    if lib.tafv_level_smooth(C.byref(mv), _ptr(t)) != 0:
        raise ValueError(lib.tafv_shard_last_error().decode())
    return t


def initial_levels(mesh, w, opt, gamma=1.4):
    """The levels plan_iteration would assign to the Euler state w (host,
    for slab cut weights only -- not bit-exact: the device plan is the
    authority): dt_max = cfl h / (|u| + c) (kernels.cpp:247-254), raw =
    ilogb(dt_max / dt_min) clamped to [0, theta_max] (levels.cpp:18-25),
    smoothed to the fixpoint."""
    w = np.asarray(w, dtype=np.float64).reshape(len(mesh["vol"]), -1)
    rho = w[:, 0]
    u = w[:, 1:4] / rho[:, None]
    p = (gamma - 1.0) * (w[:, 4] - 0.5 * rho * (u * u).sum(axis=1))
    speed = np.sqrt((u * u).sum(axis=1)) + np.sqrt(gamma * np.maximum(p, 0.0) / rho)
    with np.errstate(divide="ignore", invalid="ignore"):
        dtm = np.where(speed > 0, np.minimum(opt.dt_cap, opt.cfl * mesh["chl"] / speed), opt.dt_cap)
    ratio = dtm / dtm.min()
    raw = np.frexp(ratio)[1] - 1  # ilogb for ratio >= 1
    raw = np.clip(np.where(ratio >= 1.0, raw, 0), 0, opt.theta_max).astype(np.int32)
    return smooth_levels(mesh, raw)


def initial_level_cost(mesh, w, opt):
    """Per-cell level cost 2^(theta - tau) of the initial plan: the weights
    of the slab cut (DistDriver::repartition, exchange.cpp:598-603)."""
    return level_cost_weights(initial_levels(mesh, w, opt))


# ---- per-rank slab windows (no rank builds the global mesh) -----------------

def _dt_max_host(mesh, w, opt, gamma=1.4):
    """dt_max = cfl h / (|u| + c) on the host (slab-cut weights only)."""
    w = np.asarray(w, dtype=np.float64).reshape(len(mesh["vol"]), -1)
    rho = w[:, 0]
    u = w[:, 1:4] / rho[:, None]
    p = (gamma - 1.0) * (w[:, 4] - 0.5 * rho * (u * u).sum(axis=1))
    speed = np.sqrt((u * u).sum(axis=1)) + np.sqrt(gamma * np.maximum(p, 0.0) / rho)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(speed > 0, np.minimum(opt.dt_cap, opt.cfl * mesh["chl"] / speed), opt.dt_cap)


def plane_costs(cfg, opt, i0, i1, allreduce_min, allreduce_max, allreduce_sum):
    """Level cost 2^(theta - raw) of the initial state summed per x plane of
    a tensor-product config, each rank generating only the planes [i0, i1)
    (a provisional slab) and the collectives combining them (the raw levels,
    unsmoothed: smoothing only raises the cost near level jumps; the cut
    needs balance, not bits). Returns the per-plane costs of the whole
    lattice on every rank."""
    nx, ny, nz = cfg.n
    m = cfg.mesh(window=(i0, i1, 0, ny, 0, nz))
    dtm = _dt_max_host(m, cfg.initial_state(m), opt)
    dmin = allreduce_min(float(dtm.min()) if len(dtm) else float("inf"))
    ratio = dtm / dmin
    raw = np.clip(np.where(ratio >= 1.0, np.frexp(ratio)[1] - 1, 0), 0, opt.theta_max).astype(np.int64)
    theta = int(allreduce_max(float(raw.max()) if len(raw) else 0.0))
    cost = np.ldexp(1.0, theta - raw)
    plane = np.arange(len(cost)) % max(1, i1 - i0) + i0
    mine = np.bincount(plane, weights=cost, minlength=nx)
    return allreduce_sum(mine)


def slab_cuts(costs, nranks):
    """Contiguous plane ranges of balanced cost: cuts[r] .. cuts[r + 1]."""
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    cuts = [0]
    for r in range(1, nranks):
        cuts.append(int(np.clip(np.searchsorted(cum, cum[-1] * r / nranks), cuts[-1] + 1, len(costs) - (nranks - r))))
    cuts.append(len(costs))
    return np.asarray(cuts, dtype=np.int64)


def slab_window(cfg, cuts, rank, rings=2):
    """Rank `rank`'s x slab [cuts[rank], cuts[rank + 1]) of a tensor-product
    (unpermuted) config plus `rings` planes on each side, generated as a
    window of the lattice (tafv_mesh_hex_window: the cells and faces are
    bitwise the full mesh's, in the same relative order, so the shard built
    from it is bitwise the shard of the global mesh). Returns (window mesh,
    rank_of_cell over the window's cells, global ids of the window's cells)."""
    if cfg.permute:
        raise ValueError("slab_window: permuted configs have no lattice windows")
    nx, ny, nz = cfg.n
    i0, i1 = max(0, int(cuts[rank]) - rings), min(nx, int(cuts[rank + 1]) + rings)
    mesh = cfg.mesh(window=(i0, i1, 0, ny, 0, nz))
    wx = i1 - i0
    ids = np.arange(wx * ny * nz, dtype=np.int64)
    plane = ids % wx + i0
    roc = (np.searchsorted(np.asarray(cuts), plane, side="right") - 1).astype(np.int32)
    gid = (ids // wx) * nx + plane
    return mesh, roc, gid


def distributed_slab_window(cfg, opt, rank, nranks, allreduce):
    """The rank's slab window of a multi-process run: provisional uniform
    slabs, per-plane level costs combined with `allreduce(value, op)` (op in
    "min", "max", "sum"; value a float or a numpy array), balanced cuts,
    then the rank's own window. Returns (mesh, rank_of_cell, global ids,
    cuts); every rank gets the same cuts."""
    nx = cfg.n[0]
    b = [round(r * nx / nranks) for r in range(nranks + 1)]
    costs = plane_costs(cfg, opt, b[rank], b[rank + 1], lambda v: allreduce(v, "min"),
                        lambda v: allreduce(v, "max"), lambda v: allreduce(v, "sum"))
    cuts = slab_cuts(costs, nranks)
    mesh, roc, gid = slab_window(cfg, cuts, rank)
    return mesh, roc, gid, cuts

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

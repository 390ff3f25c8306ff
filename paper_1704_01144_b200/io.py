"""Mesh / snapshot formats (C ABI in include/tafv_gpu.h; host code): TFVM
mesh files (v1 = the reference's 2D format, read; v2 = Vec3, written),
Mesh::hash, reference-compatible text snapshots, binary snapshots and
compare_snapshots (proj/core/src/mesh.cpp:326-428, state.cpp:77-132)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .api import InvalidArgument, TafvError
from .shard import mesh_view


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc):
    if rc != 0:
        msg = N.lib().tafv_io_last_error().decode()
        raise (InvalidArgument if rc == N.TAFV_EINVAL else TafvError)(msg)


def mesh_hash(mesh):
    mv, keep = mesh_view(mesh)
    return int(N.lib().tafv_mesh_hash(C.byref(mv)))


def save_mesh(path, mesh):
    mv, keep = mesh_view(mesh)
    _check(N.lib().tafv_mesh_save(str(path).encode(), C.byref(mv)))


def load_mesh(path):
    L = N.lib()
    dim, nc, nf = C.c_int32(), C.c_int32(), C.c_int32()
    _check(L.tafv_mesh_load(str(path).encode(), C.byref(dim), C.byref(nc), C.byref(nf), *([None] * 9)))
    nc, nf = nc.value, nf.value
    m = {"dim": dim.value, "vol": np.empty(nc), "cen": np.empty((nc, 3)), "chl": np.empty(nc),
         "fl": np.empty(nf, dtype=np.int32), "fr": np.empty(nf, dtype=np.int32), "fp": np.empty(nf, dtype=np.int32),
         "fn": np.empty((nf, 3)), "fa": np.empty(nf), "fc": np.empty((nf, 3))}
    _check(L.tafv_mesh_load(str(path).encode(), None, None, None,
                            *[_ptr(m[k]) for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc")]))
    return m


def save_snapshot(path, mesh_or_hash, w, W, time=0.0, iteration=0, binary=False):
    h = mesh_or_hash if isinstance(mesh_or_hash, int) else mesh_hash(mesh_or_hash)
    w = np.ascontiguousarray(w, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    nc = w.shape[0]
    nv = 1 if w.ndim == 1 else w.shape[1]
    _check(N.lib().tafv_snapshot_save(str(path).encode(), int(binary), h, nc, nv, float(time), int(iteration),
                                      _ptr(w), _ptr(W)))


def load_snapshot(path):
    L = N.lib()
    h, nc, nv, t, it = C.c_uint64(), C.c_int32(), C.c_int32(), C.c_double(), C.c_int32()
    _check(L.tafv_snapshot_load(str(path).encode(), C.byref(h), C.byref(nc), C.byref(nv), C.byref(t),
                                C.byref(it), None, None))
    w = np.empty((nc.value, nv.value))
    W = np.empty((nc.value, nv.value))
    _check(L.tafv_snapshot_load(str(path).encode(), None, None, None, None, None, _ptr(w), _ptr(W)))
    if nv.value == 1:
        w, W = w[:, 0], W[:, 0]
    return {"mesh_hash": h.value, "time": t.value, "iteration": it.value, "w": w, "W": W}


def compare_snapshots(path_a, path_b):
    worst = C.c_double()
    _check(N.lib().tafv_snapshot_compare(str(path_a).encode(), str(path_b).encode(), C.byref(worst)))
    return worst.value

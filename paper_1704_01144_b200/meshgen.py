"""3D hexahedral meshes for the BASELINE.json configs (tafv_mesh_hex).

The reference generator is 1D/2D only (proj/core/src/mesh.cpp:302-317); this
is the 3D generator the configs need. It returns the canonical mesh dict
(reference Mesh layout, Vec3) that the GPU solver and the CPU oracle both
consume unchanged.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _empty_mesh(nc, nf):
    return {
        "dim": 3,
        "vol": np.empty(nc), "cen": np.empty((nc, 3)), "chl": np.empty(nc),
        "fl": np.empty(nf, dtype=np.int32), "fr": np.empty(nf, dtype=np.int32),
        "fp": np.empty(nf, dtype=np.int32), "fn": np.empty((nf, 3)), "fa": np.empty(nf),
        "fc": np.empty((nf, 3)),
    }


_KEYS = ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc")


def hex_mesh(x, y, z, jitter=0.0, seed=0, permute=False, window=None, lib=None):
    """Tensor-product hex mesh on node coordinates x[nx+1], y[ny+1], z[nz+1].

    window = (i0, i1, j0, j1, k0, k1): only those cells of the same lattice
    (tafv_mesh_hex_window), bitwise the full mesh's cells there. `lib` is
    any ctypes library exporting the generator (default: the product
    library; the oracle's checker library compiles the same generator)."""
    L = lib if lib is not None else N.lib()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    nx, ny, nz = len(x) - 1, len(y) - 1, len(z) - 1
    sd = int(seed) & (2**64 - 1)
    if window is None:
        def call(nc, nf, arrs):
            return L.tafv_mesh_hex(nx, ny, nz, _ptr(x), _ptr(y), _ptr(z), float(jitter), sd,
                                   int(bool(permute)), nc, nf, *arrs)
    else:
        if permute:
            raise ValueError("hex_mesh: a window of a permuted mesh is not defined")
        box = np.ascontiguousarray(window, dtype=np.int32)

        def call(nc, nf, arrs):
            return L.tafv_mesh_hex_window(nx, ny, nz, _ptr(x), _ptr(y), _ptr(z), _ptr(box), float(jitter),
                                          sd, nc, nf, *arrs)
    nc, nf = C.c_int32(), C.c_int32()
    if call(C.byref(nc), C.byref(nf), [None] * 9) != 0:
        raise ValueError("tafv_mesh_hex: invalid spec")
    m = _empty_mesh(nc.value, nf.value)
    if call(C.byref(C.c_int32()), C.byref(C.c_int32()), [_ptr(m[k]) for k in _KEYS]) != 0:
        raise ValueError("tafv_mesh_hex: invalid spec")
    return m


def make_periodic(mesh, axes, tol=1e-12):
    """Link the boundary faces of opposite domain sides along `axes` as
    periodic partners (Face::periodic_partner, mesh.hpp:26-65; the reference
    2D generator's torus, mesh.cpp:302-317): face f on the low side and face
    g on the high side with the same centroid in the other coordinates get
    fp[f] = g, fp[g] = f; both keep their single cell (right = -1). Needs
    matching boundary nodes on the two sides (no boundary jitter)."""
    m = dict(mesh)
    fp = mesh["fp"].copy()
    fc, fr = mesh["fc"], mesh["fr"]
    bnd = np.flatnonzero(fr < 0)
    for a in axes:
        lo, hi = fc[bnd, a].min(), fc[bnd, a].max()
        low = bnd[np.abs(fc[bnd, a] - lo) < tol]
        high = bnd[np.abs(fc[bnd, a] - hi) < tol]
        others = [d for d in range(3) if d != a]
        key = lambda f: tuple(np.round(fc[f, others], 9))
        index = {key(g): g for g in high}
        if len(index) != len(high) or len(low) != len(high):
            raise ValueError("make_periodic: sides do not match")
        for f in low:
            g = index[key(f)]
            fp[f], fp[g] = g, f
    m["fp"] = fp
    return m


def uniform_nodes(n):
    return np.linspace(0.0, 1.0, n + 1)


def geometric_nodes(n, ratio):
    """Spacing multiplied by `ratio` per cell away from 0, normalised to [0, 1]."""
    h = ratio ** np.arange(n, dtype=np.float64)
    x = np.concatenate([[0.0], np.cumsum(h)])
    x /= x[-1]
    x[-1] = 1.0
    return x


def centre_graded_nodes(n, ratio, core):
    """Symmetric grading: spacing 1 inside |u - 0.5| < core, growing
    geometrically by `ratio` per cell outside (fine centre, coarse walls)."""
    half = n // 2
    h = np.ones(n)
    u = (np.arange(n) + 0.5) / n - 0.5
    k = np.maximum(0, np.abs(u) - core) * n  # cells beyond the core
    h = ratio ** k
    x = np.concatenate([[0.0], np.cumsum(h)])
    x /= x[-1]
    x[-1] = 1.0
    del half
    return x

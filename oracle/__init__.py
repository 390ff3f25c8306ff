"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* :class:`OracleSolver` drives ``oracle/libtafv_oracle.so``, our C++
  restatement of the reference algorithm (``oracle/tafv_oracle.cpp``).
* :class:`RefSolver` / :func:`ref_generate_mesh` drive
  ``oracle/_ref/libtafv_ref.so``, the unmodified reference library compiled
  from ``/root/reference/proj/core`` (scalar 2D only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package; the product path never does.

Meshes travel as the canonical "mesh dict" (reference ``Mesh`` layout of
``proj/core/include/tafv/mesh.hpp:26-65`` generalised to Vec3)::

    dim, vol[nc], cen[nc,3], chl[nc], fl[nf], fr[nf], fp[nf],
    fn[nf,3], fa[nf], fc[nf,3]
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtafv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtafv_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class Record(C.Structure):
    """Mirror of ``tafv_record`` (include/tafv_gpu.h) / IterationRecord
    (proj/core/include/tafv/reference.hpp:20-29)."""

    _fields_ = [
        ("iteration", C.c_int32),
        ("theta", C.c_int32),
        ("t_start", C.c_double),
        ("dt", C.c_double),
        ("advance", C.c_double),
        ("cost_ratio", C.c_double),
        ("total_extensive", C.c_double * 8),
        ("level_cells", C.c_int64 * 16),
        ("n_levels", C.c_int32),
        ("nv", C.c_int32),
    ]

    def as_dict(self):
        return {
            "iteration": self.iteration,
            "theta": self.theta,
            "t_start": self.t_start,
            "dt": self.dt,
            "advance": self.advance,
            "cost_ratio": self.cost_ratio,
            "total_extensive": list(self.total_extensive[: self.nv]),
            "level_cells": list(self.level_cells[: self.n_levels]),
        }


class InvalidArgument(ValueError):
    """std::invalid_argument (proj/core/include/tafv/common.hpp:9-11)."""


class LogicError(RuntimeError):
    """std::logic_error (TAFV_ASSERT, common.hpp:15-19)."""


class Diverged(RuntimeError):
    """std::runtime_error (reference.cpp:124 and others)."""


_EXC = {1: InvalidArgument, 2: LogicError, 3: Diverged}


def _check(lib, rc, err_fn):
    if rc != 0:
        msg = getattr(lib, err_fn)().decode()
        raise _EXC.get(rc, RuntimeError)(msg)


_LIBS: dict = {}


def _load(path, kind):
    if path in _LIBS:
        return _LIBS[path]
    if not os.path.exists(path):
        raise OSError(f"{kind} library missing: {path} (run `make -C oracle`)")
    lib = C.CDLL(path)
    p = "orc_" if kind == "oracle" else "ref_"
    getattr(lib, p + "last_error").restype = C.c_char_p
    getattr(lib, p + "minmod").restype = C.c_double
    getattr(lib, p + "minmod").argtypes = [C.c_double, C.c_double]
    if kind == "ref":
        lib.ref_mesh_hash.restype = C.c_uint64
        lib.ref_mesh_save.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_snapshot_save.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_snapshot_compare.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p]
        lib.ref_total_extensive.restype = C.c_double
        lib.ref_total_extensive.argtypes = [C.c_void_p]
    _LIBS[path] = lib
    return lib


def oracle_lib():
    return _load(ORACLE_SO, "oracle")


def ref_lib():
    return _load(REF_SO, "ref")


def ref_available():
    return os.path.exists(REF_SO)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ---------------------------------------------------------------------------
# Reference (oracle/_ref) mesh generation: proj/core/src/mesh.cpp:302-317
# ---------------------------------------------------------------------------


def ref_generate_mesh(dim=2, nx=1, ny=1, domain=(0.0, 0.0, 1.0, 1.0), periodic_x=False,
                      periodic_y=False, regions=()):
    """Run the reference ``generate_mesh`` and export it as a mesh dict
    (plus the reference's own adjacency and hash, for cross-checks)."""
    lib = ref_lib()
    boxes = np.array([list(b) for b, _ in regions], dtype=np.float64).reshape(-1)
    scales = np.array([s for _, s in regions], dtype=np.int32)
    h = C.c_void_p()
    dom = np.asarray(domain, dtype=np.float64)
    rc = lib.ref_mesh_generate(
        dim, nx, ny, dom.ctypes.data_as(C.c_void_p), int(periodic_x), int(periodic_y),
        len(regions), boxes.ctypes.data_as(C.c_void_p) if len(regions) else None,
        scales.ctypes.data_as(C.c_void_p) if len(regions) else None, C.byref(h))
    _check(lib, rc, "ref_last_error")
    nc, nf, na = C.c_int(), C.c_int(), C.c_int()
    lib.ref_mesh_counts(h, C.byref(nc), C.byref(nf), C.byref(na))
    nc, nf, na = nc.value, nf.value, na.value
    cell = np.zeros((nc, 4))
    fi = np.zeros((nf, 3), dtype=np.int32)
    fd = np.zeros((nf, 5))
    off = np.zeros(nc + 1, dtype=np.int32)
    af = np.zeros(na, dtype=np.int32)
    an = np.zeros(na, dtype=np.int32)
    asg = np.zeros(na)
    lib.ref_mesh_export(h, *[x.ctypes.data_as(C.c_void_p) for x in (cell, fi, fd, off, af, an, asg)])
    mesh = {
        "dim": dim,
        "vol": cell[:, 2].copy(),
        "cen": np.stack([cell[:, 0], cell[:, 1], np.zeros(nc)], axis=1),
        "chl": cell[:, 3].copy(),
        "fl": fi[:, 0].copy(),
        "fr": fi[:, 1].copy(),
        "fp": fi[:, 2].copy(),
        "fn": np.stack([fd[:, 0], fd[:, 1], np.zeros(nf)], axis=1),
        "fa": fd[:, 2].copy(),
        "fc": np.stack([fd[:, 3], fd[:, 4], np.zeros(nf)], axis=1),
    }
    adj = {"off": off, "face": af, "nb": an, "sign": asg, "hash": int(lib.ref_mesh_hash(h))}
    return mesh, adj, h


class _SolverBase:
    prefix = ""

    def _c(self, rc):
        _check(self.lib, rc, self.prefix + "last_error")

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def set_options(self, theta_max=3, cfl=0.9, dt_cap=1.0):
        f = self._fn("set_options")
        f.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double]
        f(self.h, theta_max, cfl, dt_cap)

    def init_values(self, w):
        w = _f64(w)
        self._c(self._fn("init_values")(self.h, w.ctypes.data_as(C.c_void_p)))

    def get(self, name):
        out = np.zeros(self._size(name), dtype=np.int32 if name in self.INT_ARRAYS else np.float64)
        self._c(self._fn("get")(self.h, name.encode(), out.ctypes.data_as(C.c_void_p)))
        return out

    def set(self, name, values):
        dt = np.int32 if name in self.INT_ARRAYS else np.float64
        v = np.ascontiguousarray(values, dtype=dt).reshape(-1)
        assert v.size == self._size(name), (name, v.size, self._size(name))
        self._c(self._fn("set")(self.h, name.encode(), v.ctypes.data_as(C.c_void_p)))

    def time(self):
        t0, it = C.c_double(), C.c_int()
        self._fn("time")(self.h, C.byref(t0), C.byref(it))
        return t0.value, it.value

    def plan_iteration(self):
        self._c(self._fn("plan_iteration")(self.h))
        return self.plan_info()

    def inject_plan(self, tau, dt):
        tau = _i32(tau)
        f = self._fn("inject_plan")
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        self._c(f(self.h, tau.ctypes.data_as(C.c_void_p), dt))
        return self.plan_info()

    def plan_info(self):
        th, dt, cr = C.c_int(), C.c_double(), C.c_double()
        a, b, c = (np.zeros(16, dtype=np.int64) for _ in range(3))
        self._fn("plan_info")(self.h, C.byref(th), C.byref(dt), C.byref(cr),
                              *[x.ctypes.data_as(C.c_void_p) for x in (a, b, c)])
        t = th.value
        return {"theta": t, "dt": dt.value, "cost_ratio": cr.value,
                "cells_per_level": a[: t + 1].copy(), "faces_per_cadence": b[: t + 1].copy(),
                "fringe_per_level": c[:t].copy()}

    def plan_lists(self):
        info = self.plan_info()
        tau = np.zeros(self.nc, dtype=np.int32)
        cad = np.zeros(self.nf, dtype=np.int32)
        cells = np.zeros(self.nc, dtype=np.int32)
        faces = np.zeros(self.nf, dtype=np.int32)
        fr = np.zeros(max(1, int(info["fringe_per_level"].sum())), dtype=np.int32)
        self._fn("plan_lists")(self.h, *[x.ctypes.data_as(C.c_void_p) for x in (tau, cad, cells, faces, fr)])

        def split(flat, counts):
            out, o = [], 0
            for n in counts:
                out.append(flat[o:o + n].copy())
                o += n
            return out

        return {
            "tau": tau, "face_cadence": cad,
            "cells_of_level": split(cells, info["cells_per_level"]),
            "faces_of_cadence": split(faces, info["faces_per_cadence"]),
            "fringe": split(fr, info["fringe_per_level"]),
            "theta": info["theta"], "dt": info["dt"], "cost_ratio": info["cost_ratio"],
        }

    def run_iteration(self):
        r = Record()
        self._c(self._fn("run_iteration")(self.h, C.byref(r)))
        return r.as_dict()

    def integrate(self, n):
        recs = (Record * max(1, n))()
        self._c(self._fn("integrate")(self.h, n, recs))
        return [recs[i].as_dict() for i in range(n)]

    def plain_heun(self, n):
        recs = (Record * max(1, n))()
        self._c(self._fn("plain_heun")(self.h, n, recs))
        return [recs[i].as_dict() for i in range(n)]

    def kernel(self, name, items=(), front=0, phase=1, tau=None, cadence=None, dt=0.0, cfl=0.9,
               dt_cap=1.0, theta_max=3):
        """Call one reference kernel over an explicit item list
        (kernels.hpp:31-111). phase: 0 corrector, 1 predictor."""
        it = _i32(items)
        tau_a = _i32(tau) if tau is not None else None
        cad_a = _i32(cadence) if cadence is not None else None
        out = C.c_double(0.0)
        f = self._fn("kernel")
        f.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                      C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_void_p]
        self._c(f(self.h, name.encode(), it.ctypes.data_as(C.c_void_p) if it.size else None, it.size,
                  front, phase, tau_a.ctypes.data_as(C.c_void_p) if tau_a is not None else None,
                  cad_a.ctypes.data_as(C.c_void_p) if cad_a is not None else None,
                  dt, cfl, dt_cap, theta_max, C.byref(out)))
        return out.value


class RefSolver(_SolverBase):
    """SolverState + SolverOptions of the real reference (scalar 2D)."""

    prefix = "ref_"
    INT_ARRAYS = {"raw_level", "committed_front", "staged_front", "face_staged", "face_front"}

    def __init__(self, mesh_handle, model="advection", a=(1.0, 0.0)):
        self.lib = ref_lib()
        self.mesh_handle = mesh_handle
        nc, nf, na = C.c_int(), C.c_int(), C.c_int()
        self.lib.ref_mesh_counts(mesh_handle, C.byref(nc), C.byref(nf), C.byref(na))
        self.nc, self.nf = nc.value, nf.value
        self.nv = 1
        h = C.c_void_p()
        f = self.lib.ref_solver_create
        f.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double, C.c_void_p]
        self._c(f(mesh_handle, model.encode(), a[0], a[1], C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.lib.ref_solver_free(self.h)
        except Exception:
            pass

    def _size(self, name):
        return self.nf if name.startswith("face_") or name in ("phi_pred", "int_substep", "int_window") else self.nc

    def init_gaussian(self, base=1.0, amplitude=1.0, center=(0.5, 0.5), sigma=0.1):
        f = self.lib.ref_init_gaussian
        f.argtypes = [C.c_void_p] + [C.c_double] * 5
        self._c(f(self.h, base, amplitude, center[0], center[1], sigma))

    def total_extensive(self):
        return self.lib.ref_total_extensive(self.h)

    def task_integrate(self, n, workers, ces):
        """The reference's task-parallel path: TaskEngine::integrate
        (taskgen.cpp:663-675) on `workers` single-lane workers, `ces`
        computation elements, prio scheduler, task packing on."""
        recs = (Record * max(1, n))()
        self._c(self.lib.ref_taskengine_integrate(self.h, n, workers, ces, recs))
        return [recs[i].as_dict() for i in range(n)]


class OracleMesh:
    def __init__(self, mesh, closure_mask=None):
        self.lib = oracle_lib()
        self.mesh = mesh
        self.nc = int(len(mesh["vol"]))
        self.nf = int(len(mesh["fa"]))
        arrs = [_f64(mesh["vol"]), _f64(mesh["cen"]), _f64(mesh["chl"]), _i32(mesh["fl"]),
                _i32(mesh["fr"]), _i32(mesh["fp"]), _f64(mesh["fn"]), _f64(mesh["fa"]),
                _f64(mesh["fc"])]
        self._keep = arrs
        h = C.c_void_p()
        mask = None if closure_mask is None else np.ascontiguousarray(closure_mask, dtype=np.uint8)
        self._mask = mask
        rc = self.lib.orc_mesh_create_masked(int(mesh["dim"]), self.nc, self.nf,
                                             *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                             mask.ctypes.data_as(C.c_void_p) if mask is not None else None,
                                             C.byref(h))
        _check(self.lib, rc, "orc_last_error")
        self.h = h

    def adjacency(self):
        na = self.lib.orc_mesh_nadj(self.h)
        off = np.zeros(self.nc + 1, dtype=np.int32)
        face = np.zeros(na, dtype=np.int32)
        nb = np.zeros(na, dtype=np.int32)
        sign = np.zeros(na)
        self.lib.orc_mesh_adjacency(self.h, *[x.ctypes.data_as(C.c_void_p) for x in (off, face, nb, sign)])
        return {"off": off, "face": face, "nb": nb, "sign": sign}

    def smooth_to_fixpoint(self, tau):
        t = _i32(tau).copy()
        sweeps = self.lib.orc_smooth_to_fixpoint(self.h, t.ctypes.data_as(C.c_void_p))
        return t, sweeps

    def __del__(self):
        try:
            self.lib.orc_mesh_free(self.h)
        except Exception:
            pass


class OracleSolver(_SolverBase):
    """Our restatement: SolverState + SolverOptions + the sequential driver."""

    prefix = "orc_"
    INT_ARRAYS = {"raw_level", "committed_front", "staged_front", "face_staged", "face_front"}

    def __init__(self, mesh, model="euler", a=(1.0, 0.0), gamma=1.4, threads=1):
        self.lib = oracle_lib()
        self.omesh = mesh if isinstance(mesh, OracleMesh) else OracleMesh(mesh)
        self.nc, self.nf = self.omesh.nc, self.omesh.nf
        self.nv = 5 if model == "euler" else 1
        h = C.c_void_p()
        f = self.lib.orc_solver_create
        f.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double, C.c_double, C.c_void_p]
        self._c(f(self.omesh.h, model.encode(), a[0], a[1], gamma, C.byref(h)))
        self.h = h
        if threads != 1:
            self.set_threads(threads)

    def set_threads(self, n):
        self.lib.orc_set_threads(self.h, int(n))

    def __del__(self):
        try:
            self.lib.orc_solver_free(self.h)
        except Exception:
            pass

    def _size(self, name):
        per = self.nv
        if name == "dt_max" or name in self.INT_ARRAYS and not name.startswith("face_"):
            return self.nc
        if name in ("face_staged", "face_front"):
            return self.nf
        if name == "grad":
            return self.nc * per * 3
        if name.startswith("face_") or name in ("phi_pred", "int_substep", "int_window"):
            return self.nf * per
        return self.nc * per

    def set_time(self, t0, iteration):
        f = self.lib.orc_set_time
        f.argtypes = [C.c_void_p, C.c_double, C.c_int]
        f(self.h, t0, iteration)

    def rusanov(self, wl, wr, n):
        out = np.zeros(self.nv)
        wl, wr, n = _f64(wl), _f64(wr), _f64(n)
        self._c(self.lib.orc_rusanov(self.h, *[x.ctypes.data_as(C.c_void_p) for x in (wl, wr, n, out)]))
        return out


def orc_subiteration_level(s, theta):
    lib = oracle_lib()
    out = C.c_int()
    _check(lib, lib.orc_subiteration_level(s, theta, C.byref(out)), "orc_last_error")
    return out.value


def orc_classify_raw(dt_max, dt_min, theta_max):
    lib = oracle_lib()
    f = lib.orc_classify_raw
    f.argtypes = [C.c_double, C.c_double, C.c_int, C.c_void_p]
    out = C.c_int()
    _check(lib, f(dt_max, dt_min, theta_max, C.byref(out)), "orc_last_error")
    return out.value


def orc_cost_shares(cell_shares):
    lib = oracle_lib()
    v = _f64(cell_shares)
    cost = np.zeros(len(v))
    ratio = C.c_double()
    _check(lib, lib.orc_cost_shares(v.ctypes.data_as(C.c_void_p), len(v), cost.ctypes.data_as(C.c_void_p),
                                    C.byref(ratio)), "orc_last_error")
    return cost, ratio.value


def orc_minmod(x, y):
    return oracle_lib().orc_minmod(x, y)

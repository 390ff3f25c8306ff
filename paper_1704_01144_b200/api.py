"""Host-side mirror of the reference solver interface over the C ABI.

Names, argument meaning and error behaviour follow the reference's C++
entry points (proj/core/include/tafv/reference.hpp:13-58):

==========================  ==================================================
reference                   here
==========================  ==================================================
SolverOptions               :class:`SolverOptions` (model moves to Physics)
plan_iteration(m, st, opt)  :meth:`Solver.plan_iteration`
run_iteration(.., plan)     :meth:`Solver.inject_levels` + :meth:`Solver.run_iteration`
reference_iteration         :meth:`Solver.reference_iteration`
reference_integrate         :meth:`Solver.reference_integrate`
SolverState w / W / t0      :meth:`Solver.set_state` / :meth:`Solver.get_state`
std::invalid_argument       :class:`InvalidArgument` (ValueError)
std::logic_error            :class:`LogicError`
std::runtime_error          :class:`Diverged`
==========================  ==================================================

Every compute call runs on the GPU through ``libtafv_gpu.so``; there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


class TafvError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument (tafv::require, common.hpp:9-11)."""


class LogicError(TafvError):
    """std::logic_error (TAFV_ASSERT, common.hpp:15-19)."""


class Diverged(TafvError):
    """std::runtime_error("integrate: solution diverged ...") (reference.cpp:124)."""


class CudaError(TafvError):
    pass


_EXC = {N.TAFV_EINVAL: InvalidArgument, N.TAFV_ELOGIC: LogicError,
        N.TAFV_EDIVERGED: Diverged, N.TAFV_ECUDA: CudaError, N.TAFV_ENCCL: CudaError}

MODELS = {"advection": N.TAFV_ADVECTION, "burgers": N.TAFV_BURGERS, "euler": N.TAFV_EULER}


@dataclass
class SolverOptions:
    """SolverOptions (reference.hpp:13-18) without the model."""

    theta_max: int = 3
    cfl: float = 0.9
    dt_cap: float = 1.0

    def c(self):
        return N.Options(int(self.theta_max), float(self.cfl), float(self.dt_cap))


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Comm:
    """Communicator of a decomposed run (tafv_comm): NCCL across processes or
    an in-process loopback for ranks run as threads."""

    def __init__(self, h):
        self.lib = N.lib()
        self.h = h

    @staticmethod
    def nccl_unique_id():
        buf = (C.c_uint8 * 128)()
        if N.lib().tafv_comm_nccl_unique_id(buf) != 0:
            raise CudaError("ncclGetUniqueId failed")
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id, rank, nranks, device=0):
        lib = N.lib()
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        rc = lib.tafv_comm_create_nccl(buf, rank, nranks, device, C.byref(h))
        if rc != 0:
            raise _EXC.get(rc, TafvError)(lib.tafv_gpu_last_error(None).decode())
        return cls(h)

    @classmethod
    def loopback(cls, nranks):
        h = C.c_void_p()
        if N.lib().tafv_comm_create_loopback(nranks, C.byref(h)) != 0:
            raise InvalidArgument("loopback: nranks must be >= 1")
        return cls(h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.tafv_comm_destroy(self.h)
            self.h = None


class Solver:
    """One mesh + SolverState resident on one GPU (a ``tafv_gpu`` handle).

    ``mesh`` is a mesh dict (reference Mesh layout, Vec3):
    ``dim, vol, cen, chl, fl, fr, fp, fn, fa, fc``.
    """

    def __init__(self, mesh, model="euler", a=(1.0, 0.0), gamma=1.4, device=0, shard=None):
        """shard=(rank_of_cell, rank, comm): one rank of a decomposed run
        over the GLOBAL mesh (tafv_gpu_create_shard)."""
        self.lib = N.lib()
        self.model = model
        self.nv = 5 if model == "euler" else 1
        self.nc = int(len(mesh["vol"]))
        self.nf = int(len(mesh["fa"]))
        arrs = dict(
            cell_volume=_f64(mesh["vol"]), cell_centroid=_f64(mesh["cen"]),
            cell_char_length=_f64(mesh["chl"]), face_left=_i32(mesh["fl"]),
            face_right=_i32(mesh["fr"]), face_partner=_i32(mesh["fp"]),
            face_normal=_f64(mesh["fn"]), face_area=_f64(mesh["fa"]),
            face_centroid=_f64(mesh["fc"]))
        assert arrs["cell_centroid"].size == 3 * self.nc and arrs["face_normal"].size == 3 * self.nf
        mv = N.MeshView(int(mesh["dim"]), self.nc, self.nf, *[_ptr(arrs[k]) for k in (
            "cell_volume", "cell_centroid", "cell_char_length", "face_left", "face_right",
            "face_partner", "face_normal", "face_area", "face_centroid")])
        ph = N.Physics(MODELS[model], (C.c_double * 3)(a[0], a[1], a[2] if len(a) > 2 else 0.0), gamma)
        h = C.c_void_p()
        if shard is None:
            rc = self.lib.tafv_gpu_create(C.byref(mv), C.byref(ph), device, C.byref(h))
        else:
            roc, rank, comm = shard
            self._roc = np.ascontiguousarray(roc, dtype=np.int32)
            rc = self.lib.tafv_gpu_create_shard(C.byref(mv), C.byref(ph), device, _ptr(self._roc), int(rank),
                                                comm.h, C.byref(h))
            self.rank = int(rank)
            self.owned = self._roc == self.rank
            # the GLOBAL mesh view stays alive for in-library repartitions
            # (DistDriver keeps its const Mesh&)
            self._mesh_arrs, self._mv = arrs, mv
        if rc != 0:
            raise _EXC.get(rc, TafvError)(self.lib.tafv_gpu_last_error(None).decode())
        self.h = h
        self.vol = arrs["cell_volume"]
        self._plan = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.tafv_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, rc):
        if rc != 0:
            raise _EXC.get(rc, TafvError)(self.lib.tafv_gpu_last_error(self.h).decode())

    # -- state ---------------------------------------------------------------
    def set_state(self, w, W=None, t0=0.0, iteration=0):
        """SolverState w/W/t0/iteration; W=None -> W = w*V (sync_extensive);
        w=None -> w = W/V (the relation every corrector leaves)."""
        if w is None and W is None:
            raise InvalidArgument("set_state: w and W are both None")
        wa = None if w is None else _f64(w).reshape(-1)
        Wa = None if W is None else _f64(W).reshape(-1)
        for a in (wa, Wa):
            if a is not None and a.size != self.nc * self.nv:
                raise InvalidArgument("set_state: wrong state size")
        self._c(self.lib.tafv_gpu_set_state(self.h, _ptr(wa), _ptr(Wa), float(t0), int(iteration)))

    def repartition(self, rank_of_cell=None, axis=0):
        """DistDriver::repartition (exchange.cpp:595-609), collective over
        the shard's ranks, in place (tafv_gpu_repartition): the committed
        state migrates, the shard is rebuilt on the device. rank_of_cell=None:
        level-cost slabs along `axis` from the last plan. Returns the
        partition now in force."""
        if not hasattr(self, "_mv"):
            raise InvalidArgument("repartition: not a shard")
        roc = None if rank_of_cell is None else np.ascontiguousarray(rank_of_cell, dtype=np.int32)
        out = np.empty(self.nc, dtype=np.int32)
        self._c(self.lib.tafv_gpu_repartition(self.h, C.byref(self._mv), _ptr(roc), int(axis), _ptr(out)))
        self._roc = out
        self.owned = out == self.rank
        return out

    def set_repartition(self, every, axis=0):
        """DistOptions::repartition_every: reference_integrate repartitions
        by level cost every `every` iterations (0: off)."""
        if not hasattr(self, "_mv"):
            raise InvalidArgument("set_repartition: not a shard")
        self._c(self.lib.tafv_gpu_set_repartition(self.h, C.byref(self._mv), int(every), int(axis)))

    def get_state(self):
        """(w, W, t0, iteration); a shard fills only its owned rows (zeros elsewhere)."""
        w = np.zeros((self.nc, self.nv))
        W = np.zeros((self.nc, self.nv))
        t0, it = C.c_double(), C.c_int32()
        self._c(self.lib.tafv_gpu_get_state(self.h, _ptr(w), _ptr(W), C.byref(t0), C.byref(it)))
        if self.nv == 1:
            w, W = w[:, 0], W[:, 0]
        return w, W, t0.value, it.value

    def run_batch(self, W_in, W_out, opt: SolverOptions, iterations=1):
        """tafv_gpu_run_batch: independent inputs W_in[j] (extensive rows,
        original cell order -- a shard: its local cells in
        shard.describe()["cells"] order; w = W / V) each advanced `iterations`
        iterations into W_out[j], copies overlapped with compute. Buffers are
        numpy arrays or host tensors exposing data_ptr() (pin them for the
        overlap). Returns the record of the last iteration."""
        def ptr(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        n = len(W_in)
        if len(W_out) != n:
            raise InvalidArgument("run_batch: W_in and W_out differ in length")
        # a shard's arrays hold its local cells (shard.describe()["cells"] order)
        rows = self.mesh_info()["n_cells"] if hasattr(self, "rank") else self.nc
        for a in list(W_in) + list(W_out):
            # the library copies rows*nv*8 bytes through the raw pointer: only
            # C-contiguous float64 HOST buffers of exactly that size are safe
            if hasattr(a, "data_ptr"):  # torch tensor
                import torch
                ok = (a.dtype == torch.float64 and a.is_contiguous() and a.device.type == "cpu"
                      and a.numel() == rows * self.nv)
            else:
                ok = (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                      and a.size == rows * self.nv)
            if not ok:
                raise InvalidArgument("run_batch: buffers must be C-contiguous float64 host arrays of "
                                      f"{rows} x {self.nv} values")
        for a in W_out:
            if not (a.flags.writeable if isinstance(a, np.ndarray) else True):
                raise InvalidArgument("run_batch: output buffer is read-only")
        pin = (C.c_void_p * max(1, n))(*[ptr(a) for a in W_in])
        pout = (C.c_void_p * max(1, n))(*[ptr(a) for a in W_out])
        rec = N.Record()
        self._c(self.lib.tafv_gpu_run_batch(self.h, C.byref(opt.c()), n, int(iterations), pin, pout,
                                           C.byref(rec)))
        self._plan = None
        return rec.as_dict()

    def iterate_host(self, W_host, opt: SolverOptions, n=1):
        """tafv_gpu_iterate_host: reference_integrate with the state held in
        the caller's HOST buffer W_host (extensive rows, original cell order;
        a shard: its local cells in shard.describe()["cells"] order), which
        every iteration uploads and receives the new W. Returns the records."""
        rows = self.mesh_info()["n_cells"] if hasattr(self, "rank") else self.nc
        if hasattr(W_host, "data_ptr"):
            import torch
            ok = (W_host.dtype == torch.float64 and W_host.is_contiguous() and W_host.device.type == "cpu"
                  and W_host.numel() == rows * self.nv)
            p = W_host.data_ptr()
        else:
            ok = (isinstance(W_host, np.ndarray) and W_host.dtype == np.float64 and W_host.flags.c_contiguous
                  and W_host.flags.writeable and W_host.size == rows * self.nv)
            p = W_host.ctypes.data if ok else None
        if not ok:
            raise InvalidArgument("iterate_host: W_host must be a writable C-contiguous float64 host array of "
                                  f"{rows} x {self.nv} values")
        recs = (N.Record * max(1, n))()
        self._c(self.lib.tafv_gpu_iterate_host(self.h, C.byref(opt.c()), int(n), C.c_void_p(p), recs))
        self._plan = None
        return [recs[i].as_dict() for i in range(n)]

    def get_array(self, name):
        if name in ("raw_level", "tau"):
            out = np.zeros(self.nc, dtype=np.int32)
        elif name == "mesh_digest":
            out = np.zeros(20, dtype=np.uint64)
        elif name == "repartition_ms":
            out = np.zeros(1)
        elif name == "brick_info":
            out = np.zeros(4)
        elif name == "brick_counts":
            out = np.zeros((int(self.get_array("brick_info")[0]), 4), dtype=np.int32)
        else:
            rows = self.nf if name in ("phi_pred", "int_substep", "int_window") else self.nc
            width = {"grad": self.nv * 3, "dt_max": 1}.get(name, self.nv)
            out = np.empty((rows, width))
        self._c(self.lib.tafv_gpu_get_array(self.h, name.encode(), _ptr(out)))
        return out

    # -- plan ----------------------------------------------------------------
    def plan_iteration(self, opt: SolverOptions):
        """plan_iteration (reference.cpp:89-98), on the device."""
        info = N.PlanInfo()
        self._plan = None
        self._c(self.lib.tafv_gpu_plan(self.h, C.byref(opt.c()), C.byref(info)))
        self._plan = info.as_dict()
        return self._plan

    def inject_levels(self, tau, dt, opt: SolverOptions | None = None):
        """build_iteration_plan(mesh, make_level_map(tau, dt)) (levels.cpp).
        dt <= 0: dt = min_c dt_max_c / 2^tau_c using opt's cfl/dt_cap."""
        info = N.PlanInfo()
        t = _i32(tau)
        assert t.size == self.nc
        o = opt.c() if opt is not None else None
        self._plan = None
        self._c(self.lib.tafv_gpu_inject_levels(self.h, _ptr(t), float(dt),
                                                C.byref(o) if o is not None else None, C.byref(info)))
        self._plan = info.as_dict()
        return self._plan

    def plan_lists(self):
        """tau, face_cadence, cells_of_level, faces_of_cadence, fringe in
        original ids (ascending within each level), from the device lists."""
        info = self._plan
        if info is None:
            raise InvalidArgument("get_plan_lists: no plan")
        tau = np.empty(self.nc, dtype=np.int32)
        cad = np.empty(self.nf, dtype=np.int32)
        cells = np.empty(self.nc, dtype=np.int32)
        faces = np.empty(self.nf, dtype=np.int32)
        fringe = np.empty(max(1, int(sum(info["fringe_per_level"]))), dtype=np.int32)
        self._c(self.lib.tafv_gpu_get_plan_lists(self.h, _ptr(tau), _ptr(cad), _ptr(cells),
                                                 _ptr(faces), _ptr(fringe)))

        def split(flat, counts):
            out, o = [], 0
            for n in counts:
                out.append(flat[o:o + int(n)].copy())
                o += int(n)
            return out

        return {
            "tau": tau, "face_cadence": cad, "theta": info["theta"], "dt": info["dt"],
            "cost_ratio": info["cost_ratio"],
            "cells_of_level": split(cells, info["cells_per_level"]),
            "faces_of_cadence": split(faces, info["faces_per_cadence"]),
            "fringe": split(fringe, info["fringe_per_level"]),
        }

    # -- iteration -----------------------------------------------------------
    def run_iteration(self):
        """run_iteration under the current plan (reference.cpp:100-129)."""
        r = N.Record()
        self._c(self.lib.tafv_gpu_run_iteration(self.h, C.byref(r)))
        return r.as_dict()

    def reference_iteration(self, opt: SolverOptions):
        self.plan_iteration(opt)
        return self.run_iteration()

    def reference_integrate(self, opt: SolverOptions, iterations: int):
        """reference_integrate (reference.cpp:135-142)."""
        if iterations < 0:
            raise InvalidArgument("integrate: negative iteration count")
        recs = (N.Record * max(1, iterations))()
        self._plan = None
        self._c(self.lib.tafv_gpu_iterate(self.h, C.byref(opt.c()), int(iterations), recs))
        return [recs[i].as_dict() for i in range(iterations)]

    integrate = reference_integrate

    def advance(self, opt: SolverOptions, iterations: int):
        r = N.Record()
        self._c(self.lib.tafv_gpu_advance(self.h, C.byref(opt.c()), int(iterations), C.byref(r)))
        return r.as_dict()

    def stats(self):
        n = C.c_int64()
        ms = (C.c_double * 3)()
        self.lib.tafv_gpu_stats(self.h, C.byref(n), ms)
        return {"launches": n.value, "ms_total": ms[0], "ms_plan": ms[1], "ms_sweep": ms[2]}

    KERNEL_KINDS = ("K1_grad_limit", "K2_face_pred", "K2_face_corr", "K3_update_pred",
                    "K3_update_corr", "plan")

    def kernel_times(self):
        ms = (C.c_double * 6)()
        n = (C.c_int64 * 6)()
        it = (C.c_int64 * 18)()
        self.lib.tafv_gpu_kernel_times(self.h, ms, n, it)
        return {k: {"ms": ms[i], "launches": n[i], "cells": it[3 * i], "faces": it[3 * i + 1],
                    "fringe": it[3 * i + 2]} for i, k in enumerate(self.KERNEL_KINDS)}

    def mesh_info(self):
        v = (C.c_int64 * 4)()
        self.lib.tafv_gpu_mesh_info(self.h, v)
        return {"n_cells": v[0], "n_faces": v[1], "adj_slots": v[2], "nv": v[3]}

    def set_flag(self, name, value):
        self._c(self.lib.tafv_gpu_set_flag(self.h, name.encode(), int(value)))

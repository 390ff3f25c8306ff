"""ctypes binding of the C ABI in include/tafv_gpu.h (libtafv_gpu.so).

The product path has no CPU fallback: if the in-tree library is missing the
import fails loudly (run ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1704_01144_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TAFV_GPU_LIB overrides the in-tree library (A/B of two builds in one run).
LIB_PATH = os.environ.get("TAFV_GPU_LIB") or os.path.join(HERE, "libtafv_gpu.so")

TAFV_OK, TAFV_EINVAL, TAFV_ELOGIC, TAFV_EDIVERGED, TAFV_ECUDA, TAFV_ENCCL = range(6)
TAFV_ADVECTION, TAFV_BURGERS, TAFV_EULER = 0, 1, 2
MAX_LEVELS = 16


class MeshView(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("n_cells", C.c_int32),
        ("n_faces", C.c_int32),
        ("cell_volume", C.c_void_p),
        ("cell_centroid", C.c_void_p),
        ("cell_char_length", C.c_void_p),
        ("face_left", C.c_void_p),
        ("face_right", C.c_void_p),
        ("face_partner", C.c_void_p),
        ("face_normal", C.c_void_p),
        ("face_area", C.c_void_p),
        ("face_centroid", C.c_void_p),
    ]


class Physics(C.Structure):
    _fields_ = [("model", C.c_int32), ("a", C.c_double * 3), ("gamma", C.c_double)]


class Options(C.Structure):
    _fields_ = [("theta_max", C.c_int32), ("cfl", C.c_double), ("dt_cap", C.c_double)]


class Record(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32),
        ("theta", C.c_int32),
        ("t_start", C.c_double),
        ("dt", C.c_double),
        ("advance", C.c_double),
        ("cost_ratio", C.c_double),
        ("total_extensive", C.c_double * 8),
        ("level_cells", C.c_int64 * MAX_LEVELS),
        ("n_levels", C.c_int32),
        ("nv", C.c_int32),
        ("boundary_flux", C.c_double * 8),
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
            "boundary_flux": list(self.boundary_flux[: self.nv]),
        }


class PlanInfo(C.Structure):
    _fields_ = [
        ("theta", C.c_int32),
        ("n_levels", C.c_int32),
        ("dt", C.c_double),
        ("cost_ratio", C.c_double),
        ("cells_per_level", C.c_int64 * MAX_LEVELS),
        ("faces_per_cadence", C.c_int64 * MAX_LEVELS),
        ("fringe_per_level", C.c_int64 * MAX_LEVELS),
        ("c_eff", C.c_int64),
        ("f_eff", C.c_int64),
        ("r_eff", C.c_int64),
    ]

    def as_dict(self):
        t = self.theta
        return {
            "theta": t,
            "dt": self.dt,
            "cost_ratio": self.cost_ratio,
            "cells_per_level": list(self.cells_per_level[: t + 1]),
            "faces_per_cadence": list(self.faces_per_cadence[: t + 1]),
            "fringe_per_level": list(self.fringe_per_level[:t]),
            "c_eff": self.c_eff,
            "f_eff": self.f_eff,
            "r_eff": self.r_eff,
        }


# Exported symbols (declared in include/tafv_gpu.h); tests check every one.
EXPORTS = [
    "tafv_gpu_create", "tafv_gpu_destroy", "tafv_gpu_last_error", "tafv_gpu_set_state",
    "tafv_gpu_get_state", "tafv_gpu_plan", "tafv_gpu_inject_levels", "tafv_gpu_get_plan_lists",
    "tafv_gpu_run_iteration", "tafv_gpu_iterate", "tafv_gpu_advance", "tafv_gpu_run_batch", "tafv_gpu_iterate_host", "tafv_gpu_get_array",
    "tafv_gpu_set_flag", "tafv_gpu_stats", "tafv_gpu_kernel_times", "tafv_gpu_mesh_info", "tafv_mesh_hex", "tafv_mesh_hex_window",
    "tafv_partition_slabs", "tafv_shard_describe", "tafv_level_smooth", "tafv_shard_last_error",
    "tafv_comm_nccl_unique_id", "tafv_comm_create_nccl", "tafv_comm_create_loopback",
    "tafv_comm_destroy", "tafv_gpu_create_shard", "tafv_gpu_repartition", "tafv_gpu_set_repartition",
    "tafv_mesh_save", "tafv_mesh_load", "tafv_mesh_hash", "tafv_snapshot_save", "tafv_snapshot_load",
    "tafv_snapshot_compare", "tafv_io_last_error",
]

_lib = None


def bind_meshgen(L):
    """argtypes of the mesh generator entry points (csrc/meshgen.cpp), which
    the CPU checker library (oracle/) also compiles in, so a reference-arm
    process can build a config's mesh without mapping this library."""
    vp, i32, dbl = C.c_void_p, C.c_int32, C.c_double
    L.tafv_mesh_hex.argtypes = [i32, i32, i32, vp, vp, vp, dbl, C.c_uint64, i32,
                                C.POINTER(i32), C.POINTER(i32)] + [vp] * 9
    L.tafv_mesh_hex_window.argtypes = [i32, i32, i32, vp, vp, vp, vp, dbl, C.c_uint64,
                                       C.POINTER(i32), C.POINTER(i32)] + [vp] * 9
    return L


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"CUDA library missing: {LIB_PATH}; build it with __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    if os.environ.get("TAFV_GPU_LIB"):  # A/B against an older build: bind what it has
        class _Tolerant:
            def __init__(self, lib):
                self.__dict__["_lib"] = lib

            def __getattr__(self, name):
                try:
                    return getattr(self._lib, name)
                except AttributeError:
                    return type("Missing", (), {"argtypes": None, "restype": None})()

            def __setattr__(self, name, value):
                setattr(self._lib, name, value)
        L = _Tolerant(L)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.tafv_gpu_create.argtypes = [C.POINTER(MeshView), C.POINTER(Physics), C.c_int, C.POINTER(vp)]
    L.tafv_gpu_destroy.argtypes = [vp]
    L.tafv_gpu_destroy.restype = None
    L.tafv_gpu_last_error.argtypes = [vp]
    L.tafv_gpu_last_error.restype = C.c_char_p
    L.tafv_gpu_run_batch.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    L.tafv_gpu_iterate_host.argtypes = [vp, C.POINTER(Options), i32, vp, vp]
    L.tafv_gpu_set_state.argtypes = [vp, vp, vp, dbl, i32]
    L.tafv_gpu_get_state.argtypes = [vp, vp, vp, C.POINTER(dbl), C.POINTER(i32)]
    L.tafv_gpu_plan.argtypes = [vp, C.POINTER(Options), C.POINTER(PlanInfo)]
    L.tafv_gpu_inject_levels.argtypes = [vp, vp, dbl, C.POINTER(Options), C.POINTER(PlanInfo)]
    L.tafv_gpu_get_plan_lists.argtypes = [vp, vp, vp, vp, vp, vp]
    L.tafv_gpu_run_iteration.argtypes = [vp, C.POINTER(Record)]
    L.tafv_gpu_iterate.argtypes = [vp, C.POINTER(Options), i32, C.POINTER(Record)]
    L.tafv_gpu_advance.argtypes = [vp, C.POINTER(Options), i32, C.POINTER(Record)]
    L.tafv_gpu_get_array.argtypes = [vp, C.c_char_p, vp]
    L.tafv_gpu_set_flag.argtypes = [vp, C.c_char_p, i64]
    L.tafv_gpu_stats.argtypes = [vp, C.POINTER(i64), vp]
    L.tafv_gpu_kernel_times.argtypes = [vp, vp, vp, vp]
    L.tafv_gpu_mesh_info.argtypes = [vp, vp]
    bind_meshgen(L)
    L.tafv_partition_slabs.argtypes = [C.POINTER(MeshView), i32, i32, vp, vp]
    L.tafv_shard_describe.argtypes = [C.POINTER(MeshView), vp, i32, i32] + [vp] * 8
    L.tafv_level_smooth.argtypes = [C.POINTER(MeshView), vp]
    L.tafv_shard_last_error.restype = C.c_char_p
    L.tafv_comm_nccl_unique_id.argtypes = [vp]
    L.tafv_comm_create_nccl.argtypes = [vp, i32, i32, C.c_int, C.POINTER(vp)]
    L.tafv_comm_create_loopback.argtypes = [i32, C.POINTER(vp)]
    L.tafv_comm_destroy.argtypes = [vp]
    L.tafv_comm_destroy.restype = None
    L.tafv_gpu_create_shard.argtypes = [C.POINTER(MeshView), C.POINTER(Physics), C.c_int, vp, i32, vp,
                                        C.POINTER(vp)]
    L.tafv_gpu_repartition.argtypes = [vp, C.POINTER(MeshView), vp, i32, vp]
    L.tafv_gpu_set_repartition.argtypes = [vp, C.POINTER(MeshView), i32, i32]
    L.tafv_mesh_save.argtypes = [C.c_char_p, C.POINTER(MeshView)]
    L.tafv_mesh_load.argtypes = [C.c_char_p, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)] + [vp] * 9
    L.tafv_mesh_hash.argtypes = [C.POINTER(MeshView)]
    L.tafv_mesh_hash.restype = C.c_uint64
    L.tafv_snapshot_save.argtypes = [C.c_char_p, i32, C.c_uint64, i32, i32, dbl, i32, vp, vp]
    L.tafv_snapshot_load.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(i32), C.POINTER(i32),
                                     C.POINTER(dbl), C.POINTER(i32), vp, vp]
    L.tafv_snapshot_compare.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(dbl)]
    L.tafv_io_last_error.restype = C.c_char_p
    _lib = L
    return L

"""Mesh / snapshot formats, CPU only.

Against the real reference where it is available (oracle/_ref): meshes the
reference writes with Mesh::save (TFVM v1) load unchanged and hash to the
reference's Mesh::hash; our scalar text snapshot is byte-identical to
save_snapshot; compare_snapshots agrees with the reference's."""
import ctypes as C

import numpy as np
import pytest

from oracle import RefSolver, ref_available, ref_generate_mesh, ref_lib
from paper_1704_01144_b200 import InvalidArgument, configs
from paper_1704_01144_b200 import io as fio

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("spec", [dict(dim=2, nx=8, ny=6, periodic_x=True, regions=[((0.25, 0.25, 0.75, 0.75), 2)]),
                                  dict(dim=1, nx=10, periodic_x=False, regions=[((0.5, 0.0, 1.0, 1.0), 4)])])
def test_reference_mesh_file_loads_and_hashes(tmp_path, spec):
    mesh, adj, mh = ref_generate_mesh(**spec)
    path = tmp_path / "ref.tfvm"
    assert ref_lib().ref_mesh_save(mh, str(path).encode()) == 0
    m = fio.load_mesh(path)
    for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc"):
        np.testing.assert_array_equal(m[k], mesh[k])
    assert m["dim"] == spec["dim"]
    assert fio.mesh_hash(m) == adj["hash"]          # == Mesh::hash (mesh.cpp:326-343)


def test_mesh_v2_round_trip(tmp_path):
    m = configs.get(2, 10).mesh()
    p = tmp_path / "m.tfvm"
    fio.save_mesh(p, m)
    r = fio.load_mesh(p)
    for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc"):
        np.testing.assert_array_equal(r[k], m[k])
    assert fio.mesh_hash(r) == fio.mesh_hash(m)
    m2 = dict(m)
    m2["vol"] = m["vol"].copy()
    m2["vol"][0] = np.nextafter(m2["vol"][0], 1.0)
    assert fio.mesh_hash(m2) != fio.mesh_hash(m)


_REF_WRITER = r"""
import ctypes as C, sys
L = C.CDLL(sys.argv[1])
dom = (C.c_double * 4)(0, 0, 1, 1)
m, s = C.c_void_p(), C.c_void_p()
assert L.ref_mesh_generate(2, 6, 5, dom, 1, 1, 0, None, None, C.byref(m)) == 0
assert L.ref_solver_create(m, b"advection", C.c_double(1.0), C.c_double(0.5), C.byref(s)) == 0
L.ref_init_gaussian.argtypes = [C.c_void_p] + [C.c_double] * 5
assert L.ref_init_gaussian(s, 1.0, 1.0, 0.5, 0.5, 0.15) == 0
L.ref_set_options.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double]
L.ref_set_options(s, 3, 0.5, 1.0)
recs = (C.c_byte * (4096 * 3))()
assert L.ref_integrate(s, 3, recs) == 0
assert L.ref_snapshot_save(s, sys.argv[2].encode()) == 0
assert L.ref_mesh_save(m, sys.argv[3].encode()) == 0
"""


@needs_ref
def test_scalar_text_snapshot_byte_identical_to_reference(tmp_path):
    """Our text writer == the reference's save_snapshot (state.cpp:77-91) byte
    for byte. The reference writer runs in a numpy-free subprocess (its
    iostream output crashes in a process that has numpy's bundled runtime
    libraries loaded; unrelated to the code under test)."""
    import subprocess
    import sys
    from oracle import REF_SO
    a, mpath, b = tmp_path / "ref.snap", tmp_path / "ref.tfvm", tmp_path / "ours.snap"
    subprocess.run([sys.executable, "-c", _REF_WRITER, REF_SO, str(a), str(mpath)], check=True)
    mesh = fio.load_mesh(mpath)
    s = fio.load_snapshot(a)
    assert s["mesh_hash"] == fio.mesh_hash(mesh)
    fio.save_snapshot(b, mesh, s["w"], s["W"], s["time"], s["iteration"])
    assert a.read_bytes() == b.read_bytes()
    # compare_snapshots agrees with the reference's
    w2 = s["w"].copy()
    w2[3] *= 1.0 + 1e-9
    c = tmp_path / "perturbed.snap"
    fio.save_snapshot(c, mesh, w2, s["W"], s["time"], s["iteration"])
    cmp = ("import ctypes as C, sys; L = C.CDLL(sys.argv[1]); w = C.c_double(); "
           "assert L.ref_snapshot_compare(sys.argv[2].encode(), sys.argv[3].encode(), C.byref(w)) == 0; "
           "print(repr(w.value))")
    out = subprocess.run([sys.executable, "-c", cmp, REF_SO, str(a), str(c)], check=True,
                         capture_output=True, text=True).stdout
    worst = float(out.strip())
    assert fio.compare_snapshots(a, c) == worst
    assert 5e-10 < worst < 2e-9


@pytest.mark.parametrize("binary", [False, True])
def test_euler_snapshot_round_trip_and_compare(tmp_path, binary):
    cfg = configs.get(1, 16)
    m = cfg.mesh()
    w = cfg.initial_state(m)
    W = w * m["vol"][:, None]
    p = tmp_path / "s"
    fio.save_snapshot(p, m, w, W, 0.125, 7, binary=binary)
    s = fio.load_snapshot(p)
    np.testing.assert_array_equal(s["w"], w)
    np.testing.assert_array_equal(s["W"], W)
    assert (s["time"], s["iteration"], s["mesh_hash"]) == (0.125, 7, fio.mesh_hash(m))
    q = tmp_path / "q"
    w2 = w.copy()
    w2[5, 4] *= 1.0 + 3e-12
    fio.save_snapshot(q, m, w2, W, 0.125, 7, binary=not binary)
    assert 2e-12 < fio.compare_snapshots(p, q) < 4e-12
    assert fio.compare_snapshots(p, p) == 0.0


def test_compare_rejects_different_meshes(tmp_path):
    a, b = configs.get(1, 16).mesh(), configs.get(2, 16).mesh()
    for m, name in ((a, "a"), (b, "b")):
        w = np.ones((len(m["vol"]), 5))
        fio.save_snapshot(tmp_path / name, m, w, w, binary=True)
    with pytest.raises(InvalidArgument):
        fio.compare_snapshots(tmp_path / "a", tmp_path / "b")


def test_bad_files_raise(tmp_path):
    p = tmp_path / "junk"
    p.write_bytes(b"not a mesh")
    with pytest.raises(InvalidArgument):
        fio.load_mesh(p)
    with pytest.raises(InvalidArgument):
        fio.load_snapshot(p)

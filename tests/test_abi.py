"""CPU tests of the product's boundary and host logic (no GPU needed):
the C-ABI library loads and exports every symbol include/tafv_gpu.h
declares, the host-side 3D mesh generator (tafv_mesh_hex) produces closed,
consistent reference-layout meshes, and the config generators are sane."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1704_01144_b200 import _native as N
from paper_1704_01144_b200 import configs, meshgen


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tafv_gpu.h")).read()
    return sorted(set(re.findall(r"\b(tafv_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    for sym in declared:
        assert hasattr(lib, sym), f"{sym} declared in tafv_gpu.h but not exported"
    assert sorted(N.EXPORTS) == declared


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors have the C compiler's layout of the header's
    structs: sizeof and every field offset (gcc on include/tafv_gpu.h)."""
    import subprocess
    structs = {"tafv_mesh_view": N.MeshView, "tafv_record": N.Record, "tafv_options": N.Options,
               "tafv_plan_info": N.PlanInfo, "tafv_physics": N.Physics}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tafv_gpu.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {(a, b): int(c) for a, b, c in (l.split() for l in out if l.strip())}
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
    import oracle
    assert C.sizeof(oracle.Record) == C.sizeof(N.Record)


def test_create_without_gpu_fails_loudly_or_succeeds():
    """No silent CPU fallback: without a device, create reports a CUDA error."""
    try:
        import torch
        has = torch.cuda.is_available()
    except Exception:
        has = False
    if has:
        pytest.skip("GPU present: covered by the gpu suite")
    m = meshgen.hex_mesh(*(np.linspace(0, 1, 3),) * 3)
    from paper_1704_01144_b200 import CudaError, Solver
    with pytest.raises(CudaError):
        Solver(m, "euler")


def closure(m):
    nc = len(m["vol"])
    acc = np.zeros((nc, 3))
    s = m["fn"] * m["fa"][:, None]
    np.add.at(acc, m["fl"], s)
    inner = m["fr"] >= 0
    np.add.at(acc, m["fr"][inner], -s[inner])
    return np.abs(acc).max()


@pytest.mark.parametrize("jitter,permute", [(0.0, False), (0.15, True)])
def test_hex_mesh_geometry(jitter, permute):
    x = meshgen.geometric_nodes(9, 1.1)
    y = meshgen.uniform_nodes(7)
    z = meshgen.centre_graded_nodes(8, 1.2, 0.1)
    m = meshgen.hex_mesh(x, y, z, jitter=jitter, seed=5, permute=permute)
    nc, nf = 9 * 7 * 8, 10 * 7 * 8 + 9 * 8 * 8 + 9 * 7 * 9
    assert len(m["vol"]) == nc and len(m["fa"]) == nf
    assert closure(m) <= 1e-12                      # mesh.cpp:273-284 criterion
    assert abs(m["vol"].sum() - 1.0) <= 1e-12       # unit cube
    assert (m["vol"] > 0).all() and (m["chl"] > 0).all()
    np.testing.assert_allclose(np.linalg.norm(m["fn"], axis=1), 1.0, atol=1e-14)
    bnd = m["fr"] < 0
    assert bnd.sum() == 2 * (9 * 7 + 9 * 8 + 7 * 8)
    assert (m["fp"] == -1).all()
    # every cell has exactly 6 faces
    deg = np.bincount(m["fl"], minlength=nc) + np.bincount(m["fr"][~bnd], minlength=nc)
    assert (deg == 6).all()
    # normals point from left to right cell
    d = m["cen"][m["fr"][~bnd]] - m["cen"][m["fl"][~bnd]]
    assert ((d * m["fn"][~bnd]).sum(1) > 0).all()


def test_hex_mesh_permutation_is_a_relabelling():
    x = y = z = meshgen.uniform_nodes(5)
    a = meshgen.hex_mesh(x, y, z, jitter=0.1, seed=3, permute=False)
    b = meshgen.hex_mesh(x, y, z, jitter=0.1, seed=3, permute=True)
    ka = np.lexsort(a["cen"].T)
    kb = np.lexsort(b["cen"].T)
    assert np.array_equal(a["cen"][ka], b["cen"][kb])
    assert np.array_equal(a["vol"][ka], b["vol"][kb])
    fa = np.lexsort(a["fc"].T)
    fb = np.lexsort(b["fc"].T)
    assert np.array_equal(a["fn"][fa], b["fn"][fb])
    assert np.array_equal(a["fa"][fa], b["fa"][fb])


def test_hex_mesh_deterministic_and_seeded():
    x = y = z = meshgen.uniform_nodes(4)
    a = meshgen.hex_mesh(x, y, z, jitter=0.15, seed=11, permute=True)
    b = meshgen.hex_mesh(x, y, z, jitter=0.15, seed=11, permute=True)
    c = meshgen.hex_mesh(x, y, z, jitter=0.15, seed=12, permute=True)
    for k in ("cen", "vol", "fl", "fr", "fn"):
        assert np.array_equal(a[k], b[k])
    assert not np.array_equal(a["cen"], c["cen"])


def test_hex_mesh_rejects_bad_specs():
    with pytest.raises(ValueError):
        meshgen.hex_mesh([0.0, 0.5, 0.4], [0, 1], [0, 1])


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_configs_scaled(cid):
    cfg = configs.get(cid, 12)
    m = cfg.mesh()
    w = cfg.initial_state(m)
    assert w.shape == (len(m["vol"]), 5)
    assert (w[:, 0] > 0).all() and (w[:, 4] > 0).all()
    assert closure(m) <= 1e-12
    if cfg.synthetic_levels:
        tau = cfg.levels(m)
        assert tau.max() <= cfg.theta_max and tau.min() == 0
        inner = m["fr"] >= 0
        assert np.abs(tau[m["fl"][inner]] - tau[m["fr"][inner]]).max() <= 1


def test_config_sizes_match_baseline():
    assert configs.get(1).n_cells == 262144
    assert configs.get(2).n_cells == 1_000_000
    assert configs.get(3).n_cells == 8_000_000
    assert configs.get(4).n_cells == 80_062_991
    assert configs.get(5).n_cells == 16_003_008


def test_observe_tables_and_csv(tmp_path):
    """Paper Table 1 shares through the observability helpers."""
    from paper_1704_01144_b200 import observe
    rec = {"theta": 2, "level_cells": [5, 242, 9753], "cost_ratio": 3.9, "iteration": 1, "t_start": 0.0,
           "dt": 0.1, "advance": 0.4, "total_extensive": [1.0, 2.0]}
    tab = observe.level_table(rec)
    for got, want in zip([x[3] for x in tab], [0.20, 4.72, 95.08]):  # PAPER.md:570-583, test_levels.cpp:69-77
        assert abs(got - want) <= 0.01
    p = tmp_path / "r.csv"
    observe.records_to_csv([rec, rec], p, kernel_times={"K1": {"ms": 1.0, "launches": 2}})
    lines = p.read_text().splitlines()
    assert lines[0].startswith("iteration,t_start,dt,theta") and len(lines) >= 3

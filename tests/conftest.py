import glob
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def _ensure_built():
    """Build the in-tree libraries if a fresh checkout lacks them (no-op when
    __graft_entry__.build() already ran)."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "libtafv_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_1704_01144_b200", "libtafv_gpu.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1704_01144_b200", "csrc")], check=True)


_ensure_built()


def load_golden(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    mesh = {"dim": int(d["mesh_dim"])}
    for k in ("vol", "cen", "chl", "fl", "fr", "fp", "fn", "fa", "fc"):
        mesh[k] = d["mesh_" + k]
    d["mesh"] = mesh
    d["model"] = str(d["model"])
    return d


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def golden_plan_lists(d):
    th = int(d["plan_theta"])
    return {
        "tau": d["plan_tau"], "face_cadence": d["plan_cadence"],
        "cells_of_level": [d[f"plan_cells_{l}"] for l in range(th + 1)],
        "faces_of_cadence": [d[f"plan_faces_{l}"] for l in range(th + 1)],
        "fringe": [d[f"plan_fringe_{l}"] for l in range(th)],
    }


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    return 0

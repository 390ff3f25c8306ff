"""Multi-GPU (N >= 2 devices on one node): NCCL shards with the halo
exchange captured inside the sweep graphs, bitwise against the single-domain
run. Skips cleanly on boxes with fewer than 2 GPUs (every gpurun box here
has one); the SCALE run's 2/4/8-GPU path is exercised by it before any
timing."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("nproc,config,scale,rep", [(2, 2, 2, 0), (0, 3, 4, 0), (2, 3, 10, 1)])
def test_nccl_shards_bitwise(nproc, config, scale, rep, tmp_path):
    """rep > 0: in-library repartition (tafv_gpu_repartition, state migrated
    by NCCL all-reduces) before every rep-th iteration."""
    n = _ngpus()
    if n < 2:
        pytest.skip(f"needs >= 2 GPUs (found {n})")
    nproc = nproc or n  # 0: every GPU of the node
    out = tmp_path / "verdict.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tools", "multigpu_worker.py"),
           "--config", str(config), "--scale", str(scale), "--iters", "3", "--repartition-every", str(rep), "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(out.read_text())
    assert d["ok"], d

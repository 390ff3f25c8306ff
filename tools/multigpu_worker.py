#!/usr/bin/env python3
"""One rank of the multi-GPU parity check (tests/test_multigpu.py), launched
by torchrun with one process per GPU: NCCL shards of a config cut into
level-cost slabs, the sweeps captured as CUDA graphs with the halo exchange
inside (NCCL send/recv on the priority comm stream), `--iters` iterations.
Rank 0 then runs the single-domain solver on its GPU and checks bitwise
equality of the assembled owned rows (w, W) and of every record's dt,
level counts and cost ratio, plus the ledger totals within 1e-12. Writes a
JSON verdict to --out. --repartition-every k re-cuts the slabs in the library
(tafv_gpu_repartition over NCCL) before every k-th iteration."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1704_01144_b200 import Solver, configs, shard  # noqa: E402
from paper_1704_01144_b200.api import Comm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=int, default=2)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--repartition-every", type=int, default=0,
                help="DistOptions::repartition_every: in-library level-cost repartition (NCCL state migration)")
ap.add_argument("--out", required=True)
a = ap.parse_args()

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = configs.get(a.config, a.scale)
mesh = cfg.mesh()
w0 = cfg.initial_state(mesh)
opt = cfg.options()
roc = shard.partition_slabs(mesh, world, axis=0, weight=shard.initial_level_cost(mesh, w0, opt))
uid = [Comm.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = Comm.nccl(uid[0], rank, world, device=local)
s = Solver(mesh, "euler", device=local, shard=(roc, rank, comm))
s.set_state(w0)
if a.repartition_every:
    s.set_repartition(a.repartition_every, axis=0)
recs = s.reference_integrate(opt, a.iters)
w, W, t0, it = s.get_state()  # owned rows, zeros elsewhere
pair = torch.from_numpy(np.stack([w, W])).cuda()
dist.all_reduce(pair)
s.close()
comm.close()
out = {"world": world, "ok": True}
if rank == 0:
    wa, Wa = (x.cpu().numpy() for x in pair)
    g = Solver(mesh, "euler", device=local)
    g.set_state(w0)
    ref = g.reference_integrate(opt, a.iters)
    wr, Wr, t0r, _ = g.get_state()
    out["w_bitwise"] = wa.tobytes() == wr.tobytes()
    out["W_bitwise"] = Wa.tobytes() == Wr.tobytes()
    out["t_equal"] = t0 == t0r
    out["records_equal"] = all(x["dt"] == y["dt"] and x["level_cells"] == y["level_cells"] and
                               x["cost_ratio"] == y["cost_ratio"] for x, y in zip(recs, ref))
    out["totals_close"] = all(abs(p - q) <= 1e-12 * max(1.0, abs(q)) for x, y in zip(recs, ref)
                              for p, q in zip(x["total_extensive"] + x["boundary_flux"],
                                              y["total_extensive"] + y["boundary_flux"]))
    out["theta"] = [r["theta"] for r in recs]
    out["ok"] = all(out[k] for k in ("w_bitwise", "W_bitwise", "t_equal", "records_equal", "totals_close"))
    g.close()
    with open(a.out, "w") as f:
        json.dump(out, f)
dist.barrier()
dist.destroy_process_group()

"""Multi-rank path on CPU (gloo, world size 2 and 3): the decomposition the
multi-GPU solver uses, executed with the oracle's kernels per rank and real
torch.distributed (gloo) messages, must reproduce the single-domain run
bitwise.

Per rank: owned cells O + rings R1, R2 (tafv_shard_describe,
the product's host C++), faces touching O u R1. Plan: dt_max on O, all-reduce
MIN (exact, exchange.cpp:155-192); classification on O; theta_max Jacobi
sweeps with a tau halo exchange after each; theta = all-reduce MAX. Each
phase: stage every local active/fringe cell; gradients + limiter on active
O u R1 (ring-1 gradients recomputed locally from ring-2 values instead of the
reference's second exchange round, exchange.cpp:363-375); fluxes on active
faces touching O (duplicated across ranks, bitwise mirrors); updates on
active O; then the just-updated rows (w_pred after a predictor, w after a
corrector) of owned cells go to every peer holding them in its halo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(arr, nv, sh, rank):
    """Send owned rows to peers, receive halo rows (ascending global id)."""
    view = arr.reshape(-1, nv)
    reqs, bufs = [], {}
    for q in sorted(sh["send"]):
        t = torch.from_numpy(np.ascontiguousarray(view[sh["send"][q]]))
        reqs.append(dist.isend(t, dst=q))
    for q in sorted(sh["recv"]):
        bufs[q] = torch.empty((len(sh["recv"][q]), nv), dtype=torch.float64 if arr.dtype == np.float64 else torch.int32)
        reqs.append(dist.irecv(bufs[q], src=q))
    for r in reqs:
        r.wait()
    for q, b in bufs.items():
        view[sh["recv"][q]] = b.numpy()
    return arr


def _allreduce(x, op):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=op)
    return float(t.item())


def _rank_main(rank, world, port, cid, scale, iters, out, rep_every=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleMesh, OracleSolver
    from paper_1704_01144_b200 import configs, shard
    cfg = configs.periodic_blast() if cid == "P" else configs.get(cid, scale)
    mesh = cfg.mesh()
    w0 = cfg.initial_state(mesh)
    opt = cfg.options()
    nv = 5
    NG = len(mesh["vol"])

    def build(roc, w_global=None, W_global=None):
        sh = shard.describe(mesh, roc, rank, world)
        lm = shard.local_mesh(mesh, sh)
        cls = sh["cls"]
        own = np.flatnonzero(cls == 0).astype(np.int32)
        o = OracleSolver(OracleMesh(lm, closure_mask=cls <= 1), "euler")
        if W_global is None:
            o.init_values(w_global[sh["cells"]].reshape(-1))
        else:  # a repartition: the committed W carries over, w = W / V (intensive_correct)
            Wl = W_global[sh["cells"]]
            o.init_values((Wl / lm["vol"][:, None]).reshape(-1))
            o.set("W", Wl.reshape(-1))
            o.set("w", (Wl / lm["vol"][:, None]).reshape(-1))
        return sh, lm, cls, own, o

    roc = shard.partition_slabs(mesh, world, axis=0)
    sh, lm, cls, own, o = build(roc, w_global=w0)
    totals = []
    tau = None
    for it in range(iters):
        if rep_every and it > 0 and it % rep_every == 0:
            # DistDriver::repartition (exchange.cpp:595-609) as the library
            # does it (tafv_gpu_repartition): owned W rows as bit patterns and
            # the last plan's levels all-reduced, level-cost slabs re-cut
            Wb = np.zeros((NG, nv), dtype=np.int64)
            Wb[sh["cells"][own]] = o.get("W").reshape(-1, nv)[own].view(np.int64)
            tg = np.full(NG, -1, dtype=np.int32)
            tg[sh["cells"][own]] = tau[own]
            Wt, tt = torch.from_numpy(Wb), torch.from_numpy(tg)
            dist.all_reduce(Wt, op=dist.ReduceOp.SUM)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tg = tt.numpy()
            assert (tg >= 0).all()
            roc = shard.partition_slabs(mesh, world, axis=0, weight=shard.level_cost_weights(tg))
            sh, lm, cls, own, o = build(roc, W_global=Wt.numpy().view(np.float64))
        nloc = len(sh["cells"])
        fl, fr = lm["fl"], lm["fr"]
        inner = fr >= 0
        touch_own = (cls[fl] == 0) | (inner & (cls[np.maximum(fr, 0)] == 0))
        # ---- plan (reference.cpp:89-98, distributed) ----
        o.kernel("compute_dt_max", own, cfl=opt.cfl, dt_cap=opt.dt_cap)
        dt = _allreduce(o.kernel("min_dt", own), dist.ReduceOp.MIN)
        o.kernel("classify_cells", own, dt=dt, theta_max=opt.theta_max)
        tau = np.zeros(nloc, dtype=np.int32)
        tau[own] = o.get("raw_level")[own]
        tau = _exchange(tau.reshape(-1, 1), 1, sh, rank).reshape(-1)
        for _ in range(opt.theta_max):  # Jacobi sweeps on owned cells + halo refresh
            bound = tau.copy()
            a, b = fl[inner], fr[inner]
            np.minimum.at(bound, a, tau[b] + 1)
            np.minimum.at(bound, b, tau[a] + 1)
            new = tau.copy()
            new[own] = bound[own]
            tau = _exchange(new.reshape(-1, 1), 1, sh, rank).reshape(-1)
        theta = int(_allreduce(float(tau[own].max()), dist.ReduceOp.MAX))
        o.inject_plan(tau, dt)  # local LevelMap + cadences over the local faces
        cad = o.plan_lists()["face_cadence"]
        # ---- run_iteration (reference.cpp:100-129, distributed) ----
        o.kernel("reset_fronts")

        def phase(pred, level, front, last=False):
            act = np.flatnonzero(tau <= level).astype(np.int32)
            fringe = np.flatnonzero(tau == level + 1).astype(np.int32) if level < theta and not last else \
                np.zeros(0, dtype=np.int32)
            act_k1 = act[cls[act] <= 1]
            act_own = act[cls[act] == 0]
            faces = np.flatnonzero((cad <= level) & touch_own).astype(np.int32)
            ph = 1 if pred else 0
            if pred:
                o.kernel("stage_committed", act, front=front)
            else:
                o.kernel("stage_predicted", act, front=front, tau=tau)
            o.kernel("stage_interpolated", fringe, front=front, phase=ph, tau=tau)
            o.kernel("green_gauss_gradient", act_k1, front=front, phase=ph)
            o.kernel("limit_gradients", act_k1, front=front, phase=ph)
            if pred:
                o.kernel("reset_windows", faces, front=front)
            o.kernel("reconstruct_faces", faces, front=front, phase=ph)
            if pred:
                o.kernel("riemann_predict", faces, front=front)
                o.kernel("flux_sum_predict", act_own, front=front)
                o.kernel("extensive_predict", act_own, tau=tau, dt=dt)
                o.kernel("intensive_predict", act_own)
                o.set("w_pred", _exchange(o.get("w_pred"), nv, sh, rank))
            else:
                o.kernel("riemann_correct", faces, front=front, cadence=cad, dt=dt)
                o.kernel("flux_sum_correct", act_own, front=front, tau=tau, cadence=cad)
                o.kernel("extensive_correct", act_own)
                o.kernel("intensive_correct", act_own, front=front, tau=tau)
                o.set("w", _exchange(o.get("w"), nv, sh, rank))
                cf = o.get("committed_front")
                halo_act = act[cls[act] > 0]
                cf[halo_act] = front  # the owner committed them at this front
                o.set("committed_front", cf)

        from oracle import orc_subiteration_level
        subs = 1 << theta
        for s in range(1, subs + 1):
            level = orc_subiteration_level(s, theta)
            if s > 1:
                phase(False, level, s - 1)
            phase(True, level, s - 1)
        phase(False, theta, subs, last=True)
        W = o.get("W").reshape(-1, nv)
        totals.append([_allreduce(float(W[own, k].sum()), dist.ReduceOp.SUM) for k in range(nv)])
    w = o.get("w").reshape(-1, nv)
    W = o.get("W").reshape(-1, nv)
    out[rank] = (sh["cells"][own], w[own], W[own], totals)
    dist.destroy_process_group()


def _run(world, cid, scale, iters, rep_every=0):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rank_main, args=(world, port, cid, scale, iters, out, rep_every), nprocs=world,
                       join=True, start_method="fork")
    return dict(out)


@pytest.mark.parametrize("world,cid,scale,iters,rep_every", [(2, 2, 5, 3, 0), (3, 3, 10, 2, 0), (2, 4, 20, 2, 0),
                                                             (2, "P", 1, 3, 0), (2, 3, 10, 3, 2), (3, 2, 5, 3, 1)])
def test_decomposed_run_matches_single_domain_bitwise(world, cid, scale, iters, rep_every):
    """rep_every > 0: level-cost repartitions in between (state migrated by
    all-reduces of the owned rows' bit patterns, as tafv_gpu_repartition)."""
    from oracle import OracleSolver
    from paper_1704_01144_b200 import configs
    cfg = configs.periodic_blast() if cid == "P" else configs.get(cid, scale)
    mesh = cfg.mesh()
    w0 = cfg.initial_state(mesh)
    ref = OracleSolver(mesh, "euler")
    ref.init_values(w0.reshape(-1))
    opt = cfg.options()
    ref.set_options(opt.theta_max, opt.cfl, opt.dt_cap)
    recs = ref.integrate(iters)
    res = _run(world, cid, scale, iters, rep_every)
    w = np.full((len(mesh["vol"]), 5), np.nan)
    W = np.full((len(mesh["vol"]), 5), np.nan)
    for r in range(world):
        g, wl, Wl, totals = res[r]
        w[g] = wl
        W[g] = Wl
        for rt, rr in zip(totals, recs):   # sums in a different order: tolerance (test_dist.cpp:394-395)
            for a, b in zip(rt, rr["total_extensive"]):
                assert abs(a - b) <= 1e-12 * max(1.0, abs(b))
    np.testing.assert_array_equal(w.reshape(-1), ref.get("w"))
    np.testing.assert_array_equal(W.reshape(-1), ref.get("W"))


def test_partition_balances_level_cost():
    from paper_1704_01144_b200 import configs, shard
    cfg = configs.get(3, 10)
    mesh = cfg.mesh()
    wgt = np.where(mesh["cen"][:, 0] < 0.3, 8.0, 1.0)
    roc = shard.partition_slabs(mesh, 4, axis=0, weight=wgt)
    loads = np.bincount(roc, weights=wgt, minlength=4)
    assert loads.max() / loads.mean() < 1.1
    # slabs are contiguous along x
    xs = [mesh["cen"][roc == r, 0] for r in range(4)]
    for a, b in zip(xs, xs[1:]):
        assert a.max() <= b.min() + 1e-12


def test_shard_lists_are_consistent():
    from paper_1704_01144_b200 import configs, shard
    cfg = configs.get(2, 6)
    mesh = cfg.mesh()
    world = 3
    roc = shard.partition_slabs(mesh, world, axis=2)
    shs = [shard.describe(mesh, roc, r, world) for r in range(world)]
    for r in range(world):
        for q, snd in shs[r]["send"].items():
            rcv = shs[q]["recv"][r]
            assert np.array_equal(shs[r]["cells"][snd], shs[q]["cells"][rcv])   # same global cells, same order
            assert (roc[shs[r]["cells"][snd]] == r).all()
        halo = shs[r]["cls"] > 0
        assert sum(len(v) for v in shs[r]["recv"].values()) == int(halo.sum())


def _window_rank(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1704_01144_b200 import configs, shard
    ops = {"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}

    def allreduce(v, op):
        t = torch.tensor(v, dtype=torch.float64)
        dist.all_reduce(t, op=ops[op])
        return t.numpy() if t.dim() else float(t.item())

    cfg = configs.get(4, 20)
    mesh, roc, gid, cuts = shard.distributed_slab_window(cfg, cfg.options(), rank, world, allreduce)
    out[rank] = (cuts.tolist(), gid[roc == rank], mesh["vol"][roc == rank])
    dist.destroy_process_group()


def test_distributed_slab_windows_partition_the_lattice():
    """The bench's multi-process setup without a global mesh
    (shard.distributed_slab_window over gloo, world size 3): every rank
    derives the same level-cost cuts, the owned cells of the rank windows
    partition the lattice, and they are bitwise the global mesh's cells."""
    from paper_1704_01144_b200 import configs
    world, port = 3, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_window_rank, args=(world, port, out), nprocs=world, join=True, start_method="fork")
    res = dict(out)
    assert all(res[r][0] == res[0][0] for r in range(world))
    cfg = configs.get(4, 20)
    full = cfg.mesh()
    gids = np.concatenate([res[r][1] for r in range(world)])
    assert np.array_equal(np.sort(gids), np.arange(len(full["vol"])))
    for r in range(world):
        assert np.array_equal(res[r][2], full["vol"][res[r][1]])

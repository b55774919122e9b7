"""Batch / multi-GPU plumbing.

CPU: shard arithmetic and the label/objective all-gather over gloo with
world_size 2 (the same code runs over NCCL on the GPU box).
GPU: the concurrent batch solve equals one solve per instance, bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_01838_b200 import batch


def test_shard_range_covers_batch():
    for count in (0, 1, 5, 64, 65):
        for world in (1, 2, 3, 4, 8):
            spans = [batch.shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        batch.shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, count, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = batch.shard_range(count, rank, world)
        # instance i's labels are all i, its objectives (i, -i)
        lab = torch.cat([torch.full((n,), i, dtype=torch.int32) for i in range(lo, hi)]) if hi > lo else \
            torch.empty(0, dtype=torch.int32)
        obj = torch.tensor([[float(i), -float(i)] for i in range(lo, hi)], dtype=torch.float64).reshape(-1, 2)
        L, O = batch.gather_results(lab, obj, n, count)
        out[rank] = (L.numpy().copy(), O.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("count", [5, 64])
def test_gather_results_gloo_world2(count):
    world, n = 2, 7
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), count, n, out), nprocs=world, join=True)
    for r in range(world):
        L, O = out[r]
        assert L.shape == (count, n) and O.shape == (count, 2)
        assert np.array_equal(L, np.repeat(np.arange(count, dtype=np.int32)[:, None], n, axis=1))
        assert np.array_equal(O[:, 0], np.arange(count)) and np.array_equal(O[:, 1], -np.arange(count))


def _trace_key(sol):
    return [(r.round_index, r.phase, r.nodes, r.edges, r.triplets, r.lb, r.lb_valid, r.contracted) for r in sol.trace]


@pytest.mark.gpu
def test_batch_solve_equals_single_solves():
    """The union batch solve (batch.cu) reproduces every instance's single
    solve bit for bit: labels, primal, LB and the whole trace -- across
    instances that stop in different rounds, switch to the forest policy in
    different rounds, or have no positive edge at all."""
    import paper_2109_01838_b200 as P
    from paper_2109_01838_b200 import instances

    graphs = [P.WeightedGraph(*instances.grid_coo(96, 128, 0, seed=s)) for s in range(4)]
    graphs.append(P.WeightedGraph(*instances.grid8_coo(40, 50, strides=(2, 3), seed=9)))
    graphs.append(P.WeightedGraph(5))  # no edges
    graphs.append(P.WeightedGraph(1))  # one node
    graphs += [P.WeightedGraph(*instances.random_coo(120, 0.08, seed=s)) for s in range(3)]
    n, u, v, c = instances.grid_coo(20, 30, 0, seed=3)
    graphs.append(P.WeightedGraph(n, u, v, -np.abs(c)))  # all repulsive: stops in round 1
    graphs += [P.WeightedGraph(*instances.chung_lu_coo(800, 2.1, 9000, seed=s)) for s in range(2)]
    graphs.append(P.WeightedGraph(*instances.grid_coo(64, 64, 3, seed=5)))
    for mode in ("PD", "P", "PD+"):
        cfg = P.SolverConfig(mode=mode)
        singles = [P.solve(g, cfg) for g in graphs]
        for workers in (1, 3):
            got = P.solve_batch(graphs, cfg, workers=workers)
            for i, (a, b) in enumerate(zip(singles, got)):
                assert np.array_equal(a.labeling, b.labeling), (mode, workers, i)
                assert a.primal_cost == b.primal_cost and a.lower_bound == b.lower_bound, (mode, workers, i)
                assert _trace_key(a) == _trace_key(b), (mode, workers, i)


@pytest.mark.gpu
def test_batch_solve_modes_d_and_gaec():
    import paper_2109_01838_b200 as P
    from paper_2109_01838_b200 import instances

    graphs = [P.WeightedGraph(*instances.grid_coo(24, 32, 0, seed=s)) for s in range(3)]
    for cfg in (P.SolverConfig(mode="D", separation_rounds=2), P.SolverConfig(mode="GAEC")):
        got = P.solve_batch(graphs, cfg, workers=2)
        for g, b in zip(graphs, got):
            a = P.solve(g, cfg)
            assert np.array_equal(a.labeling, b.labeling)
            assert a.primal_cost == b.primal_cost and a.lower_bound == b.lower_bound
            assert _trace_key(a) == _trace_key(b)


@pytest.mark.gpu
def test_batch_solve_reports_bad_instance():
    import paper_2109_01838_b200 as P

    cfg = P.SolverConfig(mode="PD")
    with pytest.raises(ValueError):
        P.solve_batch_device(np.array([0, 4, 2]), np.array([0, 0, 0]), P._lib.empty_i32(1), P._lib.empty_i32(1),
                             P._lib.empty_f64(1), cfg)


@pytest.mark.gpu
def test_solve_sharded_over_nccl_single_rank():
    """batch.solve_sharded end to end through a real NCCL process group (one
    rank: the box has one GPU; the gather is the same all_gather_into_tensor
    the 2/4/8-GPU runs use): every instance equals its single solve."""
    import paper_2109_01838_b200 as P
    from paper_2109_01838_b200 import instances

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        insts = [instances.grid_coo(64, 80, 0, seed=s) for s in range(5)]
        cfg = P.SolverConfig(mode="PD")
        labels, objs = batch.solve_sharded(insts, cfg)
        assert labels.is_cuda and labels.shape == (5, 64 * 80) and objs.shape == (5, 2)
        for s, inst in enumerate(insts):
            one = P.solve(P.WeightedGraph(*inst), cfg)
            assert np.array_equal(labels[s].cpu().numpy(), one.labeling)
            assert objs[s, 0].item() == one.primal_cost and objs[s, 1].item() == one.lower_bound
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_union_batch_many_small_instances():
    """A few hundred tiny instances in one union (per-instance segments of
    every reduction and bound): each equals its single solve."""
    import paper_2109_01838_b200 as P
    from paper_2109_01838_b200 import instances

    graphs = [P.WeightedGraph(*instances.grid_coo(5 + s % 4, 6 + s % 3, 0, seed=s)) for s in range(300)]
    cfg = P.SolverConfig(mode="PD")
    got = P.solve_batch(graphs, cfg)
    for s in (0, 1, 77, 150, 299):
        a = P.solve(graphs[s], cfg)
        assert np.array_equal(a.labeling, got[s].labeling)
        assert a.primal_cost == got[s].primal_cost and a.lower_bound == got[s].lower_bound
        assert _trace_key(a) == _trace_key(got[s])

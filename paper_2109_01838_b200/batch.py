"""Multi-GPU batch solve of independent instances.

One process per GPU.  Rank r solves instances [lo_r, hi_r) of the batch
(contiguous shards, sizes differing by at most one) with the concurrent
batch solver, then the only exchange of the whole job: one
``all_gather_into_tensor`` of the int32 labels and one of the float64
(primal, lower bound) pairs, padded to the largest shard.  No collective
touches the data path; the reference has no multi-process design at all
(its ``--threads`` is ignored, cli.py:23-32).
"""

import numpy as np


def shard_range(count, rank, world):
    """[lo, hi) of the instances owned by ``rank`` (balanced, contiguous)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_results(labels, objectives, nodes_per_instance, count, group=None):
    """All-gather every rank's shard results.

    labels: int32 tensor [k_local * nodes_per_instance] (this rank's
    instances in order); objectives: float64 tensor [k_local, 2].  Works on
    any backend (NCCL on the GPU box, gloo on CPU tensors in the tests).
    Returns (labels [count, nodes_per_instance], objectives [count, 2]).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    kmax = -(-count // world)
    dev = labels.device
    lab = torch.full((kmax * nodes_per_instance,), -1, dtype=torch.int32, device=dev)
    lab[: labels.numel()] = labels
    obj = torch.zeros((kmax, 2), dtype=torch.float64, device=dev)
    obj[: objectives.shape[0]] = objectives
    all_lab = torch.empty(world * lab.numel(), dtype=torch.int32, device=dev)
    all_obj = torch.empty((world * kmax, 2), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(all_lab, lab, group=group)
    dist.all_gather_into_tensor(all_obj, obj, group=group)
    all_lab = all_lab.view(world, kmax, nodes_per_instance)
    all_obj = all_obj.view(world, kmax, 2)
    keep_l, keep_o = [], []
    for r in range(world):
        lo, hi = shard_range(count, r, world)
        keep_l.append(all_lab[r, : hi - lo])
        keep_o.append(all_obj[r, : hi - lo])
    return torch.cat(keep_l), torch.cat(keep_o)


def solve_sharded(instances, cfg, workers=1, group=None):
    """Solve a batch of equally sized instances across all ranks.

    instances: list of (n, u, v, cost) raw COO (every rank holds the list;
    only its shard is built and solved).  Returns (labels [count, n],
    objectives [count, 2]) on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import graph as G
    from . import solver as S

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    count = len(instances)
    n = instances[0][0]
    lo, hi = shard_range(count, rank, world)
    graphs = [G.WeightedGraph(*instances[i]) for i in range(lo, hi)]
    sols = S.solve_batch(graphs, cfg, workers=workers)
    dev = torch.device("cuda", torch.cuda.current_device())
    lab = torch.from_numpy(np.concatenate([s.labeling for s in sols]).astype(np.int32)).to(dev) if sols else \
        torch.empty(0, dtype=torch.int32, device=dev)
    obj = torch.tensor([[s.primal_cost, s.lower_bound] for s in sols], dtype=torch.float64, device=dev).reshape(-1, 2)
    return gather_results(lab, obj, n, count, group)

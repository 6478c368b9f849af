"""Box -> rank distribution with measured per-box chemistry cost (PAPER.md P:127
"users can calculate computational costs ... and provide these to AMReX's load balancing").

Cells are independent 0-D reactors during chemistry, so the path shards by box with no
data-path collective.  NCCL (torch.distributed) carries only:
  (1) all_gather of the per-box cost vector (nboxes x 8 B) after a calibration call,
  (2) all_reduce SUM/MAX of the stats vector (convergence: unfinished cells; time),
  (3) all_reduce MIN of a proposed dt (stand-in for the CFL reduction).
The partition is deterministic and identical on every rank; owners regenerate their boxes from
the pure synthetic generator, so no box data migrates (a real AMR code would migrate through its
framework: out of scope).
"""
from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(costs, nranks):
    """Longest-processing-time-first: boxes by cost descending (ties: lower box id first), each to
    the least-loaded rank (ties: lowest rank).  Returns owner[nboxes] (int)."""
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(len(costs)), key=lambda b: (-costs[b], b))
    heap = [(0.0, r) for r in range(nranks)]
    heapq.heapify(heap)
    owner = np.empty(len(costs), dtype=np.int64)
    for b in order:
        load, r = heapq.heappop(heap)
        owner[b] = r
        heapq.heappush(heap, (load + costs[b], r))
    return owner


def loads(costs, owner, nranks):
    out = np.zeros(nranks)
    np.add.at(out, np.asarray(owner), np.asarray(costs, dtype=np.float64))
    return out


def imbalance(costs, owner, nranks):
    """max/mean of the per-rank load (1.0 = perfect balance)."""
    ld = loads(costs, owner, nranks)
    return float(ld.max() / ld.mean()) if ld.mean() > 0 else 1.0


def gather_costs(local_costs, group=None):
    """all_gather of equal-length per-rank cost vectors -> the global vector (rank-major)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.asarray(local_costs, dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    world = dist.get_world_size(group)
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.cpu().numpy()


def reduce_stats(vec, op="sum", group=None):
    """all_reduce of a small stats vector (SUM for counts, MAX for times, MIN for dt)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.asarray(vec, dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}[op],
                    group=group)
    return t.cpu().numpy()


def balance(local_costs, group=None):
    """Gather every rank's per-box costs and compute the same LPT owner map on all ranks."""
    import torch.distributed as dist
    costs = gather_costs(local_costs, group)
    return costs, lpt_partition(costs, dist.get_world_size(group))


def plan(home, local_costs, nboxes, world, balance="lpt", group=None):
    """The bench's cost-weighted box -> rank plan.  `home(r)` lists the global box ids
    rank r integrated in its calibration call (in the order of its local cost vector); every rank
    passes its own costs.  The costs are all-gathered (equal lengths: each rank calibrates the same
    number of boxes), put back in global box order, and every rank computes the same owner map:
    LPT on the measured cost, or (balance="none") each box stays on its home rank.
    Returns (global costs, owner[nboxes], max/mean imbalance with this owner map, imbalance of the
    home map)."""
    home_owner = np.empty(nboxes, dtype=np.int64)
    for r in range(world):
        home_owner[np.asarray(home(r), dtype=np.int64)] = r
    if world == 1:
        costs = np.asarray(local_costs, dtype=np.float64)
        return costs, np.zeros(nboxes, dtype=np.int64), 1.0, 1.0
    rank_major = gather_costs(local_costs, group)
    costs = np.zeros(nboxes)
    k = 0
    for r in range(world):
        ids = list(home(r))
        costs[ids] = rank_major[k:k + len(ids)]
        k += len(ids)
    owner = lpt_partition(costs, world) if balance == "lpt" else home_owner
    return costs, owner, imbalance(costs, owner, world), imbalance(costs, home_owner, world)


def step_reductions(n_unfinished, substeps, dt_proposed, group=None):
    """SURVEY §8(e) (2)-(3), once per CFD step: SUM of unfinished cells and attempted substeps
    (convergence), MIN of the proposed next dt (stand-in for the CFL reduction)."""
    tot = reduce_stats([n_unfinished, substeps], "sum", group)
    dtg = reduce_stats([dt_proposed], "min", group)
    return dict(n_unfinished=int(tot[0]), substeps=int(tot[1]), dt_next=float(dtg[0]))

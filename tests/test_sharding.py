"""Host logic of the multi-GPU path: LPT partition and the collective plumbing,
exercised with torch.distributed gloo, world_size 2, on CPU."""
import os
import socket

import numpy as np
import pytest

from paper_2510_23993_b200.sharding import imbalance, loads, lpt_partition


def test_lpt_deterministic_and_tie_breaking():
    costs = [5.0, 5.0, 3.0, 3.0, 1.0]
    own = lpt_partition(costs, 2)
    assert list(own) == [0, 1, 0, 1, 0]          # ties: lower box id first, lowest rank first
    assert list(lpt_partition(costs, 2)) == list(own)


def test_lpt_bound():
    """Graham's bound: LPT makespan <= (4/3 - 1/(3m)) OPT; OPT >= max(mean, max cost)."""
    rng = np.random.default_rng(0)
    for m in (2, 4, 8):
        c = rng.lognormal(0, 1.5, 200)
        own = lpt_partition(c, m)
        lb = max(c.sum() / m, c.max())
        assert loads(c, own, m).max() <= (4 / 3 - 1 / (3 * m)) * lb + 1e-9
        assert imbalance(c, own, m) >= 1.0


def test_lpt_single_rank_and_empty():
    assert list(lpt_partition([1, 2, 3], 1)) == [0, 0, 0]
    assert len(lpt_partition([], 4)) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2510_23993_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = np.arange(3, dtype=float) + 10 * rank        # rank r owns boxes 3r..3r+2
        costs, owner = sharding.balance(local)
        s = sharding.reduce_stats([rank + 1, 2.0], "sum")
        mx = sharding.reduce_stats([rank * 1.5], "max")
        mn = sharding.reduce_stats([1e-7 * (rank + 1)], "min")
        q.put((rank, costs.tolist(), owner.tolist(), s.tolist(), mx.tolist(), mn.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_balance_and_reductions():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, c0, o0, s0, m0, n0), (_, c1, o1, s1, m1, n1) = res
    assert c0 == c1 == [0.0, 1.0, 2.0, 10.0, 11.0, 12.0]
    assert o0 == o1 == list(lpt_partition(c0, 2))
    assert s0 == s1 == [3.0, 4.0]
    assert m0 == m1 == [1.5]
    assert n0 == n1 == [1e-7]


def _plan_worker(rank, world, port, q):
    """The bench's balancing logic (sharding.plan) on the cfg4 layout (P copies of 192 boxes, copy p
    calibrated on rank p) and the cfg5 layout (128 boxes round-robin), with a fake cost vector that
    is a pure function of the global box id, plus the per-step reductions."""
    import torch.distributed as dist
    from paper_2510_23993_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = lambda b: float(1 + (b * 2654435761) % 997) * (50.0 if b % 192 >= 128 else 1.0)  # noqa: E731
        out = {}
        home4 = lambda r: list(range(192 * r, 192 * (r + 1)))                           # noqa: E731
        home5 = lambda r: list(range(r, 128, world))                                   # noqa: E731
        for name, home, nb in (("cfg4", home4, 192 * world), ("cfg5", home5, 128)):
            for bal in ("lpt", "none"):
                c, own, imb, imb_home = sharding.plan(home, [fake(b) for b in home(rank)], nb, world, bal)
                out[(name, bal)] = (c.tolist(), own.tolist(), imb, imb_home)
        red = sharding.step_reductions(rank, 100 * (rank + 1), 1e-7 / (rank + 1))
        q.put((rank, out, red))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bench_plan_cfg4_cfg5():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    ps = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    fake = lambda b: float(1 + (b * 2654435761) % 997) * (50.0 if b % 192 >= 128 else 1.0)  # noqa: E731
    for key in res[0][1]:
        c0, o0, i0, h0 = res[0][1][key]
        c1, o1, i1, h1 = res[1][1][key]
        assert c0 == c1 and o0 == o1 and i0 == i1          # identical plan on every rank
        nb = len(c0)
        assert c0 == [fake(b) for b in range(nb)]           # costs back in global box order
        assert set(o0) <= set(range(world))
        if key[1] == "lpt":
            assert o0 == list(lpt_partition(c0, world))
            assert i0 <= h0 + 1e-12                         # LPT never worse than the home map
            assert i0 < 1.02
        else:
            assert i0 == h0
    # the cfg4 copies differ in cost only by id: LPT beats "copy p -> rank p"
    assert res[0][1][("cfg4", "lpt")][2] <= res[0][1][("cfg4", "none")][2]
    for _, _, red in res:
        assert red == dict(n_unfinished=1, substeps=300, dt_next=5e-8)

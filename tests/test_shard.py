"""Multi-process (gloo, world size 2, CPU) tests of the sub-region sharding host logic
(PAPER.md:51/112/146: sub-regions are optimised independently in parallel)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_01677_b200 import shard


def test_assign_equal_regions_balanced():
    own = shard.assign_subregions(8, 4)
    assert sorted(sum(own, [])) == list(range(8))
    assert all(len(o) == 2 for o in own)
    assert shard.assign_subregions(8, 8) == [[k] for k in range(8)]
    assert shard.assign_subregions(8, 1) == [list(range(8))]


def test_assign_lpt_bound():
    costs = [5, 1, 4, 2, 3, 3, 2, 1]
    own = shard.assign_subregions(8, 3, costs)
    loads = [sum(costs[k] for k in o) for o in own]
    assert sorted(sum(own, [])) == list(range(8))
    assert max(loads) - min(loads) <= max(costs)
    with pytest.raises(ValueError):
        shard.assign_subregions(2, 0)


def test_weak_region():
    assert [shard.weak_region(r) for r in range(10)] == [0, 1, 2, 3, 4, 5, 6, 7, 0, 1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        own = shard.assign_subregions(8, world)[rank]
        rec = shard.stats_record(rank=rank, ms=10.0 + rank, masked_pixels=1e6 * len(own), blends=5e7 * (rank + 1),
                                 views=len(own))
        st = shard.gather_stats(rec)
        agg = shard.aggregate(st)
        q.put((rank, own, st.numpy().tolist(), agg))
    finally:
        dist.destroy_process_group()


def test_gather_stats_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    owned = [r[1] for r in res]
    assert sorted(sum(owned, [])) == list(range(8)) and owned[0] != owned[1]
    # every rank sees the same gathered table, rank-ordered
    assert res[0][2] == res[1][2]
    table = torch.tensor(res[0][2])
    assert table[:, 0].tolist() == [0.0, 1.0]
    agg = res[0][3]
    assert agg["ms_max"] == 11.0  # device time = max over ranks
    assert agg["masked_pixels"] == 8e6
    assert abs(agg["mpix_per_s"] - 8.0 / 0.011) < 1e-6


# ------------------------------------------------ group training layout / view-parallel DP (NEXT-4)
def test_rank_layout():
    lay = shard.rank_layout(8, 4)
    assert [l[0] for l in lay] == shard.assign_subregions(8, 4) and all(l[1] == [r] for r, l in enumerate(lay))
    lay = shard.rank_layout(2, 5)
    assert [l[0] for l in lay] == [[0], [1], [0], [1], [0]]
    assert lay[0][1] == [0, 2, 4] and lay[4][2] == 2 and lay[3][1] == [1, 3]
    with pytest.raises(ValueError):
        shard.rank_layout(0, 2)


def test_view_schedule():
    a = shard.view_schedule(40, 100, seed=7, region=3)
    assert a == shard.view_schedule(40, 100, seed=7, region=3)  # deterministic
    assert sorted(a[:40]) == list(range(40))                     # epoch = permutation
    assert a != shard.view_schedule(40, 100, seed=7, region=4)   # seeded per region
    m = [shard.view_schedule(40, 30, seed=7, region=3, dp_rank=k, dp_size=3) for k in range(3)]
    for t in range(30):
        assert len({m[0][t], m[1][t], m[2][t]}) == 3              # distinct views per iteration
    assert sorted(m[0][:13] + m[1][:13] + m[2][:13]) == sorted(a[:40])[:39] or \
        len(set(m[0][:13] + m[1][:13] + m[2][:13])) == 39                      # one epoch, 39 distinct views
    with pytest.raises(ValueError):
        shard.view_schedule(2, 5, seed=1, region=0, dp_rank=0, dp_size=3)


def _dp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import oracle
        g = [torch.full((3, 5), float(rank + 1)), torch.arange(4.0) * (rank + 1)]
        shard.allreduce_mean(g)
        s = [torch.ones(6) * (rank + 1)]
        shard.allreduce_sum(s)
        # identical Adam on identical parameters after the averaged gradient keeps members in sync
        p = np.linspace(-1, 1, 15)
        grad = torch.from_numpy(np.random.default_rng(rank).normal(size=15))
        shard.allreduce_mean([grad])
        p2, _, _ = oracle.adam_step(p, grad.numpy(), np.zeros(15), np.zeros(15), 1, lr=1e-2)
        q.put((rank, [t.tolist() for t in g], s[0].tolist(), p2.tolist()))
    finally:
        dist.destroy_process_group()


def test_view_parallel_allreduce_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert r[1][0] == [[1.5] * 5] * 3 and r[1][1] == [0.0, 1.5, 3.0, 4.5]
        assert r[2] == [3.0] * 6
    assert res[0][3] == res[1][3]  # members stay bit-identical

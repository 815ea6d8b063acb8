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

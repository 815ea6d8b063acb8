"""Sub-region sharding across ranks (one process per GPU).

PAPER.md:51 "Each sub-group can be independently optimized in parallel",
PAPER.md:112 "each sub-group encompassing its associated sparse points, cameras,
and refined masks": the path partitions into independent
sub-regions, so ranks own whole sub-regions and the data path has NO collective.
The only collective is the all-gather of a fixed-size per-rank statistics record
(loss / timing / counters), off the timed region.

When there are more ranks than sub-regions (not in the paper), the ranks
that share a sub-region train it view-parallel: each renders a different view of the same
iteration and the parameter gradients are averaged over the group (allreduce_mean, NCCL) before
the identical Adam step on every member.

Host logic only (no kernels): it is exercised with the gloo backend on CPU in
tests/test_shard.py and with NCCL over NVLink by bench.py at N > 1.
"""
from __future__ import annotations

import torch

STATS_LEN = 16  # floats per rank record
STATS_FIELDS = ("rank", "ms", "masked_pixels", "blends", "tile_imbalance", "views", "M", "evaluated")


def assign_subregions(n_regions: int, world: int, costs=None):
    """Owner lists: rank r -> sub-region ids.  Longest-processing-time-first greedy over
    the per-region costs (default: equal), ties to the lowest rank, so the ranks'
    loads differ by at most one region's cost (Graham's LPT bound)."""
    if world <= 0:
        raise ValueError("world must be >= 1")
    costs = [1.0] * n_regions if costs is None else [float(c) for c in costs]
    if len(costs) != n_regions:
        raise ValueError("one cost per region")
    order = sorted(range(n_regions), key=lambda k: (-costs[k], k))
    load = [0.0] * world
    owned = [[] for _ in range(world)]
    for k in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owned[r].append(k)
        load[r] += costs[k]
    return [sorted(o) for o in owned]


def weak_region(rank: int, n_regions: int = 8) -> int:
    """Weak-scaling layout used by bench.py: rank r owns sub-region r mod n_regions."""
    return rank % n_regions


def stats_record(**kw) -> torch.Tensor:
    rec = torch.zeros(STATS_LEN, dtype=torch.float64)
    for i, f in enumerate(STATS_FIELDS):
        if f in kw:
            rec[i] = float(kw[f])
    return rec


def gather_stats(rec: torch.Tensor, group=None):
    """All-gather one STATS_LEN record per rank; returns a (world, STATS_LEN) tensor on
    the record's device.  Single-process: returns rec[None]."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return rec[None].clone()
    world = dist.get_world_size(group)
    out = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(out, rec, group=group)
    return torch.stack(out)


def aggregate(stats: torch.Tensor):
    """Whole-job figures from the gathered records: time = max over ranks (device-timed),
    work = sum over ranks."""
    ms = float(stats[:, STATS_FIELDS.index("ms")].max())
    pix = float(stats[:, STATS_FIELDS.index("masked_pixels")].sum())
    bl = float(stats[:, STATS_FIELDS.index("blends")].sum())
    return {"ms_max": ms, "masked_pixels": pix, "blends": bl,
            "mpix_per_s": pix / 1e6 / (ms / 1e3) if ms > 0 else 0.0,
            "rank_imbalance": ms / max(float(stats[:, STATS_FIELDS.index("ms")].mean()), 1e-12)}


# ---------------------------------------------------------------- group training layout
def rank_layout(n_regions: int, world: int, costs=None):
    """Per rank: (owned region ids, data-parallel peer ranks, index among the peers).
    world <= n_regions: LPT ownership (assign_subregions), no peers.  world > n_regions: rank r
    trains region r mod n_regions together with the other ranks of that residue class
    (view-parallel data parallelism inside the region)."""
    if world <= 0 or n_regions <= 0:
        raise ValueError("world and n_regions must be >= 1")
    if world <= n_regions:
        own = assign_subregions(n_regions, world, costs)
        return [(own[r], [r], 0) for r in range(world)]
    out = []
    for r in range(world):
        k = r % n_regions
        peers = [q for q in range(world) if q % n_regions == k]
        out.append(([k], peers, peers.index(r)))
    return out


def view_schedule(n_views: int, iters: int, seed: int, region: int, dp_rank: int = 0, dp_size: int = 1):
    """View index of every iteration for one data-parallel member: a shuffled epoch order seeded per
    region (seed ^ region, so the result does not depend on co-scheduled regions); each epoch is cut
    into floor(n_views / dp_size) iterations of dp_size consecutive views (the remainder is dropped),
    member dp_rank taking the dp_rank-th view of each: distinct views in every iteration."""
    import numpy as np
    if n_views <= 0 or not (0 <= dp_rank < dp_size) or dp_size > n_views:
        raise ValueError("need n_views >= dp_size >= 1 and 0 <= dp_rank < dp_size")
    rng = np.random.Generator(np.random.Philox(int(seed) ^ int(region)))
    per = n_views // dp_size
    out = []
    while len(out) < iters:
        perm = rng.permutation(n_views).tolist()
        out.extend(perm[t * dp_size + dp_rank] for t in range(per))
    return out[:iters]


def allreduce_mean(tensors, group=None):
    """Average a list of same-dtype tensors over the process group with ONE coalesced all-reduce
    (NCCL over NVLink on the GPU; gloo on CPU in the tests).  In place."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return tensors
    n = dist.get_world_size(group)
    if n == 1:
        return tensors
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, group=group)
    flat.div_(n)
    o = 0
    for t in tensors:
        k = t.numel()
        t.copy_(flat[o:o + k].view_as(t))
        o += k
    return tensors


def allreduce_sum(tensors, group=None):
    """Sum over the group (used for the densification statistics), one coalesced all-reduce."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return tensors
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, group=group)
    o = 0
    for t in tensors:
        k = t.numel()
        t.copy_(flat[o:o + k].view_as(t))
        o += k
    return tensors

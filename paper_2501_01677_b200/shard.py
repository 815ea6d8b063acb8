"""Sub-region sharding across ranks (one process per GPU).

PAPER.md:51 "Each sub-group can be independently optimized in parallel",
PAPER.md:112 "each sub-group encompassing its associated sparse points, cameras,
and refined masks": the path partitions into independent
sub-regions, so ranks own whole sub-regions and the data path has NO collective.
The only collective is the all-gather of a fixed-size per-rank statistics record
(loss / timing / counters), off the timed region.

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

"""Parallel group training ("each sub-group can be independently optimized in parallel",
P:200 30 000 iterations per block; SURVEY §8 NEXT-3 "sub-region scheduler across 8 GPUs").

One process per GPU (torchrun).  shard.rank_layout decides which sub-regions a rank trains;
ranks that share a sub-region (more GPUs than sub-regions, NEXT-4) train it view-parallel with
their gradients averaged over an NCCL group.  Each region: views in a seeded shuffled epoch
order (shard.view_schedule), train.Trainer iterations (Eq. 10-11), densification every
`densify_every` iterations until `densify_until`, opacity reset every `reset_every`.  Rank 0
prints one JSON report (per region: final loss terms, Gaussian count, device time).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_2501_01677_b200.groups --regions 8 --iters 300

Inputs are the synthetic C4 sub-regions of synth/scenes.py (--small: C1-sized scenes); the
targets are synthetic photos (there is no dataset in this environment).
"""
from __future__ import annotations

import argparse
import json
import os
import time


def _region_data(k, args, dev):
    import numpy as np
    import torch
    from synth import scenes as S
    if args.small:
        sc = S.config1(seed=1000 + k, n=args.small_n, W=96, H=64)
        cams, masks = [sc.camera] * 4, [torch.from_numpy(np.ascontiguousarray(sc.mask)).to(dev)] * 4
        g = sc.gaussians
        H, W = sc.mask.shape
        tg = [torch.from_numpy(S.reference_image(H, W, 2000 + k + 7 * v)).to(dev) for v in range(4)]
    else:
        sub = S.subregion(k, n_views=args.views)
        g, cams = sub["gaussians"], sub["cameras"]
        masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev) for c in cams]
        H, W = masks[0].shape
        gen = torch.Generator(device=dev)
        gen.manual_seed(3000 + k)
        tg = [torch.rand(3, H, W, device=dev, generator=gen) for _ in cams]
    return g, cams, masks, tg


def train_region(k, args, dev, dp_group=None, dp_rank=0, dp_size=1):
    import torch
    from . import shard
    from .raster import GaussianTensors, Rasterizer, camera_from
    from .train import AdamConfig, DensifyConfig, Trainer
    gnp, cams, masks, targets = _region_data(k, args, dev)
    g = GaussianTensors.from_numpy(gnp, dev)
    H, W = masks[0].shape
    r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
    tr = Trainer(r, g, AdamConfig(lr_mean=args.lr_mean))
    ccam = [camera_from(c) for c in cams]
    extras = {}
    sched = shard.view_schedule(len(cams), args.iters, args.seed, k, dp_rank, dp_size)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    first = None
    for it, v in enumerate(sched):
        if v not in extras:
            extras[v] = (tr.r.gc_weights(targets[v], masks[v]), tr.r.boundary_band(masks[v], 1))
        tr.step(ccam[v], masks[v], targets[v], gc_w=extras[v][0], band=extras[v][1], dp_group=dp_group)
        if it == 0:
            first = tr.losses()
        if args.densify_every and (it + 1) % args.densify_every == 0 and it + 1 <= args.densify_until:
            tr.densify(DensifyConfig(grad_threshold=args.grad_threshold, dense_limit=args.dense_limit,
                                     seed=args.seed ^ k), dp_group=dp_group)
        if args.reset_every and (it + 1) % args.reset_every == 0:
            tr.reset_opacity(0.01)
    e1.record()
    torch.cuda.synchronize()
    last = tr.losses()
    import hashlib
    h = hashlib.sha256()
    for t in (tr.g.mean, tr.g.scale, tr.g.rot, tr.g.opacity, tr.g.sh, tr.m, tr.v):
        h.update(t.detach().contiguous().cpu().numpy().tobytes())
    return {"region": k, "iters": args.iters, "dp_size": dp_size, "dp_rank": dp_rank, "n_gaussians": tr.g.n,
            "ms": e0.elapsed_time(e1), "first_loss": first, "final_loss": last,
            "state_digest": h.hexdigest()[:24]}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--regions", type=int, default=8)
    ap.add_argument("--views", type=int, default=40)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1677)
    ap.add_argument("--lr-mean", type=float, default=1.6e-4)
    ap.add_argument("--densify-every", type=int, default=100)
    ap.add_argument("--densify-until", type=int, default=15000)
    ap.add_argument("--reset-every", type=int, default=3000)
    ap.add_argument("--grad-threshold", type=float, default=2e-4)
    ap.add_argument("--dense-limit", type=float, default=0.5)
    ap.add_argument("--small", action="store_true", help="C1-sized scenes (tests)")
    ap.add_argument("--small-n", type=int, default=1000)
    args = ap.parse_args(argv)
    import torch
    import torch.distributed as dist
    from . import shard
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("PGSAG_DIST_BACKEND", "nccl")  # gloo: smoke-test N ranks on one GPU
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lay = shard.rank_layout(args.regions, world)
    groups = {}
    if world > args.regions:  # every rank creates every group, in the same order
        for k in range(args.regions):
            peers = [q for q in range(world) if q % args.regions == k]
            groups[k] = dist.new_group(peers) if len(peers) > 1 else None
    own, peers, dp_rank = lay[rank]
    t0 = time.time()
    reports = [train_region(k, args, dev, groups.get(k), dp_rank, len(peers)) for k in own]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, reports)
        reports = [x for rr in allr for x in rr]
    if rank == 0:
        print(json.dumps({"world": world, "regions": args.regions, "wall_s": time.time() - t0,
                          "reports": reports}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return reports


if __name__ == "__main__":
    main()

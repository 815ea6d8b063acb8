#!/usr/bin/env python
"""Benchmark of the PG-SAG masked tile rasterizer (forward + backward) on B200.

One "step" = the whole hot path (A0-A8: preprocess, bin/sort, forward
compositor, backward compositor, preprocess backward) for one full-resolution
view of the rank's sub-region (BASELINE.json configs[3], "C4": visibility-
grouped sub-regions of 1.5M Gaussians with 40 oblique 5472x3648 views, one
sub-region per GPU; weak scaling, no collective on the data path).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c4|c3|c2|c5]

Prints ONE JSON line (rank 0).  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "masked Mpix/s fwd+bwd and Gaussian-pixel blends/s at 1/2/4/8 B200; % FP32/HBM roofline"
UNIT = "Mpix/s"

# algorithmic FP32 work per unit, FMA = 2 flops (exp/rcp on MUFU not counted)
FLOP_EVAL = 9        # per evaluated (pixel, Gaussian) pair: dx, dy, quadratic form, o*rho
FLOP_BLEND_FWD = 17  # per blended pair in A6: 1-a, T(1-a), aT, 7 channel FMAs
FLOP_BLEND_BWD = 46  # per blended pair in A7: 1-a, T recovery, G.F, dalpha, suffix, P, aT, dF, d o, d power, d conic
# SURVEY §8(d)'s roofline contract: FP32 lane-instructions per unit (MUFU not counted), against
# 148 SMs x 128 lanes x clock lane-instructions per second
INST_EVAL_FWD = 14   # A6 per evaluated pair: 2 sub, 6 quadratic form, 2 exp argument / opacity, min, 2 cmp, 1 sel
INST_BLEND_FWD = 10  # A6 per blended pair: T update, w, 7 FMA into C/N/D, termination compare
INST_VISIT_BWD = 17  # A7 per visited pair: 14 (alpha recompute) + 3 (T recovery)
INST_BLEND_BWD = 55  # A7 per blended pair: suffix update, dalpha, 7 dF, d opacity, 3 d conic, 2 d mean
BYTES_A1 = {0: 56 + 76, 1: 56 + 36 + 76, 2: 56 + 96 + 76, 3: 56 + 180 + 76}  # params read + 76 B written
SM_COUNT = 148
FP32_LANES = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--views", type=int, default=40)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-parallel", action="store_true", help="skip the whole-host oracle baseline")
    ap.add_argument("--no-train", action="store_true", help="skip the NEXT-3 training-iteration timing")
    ap.add_argument("--profile", action="store_true", help="per-kernel table on stderr")
    ap.add_argument("--n-gaussians", type=int, default=None, help="C4: Gaussians per sub-region (default 1.5M)")
    ap.add_argument("--image", default=None, help="C4: WxH of the views (default 5472x3648; f scales with W)")
    ap.add_argument("--digests", default=None, help="write per-(region, view) output digests (JSON) here "
                                                     "(the SURVEY §8(e) 1-GPU vs N-GPU equality check)")
    return ap.parse_args()


# --------------------------------------------------------------- workload
N_REGIONS = 8  # BASELINE.json configs[3]: 8 visibility-grouped sub-regions


def owned_regions(rank, world):
    """at k GPUs each rank owns 8/k whole sub-regions (shard.assign_subregions, LPT
    over equal costs): strong scaling of the fixed 8-region workload.  Ranks beyond 8 repeat a
    region (not a configuration the driver runs)."""
    from paper_2501_01677_b200 import shard
    if rank >= N_REGIONS:
        return [rank % N_REGIONS]
    return shard.assign_subregions(N_REGIONS, min(world, N_REGIONS))[rank]


def load_workload(args, rank, world, n_views, device):
    """Returns ([regions], name): each region a dict(id, g (numpy Gaussians), cams, masks (device))."""
    import torch
    from synth import scenes as S
    if args.config == "c4":
        kw = {}
        if args.n_gaussians:
            kw["n"] = int(args.n_gaussians)
        if args.image:
            W_, H_ = (int(x) for x in args.image.lower().split("x"))
            kw.update(W=W_, H=H_, f=3648.0 * W_ / 5472.0)
        regs = []
        for reg in owned_regions(rank, world):
            sub = S.subregion(reg, n_views=n_views, **kw)
            masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=device)).to(device)
                     for c in sub["cameras"]]
            regs.append({"id": reg, "g": sub["gaussians"], "cams": sub["cameras"], "masks": masks})
        n = regs[0]["g"].n
        W, H = regs[0]["cams"][0].width, regs[0]["cams"][0].height
        return regs, (f"C4: 8 visibility-grouped sub-regions x {n} Gaussians, oblique {W}x{H} views with "
                      f"building masks; one step = one view of every sub-region (rank {rank} owns regions "
                      f"{[r_['id'] for r_ in regs]})")
    sc = {"c2": S.config2, "c3": S.config3, "c5": S.config5}[args.config](device=device)
    mask = torch.from_numpy(sc.mask).to(device)
    return [{"id": 0, "g": sc.gaussians, "cams": [sc.camera], "masks": [mask]}], \
        f"{args.config.upper()}: {sc.gaussians.n} Gaussians, {sc.camera.width}x{sc.camera.height}, building mask"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms
    DURING the timed region (the same counters nvidia-smi's clocks line reads)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index):
        self.dev = dev_index
        self.sm, self.reasons, self.max = [], set(), None
        self._stop = threading.Event()
        self.h = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis and vis.split(",")[0].isdigit() else self.dev
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(idx)
            self.max = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.sm.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def _poll(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.h is not None:
            self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "NVML poll 2 ms"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# -------------------------------------------------------------- oracle arm
def oracle_sample(g, cam, mask_np, n_pix, seed=0):
    """Time the oracle (single thread, as it stands) fwd+bwd on n_pix sampled masked pixels."""
    import oracle
    from synth import scenes as S
    pix = S.sample_pixels(mask_np, n_pix, seed=seed)
    up = np.random.default_rng(seed).normal(size=(len(pix), 9))
    t0 = time.perf_counter()
    oracle.render(g, cam, mask_np, pix, upstream=up)
    return len(pix), time.perf_counter() - t0


_PAR = {}


def _oracle_shard(k):
    """Worker of the whole-host oracle baseline (forked; reads the scene from _PAR)."""
    import oracle
    g, cam, mask_np, pix, up = _PAR["g"], _PAR["cam"], _PAR["mask"], _PAR["pix"][k], _PAR["up"][k]
    t0 = time.perf_counter()
    oracle.render(g, cam, mask_np, pix, upstream=up)
    return len(pix), time.perf_counter() - t0


def oracle_sample_parallel(g, cam, mask_np, n_per, procs, seed=0):
    """SURVEY §8(d) whole-host oracle number: `procs` independent oracle processes (the oracle as it
    stands, one thread each) over disjoint shards of n_per sampled masked pixels each."""
    import multiprocessing as mproc
    from synth import scenes as S
    pix = S.sample_pixels(mask_np, n_per * procs, seed=seed)
    shards = np.array_split(pix, procs)
    rng = np.random.default_rng(seed)
    _PAR.update(g=g, cam=cam, mask=mask_np, pix=shards, up=[rng.normal(size=(len(x), 9)) for x in shards])
    t0 = time.perf_counter()
    with mproc.get_context("fork").Pool(procs) as pool:
        res = pool.map(_oracle_shard, range(procs))
    wall = time.perf_counter() - t0
    _PAR.clear()
    return sum(r[0] for r in res), wall


def cpu_model():
    """`lscpu` model name of the host (the oracle baseline's hardware)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (the only reference this paper-tier run has), rank 0 only;
    each step samples 256 masked pixels of one view of the next sub-region of the workload."""
    if rank != 0:
        return
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    regs, name = load_workload(args, 0, 1, max(1, min(args.views, args.steps + args.warmup)), dev)
    mask_np = [[m.cpu().numpy() for m in rg["masks"]] for rg in regs]
    n_pix = 256
    pick = lambda s: (regs[s % len(regs)], mask_np[s % len(regs)], (s // len(regs)) % len(regs[s % len(regs)]["cams"]))
    for s in range(args.warmup):
        rg, mn, v = pick(s)
        oracle_sample(rg["g"], rg["cams"][v], mn[v], 16, seed=s)
    tot_pix, tot_t = 0, 0.0
    for s in range(args.steps):
        rg, mn, v = pick(args.warmup + s)
        p, t = oracle_sample(rg["g"], rg["cams"][v], mn[v], n_pix, seed=100 + s)
        tot_pix += p
        tot_t += t
    val = tot_pix / 1e6 / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None,
            "dtype": "f32/f64 (CPU oracle)", "data": "synthetic",
            "config": {"workload": name, "sample": f"{n_pix} sampled masked pixels per step (one view of the "
                                                     f"next sub-region)"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{n_pix} sampled masked pixels per step, fwd+bwd, full-scene projection"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def digest(t):
    import hashlib
    return hashlib.sha256(t.detach().contiguous().cpu().numpy().tobytes()).hexdigest()[:16]


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    # NCCL over NVLink for the (off-path) statistics collectives; PGSAG_DIST_BACKEND=gloo runs the
    # same multi-rank code with host collectives (used to test N>1 on a single test GPU).
    backend = os.environ.get("PGSAG_DIST_BACKEND", "nccl")
    if backend != "nccl" and torch.cuda.is_available():
        local = local % torch.cuda.device_count()
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cdev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2501_01677_b200 import _lib as L
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

    nsteps_all = args.steps + args.warmup
    n_views = max(1, min(args.views, nsteps_all)) if args.config == "c4" else 1
    regs, wname = load_workload(args, rank, world, n_views, dev)
    for rg in regs:
        rg["gt"] = GaussianTensors.from_numpy(rg["g"], dev)
        rg["ccam"] = [camera_from(c) for c in rg["cams"]]
        rg["npix"] = [int(m.count_nonzero().item()) for m in rg["masks"]]
    g0 = regs[0]["gt"]
    H, W = regs[0]["masks"][0].shape
    r = Rasterizer(max(rg["gt"].n for rg in regs), W, H, g0.sh_degree, capacity=24 * g0.n, device=dev,
                   counters=True, sat=False)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1677)  # the same synthetic upstream on every rank (the 1-vs-N region check compares them)
    up = {"dC": torch.randn(3, H, W, device=dev, generator=gen), "dN": torch.randn(3, H, W, device=dev, generator=gen),
          "dD": torch.randn(H, W, device=dev, generator=gen), "dA": torch.randn(H, W, device=dev, generator=gen),
          "dDep": torch.randn(H, W, device=dev, generator=gen)}

    def run_view(ri, v):
        rg = regs[ri]
        r.forward(rg["gt"], rg["ccam"][v], rg["masks"][v])
        r.backward(**up)

    # one step = one view of every owned sub-region (step s: view s mod n_views of each)
    step_views = lambda s: [(ri, s % len(regs[ri]["cams"])) for ri in range(len(regs))]

    def step(s):
        for ri, v in step_views(s):
            run_view(ri, v)

    # counting pass (untimed): E, B, V and M per (region, view)
    per_view = {}
    for s in range(nsteps_all):
        for ri, v in step_views(s):
            if (ri, v) in per_view:
                continue
            r.counters.zero_()
            run_view(ri, v)
            torch.cuda.synchronize()
            per_view[(ri, v)] = r.stats()
    # tile imbalance of the first view: max / mean blends per active tile
    m00 = regs[0]["masks"][0]
    r.forward(g0, regs[0]["ccam"][0], m00)
    gtile = torch.nn.functional.pad(r.img_g.clamp(min=0).float() * (m00 > 0),
                                    (0, (16 - W % 16) % 16, 0, (16 - H % 16) % 16))
    tb = gtile.reshape(gtile.shape[0] // 16, 16, gtile.shape[1] // 16, 16).sum(dim=(1, 3))
    act = tb[tb > 0]
    imbalance = float(act.max() / act.mean()) if act.numel() else 0.0
    # SURVEY §8(d) C5 statistics, for every config: entries per active tile (p50 / p99 / max)
    rl = (r.ranges.view(-1, 2)[:, 1] - r.ranges.view(-1, 2)[:, 0]).double()
    rl = rl[rl > 0]
    tile_entries = ([float(torch.quantile(rl, 0.5)), float(torch.quantile(rl, 0.99)), float(rl.max())]
                    if rl.numel() else [0.0, 0.0, 0.0])
    # timed steps use the sync-free sort (no host synchronisation inside a step); the counting pass
    # above read every view's M: size the entry buffers to the largest (+15 %), which also bounds the
    # sync-free sort's grids
    r._alloc_bins(int(1.15 * max(st["M"] for st in per_view.values())) + 4096)
    r._build_bins()
    r._img.counters = None  # timed steps run the non-counting kernels
    r.sync_free = True

    tsteps = [args.warmup + s for s in range(args.steps)]
    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    # per-kernel split: one untimed pass over the same steps with every kernel bracketed by CUDA
    # events (pgsag_timing_*); it names the dominant kernel
    L.timing_filter(None)
    L.timing_enable(True)
    L.timing_collect()
    for s in tsteps:
        step(s)
    torch.cuda.synchronize()
    L.timing_enable(False)
    ksplit = L.timing_collect()
    dom = max(ksplit.items(), key=lambda kv: kv[1][0])[0] if ksplit else None
    if world > 1:
        dist.barrier()
    # the timed region: only the dominant kernel carries an event pair (its live launch time for the
    # roofline), so the other launches run without event records
    L.timing_filter(dom)
    L.timing_enable(dom is not None)
    L.timing_collect()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in tsteps]
        ev0.record()
        for s, e in zip(tsteps, evs):
            step(s)
            e.record()
        ev1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    L.timing_enable(False)
    L.timing_filter(None)
    kdom = L.timing_collect()
    # capacity check of the sync-free timed views (the counting pass sized the buffers from every
    # view's M, so this must hold; an overflowed view would have been rendered empty)
    assert r.check_capacity(), "sync-free entry capacity exceeded in the timed region"
    ms = ev0.elapsed_time(ev1)
    per_step = [ev0.elapsed_time(evs[0])] + [evs[k - 1].elapsed_time(evs[k]) for k in range(1, len(evs))]
    pct = lambda q: float(np.percentile(per_step, q))
    timed_views = [rv for s in tsteps for rv in step_views(s)]
    pix = float(sum(regs[ri]["npix"][v] for ri, v in timed_views))
    blends = float(sum(per_view[rv]["blended"] for rv in timed_views))
    if world > 1:
        t = torch.tensor([ms], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        agg = torch.tensor([pix, blends], device=cdev, dtype=torch.float64)
        dist.all_reduce(agg)
        pix_all, blends_all = float(agg[0]), float(agg[1])
        # per-rank statistics record all-gathered over NVLink (off the timed region)
        from paper_2501_01677_b200 import shard
        rec = shard.stats_record(rank=rank, ms=ms, masked_pixels=pix, blends=blends, tile_imbalance=imbalance,
                                 views=len(timed_views)).to(cdev)
        rank_table = shard.gather_stats(rec).cpu()
    else:
        ms_max, pix_all, blends_all = ms, pix, blends
    value = pix_all / 1e6 / (ms_max / 1e3)

    # ---------------------------------------------------- roofline (dominant kernel)
    peaks = measured_peaks()
    ksteps = {k: (v[0] / args.steps, v[1] // max(args.steps, 1)) for k, v in ksplit.items()}
    launches = int(sum(v[1] for v in ksplit.values()))
    nviews_step = len(timed_views) / max(args.steps, 1)
    mean_over = lambda key: sum(per_view[rv][key] for rv in timed_views) / max(len(timed_views), 1)
    Ev, Bv, Vv, Mv = mean_over("evaluated"), mean_over("blended"), mean_over("bwd_visited"), mean_over("M")
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    inst_peak = SM_COUNT * FP32_LANES * sm_mhz * 1e6 / 1e12  # T FP32 lane-instructions / s
    fp32_peak = 2 * inst_peak  # TFLOP/s (FMA = 2)
    roof, roof_flops = None, None
    if dom and dom in kdom:
        tot_ms, nl = kdom[dom]
        avg_s = tot_ms / 1e3 / max(nl, 1)
        per_launch = lambda x: x * nviews_step * args.steps / max(nl, 1)  # units per launch of the kernel
        if dom.startswith(("A6", "A7")):
            inst = (INST_EVAL_FWD * Ev + INST_BLEND_FWD * Bv) if dom.startswith("A6") else \
                (INST_VISIT_BWD * Vv + INST_BLEND_BWD * Bv)
            flops = (FLOP_EVAL * Ev + FLOP_BLEND_FWD * Bv) if dom.startswith("A6") else \
                (FLOP_EVAL * Vv + FLOP_BLEND_BWD * Bv)
            roof = {"kernel": dom, "bound": "alu", "achieved": per_launch(inst) / avg_s / 1e12, "peak": inst_peak,
                    "unit": "T FP32 lane-instr/s",
                    "convention": "SURVEY §8(d): A6 14 per evaluated + 10 per blended pair, A7 17 per visited + "
                                  "55 per blended pair; peak 148 SMs x 128 lanes x sm_max_mhz"}
            roof_flops = {"achieved": per_launch(flops) / avg_s / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
                          "convention": "the kernel's own FP32 flops, FMA = 2 (DESIGN.md §5)"}
            roof_flops["frac"] = roof_flops["achieved"] / roof_flops["peak"]
        elif dom.startswith("A1"):
            roof = {"kernel": dom, "bound": "hbm", "achieved": per_launch(BYTES_A1[g0.sh_degree] * g0.n) / avg_s / 1e9,
                    "peak": float(peaks.get("hbm_gbs", 6551.4)), "unit": "GB/s"}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": None, "peak": float(peaks.get("hbm_gbs", 6551.4)),
                    "unit": "GB/s"}
        if roof["achieved"] is not None:
            roof["frac"] = roof["achieved"] / roof["peak"]
        roof["peak_source"] = ("148 SMs x 128 FP32 lanes x sm_max_mhz (MEASURED_PEAKS.json)"
                               if roof["bound"] == "alu" else "MEASURED_PEAKS.json hbm_gbs")
        if roof["bound"] == "alu":  # cross-check of the derived FP32 peak: FFMA2 chains, all SMs
            scratch = torch.empty(256, device=dev)
            st_ = torch.cuda.current_stream().cuda_stream
            roof["peak_measured"] = {"ffma2_tflops": L.microbench_fp32(1, 16384, scratch.data_ptr(), st_),
                                     "ffma_tflops": L.microbench_fp32(0, 16384, scratch.data_ptr(), st_),
                                     "source": "pgsag_microbench_fp32: 16 independent FMA chains per thread, 8 CTAs/SM"}
        roof["traffic"] = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            if tr.get("config") == args.config and dom in tr.get("bytes_per_launch", {}):
                roof["traffic"] = tr["bytes_per_launch"][dom]
        except Exception:
            pass
        roof["share_of_step"] = tot_ms / max(ms, 1e-9)

    # every kernel of the step against its own roof: algorithmic bytes (HBM) or
    # FP32 lane-instructions (§8(d) counts) per view / its mean time per view in the split pass
    rooflines_all = {}
    if ksplit:
        n_, px_, tiles_ = g0.n, W * H, ((W + 15) // 16) * ((H + 15) // 16)
        tile_bits = max(1, (tiles_ - 1).bit_length())
        alg = {  # (bound, units per view over all launches of the kernel)
            "A0_tilemask_count": ("hbm", px_ + 4 * tiles_),
            "A1_preprocess": ("hbm", BYTES_A1[g0.sh_degree] * n_),
            "A2_scan": ("hbm", 8 * n_),
            "A3_duplicate": ("hbm", 8 * Mv + 20 * n_),
            # stage 1 (depth, 32 bits, 4 passes over n) and stage 2 (tile, 2 passes over M): per pass
            # key + value read and written (16 B per key)
            "A4_radix_onesweep_s1": ("hbm", 4 * 16 * n_),
            "A4_radix_onesweep_s2": ("hbm", (2 if tile_bits > 9 else 1) * 16 * Mv),
            "A4_radix_hist_s1": ("hbm", 8 * n_ + 8 * n_),  # depth + tiles_touched read, keys + ids written
            "A4_radix_hist_s2": ("hbm", 4 * Mv),
            "A5_ranges": ("hbm", 4 * Mv + 8 * tiles_),
            "A6_render_fwd": ("alu", INST_EVAL_FWD * Ev + INST_BLEND_FWD * Bv),
            "A7_render_bwd": ("alu", INST_VISIT_BWD * Vv + INST_BLEND_BWD * Bv),
            "A8_preprocess_bwd": ("hbm", 536 * n_),  # 236 B params + 64 B 2D gradients read, 236 B written
        }
        hbm = float(peaks.get("hbm_gbs", 6551.4))
        for k, (b_, units) in alg.items():
            if k not in ksteps:
                continue
            t_s = ksteps[k][0] / 1e3 / max(nviews_step, 1e-9)  # s per view
            if b_ == "hbm":
                a_ = units / t_s / 1e9
                rooflines_all[k] = {"bound": "hbm", "achieved_gbs": round(a_, 1), "frac": round(a_ / hbm, 4)}
            else:
                a_ = units / t_s / 1e12
                rooflines_all[k] = {"bound": "alu", "achieved_tinst": round(a_, 3), "frac": round(a_ / inst_peak, 4)}

    def dmax(x):  # max over ranks of a device time
        if world > 1:
            t = torch.tensor([x], device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    def dsum(x):
        if world > 1:
            t = torch.tensor([x], device=cdev, dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())
        return x

    # ------------------------------------------- SURVEY §8(e) check: per-(region, view) output digests
    if args.digests:
        r.sync_free = False
        rec = []
        for ri, rg in enumerate(regs):
            for v in range(len(rg["cams"])):
                r.forward(rg["gt"], rg["ccam"][v], rg["masks"][v])
                gr = r.backward(**up)
                torch.cuda.synchronize()
                m = rg["masks"][v] > 0
                rec.append({"region": rg["id"], "view": v, "M": r.M,
                            "fwd": {k: digest(getattr(r, "img_" + k)[..., m] if getattr(r, "img_" + k).dim() == 3
                                              else getattr(r, "img_" + k)[m]) for k in ("C", "N", "D", "T", "g")},
                            "grad_sums": {k: float(gr[k].double().abs().sum()) for k in ("dmean", "dscale", "drot",
                                                                                      "dopacity", "dsh")}})
        if world > 1:
            allr = [None] * world
            dist.all_gather_object(allr, rec)
            rec = [x for rr in allr for x in rr]
        if rank == 0:
            with open(args.digests, "w") as f:
                json.dump(rec, f)

    # ------------------------------------------- e2e_raster: rasterizer fwd+bwd from host buffers
    # (every input of pgsag_* copied in each step: Gaussians, mask, upstream planes; gradients out)
    # over the first owned region's views
    R0 = regs[0]
    r.sync_free = False
    e2e_raster = None
    if not args.no_e2e:
        pin = lambda t: t.detach().cpu().pin_memory()
        hg = {k: pin(getattr(g0, k)) for k in ("mean", "scale", "rot", "opacity", "sh")}
        hm = [pin(m) for m in R0["masks"]]
        hup = {k: pin(v) for k, v in up.items()}
        hgrad = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in
                 (("dmean", r.dmean), ("dscale", r.dscale), ("drot", r.drot), ("dopacity", r.dopacity),
                  ("dsh", r.dsh))}
        dg = GaussianTensors(*(torch.empty_like(getattr(g0, k)) for k in ("mean", "scale", "rot", "opacity", "sh")),
                             g0.sh_degree)
        dmask = torch.empty_like(R0["masks"][0])
        dup = {k: torch.empty_like(v) for k, v in up.items()}
        h2d = sum(t.numel() * t.element_size() for t in hg.values()) + hm[0].numel() + \
            sum(t.numel() * t.element_size() for t in hup.values())
        d2h = sum(t.numel() * t.element_size() for t in hgrad.values())
        ke = min(args.steps, 5)
        eviews = [s % len(R0["cams"]) for s in tsteps[:ke]]

        def e2e_step(v):
            for k in hg:
                getattr(dg, k).copy_(hg[k], non_blocking=True)
            dmask.copy_(hm[v], non_blocking=True)
            for k in hup:
                dup[k].copy_(hup[k], non_blocking=True)
            r.forward(dg, R0["ccam"][v], dmask)
            gr = r.backward(**dup)
            for k in hgrad:
                hgrad[k].copy_(gr[k], non_blocking=True)
        e2e_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for v in eviews:
            e2e_step(v)
        e1.record()
        torch.cuda.synchronize()
        ems = dmax(e0.elapsed_time(e1))
        epix = dsum(float(sum(R0["npix"][v] for v in eviews)))
        e2e_raster = {"value": epix / 1e6 / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(d2h), "steps": ke,
                      "note": "per view: pinned host Gaussians+mask+upstream planes -> device, fwd+bwd, "
                              "gradients -> host"}
        del dg, dup, hg, hup, hgrad

    # ------------------------------------------- NEXT-3: full training iteration (Eq. 10-11)
    # train_step: device-resident inputs; e2e: the same iterations through the public API
    # (train.Trainer.step) with each step's inputs (target photo + building mask) copied from
    # pinned host memory on a copy stream (double-buffered, prefetching the next view while the
    # current one trains) and the loss terms read back to the host every step.
    train, e2e = None, None
    if not (args.no_train and args.no_e2e):
        from paper_2501_01677_b200.train import Trainer
        gt_ = GaussianTensors(*(getattr(g0, k).clone() for k in ("mean", "scale", "rot", "opacity", "sh")),
                              g0.sh_degree)
        rt = Rasterizer(g0.n, W, H, g0.sh_degree, capacity=r.capacity, device=dev, counters=False, sat=False,
                        sync_free=True)
        tr = Trainer(rt, gt_)
        kt = args.steps  # K iterations over the first owned region's views
        tviews = [s % len(R0["cams"]) for s in tsteps]
        masks0, ccam0, npix0 = R0["masks"], R0["ccam"], R0["npix"]
        tgt = torch.rand(3, H, W, device=dev, generator=gen)  # synthetic target photo
        for v in tviews[:2]:  # warm-up
            tr.step(ccam0[v], masks0[v], tgt, gc_w=rt.gc_weights(tgt, masks0[v]), band=rt.boundary_band(masks0[v], 1))
        torch.cuda.synchronize()
        if not args.no_train:
            extras = {v: (rt.gc_weights(tgt, masks0[v]), rt.boundary_band(masks0[v], 1)) for v in set(tviews)}
            if world > 1:
                dist.barrier()
            L.timing_enable(True)
            L.timing_collect()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for v in tviews:
                tr.step(ccam0[v], masks0[v], tgt, gc_w=extras[v][0], band=extras[v][1])
            t1.record()
            torch.cuda.synchronize()
            L.timing_enable(False)
            tk = L.timing_collect()
            tms = dmax(t0.elapsed_time(t1))
            tpix = dsum(float(sum(npix0[v] for v in tviews)))
            lo = tr.losses()
            train = {"ms_per_iter": tms / kt, "value": tpix / 1e6 / (tms / 1e3), "unit": UNIT, "iters": kt,
                     "terms": "L_rgb (L1+SSIM) + L_s + L_ban + L_GC-load with P:179 weights; Adam on raw params",
                     "gpu_launches": int(sum(v[1] for v in tk.values())),
                     "kernels_ms_per_iter": {k: round(v[0] / kt, 4) for k, v in sorted(tk.items())},
                     "last_loss": {k: round(float(x), 6) for k, x in lo.items()},
                     "losses_finite": bool(all(math.isfinite(float(x)) for x in lo.values()))}
            del extras
        if not args.no_e2e:
            # the photo as captured: 8-bit interleaved RGB (pgsag_unpack_rgb8 makes the float planes)
            htgt = (tgt * 255.0).round().to(torch.uint8).permute(1, 2, 0).contiguous().cpu().pin_memory()
            hmask = [m.cpu().pin_memory() for m in masks0]
            dt8 = [torch.empty(H, W, 3, dtype=torch.uint8, device=dev) for _ in range(2)]
            dt = [torch.empty_like(tgt) for _ in range(2)]
            dm = [torch.empty_like(masks0[0]) for _ in range(2)]
            hloss = torch.empty(kt, 6, dtype=torch.float64, pin_memory=True)
            cs = torch.cuda.Stream(device=dev)
            main = torch.cuda.current_stream()
            ready = [torch.cuda.Event() for _ in range(2)]
            free = [torch.cuda.Event() for _ in range(2)]

            def fetch(slot, v):
                with torch.cuda.stream(cs):
                    cs.wait_event(free[slot])
                    dt8[slot].copy_(htgt, non_blocking=True)
                    dm[slot].copy_(hmask[v], non_blocking=True)
                    ready[slot].record(cs)

            for k in range(2):
                free[k].record(main)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            fetch(0, tviews[0])
            for s_, v in enumerate(tviews):
                cur = s_ & 1
                if s_ + 1 < kt:
                    fetch(cur ^ 1, tviews[s_ + 1])
                main.wait_event(ready[cur])
                L.unpack_rgb8(dt8[cur].data_ptr(), W, H, dt[cur].data_ptr(), main.cuda_stream)
                tr.step_photo(ccam0[v], dm[cur], dt[cur])
                hloss[s_].copy_(tr.loss_rgb, non_blocking=True)
                free[cur].record(main)
            e1.record(main)
            torch.cuda.synchronize()
            assert not tr.losses()["overflowed"]
            ems = dmax(e0.elapsed_time(e1))
            epix = dsum(float(sum(npix0[v] for v in tviews)))
            e2e = {"value": epix / 1e6 / (ems / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(htgt.numel() + hmask[0].numel()),
                   "d2h_bytes_per_step": int(hloss[0].numel() * 8), "steps": kt,
                   "note": "train.Trainer.step per view: pinned host photo (8-bit HxWx3) + building mask -> device "
                           "(copy stream, prefetched), pgsag_unpack_rgb8, Eq. 9 weights + boundary band, A0-A8 + "
                           "L_rgb + L_ban + L_GC-load + L_s/Adam, loss terms -> host; Gaussians and optimiser state "
                           "are resident model state; a step here is one view (the bench step's unit of work)"}
        del tr, gt_, rt

    # ------------------------------------------------------------- CPU oracle baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v0 = tsteps[0] % len(R0["cams"])
        n_s = 1024 if args.config in ("c4", "c3", "c5") else 4096
        mnp = R0["masks"][v0].cpu().numpy()
        p, t = oracle_sample(R0["g"], R0["cams"][v0], mnp, n_s)
        # C1 (the oracle's full-frame config) fwd+bwd over every mask pixel, same thread
        from synth import scenes as S
        c1 = S.config1()
        c1p, c1t = oracle_sample(c1.gaussians, c1.camera, c1.mask, int(c1.mask.sum()))
        cpu = {"value": p / 1e6 / t, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{p} sampled masked pixels of view {v0} of region {R0['id']}, fwd+bwd, single thread, "
                         f"incl. full-scene projection ({t:.1f} s)",
               "full_frame_extrapolated_s": R0["npix"][v0] / p * t,
               "c1_full_frame": {"pixels": c1p, "seconds": c1t, "note": "C1: 1000 Gaussians, 64x64, every mask "
                                                                         "pixel fwd+bwd, single thread"}}
        if not args.no_cpu_parallel:
            procs = max(1, min(os.cpu_count() or 1, 64))
            pp, tw = oracle_sample_parallel(R0["g"], R0["cams"][v0], mnp, n_s // 2, procs, seed=1)
            cpu["whole_host"] = {"value": pp / 1e6 / tw, "unit": UNIT, "cores": procs, "kind": "oracle",
                                 "sample": f"{procs} forked oracle processes x {n_s // 2} disjoint sampled pixels "
                                           f"({pp} total, wall {tw:.1f} s, each incl. its full-scene projection)"}

    if rank == 0:
        st0 = per_view[timed_views[0]]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wname, "views_per_step": int(round(len(timed_views) / args.steps)) * world
                       if args.config == "c4" else world,
                       "views_per_step_per_rank": nviews_step,
                       "l2": "inputs larger than L2 (Gaussians 1.5M x 236 B = 354 MB per sub-region, a new view and "
                             "sub-region every view)",
                       "sh_degree": g0.sh_degree, "n_gaussians_per_region": g0.n, "image": [W, H],
                       "regions_rank0": [rg["id"] for rg in regs]},
            "blends_per_s": blends_all / (ms_max / 1e3),
            "masked_pixels_per_step": pix_all / args.steps,
            "tile_imbalance_max_over_mean": imbalance,
            "tile_entries_p50_p99_max": tile_entries,
            "M_per_view": Mv, "evaluated_per_view": Ev, "blended_per_view": Bv, "bwd_visited_per_view": Vv,
            "inst_per_unit": {"evaluated_fwd": INST_EVAL_FWD, "blended_fwd": INST_BLEND_FWD,
                              "visited_bwd": INST_VISIT_BWD, "blended_bwd": INST_BLEND_BWD},
            "flop_per_unit": {"evaluated": FLOP_EVAL, "blended_fwd": FLOP_BLEND_FWD, "blended_bwd": FLOP_BLEND_BWD},
            "roofline": roof, "roofline_flops": roof_flops, "rooflines_all_kernels": rooflines_all,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_raster": e2e_raster, "gpu_launches": launches,
            "train_step": train,
            "kernels_ms_per_step": {k: round(v[0], 4) for k, v in sorted(ksteps.items())},
            "kernels_ms_per_view": {k: round(v[0] / max(nviews_step, 1e-9), 4) for k, v in sorted(ksteps.items())},
            "kernels_split_source": "untimed pass over the same steps with every kernel event-bracketed; inside "
                                    "the timed region only the dominant kernel is (roofline.achieved)",
            "clocks": clk.summary(),
            "per_rank_ms": (rank_table[:, 1].tolist() if world > 1 else [ms]),
            "step_ms_p10_p50_p90": [round(pct(10), 4), round(pct(50), 4), round(pct(90), 4)],
        }
        print(json.dumps(line), flush=True)
        if args.profile:
            tot = sum(v[0] for v in ksteps.values())
            for k, v in sorted(ksteps.items(), key=lambda kv: -kv[1][0]):
                sys.stderr.write(f"{k:24s} {v[0]:9.3f} ms/step  {100 * v[0] / max(tot, 1e-9):5.1f}%  x{v[1]}\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

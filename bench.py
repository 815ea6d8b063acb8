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
    return ap.parse_args()


# --------------------------------------------------------------- workload
def load_workload(cfg, rank, n_views, device):
    """Returns (numpy Gaussians, [cameras], [mask tensors on device], name)."""
    import torch
    from synth import scenes as S
    if cfg == "c4":
        from paper_2501_01677_b200 import shard
        reg = shard.weak_region(rank)
        sub = S.subregion(reg, n_views=n_views)
        cams = sub["cameras"]
        masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=device)).to(device) for c in cams]
        return sub["gaussians"], cams, masks, (f"C4: one visibility-grouped sub-region per GPU (rank 0: region {reg}), "
                                               f"1.5M Gaussians, {len(cams)} oblique 5472x3648 views, building mask")
    sc = {"c2": S.config2, "c3": S.config3, "c5": S.config5}[cfg](device=device)
    mask = torch.from_numpy(sc.mask).to(device)
    return sc.gaussians, [sc.camera], [mask], f"{cfg.upper()}: {sc.gaussians.n} Gaussians, " \
                                                 f"{sc.camera.width}x{sc.camera.height}, building mask"


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


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (the only reference this paper-tier run has), rank 0 only."""
    if rank != 0:
        return
    import torch
    from synth import scenes as S
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g, cams, masks, name = load_workload(args.config, 0, min(args.views, args.steps + args.warmup), dev)
    mask_np = [m.cpu().numpy() for m in masks]
    n_pix = 256
    for s in range(args.warmup):
        oracle_sample(g, cams[s % len(cams)], mask_np[s % len(cams)], 16, seed=s)
    tot_pix, tot_t = 0, 0.0
    for s in range(args.steps):
        v = (args.warmup + s) % len(cams)
        p, t = oracle_sample(g, cams[v], mask_np[v], n_pix, seed=100 + s)
        tot_pix += p
        tot_t += t
    val = tot_pix / 1e6 / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (CPU oracle)",
            "data": "synthetic", "config": {"workload": name, "sample": f"{n_pix} sampled masked pixels per step"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{n_pix} sampled masked pixels per step, fwd+bwd, full-scene projection"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    # NCCL over NVLink for the (off-path) statistics collectives; PGSAG_DIST_BACKEND=gloo runs the
    # same multi-rank code with host collectives (used to smoke-test N>1 on a single test GPU).
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

    n_views = min(args.views, args.steps + args.warmup) if args.config == "c4" else 1
    g_np, cams, masks, wname = load_workload(args.config, rank, n_views, dev)
    g = GaussianTensors.from_numpy(g_np, dev)
    H, W = masks[0].shape
    ccam = [camera_from(c) for c in cams]
    r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=True, sat=False)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1677 + rank)
    up = {"dC": torch.randn(3, H, W, device=dev, generator=gen), "dN": torch.randn(3, H, W, device=dev, generator=gen),
          "dD": torch.randn(H, W, device=dev, generator=gen), "dA": torch.randn(H, W, device=dev, generator=gen),
          "dDep": torch.randn(H, W, device=dev, generator=gen)}
    npix = [int(m.count_nonzero().item()) for m in masks]

    def step(v):
        r.forward(g, ccam[v], masks[v])
        r.backward(**up)

    # counting pass (untimed): E, B, V and M per view
    per_view = {}
    for v in range(len(cams)):
        r.counters.zero_()
        step(v)
        torch.cuda.synchronize()
        st = r.stats()
        per_view[v] = st
    # tile imbalance of view 0: max / mean blends per active tile
    r.forward(g, ccam[0], masks[0])
    gt = torch.nn.functional.pad(r.img_g.clamp(min=0).float() * (masks[0] > 0),
                                 (0, (16 - W % 16) % 16, 0, (16 - H % 16) % 16))
    tb = gt.reshape(gt.shape[0] // 16, 16, gt.shape[1] // 16, 16).sum(dim=(1, 3))
    act = tb[tb > 0]
    imbalance = float(act.max() / act.mean()) if act.numel() else 0.0
    # SURVEY §8(d) C5 statistics, for every config: entries per active tile (p50 / p99 / max)
    rl = (r.ranges.view(-1, 2)[:, 1] - r.ranges.view(-1, 2)[:, 0]).double()
    rl = rl[rl > 0]
    tile_entries = ([float(torch.quantile(rl, 0.5)), float(torch.quantile(rl, 0.99)), float(rl.max())]
                    if rl.numel() else [0.0, 0.0, 0.0])
    r._img.counters = None  # timed steps run the non-counting kernels
    # timed steps use the sync-free sort (no host synchronisation inside a step); the counting pass
    # above read every view's M: size the entry buffers to the largest (+15 %), which also bounds the
    # sync-free sort's grids
    r._alloc_bins(int(1.15 * max(per_view[v]["M"] for v in per_view)) + 4096)
    r._build_structs()
    r._img.counters = None
    r.sync_free = True

    views = [(args.warmup + s) % len(cams) for s in range(args.steps)]
    for s in range(args.warmup):
        step(s % len(cams))
    torch.cuda.synchronize()
    # per-kernel split: one untimed pass over the same views with every kernel bracketed by CUDA
    # events (pgsag_timing_*); it names the dominant kernel
    L.timing_filter(None)
    L.timing_enable(True)
    L.timing_collect()
    for v in views:
        step(v)
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
        evs = [torch.cuda.Event(enable_timing=True) for _ in views]
        ev0.record()
        for v, e in zip(views, evs):
            step(v)
            e.record()
        ev1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    L.timing_enable(False)
    L.timing_filter(None)
    kdom = L.timing_collect()
    ms = ev0.elapsed_time(ev1)
    per_step = [ev0.elapsed_time(evs[0])] + [evs[k - 1].elapsed_time(evs[k]) for k in range(1, len(evs))]
    pct = lambda q: float(np.percentile(per_step, q))
    pix = float(sum(npix[v] for v in views))
    blends = float(sum(per_view[v]["blended"] for v in views))
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
                                 views=len(views)).to(cdev)
        rank_table = shard.gather_stats(rec).cpu()
    else:
        ms_max, pix_all, blends_all = ms, pix, blends
    value = pix_all / 1e6 / (ms_max / 1e3)

    # ---------------------------------------------------- roofline (dominant kernel)
    peaks = measured_peaks()
    ksteps = {k: (v[0] / args.steps, v[1] // max(args.steps, 1)) for k, v in ksplit.items()}
    launches = int(sum(v[1] for v in ksplit.values()))
    roof = None
    if dom and dom in kdom:
        tot_ms, nl = kdom[dom]
        avg_s = tot_ms / 1e3 / max(nl, 1)
        E = sum(per_view[v]["evaluated"] for v in views) / len(views)
        B = sum(per_view[v]["blended"] for v in views) / len(views)
        V = sum(per_view[v]["bwd_visited"] for v in views) / len(views)
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = SM_COUNT * FP32_LANES * 2 * sm_mhz * 1e6 / 1e12
        if dom.startswith("A6"):
            roof = {"kernel": dom, "bound": "alu", "achieved": (FLOP_EVAL * E + FLOP_BLEND_FWD * B) / avg_s / 1e12,
                    "peak": fp32_peak, "unit": "TFLOP/s"}
        elif dom.startswith("A7"):
            roof = {"kernel": dom, "bound": "alu", "achieved": (FLOP_EVAL * V + FLOP_BLEND_BWD * B) / avg_s / 1e12,
                    "peak": fp32_peak, "unit": "TFLOP/s"}
        elif dom.startswith("A1"):
            roof = {"kernel": dom, "bound": "hbm", "achieved": BYTES_A1[g.sh_degree] * g.n / avg_s / 1e9,
                    "peak": float(peaks.get("hbm_gbs", 6551.4)), "unit": "GB/s"}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": None, "peak": float(peaks.get("hbm_gbs", 6551.4)),
                    "unit": "GB/s"}
        if roof["achieved"] is not None:
            roof["frac"] = roof["achieved"] / roof["peak"]
        roof["peak_source"] = ("148 SMs x 128 FP32 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json)"
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
    # flops (FP32) per launch / its mean launch time in the split pass
    rooflines_all = {}
    if ksplit:
        Mv = sum(per_view[v]["M"] for v in views) / len(views)
        Ev = sum(per_view[v]["evaluated"] for v in views) / len(views)
        Bv = sum(per_view[v]["blended"] for v in views) / len(views)
        Vv = sum(per_view[v]["bwd_visited"] for v in views) / len(views)
        n_, px_, tiles_ = g.n, W * H, ((W + 15) // 16) * ((H + 15) // 16)
        tile_bits = max(1, (tiles_ - 1).bit_length())
        alg = {  # (bound, units per view over all launches of the kernel)
            "A0_tilemask_count": ("hbm", px_ + 4 * tiles_),
            "A1_preprocess": ("hbm", BYTES_A1[g.sh_degree] * n_),
            "A2_scan": ("hbm", 8 * n_),
            "A3_duplicate": ("hbm", 8 * Mv + 20 * n_),
            "A4_radix_onesweep": ("hbm", 4 * 16 * n_ + (2 if tile_bits > 9 else 1) * 16 * Mv),
            "A4_radix_hist": ("hbm", 4 * n_ + 4 * Mv),
            "A5_ranges": ("hbm", 4 * Mv + 8 * tiles_),
            "A6_render_fwd": ("alu", FLOP_EVAL * Ev + FLOP_BLEND_FWD * Bv),
            "A7_render_bwd": ("alu", FLOP_EVAL * Vv + FLOP_BLEND_BWD * Bv),
            "A8_preprocess_bwd": ("hbm", 536 * n_),  # 236 B params + 64 B 2D gradients read, 236 B written
        }
        hbm = float(peaks.get("hbm_gbs", 6551.4))
        fp32 = SM_COUNT * FP32_LANES * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        for k, (b_, units) in alg.items():
            if k not in ksteps:
                continue
            t_s = ksteps[k][0] / 1e3  # ms per step -> s
            if b_ == "hbm":
                a_ = units / t_s / 1e9
                rooflines_all[k] = {"bound": "hbm", "achieved_gbs": round(a_, 1), "frac": round(a_ / hbm, 4)}
            else:
                a_ = units / t_s / 1e12
                rooflines_all[k] = {"bound": "alu", "achieved_tflops": round(a_, 3), "frac": round(a_ / fp32, 4)}

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

    # ------------------------------------------- e2e_raster: rasterizer fwd+bwd from host buffers
    # (every input of pgsag_* copied in each step: Gaussians, mask, upstream planes; gradients out)
    e2e_raster = None
    if not args.no_e2e:
        pin = lambda t: t.detach().cpu().pin_memory()
        hg = {k: pin(getattr(g, k)) for k in ("mean", "scale", "rot", "opacity", "sh")}
        hm = [pin(m) for m in masks]
        hup = {k: pin(v) for k, v in up.items()}
        hgrad = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in
                 (("dmean", r.dmean), ("dscale", r.dscale), ("drot", r.drot), ("dopacity", r.dopacity),
                  ("dsh", r.dsh))}
        dg = GaussianTensors(*(torch.empty_like(getattr(g, k)) for k in ("mean", "scale", "rot", "opacity", "sh")),
                             g.sh_degree)
        dmask = torch.empty_like(masks[0])
        dup = {k: torch.empty_like(v) for k, v in up.items()}
        h2d = sum(t.numel() * t.element_size() for t in hg.values()) + hm[0].numel() + \
            sum(t.numel() * t.element_size() for t in hup.values())
        d2h = sum(t.numel() * t.element_size() for t in hgrad.values())
        ke = min(args.steps, 5)

        def e2e_step(v):
            for k in hg:
                getattr(dg, k).copy_(hg[k], non_blocking=True)
            dmask.copy_(hm[v], non_blocking=True)
            for k in hup:
                dup[k].copy_(hup[k], non_blocking=True)
            r.forward(dg, ccam[v], dmask)
            gr = r.backward(**dup)
            for k in hgrad:
                hgrad[k].copy_(gr[k], non_blocking=True)
        e2e_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s_ in range(ke):
            e2e_step(views[s_])
        e1.record()
        torch.cuda.synchronize()
        ems = dmax(e0.elapsed_time(e1))
        epix = dsum(float(sum(npix[views[s_]] for s_ in range(ke))))
        e2e_raster = {"value": epix / 1e6 / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                      "d2h_bytes_per_step": int(d2h), "steps": ke,
                      "note": "pinned host Gaussians+mask+upstream planes -> device, fwd+bwd, gradients -> host"}
        del dg, dup, hg, hup, hgrad

    # ------------------------------------------- NEXT-3: full training iteration (Eq. 10-11)
    # train_step: device-resident inputs; e2e: the same iterations through the public API
    # (train.Trainer.step) with each step's inputs (target photo + building mask) copied from
    # pinned host memory on a copy stream (double-buffered, prefetching the next view while the
    # current one trains) and the loss terms read back to the host every step.
    train, e2e = None, None
    if not (args.no_train and args.no_e2e):
        from paper_2501_01677_b200.train import Trainer
        gt_ = GaussianTensors(*(getattr(g, k).clone() for k in ("mean", "scale", "rot", "opacity", "sh")),
                              g.sh_degree)
        tr = Trainer(r, gt_)
        kt = args.steps  # the same K views as the timed rasterizer steps
        tviews = views[:kt]
        tgt = torch.rand(3, H, W, device=dev, generator=gen)  # synthetic target photo
        for v in tviews[:2]:  # warm-up
            tr.step(ccam[v], masks[v], tgt, gc_w=r.gc_weights(tgt, masks[v]), band=r.boundary_band(masks[v], 1))
        torch.cuda.synchronize()
        if not args.no_train:
            extras = {v: (r.gc_weights(tgt, masks[v]), r.boundary_band(masks[v], 1)) for v in set(tviews)}
            if world > 1:
                dist.barrier()
            L.timing_enable(True)
            L.timing_collect()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for v in tviews:
                tr.step(ccam[v], masks[v], tgt, gc_w=extras[v][0], band=extras[v][1])
            t1.record()
            torch.cuda.synchronize()
            L.timing_enable(False)
            tk = L.timing_collect()
            tms = dmax(t0.elapsed_time(t1))
            tpix = dsum(float(sum(npix[v] for v in tviews)))
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
            hmask = [m.cpu().pin_memory() for m in masks]
            dt8 = [torch.empty(H, W, 3, dtype=torch.uint8, device=dev) for _ in range(2)]
            dt = [torch.empty_like(tgt) for _ in range(2)]
            dm = [torch.empty_like(masks[0]) for _ in range(2)]
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
                tr.step_photo(ccam[v], dm[cur], dt[cur])
                hloss[s_].copy_(tr.loss_rgb, non_blocking=True)
                free[cur].record(main)
            e1.record(main)
            torch.cuda.synchronize()
            ems = dmax(e0.elapsed_time(e1))
            epix = dsum(float(sum(npix[v] for v in tviews)))
            e2e = {"value": epix / 1e6 / (ems / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(htgt.numel() + hmask[0].numel()),
                   "d2h_bytes_per_step": int(hloss[0].numel() * 8), "steps": kt,
                   "note": "train.Trainer.step per view: pinned host photo (8-bit HxWx3) + building mask -> device "
                           "(copy stream, prefetched), pgsag_unpack_rgb8, Eq. 9 weights + boundary band, A0-A8 + "
                           "L_rgb + L_ban + L_GC-load + L_s/Adam, loss terms -> host; Gaussians and optimiser state "
                           "are resident model state"}
        del tr, gt_

    # ------------------------------------------------------------- CPU oracle baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v0 = views[0]
        n_s = 1024 if args.config in ("c4", "c3", "c5") else 4096
        mnp = masks[v0].cpu().numpy()
        p, t = oracle_sample(g_np, cams[v0], mnp, n_s)
        cpu = {"value": p / 1e6 / t, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{p} sampled masked pixels of view {v0}, fwd+bwd, single thread, incl. full-scene "
                         f"projection ({t:.1f} s)"}
        if not args.no_cpu_parallel:
            procs = max(1, min(os.cpu_count() or 1, 64))
            pp, tw = oracle_sample_parallel(g_np, cams[v0], mnp, n_s // 2, procs, seed=1)
            cpu["whole_host"] = {"value": pp / 1e6 / tw, "unit": UNIT, "cores": procs, "kind": "oracle",
                                 "sample": f"{procs} forked oracle processes x {n_s // 2} disjoint sampled pixels "
                                           f"({pp} total, wall {tw:.1f} s, each incl. its full-scene projection)"}

    if rank == 0:
        st0 = per_view[views[0]]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wname, "views_per_step": 1, "timed_views": views,
                       "l2": "inputs larger than L2 (Gaussians 1.5M x 236 B = 354 MB per rank, new view each step)",
                       "sh_degree": g.sh_degree, "n_gaussians": g.n, "image": [W, H]},
            "blends_per_s": blends_all / (ms_max / 1e3),
            "masked_pixels_per_step": pix_all / args.steps,
            "tile_imbalance_max_over_mean": imbalance,
            "tile_entries_p50_p99_max": tile_entries,
            "M_per_view": st0["M"], "evaluated_per_view": st0["evaluated"], "blended_per_view": st0["blended"],
            "bwd_visited_per_view": st0["bwd_visited"],
            "flop_per_unit": {"evaluated": FLOP_EVAL, "blended_fwd": FLOP_BLEND_FWD, "blended_bwd": FLOP_BLEND_BWD},
            "roofline": roof, "rooflines_all_kernels": rooflines_all, "cpu_baseline": cpu, "e2e": e2e, "e2e_raster": e2e_raster, "gpu_launches": launches,
            "train_step": train,
            "kernels_ms_per_step": {k: round(v[0], 4) for k, v in sorted(ksteps.items())},
            "kernels_split_source": "untimed pass over the same views with every kernel event-bracketed; inside "
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

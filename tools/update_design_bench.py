"""Regenerate DESIGN.md section 13.0's headline paragraph and tables from profiles/r02_bench_c4.json."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "profiles/r02_bench_c4.json")))
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
i = s.index("### 13.0 Round 2")
k = s.index("| kernel | roof | achieved | fraction |", i)
k2 = s.index("\n\n", k)
rows = "\n".join(f"| {n} | {v:.4f} |" for n, v in sorted(d["kernels_ms_per_view"].items(), key=lambda kv: -kv[1]))
ra = d["rooflines_all_kernels"]
rr = "\n".join(
    f"| {n} | {v['bound']} | {v.get('achieved_gbs', v.get('achieved_tinst'))} "
    f"{'GB/s' if v['bound'] == 'hbm' else 'T inst/s'} | {100 * v['frac']:.1f} % |" for n, v in ra.items())
cb = d["cpu_baseline"]
head = f"""### 13.0 Round 2 (`profiles/r02_bench_c4.json`, default `python bench.py`, final build)

C4 workload as SURVEY §8(d) defines it: one step = one view of each of the 8 sub-regions (1.5 M Gaussians each,
5472×3648 oblique views, ray-cast building masks), {d['steps']} timed steps after {d['warmup']} warm-up steps,
SM clock {d['clocks']['sm_mhz']:.0f} MHz (max {d['clocks']['sm_max_mhz']:.0f}), throttle reasons {d['clocks']['reasons']}.

- `value` = **{d['value']:.0f} masked Mpix/s** fwd+bwd ({d['ms_per_step']:.2f} ms per 8-view step, {d['masked_pixels_per_step'] / 8 / 1e6:.2f} M mask
  pixels per view on average, {d['blends_per_s'] / 1e9:.0f}·10⁹ blends/s); {d['gpu_launches']} kernel launches in the timed region; per-step
  p10/p50/p90 = {d['step_ms_p10_p50_p90']} ms.  (Round 1 reported 1807 Mpix/s on one sub-region's views; the
  round-2 step is the 8-region step of SURVEY §8(d).)
- Dominant kernel A7: {d['roofline']['achieved']:.2f} T FP32 lane-instr/s = **{100 * d['roofline']['frac']:.1f} %** of the §8(d) peak
  ({d['roofline']['peak']:.2f} T/s); by the flop convention {d['roofline_flops']['achieved']:.2f} TFLOP/s = {100 * d['roofline_flops']['frac']:.1f} % of 74.45.
  Share of the step {100 * d['roofline']['share_of_step']:.0f} %.
- `e2e` (training iterations through `Trainer.step_photo` with the 8-bit photo and mask copied from pinned
  host memory each step) = {d['e2e']['value']:.0f} Mpix/s; `train_step` = {d['train_step']['ms_per_iter']:.2f} ms per view;
  `e2e_raster` (every rasterizer input from the host, PCIe-bound) = {d['e2e_raster']['value']:.0f} Mpix/s.
- `cpu_baseline` (the oracle, one core of "{cb['cpu_model']}") = {cb['value']:.2e} Mpix/s; full-frame
  extrapolation {cb['full_frame_extrapolated_s'] / 3600:.0f} h per view; C1 full frame {cb['c1_full_frame']['seconds'] * 1e3:.1f} ms;
  whole host ({cb['whole_host']['cores']} processes) = {cb['whole_host']['value']:.2e} Mpix/s.
- Other configs: `profiles/r02_bench_other_configs.json`.

| kernel (per view) | ms |
|---|---|
{rows}

| kernel | roof | achieved | fraction |
|---|---|---|---|
{rr}"""
s = s[:i] + head + s[k2:]
open(p, "w").write(s)
print("DESIGN.md 13.0 updated:", round(d["value"]), "Mpix/s")

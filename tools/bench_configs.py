"""Run bench.py on the non-headline configs (C2, C3, C5) and write gpurun_out/<tag>_bench_other_configs.json (copied to profiles/ by hand)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = []
for cfg in ("c2", "c3", "c5"):
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "5", "--warmup", "3", "--no-cpu",
                        "--no-e2e"], cwd=ROOT, capture_output=True, text=True)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    out.append({"config": cfg, "workload": d["config"]["workload"], "value_mpix_s": round(d["value"], 1),
                "ms_per_view": round(d["ms_per_step"] / d["config"].get("views_per_step", 1), 3),
                "tile_entries_p50_p99_max": d.get("tile_entries_p50_p99_max"),
                "tile_imbalance_max_over_mean": d.get("tile_imbalance_max_over_mean"),
                "M_per_view": d.get("M_per_view"), "blended_per_view": d.get("blended_per_view"),
                "kernels_ms_per_view": d.get("kernels_ms_per_view"),
                "roofline": {k: d["roofline"][k] for k in ("kernel", "achieved", "peak", "unit", "frac")},
                "train_ms_per_iter": (d.get("train_step") or {}).get("ms_per_iter"), "clocks": d.get("clocks")})
    print(cfg, out[-1]["value_mpix_s"], out[-1]["ms_per_view"], round(out[-1]["roofline"]["frac"], 3), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"{tag}_bench_other_configs.json"), "w"), indent=1)

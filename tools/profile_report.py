"""Write profiles/<tag>_launches.md (ncu per-launch device times of OUR kernels, grouped)
and profiles/<tag>_ncu.md (key counters of the full captures) from gpurun_out/ files."""
import collections, csv, io, subprocess, sys

STAGE = {"tilemask_count_kernel": "A0", "tilemask_prefix_kernel": "A0", "tilemask_list_kernel": "A0",
         "tilemask_satcol_kernel": "A0", "preprocess_kernel": "A1", "scan_kernel": "A2",
         "duplicate_kernel": "A3", "radix_hist_kernel": "A4", "radix_pass_kernel": "A4",
         "ranges_kernel": "A5", "lpt_class_kernel": "A5", "lpt_scatter_kernel": "A5", "render_fwd_kernel": "A6",
         "gc_finalize_kernel": "N1", "render_bwd_kernel": "A7", "preprocess_bwd_kernel": "A8",
         "finite_check_kernel": "A1", "adam_init_kernel": "N3", "loss_total_kernel": "N3",
         "sobel_kernel": "N1", "gc_normalize_kernel": "N1", "band_kernel": "N2", "band_tiled_kernel": "N2", "ban_kernel": "N2", "rgb_fwd_kernel": "N3", "rgb_bwd_kernel": "N3", "rgb_finalize_kernel": "N3",
         "adam_kernel": "N3", "unpack_rgb8_kernel": "N3", "densify_classify_kernel": "N3", "densify_scan_kernel": "N3",
         "densify_apply_kernel": "N3", "opacity_reset_kernel": "N3"}
OURS = tuple(STAGE)


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        nm = next((o for o in OURS if o in r[ki]), None)
        if not nm:
            continue
        v = float(r[vi].replace(',', ''))
        u = r[ui]
        us = v / 1e3 if u in ('nsecond', 'ns') else v * 1e3 if u in ('msecond', 'ms') else v
        tot[nm] += us
        cnt[nm] += 1
    out = []
    for title, pick in (("Rasterizer path A0-A8 (the bench step)", lambda k: STAGE[k][0] == "A"),
                        ("NEXT rows (training iteration kernels)", lambda k: STAGE[k][0] == "N")):
        sel = {k: v for k, v in tot.items() if pick(k)}
        T = sum(sel.values()) or 1.0
        out += [f"\n#### {title}\n", "| stage | kernel | launches | total us | share of the group |",
                "|---|---|---|---|---|"]
        for k, v in sorted(sel.items(), key=lambda kv: -kv[1]):
            out.append(f"| {STAGE[k]} | `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


def ncu(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    keys = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
            'smsp__thread_inst_executed_per_inst_executed.ratio', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
    res = []
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')].split('(')[0].replace('void ', '').replace('unnamed>::', '')
        res.append(f"### `{name}`\n")
        res.append("| metric | value | unit |\n|---|---|---|")
        for k in keys:
            if k in hdr:
                res.append(f"| {k} | {r[hdr.index(k)]} | {units[hdr.index(k)]} |")
        st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_')
              and h.endswith('_per_issue_active.ratio')]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:6]
        res.append("\nTop stall reasons (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
            f"{float(v):.2f}" for h, v in st) + "\n")
    return "\n".join(res)


if __name__ == "__main__":
    tag, launch_csv, rep, cmd = sys.argv[1:5]
    open(f"profiles/{tag}_launches.md", "w").write(
        f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\nCommand: `{cmd}`\n\n"
        "Per-launch times are cold-cache and serialised (ncu); compare SHARES with the bench's live CUDA-event "
        "split (`kernels_ms_per_step`), not absolutes.\n\n" + launches(launch_csv, 2) + "\n")
    open(f"profiles/{tag}_ncu.md", "w").write(
        f"# {tag}: ncu --set full captures (C4 view)\n\nCommand: `{sys.argv[5] if len(sys.argv) > 5 else cmd}`\n\n"
        + "\n".join(ncu(x) for x in rep.split(",")) + "\n")
    print("ok")

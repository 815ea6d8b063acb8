"""Markdown table of an ncu --set full report: per kernel launch, duration, DRAM bytes read / written,
DRAM throughput (% of peak), achieved DRAM GB/s, issue-active, warps-active and the top stall reasons.

    python tools/ncu_table.py report.ncu-rep [--peak-gbs 6543.7] > profiles/rNN_ncu_x.md
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--peak-gbs", type=float, default=6543.7)
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    col = lambda r, k: r[hdr.index(k)] if k in hdr else ""
    def num(r, k, scale=1.0):
        v = col(r, k).replace(",", "")
        return float(v) * scale if v else float("nan")
    uscale = lambda k, want: {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
                              "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(units[hdr.index(k)], 1.0)
    print("| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM GB/s | % of measured HBM peak | "
          "gpu__dram_throughput % | issue-active % | warps-active % | top stalls (warps/issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for i, r in enumerate(rows):
        name = col(r, "Kernel Name").split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        t = num(r, "gpu__time_duration.sum", uscale("gpu__time_duration.sum", "s"))
        rd = num(r, "dram__bytes_read.sum", uscale("dram__bytes_read.sum", "B"))
        wr = num(r, "dram__bytes_write.sum", uscale("dram__bytes_write.sum", "B"))
        gbs = (rd + wr) / t / 1e9
        st = [(h, col(r, h)) for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio")]
        st = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(v or 0)) for h, v in st), key=lambda x: -x[1])[:3]
        print(f"| {i} | `{name}` | {t * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} | "
              f"{100 * gbs / a.peak_gbs:.1f} | {num(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{num(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{num(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              + ", ".join(f"{k} {v:.2f}" for k, v in st) + " |")


if __name__ == "__main__":
    main()

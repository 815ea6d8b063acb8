"""Summarise an ncu report: key throughput metrics, stall reasons, and hot SASS blocks per kernel."""
import csv, collections, subprocess, sys, io

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_requests_srcunit_tex_op_red.sum',
        'sm__sass_thread_inst_executed_op_ffma_pred_on.sum', 'sm__sass_thread_inst_executed_op_fadd_pred_on.sum',
        'sm__sass_thread_inst_executed_op_fmul_pred_on.sum']

def main(rep, sass_for=None):
    hdr, units, rows = raw(rep)
    for r in rows:
        name = r[hdr.index('Kernel Name')]
        print('=====', name[:70])
        for k in KEYS:
            if k in hdr:
                print(f'   {k:70s} {r[hdr.index(k)]:>18s} {units[hdr.index(k)]}')
        st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:7]
        print('   stalls:', ', '.join(f"{h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={float(v):.2f}" for h, v in st))
    if sass_for:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                              f"regex:{sass_for}"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = rows[1]
        ie = hdr.index('Instructions Executed'); isrc = hdr.index('Source')
        data = [(r[isrc].strip(), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]
        tot = sum(e for _, e in data)
        blocks = collections.OrderedDict()
        for s, e in data:
            if e:
                op = s.split()[1] if s.startswith('@') else s.split()[0]
                blocks.setdefault(e, []).append(op)
        print(f'   SASS {sass_for}: total {tot}')
        for e, ins in sorted(blocks.items(), key=lambda kv: -kv[0] * len(kv[1]))[:8]:
            c = collections.Counter(ins)
            print(f"     exec {e:>11d} x{len(ins):3d} = {e*len(ins)/tot*100:5.1f}%  ", dict(c.most_common(9)))

if __name__ == '__main__':
    main(sys.argv[1], *(sys.argv[2:3]))

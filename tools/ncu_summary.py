"""Summarise an ncu --set full report (read here, no GPU needed)."""
import csv, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg.per_second', 'smsp__cycles_active.avg',
        'smsp__sass_thread_inst_executed_op_ffma_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_fmul_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_fadd_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum',
        'dram__bytes_write.sum.per_second']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')][:90]
        print(f'== {name}')
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f'  {w:70s} {vals[i]:>16s} {units[i]}')
        stall = [(h, vals[i]) for i, h in enumerate(hdr)
                 if h.startswith('smsp__average_warp_latency_issue_stalled') or
                 (h.startswith('smsp__warps_issue_stalled_') and h.endswith('_per_warp_active.pct'))]
        for h, v in sorted(stall, key=lambda x: -float(x[1] or 0))[:8]:
            print(f'  {h:70s} {v:>16s}')


if __name__ == '__main__':
    main(sys.argv[1])

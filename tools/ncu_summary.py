"""Summarise an ncu report (raw page): per launch duration, pipes, issue, stalls, DRAM bytes."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'sm__cycles_elapsed.avg.per_second']


def main(path, nlaunch=4):
    # a .ncu-rep, or its raw page already exported (ncu -i ... --page raw --csv > x.csv)
    out = open(path).read() if path.endswith('.csv') else subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    for row in r[2:2 + nlaunch]:
        print('---', row[hdr.index('Kernel Name')][:70])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print('   %-70s %s %s' % (k, row[i], units[i]))
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
                try:
                    st.append((float(row[i]), h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
                except ValueError:
                    pass
        print('   stalls/issue:', ', '.join('%s %.2f' % (n, v) for v, n in sorted(st, reverse=True)[:8]))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4)

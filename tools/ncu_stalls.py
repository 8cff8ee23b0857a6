"""Stall-reason breakdown + pipe utilisation per launch from an ncu report (raw page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio']
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')][:60]
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
            try:
                st[h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]] = float(r[i])
            except ValueError:
                pass
    print(name)
    print('   stalls:', ', '.join(f'{k} {v:.2f}' for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    for k in KEYS:
        if k in hdr:
            print(f'   {k} = {r[hdr.index(k)]} {rows[1][hdr.index(k)]}')

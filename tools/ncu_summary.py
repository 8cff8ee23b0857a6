"""Summarise an ncu report (details page) into key metrics per kernel launch."""
import csv
import subprocess
import sys

WANT = ['Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible', 'Waves Per SM', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block', 'Block Limit Shared Mem',
        'Block Limit Registers', 'One or More Eligible', 'Active Warps Per Scheduler', 'Eligible Warps Per Scheduler']

rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(x) for x in ['Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'])
cur = None
for row in rows[1:]:
    if row[ii] != cur:
        cur = row[ii]
        print(f"== launch {cur}: {row[ki][:90]}")
    if any(row[mi].startswith(w) for w in WANT):
        print(f"   {row[mi]} = {row[vi]} {row[ui]}")

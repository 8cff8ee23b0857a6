"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel + grid."""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
agg = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    key = (r[ki].split('(')[0][:48], r[gi])
    agg.setdefault(key, []).append(float(r[vi].replace(',', '')) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):6d} x {sum(v) / len(v):9.1f} us  {sum(v) / tot * 100:5.1f}%  {k[0]} {k[1]}")

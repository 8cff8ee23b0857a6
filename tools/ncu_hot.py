"""Top SASS instructions by warp-stall samples for the first launch of a kernel in an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', f'regex:{kern}',
                      '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == 'Kernel Name':
        break
    data.append(r)
si = hdr.index('Warp Stall Sampling (All Samples)')
tot = sum(int(r[si] or 0) for r in data)
top = sorted(range(len(data)), key=lambda i: -int(data[i][si] or 0))[:n]
for i in sorted(top):
    print(f"{i:5d} {int(data[i][si]) / tot * 100:5.1f}%  {data[i][1].strip()[:90]}")
print('total samples', tot, 'instructions', len(data))

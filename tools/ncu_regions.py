"""Warp-stall samples of one kernel aggregated over SASS index windows (phase
attribution), with the top stall reasons per window."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
win = int(sys.argv[3]) if len(sys.argv) > 3 else 200
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
reasons = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
num = lambda x: float(x) if x not in ('', None) else 0.0  # noqa: E731
tot = sum(num(r[si]) for r in data)
for a in range(0, len(data), win):
    seg = data[a:a + win]
    s = sum(num(r[si]) for r in seg)
    rs = {hdr[i][6:]: sum(num(r[i]) for r in seg) for i in reasons}
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:4]
    print(f"{a:5d}-{a + len(seg) - 1:5d} {s / tot * 100:5.1f}%  " +
          " ".join(f"{k}:{v / tot * 100:.1f}" for k, v in top))
print('total samples', int(tot), 'instructions', len(data))

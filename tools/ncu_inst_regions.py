"""Dynamic warp-instruction counts of one kernel per SASS window, split into
FP64 / shared / global / other (from the ncu source page)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
win = int(sys.argv[3]) if len(sys.argv) > 3 else 500
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', f'regex:{kern}',
                      '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == 'Kernel Name':
        break
    data.append(r)
ie = hdr.index('Instructions Executed')
num = lambda x: float(x) if x not in ('', None) else 0.0  # noqa: E731


def cls(src):
    t = src.strip().split()
    if not t:
        return 'other'
    op = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
    op = op.split('.')[0]
    if op in ('DFMA', 'DADD', 'DMUL'):
        return 'fp64'
    if op in ('LDS', 'STS', 'LDSM'):
        return 'smem'
    if op in ('LDG', 'STG', 'LDGSTS', 'LD', 'ST', 'CCTL'):
        return 'gmem'
    return 'other'


tot = {}
for a in range(0, len(data), win):
    seg = data[a:a + win]
    c = {}
    for r in seg:
        k = cls(r[1])
        c[k] = c.get(k, 0) + num(r[ie])
        tot[k] = tot.get(k, 0) + num(r[ie])
    s = sum(c.values())
    print(f"{a:5d}-{a + len(seg) - 1:5d} {s / 1e6:7.2f}M  " + " ".join(f"{k}:{v / max(s, 1) * 100:.0f}%" for k, v in sorted(c.items())))
s = sum(tot.values())
print(f"total {s / 1e6:.2f}M warp-instr: " + " ".join(f"{k}:{v / s * 100:.1f}%" for k, v in sorted(tot.items())))

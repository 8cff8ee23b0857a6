"""Opcode mix of one kernel launch from an ncu source-page CSV
(`ncu -i rep --page source --csv --print-source sass --launch-skip K --launch-count 1`):
warp instructions, shared-memory wavefronts, global L1 tag requests / sectors
and stall samples per opcode class, per CTA."""
import collections
import csv
import re
import sys

path, ctas = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if len(r) != len(hdr) or r[0] in ('Kernel Name', 'Address'):
        break
    data.append(r)
H = {h: i for i, h in enumerate(hdr)}
num = lambda x: float(x) if x not in ('', None) else 0.0  # noqa: E731
S = 'Warp Stall Sampling (All Samples)'
tot_samp = sum(num(r[H[S]]) for r in data)
ops, wf_sh, wf_id, l1req, sect, samp = (collections.Counter() for _ in range(6))
for r in data:
    src = r[H['Source']].strip()
    m = re.match(r'(@!?U?P\d+\s+)?([A-Z0-9_.]+)', src)
    op = m.group(2) if m else src[:10]
    base = op.split('.')[0]
    key = op if base in ('LDG', 'STG', 'LDS', 'STS', 'LDGSTS', 'LD', 'ST', 'BAR', 'SHFL') else base
    ops[key] += num(r[H['Instructions Executed']])
    wf_sh[key] += num(r[H['L1 Wavefronts Shared']])
    wf_id[key] += num(r[H['L1 Wavefronts Shared Ideal']])
    l1req[key] += num(r[H['L1 Tag Requests Global']])
    sect[key] += num(r[H['L2 Theoretical Sectors Global']])
    samp[key] += num(r[H[S]])
tot = sum(ops.values())
print(f'SASS instrs {len(data)}, warp instr/CTA {tot / ctas:.0f}, samples {tot_samp:.0f}')
print(f"{'op':28s} {'instr/CTA':>10s} {'%':>6s} {'smem wf':>9s} {'ideal':>8s} {'L1 tag':>8s} {'sectors':>9s} {'stall%':>7s}")
for k, v in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
    print(f"{k:28s} {v / ctas:10.1f} {v / tot * 100:6.1f} {wf_sh[k] / ctas:9.1f} {wf_id[k] / ctas:8.1f} "
          f"{l1req[k] / ctas:8.1f} {sect[k] / ctas:9.1f} {samp[k] / tot_samp * 100:7.1f}")
print(f"{'total':28s} {tot / ctas:10.1f} {100:6.1f} {sum(wf_sh.values()) / ctas:9.1f} {sum(wf_id.values()) / ctas:8.1f} "
      f"{sum(l1req.values()) / ctas:8.1f} {sum(sect.values()) / ctas:9.1f}")

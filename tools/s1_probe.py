"""One-vector (PCG-regime) sweep timing at a config: graph-replayed Gram
sweep per stage-step, and the per-kernel event probe (TLM stage + column pass,
ADJ stage + pass) at s = 1, to split kernel time from launch gaps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import api, scenario  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sdv.init(0)
sc = scenario.build(cfg)
prob = sc.problem
tr = prob.linearize(prob.background)
V = api.gaussian_matrix(prob.n, 1, 3)
dV = api.DeviceBuffer(V.nbytes)
dV.upload(V)
dH = api.DeviceBuffer(V.nbytes)
for _ in range(3):
    tr.gram_dev(dV.ptr.value, 1, dH.ptr.value)
prob.synchronize()
a, b = api.Event(), api.Event()
a.record(prob)
for _ in range(3):
    tr.gram_dev(dV.ptr.value, 1, dH.ptr.value)
b.record(prob)
ms = a.elapsed_ms(b) / 3
steps = prob.total_steps
print(f"cfg {cfg} s=1 gram: {ms:.2f} ms, {ms * 1e3 / (8 * steps):.2f} us per stage-step (graph replay)")
ts, tc = tr.probe_stage_kernels(1, 64)
print(f"probe TLM: stage {ts * 1e3:.2f} us, column pass {tc * 1e3:.2f} us (events around each launch)")
ta, tca = tr.probe_adj_stage_kernels(1, 64)
print(f"probe ADJ: stage {ta * 1e3:.2f} us, column pass {tca * 1e3:.2f} us")

"""Steady-state time of small-block Gram sweeps (the PCG / line-search regime,
CUDA-graph replay after the first two calls) on a config grid."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import api, scenario  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
sdv.init(0)
sc = scenario.build(cfg)
prob = sc.problem
tr = prob.linearize(prob.background)
for s in sizes:
    V = api.gaussian_matrix(prob.n, s, 3)
    dV = api.DeviceBuffer(V.nbytes)
    dV.upload(V)
    dH = api.DeviceBuffer(V.nbytes)
    for _ in range(3):
        tr.gram_dev(dV.ptr.value, s, dH.ptr.value)
    prob.synchronize()
    a, b = api.Event(), api.Event()
    reps = 3
    a.record(prob)
    for _ in range(reps):
        tr.gram_dev(dV.ptr.value, s, dH.ptr.value)
    b.record(prob)
    ms = a.elapsed_ms(b) / reps
    print(f"cfg {cfg} s={s}: {ms:.2f} ms per gram, {s / ms * 1e3:.2f} HVP/s, "
          f"{ms * 1e3 / (8 * prob.total_steps):.2f} us per stage-step", flush=True)

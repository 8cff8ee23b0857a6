"""Full-window parity at BASELINE sizes (too slow for the test suite: the CPU oracle needs minutes per
column): config C's Hessian products over its whole assimilation window on the GPU (as the bench sweeps
them: L2-resident sub-blocks on 512^2) against the CPU oracle on a few columns. Usage:
python tools/full_window_parity.py <config> <block width> <col,col,...>"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import oracle_lib as oracle  # noqa: E402
import paper_2401_15758_b200 as sdv  # noqa: E402
from test_gpu_parity import pair, rel  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cols = [int(c) for c in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, s - 1]
sdv.init(0)
osc, prob = pair(oracle, cfg)
print(f"config {cfg}: n = {osc.n}, steps = {prob.total_steps}, block {s}, sub-blocks {prob.sub_blocks(s)}", flush=True)
gtr = prob.linearize(osc.background)
V = oracle.gaussian_matrix(osc.n, s, 71)
W = oracle.gaussian_matrix(osc.m, s, 72)
t = time.time()
Y, HV, Z = gtr.misfit_apply(V), gtr.gram(V), gtr.misfit_adjoint(W)
print(f"GPU block sweeps: {time.time() - t:.1f} s", flush=True)
dot = max(abs(Y[j] @ W[j] - V[j] @ Z[j]) / (np.linalg.norm(V[j]) * np.linalg.norm(W[j])) for j in range(s))
print(f"dot test max |<Av,w> - <v,A^T w>| / (|v||w|) over {s} columns: {dot:.2e}", flush=True)
t = time.time()
otr = osc.linearize(osc.background)
Yo = otr.misfit_apply(V[cols], workers=len(cols))
HVo = otr.misfit_adjoint(Yo, workers=len(cols))
print(f"oracle ({len(cols)} columns, {len(cols)} threads): {time.time() - t:.0f} s", flush=True)
for i, j in enumerate(cols):
    print(f"column {j}: |Y_gpu - Y_oracle|/|Y| = {rel(Y[j], Yo[i]):.2e}, |HV_gpu - HV_oracle|/|HV| = {rel(HV[j], HVo[i]):.2e}",
          flush=True)

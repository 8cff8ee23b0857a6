"""C4 (BVE 256^2) adaptive SingleView GN on an 8-step window, GPU vs the CPU
oracle: PCG counts per GN iteration, final ranks, sketch counters, analysis
distance and wall times. (Too slow for the test suite: the oracle needs
~400 s on 16 threads.)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import oracle_lib as oracle  # noqa: E402
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import api, scenario  # noqa: E402
from test_gpu_parity import pair, rel  # noqa: E402

sdv.init(0)
oracle.lib()
osc, prob = pair(oracle, 4, steps=8, spi=4)
kw = scenario.CONFIGS[4].gn_kwargs()
kw.update(max_gn_iters=2, method=api.SINGLEVIEW)
t = time.time()
ro = osc.gn_solve(method=api.SINGLEVIEW, max_gn_iters=2, workers=16)
to = time.time() - t
t = time.time()
rg = prob.gn_solve(**kw)
tg = time.time() - t
print("oracle pcg", ro["log"][:, 4], "rank", ro["log"][:, 8], "counters", ro["log"][:, 14:16].tolist(), f"{to:.1f}s")
print("gpu    pcg", rg["log"][:, 4], "rank", rg["log"][:, 8], "counters", rg["log"][:, 14:16].tolist(), f"{tg:.1f}s")
print("analysis rel", rel(rg["analysis"], ro["analysis"]))

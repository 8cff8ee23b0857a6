"""One block Gram sweep (TLM + ADJ) on a config grid with a short window, for
launch-list timing under ncu (`--metrics gpu__time_duration.sum`)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import scenario  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = int(sys.argv[2]) if len(sys.argv) > 2 else 110
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sdv.init(0)
spec = scenario.with_window(scenario.CONFIGS[cfg], steps=steps, spi=steps)
sc = scenario.build(spec)
tr = sc.problem.linearize(sc.problem.background)
V = np.random.default_rng(0).standard_normal((s, sc.problem.n))
for _ in range(2):
    tr.gram(V)
print("done")

"""Tiny fused-path Gram sweeps for compute-sanitizer (memcheck / racecheck /
synccheck): one RK4 step on 64^2 (s = 37) and 512^2 (s = 5), TLM + ADJ with the
tile-carry Poisson path, checked against the column-pass path."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import api, scenario  # noqa: E402

sdv.init(0)
cases = [(64, 37), (512, 5)] if len(sys.argv) < 2 else [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
for n, s in cases:
    spec = scenario.ConfigSpec(**{**scenario.CONFIGS[2].__dict__, "name": f"bve-{n}", "n": n, "steps": 2, "spi": 1,
                                  "dt": 0.01 * 128 / n})
    sc = scenario.build(spec)
    tr = sc.problem.linearize(sc.problem.background)
    V = api.gaussian_matrix(sc.problem.n, s, 3)
    os.environ.pop("SDV_NO_FUSE", None)
    H = tr.gram(V)
    os.environ["SDV_NO_FUSE"] = "1"
    H0 = tr.gram(V)
    os.environ.pop("SDV_NO_FUSE", None)
    err = max(np.linalg.norm(H[j] - H0[j]) / np.linalg.norm(H0[j]) for j in range(s))
    print(f"n={n} s={s}: fused vs column path max rel {err:.2e}", flush=True)
    assert err < 1e-12

"""GPU gn_solve vs the oracle GN fixtures (tests/golden/gn_<name>[_alt|_pert].npz):
PCG counts per GN step, analysis / cost differences. usage: python tools/gn_vs_fixture.py c3_w8 [...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2401_15758_b200 as sdv  # noqa: E402
from paper_2401_15758_b200 import scenario  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


sdv.init(0)
for name in sys.argv[1:]:
    z = np.load(os.path.join(G, f"gn_{name}.npz"))
    meta = json.loads(str(z["meta"]))
    cfg = meta["config"]
    import oracle_lib

    osc = oracle_lib.Scenario(cfg, steps=meta["steps"], spi=meta["spi"])
    prob = scenario.from_arrays(scenario.CONFIGS[cfg], osc.indices, osc.values, osc.variances, osc.background,
                                steps=meta["steps"], spi=meta["spi"])
    kw = scenario.CONFIGS[cfg].gn_kwargs()
    kw.update(meta["gn"])
    r = prob.gn_solve(**kw)
    out = {"name": name, "pcg_gpu": r["log"][:, 4].tolist(), "pcg_oracle": z["log"][:, 4].tolist(),
           "analysis_gpu": rel(r["analysis"], z["analysis"]),
           "cost_gpu": float(np.max(np.abs(r["log"][:, 1] - z["log"][:, 1]) / np.abs(z["log"][:, 1]))),
           "eig0_gpu": (float(np.linalg.norm(r["eig0"][:len(z["eig0"])] - z["eig0"]) / np.linalg.norm(z["eig0"]))
                        if len(z["eig0"]) else None),
           "eig0_n": [len(r["eig0"]), len(z["eig0"])],
           "kappa_gpu_oracle": [r["log"][:, 9].tolist(), z["log"][:, 9].tolist()],
           "decisions_equal": bool(np.array_equal(r["log"][:, 7:9], z["log"][:, 7:9])
                                   and np.array_equal(r["log"][:, 14:16], z["log"][:, 14:16]))}
    for suf in ("alt", "pert"):
        p = os.path.join(G, f"gn_{name}_{suf}.npz")
        if os.path.exists(p):
            za = np.load(p)
            out[f"pcg_{suf}"] = za["log"][:, 4].tolist()
            out[f"analysis_{suf}"] = rel(za["analysis"], z["analysis"])
    print(json.dumps(out), flush=True)

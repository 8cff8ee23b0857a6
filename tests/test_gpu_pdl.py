"""Programmatic dependent launch is semantically transparent: every BVE kernel
waits (griddepcontrol.wait) before it touches its predecessor's output, so
sweeps launched with the PDL attribute (default) and without it (SDV_NO_PDL=1,
read once per process, hence the subprocesses) give bitwise the same results
on every path: one-vector small-block sweeps (2-row stage kernels + column
pass, CUDA-graph replay), narrow fused blocks (one lane, graph replay), two
fused lanes, the plain 128^2 path and the nonlinear forward model."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2401_15758_b200 as sdv
from paper_2401_15758_b200 import api, scenario
sdv.init(0)
out = {{}}
for cfg, steps, spi, widths in ((3, 8, 4, (1, 3, 10)), (4, 8, 4, (1, 2, 8)), (2, 8, 4, (1, 5, 20))):
    spec = scenario.with_window(scenario.CONFIGS[cfg], steps=steps, spi=spi)
    sc = scenario.build(spec)
    tr = sc.problem.linearize(sc.problem.background)
    out[f"state{{cfg}}"] = tr.state_at(steps)
    for s in widths:
        V = api.gaussian_matrix(sc.problem.n, s, 91)
        for rep in range(3):  # plain launches, graph capture, graph replay
            out[f"hv{{cfg}}_{{s}}_{{rep}}"] = tr.gram(V)
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, name, env_extra):
    path = str(tmp_path / f"{name}.npz")
    env = dict(os.environ)
    env.pop("SDV_NO_PDL", None)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], check=True, env=env, timeout=600)
    return np.load(path)


@pytest.mark.timeout(900)
def test_pdl_and_plain_launches_bitwise_equal(tmp_path):
    a = _run(tmp_path, "pdl", {})
    b = _run(tmp_path, "nopdl", {"SDV_NO_PDL": "1"})
    assert sorted(a.files) == sorted(b.files) and len(a.files) == 30
    for k in a.files:
        assert np.all(np.isfinite(a[k])), k
        assert np.array_equal(a[k], b[k]), k
    # replays reproduce the plain launches
    for k in a.files:
        if k.endswith("_0"):
            assert np.array_equal(a[k], a[k[:-2] + "_2"]), k

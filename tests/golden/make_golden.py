"""Generate the oracle golden fixtures for the long config-parity cases (row N1).

TEST INFRASTRUCTURE ONLY. The CPU oracle (oracle/, a restatement of the
reference's gn_solve, proj/src/fourdvar.cpp:213-422, and sketches,
proj/src/sketch.cpp:142-564) runs each case once, here, and the result is
committed as tests/golden/gn_<name>.npz; tests/test_gpu_config_parity.py
compares the CUDA path against it on the GPU box, where re-running these
oracle solves (minutes to tens of minutes of serial PCG on the host) would not
fit the test budget. Short cases stay live in the other parity tests.

Usage: ORACLE_THREADS=8 python tests/golden/make_golden.py [case ...]
       ORACLE_BUILD=alt ORACLE_THREADS=8 python tests/golden/make_golden.py [case ...]
The second form runs the oracle's second build (oracle/Makefile ALTFLAGS,
FMA contraction) and writes gn_<name>_alt.npz: the roundoff spread of the
reference algorithm between two valid builds, which bounds the PCG-count and
analysis agreement the GPU can be held to on long CG runs.
       ORACLE_PERTURB=1e-15 ... writes gn_<name>_pert.npz: the same case from a
background perturbed at roundoff level (relative 1e-15), a second measure of how
chaotic the case's PCG counts are.
(ORACLE_THREADS only speeds the oracle up: its threading is bitwise neutral,
tests/test_oracle.py::test_oracle_threading_bitwise_neutral.)
"""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib  # noqa: E402

# name: (config, steps, spi, gn overrides). Modes: 1 SketchPrec, 2 SketchPrecA,
# 3 PrecGamma; methods: 0 RandSVD, 1 Nystrom, 2 SingleView.
CASES = {
    # C1: the config's three methods at k = 50, p = 10 (l = 60; SingleView l2 = 121), full grid and window
    "c1_nystrom": (1, -1, -1, dict(mode=1, method=1, rank=60)),
    "c1_singleview": (1, -1, -1, dict(mode=1, method=2, rank=60, rank2=121)),
    # C2: the config's own solver (Nystrom k = 40, p = 10), full 200-step window, all 5 GN iterations
    "c2_full": (2, -1, -1, dict(mode=1, method=1, rank=50)),
    # C3: the config's own solver (RandSVD k = 100, p = 10: one block of 110 products per sketch) on the full
    # 512^2 grid over an 8-step window (2 observation intervals), 2 GN iterations
    "c3_w8": (3, 8, 4, dict(mode=1, method=0, rank=110, max_gn_iters=2)),
    # C4: the config's adaptive Nystrom (10 by 10 to 100, SketchPrecA with the reuse test) on the full
    # 256^2 grid over a 40-step window (2 intervals), 3 GN iterations so the reuse decision is taken twice
    "c4_w40": (4, 40, 20, dict(mode=2, method=1, rank=10, growth=10, max_rank=100, rank2=201, max_gn_iters=3)),
    # C4's solver on an 8-step window (2 intervals), one GN iteration: the adaptive sketch hits its cap
    "c4_w8": (4, 8, 4, dict(mode=2, method=1, rank=10, growth=10, max_rank=100, rank2=201, max_gn_iters=1)),
    # C4 with adaptive SingleView (the config's other arm), same window, 2 GN iterations
    "c4_w40_sv": (4, 40, 20, dict(mode=2, method=2, rank=10, growth=10, max_rank=100, rank2=201, max_gn_iters=2)),
}


ALT = os.environ.get("ORACLE_BUILD") == "alt"
PERT = os.environ.get("ORACLE_PERTURB")  # e.g. 1e-15: background x (1 + rel g), oracle/src/capi.cpp


def oracle_flags():
    mk = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "Makefile")
    for line in open(mk):
        if line.startswith("ALTFLAGS" if ALT else "CXXFLAGS"):
            return line.split("=", 1)[1].strip()
    return "?"


def run(name):
    cfg, steps, spi, kw = CASES[name]
    osc = oracle_lib.Scenario(cfg, steps=steps, spi=spi)
    workers = os.cpu_count() or 8
    t0 = time.time()
    r = osc.gn_solve(workers=workers, **kw)
    secs = time.time() - t0
    meta = dict(case=name, config=cfg, steps=steps, spi=spi, gn=kw, oracle_seconds=secs, workers=workers,
                oracle_threads=os.environ.get("ORACLE_THREADS", "1"), oracle_cxxflags=oracle_flags(),
                background_perturbation=PERT,
                host=platform.processor() or platform.machine(),
                git=subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                                   cwd=HERE).stdout.strip())
    out = os.path.join(HERE, f"gn_{name}{'_alt' if ALT else ''}{'_pert' if PERT else ''}.npz")
    np.savez_compressed(out, analysis=r["analysis"], log=r["log"], summary=r["summary"], eig0=r["eig0"],
                        meta=json.dumps(meta))
    print(f"{name}: {len(r['log'])} GN iterations, PCG {r['log'][:, 4].astype(int).tolist()}, "
          f"{secs:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        run(name)

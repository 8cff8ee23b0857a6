"""GPU parity of the fused Poisson path (stage kernels with tile-local
y-recurrences + the tile-carry pass, bve_carry), taken by block sweeps wide
enough for 8-row stage tiles. Blocks here are sized to take that path; the
same products through the column-pass path (SDV_NO_FUSE=1) and the CPU
oracle are the references. Tolerances as test_gpu_parity (1e-10 relative
for Hessian products, dot test 1e-10).
"""
import os

import numpy as np
import pytest

from test_gpu_parity import pair, rel

pytestmark = pytest.mark.gpu

# (config, steps, spi, s): s is the smallest block that takes the fused path
# at that grid (8-row tiles fill >= 2 CTAs per SM), plus one wider block.
CASES = [(3, 16, 8, 5), (3, 8, 4, 12), (2, 40, -1, 19), (4, 40, -1, 10), (4, 20, 10, 23)]


def _no_fuse(flag):
    if flag:
        os.environ["SDV_NO_FUSE"] = "1"
    else:
        os.environ.pop("SDV_NO_FUSE", None)


@pytest.mark.parametrize("cfg,steps,spi,s", CASES)
def test_fused_gram_matches_column_path_and_oracle(oracle, sdv, cfg, steps, spi, s):
    osc, prob = pair(oracle, cfg, steps, spi)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, s, 31)
    W = oracle.gaussian_matrix(osc.m, s, 32)
    try:
        _no_fuse(False)
        HV, Y, Z = gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)
        _no_fuse(True)
        HV0, Y0, Z0 = gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)
    finally:
        _no_fuse(False)
    for j in range(s):
        assert rel(HV[j], HV0[j]) <= 1e-12, ("HV vs column path", j)
        assert rel(Y[j], Y0[j]) <= 1e-12, ("Y vs column path", j)
        assert rel(Z[j], Z0[j]) <= 1e-12, ("Z vs column path", j)
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])
    # oracle on the first and last columns (1e-10 relative)
    for j in (0, s - 1):
        Yo = otr.misfit_apply(V[j:j + 1], workers=8)
        assert rel(Y[j], Yo[0]) <= 1e-10, ("Y vs oracle", j)
        assert rel(HV[j], otr.misfit_adjoint(Yo)[0]) <= 1e-10, ("HV vs oracle", j)
        assert rel(Z[j], otr.misfit_adjoint(W[j:j + 1], workers=8)[0]) <= 1e-10, ("Z vs oracle", j)


def test_fused_sub_range_tlm_adj(oracle, sdv):
    """tlm_range/adj_range over sub-ranges on a fused-width block (C3 grid)."""
    osc, prob = pair(oracle, 3, 8, 4)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    X = oracle.gaussian_matrix(osc.n, 6, 5)
    for b, e in [(0, 8), (3, 7), (5, 6)]:
        Tg, Ag = gtr.tlm_range(b, e, X), gtr.adj_range(b, e, X)
        for j in (0, 5):
            assert rel(Tg[j], otr.tlm_range(b, e, X[j])) <= 1e-10, (b, e, j)
            assert rel(Ag[j], otr.adj_range(b, e, X[j])) <= 1e-10, (b, e, j)


@pytest.mark.parametrize("cfg,steps,spi,s", [(2, 40, -1, 1), (2, 20, 10, 3), (4, 20, 10, 1), (4, 40, -1, 4)])
def test_cluster_sweeps_match_block_path_and_oracle(oracle, sdv, cfg, steps, spi, s):
    """Cluster-resident small-block sweeps (bve_cluster.cu, opt-in SDV_CLUSTER)
    vs the block path and the oracle: misfit apply/adjoint and Gram products."""
    osc, prob = pair(oracle, cfg, steps, spi)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, s, 41)
    W = oracle.gaussian_matrix(osc.m, s, 42)
    try:
        os.environ["SDV_CLUSTER"] = "8"
        HV, Y, Z = gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)
        os.environ.pop("SDV_CLUSTER", None)
        HV0, Y0, Z0 = gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)
    finally:
        os.environ.pop("SDV_CLUSTER", None)
    for j in range(s):
        assert rel(HV[j], HV0[j]) <= 1e-12, ("HV vs block path", j)
        assert rel(Y[j], Y0[j]) <= 1e-12, ("Y vs block path", j)
        assert rel(Z[j], Z0[j]) <= 1e-12, ("Z vs block path", j)
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])
    Yo = otr.misfit_apply(V[:1], workers=8)
    assert rel(Y[0], Yo[0]) <= 1e-10
    assert rel(HV[0], otr.misfit_adjoint(Yo)[0]) <= 1e-10
    assert rel(Z[0], otr.misfit_adjoint(W[:1], workers=8)[0]) <= 1e-10


@pytest.mark.parametrize("n,s", [(64, 37), (64, 40), (128, 21), (256, 11), (512, 7)])
def test_fused_vs_column_path_other_grids(sdv, n, s):
    """Fused path on grids without an oracle case (64^2) and on odd block widths
    (two unequal sweep lanes): Gram products equal the column-pass path to 1e-12
    and the misfit pair passes the dot test."""
    from paper_2401_15758_b200 import api, scenario

    spec = scenario.ConfigSpec(**{**scenario.CONFIGS[2].__dict__, "name": f"bve-{n}", "n": n, "steps": 8, "spi": 4,
                                  "dt": 0.01 * 128 / n})
    sc = scenario.build(spec)
    tr = sc.problem.linearize(sc.problem.background)
    V = api.gaussian_matrix(sc.problem.n, s, 51)
    W = api.gaussian_matrix(sc.problem.m, s, 52)
    try:
        _no_fuse(False)
        HV, Y, Z = tr.gram(V), tr.misfit_apply(V), tr.misfit_adjoint(W)
        _no_fuse(True)
        HV0 = tr.gram(V)
    finally:
        _no_fuse(False)
    for j in range(s):
        assert rel(HV[j], HV0[j]) <= 1e-12, j
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])


@pytest.mark.parametrize("n,s", [(64, 37), (256, 12), (512, 5)])
def test_fused_sweeps_bitwise_deterministic(sdv, n, s):
    """Repeated fused-path Gram sweeps are bitwise identical (no shared-memory
    races in the in-place FFTs / per-team barriers, deterministic reductions)."""
    from paper_2401_15758_b200 import api, scenario

    spec = scenario.ConfigSpec(**{**scenario.CONFIGS[2].__dict__, "name": f"bve-{n}", "n": n, "steps": 4, "spi": 2,
                                  "dt": 0.01 * 128 / n})
    sc = scenario.build(spec)
    tr = sc.problem.linearize(sc.problem.background)
    V = api.gaussian_matrix(sc.problem.n, s, 61)
    first = tr.gram(V)
    for _ in range(3):
        assert np.array_equal(tr.gram(V), first)

"""GPU parity for the reference's own barotropic-vorticity preset bve_2
(proj/src/harness.cpp:285-309): 64 x 129 Dirichlet BVE (RK3-TVD, Re 200,
Ro 0.0016, DST Poisson), 16 x 16 sensors, 2-D Laplacian prior (alpha 0,
beta 0.06), truth = the reference's spun-up fixture field. The oracle side is
oracle.Scenario(101), pinned through tests/test_oracle.py's fixture test.
Tolerances as test_gpu_parity.py.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NX, NY, RE, RO, DT, NT, SPI, ALPHA, BETA = 64, 129, 200.0, 0.0016, 0.001225 / 4, 8, 4, 0.0, 0.06


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def pair(oracle, sdv):
    from paper_2401_15758_b200 import api

    osc = oracle.Scenario(101)
    prob = api.Problem(api.MODEL_BVE_DIRICHLET, NX, 0.0, DT, NT, SPI, 0.0, 0.0, osc.indices, osc.values,
                       osc.variances, osc.background, prior_kind=api.PRIOR_LAPLACIAN, prior_alpha=ALPHA,
                       prior_beta=BETA, ny=NY, reynolds=RE, rossby=RO)
    assert (prob.n, prob.m, prob.n_t, prob.spi) == (osc.n, osc.m, osc.n_t, osc.spi)
    return osc, prob


def test_prior_sqrt_parity(oracle, pair):
    osc, prob = pair
    V = oracle.gaussian_matrix(osc.n, 3, 21)
    G = prob.prior_sqrt(V)
    for j in range(3):
        assert rel(G[j], osc.prior_sqrt(V[j])) <= 1e-12


def test_forward_and_linearize_parity(pair):
    osc, prob = pair
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    for i in range(1, osc.n_t + 1):
        assert rel(gtr.state_at(i * osc.spi), otr.state_at(i * osc.spi)) <= 1e-11, i
    assert rel(prob.forward(osc.truth0, 40), osc.forward(osc.truth0, 40)) <= 1e-11


def test_misfit_block_parity_and_dot(oracle, pair):
    osc, prob = pair
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    s = 4
    V = oracle.gaussian_matrix(osc.n, s, 11)
    W = oracle.gaussian_matrix(osc.m, s, 12)
    Yg, Zg = gtr.misfit_apply(V), gtr.misfit_adjoint(W)
    Yo, Zo = otr.misfit_apply(V, workers=8), otr.misfit_adjoint(W, workers=8)
    for j in range(s):
        assert rel(Yg[j], Yo[j]) <= 1e-10, ("Y", j)
        assert rel(Zg[j], Zo[j]) <= 1e-10, ("Z", j)
        assert abs(Yg[j] @ W[j] - V[j] @ Zg[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])
    HV = gtr.gram(V)
    for j in range(s):
        assert rel(HV[j], otr.misfit_adjoint(Yo[j:j + 1])[0]) <= 1e-10


def test_tlm_adj_sub_ranges(oracle, pair):
    osc, prob = pair
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    x = oracle.gaussian_matrix(osc.n, 1, 5)[0]
    T = osc.n_t * osc.spi
    for b, e in [(0, T), (3, 7), (T - 4, T)]:
        assert rel(gtr.tlm_range(b, e, x)[0], otr.tlm_range(b, e, x)) <= 1e-10
        assert rel(gtr.adj_range(b, e, x)[0], otr.adj_range(b, e, x)) <= 1e-10


def test_evaluate_xspace_parity(oracle, pair):
    osc, prob = pair
    x = osc.background + osc.prior_sqrt(0.05 * oracle.gaussian_matrix(osc.n, 1, 3)[0])
    co, go, lo, _ = osc.evaluate(x)
    cg, gg, lg = prob.evaluate(x)
    assert abs(cg - co) <= 1e-12 * abs(co)
    assert rel(gg, go) <= 1e-10
    assert rel(lg, lo) <= 1e-10


def test_sketch_eigenvalue_parity(oracle, pair):
    osc, prob = pair
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    for method in (0, 1, 2):
        eo, _, co = otr.sketch(method, 24, 77, workers=8)
        eg, _, cg = gtr.sketch(method, 24, 77)
        assert tuple(cg) == tuple(co), method
        assert np.linalg.norm(eg - eo[:len(eg)]) / np.linalg.norm(eo) <= 1e-8, method


def test_bve2_gn_parity(oracle, pair):
    """The preset's solver (SketchPrec, RandSVD rank 192, seed mix_seed(1234, 42)), 2 GN iterations."""
    osc, prob = pair
    ro = osc.gn_solve(max_gn_iters=2, workers=8)
    rg = prob.gn_solve(mode=1, method=0, rank=192, growth=64, eps_reuse=50.0, max_gn_iters=2, pcg_max_iter=4000,
                       seed=oracle.mix_seed(1234, 42))
    assert len(rg["log"]) == len(ro["log"]) == 2
    assert np.all(np.abs(rg["log"][:, 4] - ro["log"][:, 4]) <= 1)
    assert rel(rg["analysis"], ro["analysis"]) <= 1e-8
    assert np.array_equal(rg["log"][:, 14:16], ro["log"][:, 14:16])
    assert rg["log"][1][1] < rg["log"][0][1]  # the cost decreases

"""CPU oracle pins (no GPU): the oracle is checked against the reference's own
golden vector and known-answer/property tests before it is trusted as the
parity checker for the CUDA path.

Reference tests restated: proj/tests/test_{linalg,sketching,burgers,bve,fourdvar,harness}.cpp
and the Exp 1.1 acceptance bands of /root/reference/SPEC.md:604.
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_mix_seed_matches_fixture_seed(oracle):
    # proj/data/fixtures/bve_truth_64x129_s600_seed4199148429166567583_v1.csv
    assert oracle.mix_seed(1234, 7) == 4199148429166567583


def test_bve_truth_fixture_pin(oracle):
    """Reference golden vector: Dirichlet RK3-TVD BVE spin-up (harness.cpp:119-170, preset bve_2)."""
    golden = np.load(os.path.join(GOLDEN, "bve_truth_64x129_s600.npy"))
    f = oracle.bve_fixture(64, 129, 200.0, 0.0016, 0.001225 / 4.0, 600, oracle.mix_seed(1234, 7))
    assert np.linalg.norm(f - golden) <= 1e-12 * np.linalg.norm(golden)


def test_gaussian_matrix_is_deterministic_and_column_major(oracle):
    a = oracle.gaussian_matrix(7, 3, 5)
    b = oracle.gaussian_matrix(7, 3, 5)
    assert np.array_equal(a, b)
    # one sampler filled column by column: a 21-vector equals the flattened block
    v = oracle.gaussian_matrix(21, 1, 5)[0]
    assert np.array_equal(a.reshape(-1), v)
    big = oracle.gaussian_matrix(200000, 1, 9)[0]
    assert abs(big.mean()) < 0.01 and abs(big.std() - 1.0) < 0.01


def test_exp11_reproduces_paper_table(oracle):
    """Burgers Exp 1.1 (n=399, l=15): SPEC.md:604 bands, exact offline counters."""
    sc = oracle.Scenario(100)
    res = {}
    for name, mode, method in [("PrecGamma", 3, 0), ("RandSVD", 1, 0), ("Nystrom", 1, 1), ("SingleView", 1, 2),
                               ("Lanczos", 4, 0)]:
        r = sc.gn_solve(mode=mode, method=method, workers=8)
        assert len(r["log"]) == 3 and r["summary"][3] == 1, name  # 3 GN iterations, converged
        res[name] = (r["summary"][2], r["log"][-1][14], r["log"][-1][15])
    assert abs(res["PrecGamma"][0] - 44) <= 5
    assert abs(res["Lanczos"][0] - 3) <= 1
    assert abs(res["RandSVD"][0] - 6) <= 3 and res["RandSVD"][1:] == (45, 45)
    assert abs(res["Nystrom"][0] - 6) <= 3 and res["Nystrom"][1:] == (45, 45)
    assert abs(res["SingleView"][0] - 11) <= 4 and res["SingleView"][1:] == (45, 93)


@pytest.mark.parametrize("cfg,steps", [(0, -1), (1, 100), (2, 40), (4, 20)])
def test_config_misfit_dot_test(oracle, cfg, steps):
    """|<Av,w> - <v,A^T w>| <= 1e-10 |v||w| (proj/tests/test_fourdvar.cpp:265-277)."""
    sc = oracle.Scenario(cfg, steps=steps)
    tr = sc.linearize(sc.background)
    rng = np.random.default_rng(cfg)
    V = rng.standard_normal((2, sc.n))
    W = rng.standard_normal((2, sc.m))
    Y = tr.misfit_apply(V, workers=2)
    Z = tr.misfit_adjoint(W, workers=2)
    for j in range(2):
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])


@pytest.mark.parametrize("cfg,steps", [(0, 40), (2, 20)])
def test_config_tlm_matches_central_fd(oracle, cfg, steps):
    """proj/tests/test_burgers.cpp:101-120, test_bve.cpp:141-156."""
    sc = oracle.Scenario(cfg, steps=steps)
    T = sc.n_t * sc.spi
    tr = sc.linearize(sc.background)
    dx = np.random.default_rng(1).standard_normal(sc.n)
    dx /= np.linalg.norm(dx)
    tlm = tr.tlm_range(0, T, dx)
    h = 1e-6
    cen = (sc.forward(sc.background + h * dx, T) - sc.forward(sc.background - h * dx, T)) / (2 * h)
    assert np.linalg.norm(cen - tlm) <= 1e-5 * np.linalg.norm(tlm)


def test_arakawa_conservation_and_antisymmetry(oracle):
    n = 32
    rng = np.random.default_rng(3)
    a, b, c = (rng.standard_normal(n * n) for _ in range(3))
    J = lambda x, y: oracle.bve_op(n, 2, x, y)
    s = np.linalg.norm(a) * np.linalg.norm(b) * 1e-12 * n * n
    assert abs(b @ J(a, b)) <= s  # enstrophy
    assert abs(a @ J(a, b)) <= s  # energy
    assert abs(c @ J(a, b) + b @ J(a, c)) <= s  # J(a,.) antisymmetric


def test_periodic_poisson_inverts_fourier_modes(oracle):
    n = 32
    h = 2 * np.pi / n
    i = np.arange(n)
    for kx, ky in [(1, 0), (3, 2), (5, 7)]:
        mode = np.cos(kx * h * i)[None, :] * np.cos(ky * h * i)[:, None]
        mu = 4 / h ** 2 * (np.sin(np.pi * kx / n) ** 2 + np.sin(np.pi * ky / n) ** 2)
        psi = oracle.bve_op(n, 0, mu * mode.reshape(-1))
        assert np.linalg.norm(psi - mode.reshape(-1)) <= 1e-12 * np.linalg.norm(mode)
    w = np.random.default_rng(0).standard_normal(n * n)
    w -= w.mean()
    lap = oracle.bve_op(n, 1, oracle.bve_op(n, 0, w))
    assert np.linalg.norm(lap + w) <= 1e-10 * np.linalg.norm(w)


def test_woodbury_matches_dense_inverse(oracle):
    """proj/tests/test_linalg.cpp:31-80."""
    rng = np.random.default_rng(4)
    n, l = 30, 6
    V, _ = np.linalg.qr(rng.standard_normal((n, l)))
    lam = np.array([9.0, 4.0, 2.0, 1.0, 0.5, 0.0])
    v = rng.standard_normal(n)
    dense = np.linalg.solve(np.eye(n) + V @ np.diag(lam) @ V.T, v)
    assert np.linalg.norm(oracle.woodbury(V, lam, v) - dense) <= 1e-12 * np.linalg.norm(dense)
    with pytest.raises(ValueError):
        oracle.woodbury(V, lam, np.full(n, np.nan))


def test_pcg_known_answers(oracle):
    """proj/tests/test_linalg.cpp:82-160."""
    rhs = oracle.gaussian_matrix(9, 1, 4)[0]
    x, it, conv = oracle.pcg_dense(np.eye(9), rhs, tol=1e-12, max_iter=10)
    assert conv and it == 1
    d = np.arange(1.0, 11.0)
    x, it, conv = oracle.pcg_dense(np.diag(d), np.ones(10), tol=1e-9, max_iter=50)
    assert conv and it <= 10 and np.linalg.norm(x - 1 / d) <= 1e-8
    rng = np.random.default_rng(5)
    g = rng.standard_normal((15, 9))
    h = g @ g.T + np.eye(15)
    x, it, conv = oracle.pcg_dense(h, rng.standard_normal(15), minv=np.linalg.inv(h), tol=1e-10, max_iter=50)
    assert conv and it == 1
    with pytest.raises(RuntimeError):
        oracle.pcg_dense(np.diag([1.0, -1.0, 2.0]), np.ones(3), tol=1e-10, max_iter=10)
    x, it, conv = oracle.pcg_dense(np.eye(4), np.zeros(4))
    assert conv and it == 0 and not x.any()


def test_thin_qr_sign_convention_and_deficiency(oracle):
    rng = np.random.default_rng(6)
    y = rng.standard_normal((20, 5))
    q, r, nd = oracle.thin_qr(y)
    assert nd == 0
    assert np.all(np.diag(r) >= 0)
    assert np.linalg.norm(q @ r - y) <= 1e-13 * np.linalg.norm(y)
    assert np.linalg.norm(q.T @ q - np.eye(5)) <= 1e-14
    y[:, 3] = y[:, 0] + y[:, 1]
    _, _, nd = oracle.thin_qr(y)
    assert nd == 1


def _with_singular_values(m, n, sigma, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, len(sigma))))
    v, _ = np.linalg.qr(rng.standard_normal((n, len(sigma))))
    return u @ np.diag(sigma) @ v.T


def test_sketches_exact_on_low_rank(oracle):
    """proj/tests/test_sketching.cpp:46-113 (RandSVD 1e-10, Nystrom 1e-6, SingleView 1e-8)."""
    a = _with_singular_values(12, 20, [3.0, 2.0, 1.0, 0.5], 5)
    h = a.T @ a
    sn = np.linalg.norm(h, 2)
    for method, rank, tol in [(0, 8, 1e-10), (1, 6, 1e-6), (2, 9, 1e-8)]:
        eig, basis = oracle.sketch_dense(a, method, rank, 17, rank2=19)
        hat = basis @ np.diag(eig) @ basis.T
        assert np.linalg.norm(h - hat, 2) <= tol * sn, method


def test_oracle_gn_c0_runs_and_decreases_cost(oracle):
    sc = oracle.Scenario(0)
    r = sc.gn_solve(workers=4)
    costs = r["log"][:, 1]
    assert len(costs) == 5 and np.all(np.diff(costs) <= 1e-12 * costs[0])
    err_a = np.linalg.norm(r["analysis"] - sc.truth0)
    err_b = np.linalg.norm(sc.background - sc.truth0)
    assert err_a < 0.1 * err_b


def test_oracle_threading_bitwise_neutral(oracle, tmp_path):
    """ORACLE_THREADS (intra-operator par_for, oracle/src/dense.cpp) never changes a bit: the golden
    fixtures made with it (tests/golden/make_golden.py) equal a serial oracle's results."""
    import subprocess
    import sys

    code = ("import sys, numpy as np; sys.path.insert(0, %r); import oracle_lib as o; "
            "sc = o.Scenario(2, steps=8, spi=4); tr = sc.linearize(sc.background); "
            "np.save(%r, np.concatenate([tr.gram(o.gaussian_matrix(sc.n, 2, 3))[0], "
            "sc.gn_solve(max_gn_iters=1, workers=2)['analysis']]))")
    outs = []
    for th in ("1", "4"):
        f = str(tmp_path / f"o{th}.npy")
        env = dict(os.environ, ORACLE_THREADS=th)
        subprocess.run([sys.executable, "-c", code % (os.path.dirname(os.path.abspath(__file__)), f)], check=True,
                       env=env)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])

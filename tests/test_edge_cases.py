"""Edge cases of the boundary and the CUDA path, after the reference's own
tests: validation errors (proj/src/fourdvar.cpp:25-58), homogeneity
(proj/tests/test_burgers.cpp:122-129), determinism
(proj/tests/test_sketching.cpp:474-490), non-finite detection
(proj/tests/test_burgers.cpp:174-178), worker/group independence
(proj/tests/test_sketching.cpp:463-472)."""
import numpy as np
import pytest


def _args(model=1, n=64, n_t=2, spi=3, idx=(0, 4, 8), var=1e-4):
    idx = np.asarray(idx, np.int64)
    vals = np.zeros((n_t, idx.size))
    variances = np.full((n_t, idx.size), var)
    dim = n if model == 1 else n * n
    return (model, n, 1e-3, 1e-4, n_t, spi, 0.1, 0.05, idx, vals, variances, np.zeros(dim))


@pytest.mark.parametrize("bad,msg", [
    (dict(model=7), "unknown model"),
    (dict(n=100), "power of two"),
    (dict(idx=(0, 4, 4)), "strictly increasing"),
    (dict(idx=(0, 70)), "strictly increasing"),
    (dict(var=0.0), "variances must be positive"),
    (dict(n_t=0), "n_t >= 1"),
])
def test_problem_validation_raises_invalid_argument(bad, msg):
    """No GPU needed: validation precedes any CUDA call (SDV_EINVAL -> ValueError)."""
    from paper_2401_15758_b200 import api

    with pytest.raises(ValueError, match=msg):
        api.Problem(*_args(**bad))


def test_reference_bve_validation():
    """proj/src/bve.cpp BVEModel ctor checks (nx, ny >= 3, Re, Ro > 0) and the prior pairing."""
    from paper_2401_15758_b200 import api

    idx, vals, var = np.array([0, 5]), np.zeros((1, 2)), np.ones((1, 2))
    base = dict(prior_kind=1, prior_alpha=0.0, prior_beta=0.06, ny=9, reynolds=200.0, rossby=0.0016)
    args = (4, 8, 0.0, 1e-3, 1, 2, 0.0, 0.0, idx, vals, var, np.zeros(72))
    for bad, msg in [(dict(ny=2), "BVEModel"), (dict(rossby=0.0), "BVEModel"), (dict(prior_kind=0), "Laplacian")]:
        with pytest.raises(ValueError, match=msg):
            api.Problem(*args, **{**base, **bad})


@pytest.mark.parametrize("model,kind,alpha,beta,n,msg", [
    (3, 0, 0.5, 500.0, 399, "Laplacian prior"),       # Dirichlet Burgers needs the Laplacian prior
    (1, 1, 0.5, 500.0, 64, "Fourier-diagonal"),       # periodic models take the Fourier prior
    (3, 1, 0.0, 0.0, 399, "alpha \\+ beta > 0"),      # proj/src/prior.cpp:11-12
    (3, 1, -1.0, 5.0, 399, "alpha, beta >= 0"),
    (3, 1, 0.5, 500.0, 2, "3 <= n <= 4096"),
])
def test_prior_validation(model, kind, alpha, beta, n, msg):
    from paper_2401_15758_b200 import api

    a = list(_args(model=1, n=n, idx=(0, 1)))
    a[0] = model
    with pytest.raises(ValueError, match=msg):
        api.Problem(*a, prior_kind=kind, prior_alpha=alpha, prior_beta=beta)


@pytest.mark.gpu
def test_tlm_exactly_homogeneous_in_powers_of_two(oracle, sdv):
    from paper_2401_15758_b200 import scenario

    for cfg, steps in [(0, 20), (2, 8)]:
        osc = oracle.Scenario(cfg, steps=steps, spi=4 if cfg == 2 else -1)
        prob = scenario.from_arrays(scenario.CONFIGS[cfg], osc.indices, osc.values, osc.variances, osc.background,
                                    steps=steps, spi=4 if cfg == 2 else None)
        tr = prob.linearize(osc.background)
        dx = oracle.gaussian_matrix(osc.n, 1, 42)
        once = tr.tlm_range(0, steps, dx)
        twice = tr.tlm_range(0, steps, 2.0 * dx)
        assert np.array_equal(twice, 2.0 * once)
        assert not tr.tlm_range(0, steps, np.zeros_like(dx)).any()
        assert not tr.adj_range(0, steps, np.zeros_like(dx)).any()


@pytest.mark.gpu
def test_results_independent_of_group_size_and_bitwise_deterministic(oracle, sdv):
    from paper_2401_15758_b200 import scenario

    osc = oracle.Scenario(2, steps=8, spi=4)
    V = oracle.gaussian_matrix(osc.n, 7, 3)
    outs = []
    for g in (0, 1, 3, 7):
        prob = scenario.from_arrays(scenario.CONFIGS[2], osc.indices, osc.values, osc.variances, osc.background,
                                    block_group=g, steps=8, spi=4)
        outs.append(prob.linearize(osc.background).gram(V))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    prob = scenario.from_arrays(scenario.CONFIGS[2], osc.indices, osc.values, osc.variances, osc.background,
                                steps=8, spi=4)
    tr = prob.linearize(osc.background)
    e1 = tr.sketch(1, 20, 77)[0]
    e2 = tr.sketch(1, 20, 77)[0]
    assert np.array_equal(e1, e2)


@pytest.mark.gpu
def test_block_of_one_and_ragged_blocks(oracle, sdv):
    from paper_2401_15758_b200 import scenario

    osc = oracle.Scenario(2, steps=8, spi=4)
    prob = scenario.from_arrays(scenario.CONFIGS[2], osc.indices, osc.values, osc.variances, osc.background,
                                block_group=4, steps=8, spi=4)
    tr = prob.linearize(osc.background)
    otr = osc.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, 10, 9)  # 10 = 4 + 4 + 2 (ragged last group)
    G = tr.gram(V)
    one = tr.gram(V[3:4])
    assert np.array_equal(one[0], G[3])
    for j in (0, 5, 9):
        ref = otr.gram(V[j:j + 1])[0]
        assert np.linalg.norm(G[j] - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.gpu
def test_nonfinite_state_raises_runtime_error(sdv):
    """Over-CFL forward integration must fail loudly (proj/src/bve.cpp:120-124)."""
    from paper_2401_15758_b200 import api

    n = 64
    x0 = 1e3 * api.gaussian_vector(n * n, 5)
    prob = api.Problem(2, n, 1e-4, 5.0, 2, 20, 0.2, 0.3, np.zeros(0, np.int64), np.zeros(0), np.zeros(0), x0)
    with pytest.raises(sdv.SdvError, match="non-finite"):
        prob.linearize(x0)


@pytest.mark.gpu
@pytest.mark.timeout(120)
def test_problem_destroyed_before_its_trajectories(sdv):
    """Handles are reference-counted (include/sdv.h): a host language whose finalisers run in no particular
    order (Python's cyclic GC, interpreter exit) may destroy a problem before its trajectories; the
    trajectories stay usable and the last one releases the problem."""
    from paper_2401_15758_b200 import api

    prob = api.Problem(*_args(model=1, n=64))
    t1, t2 = prob.linearize(np.zeros(64)), prob.linearize(np.ones(64) * 0.1)
    v = np.ones((2, 64))
    before = t1.tlm_range(0, 3, v)
    prob.close()
    assert np.array_equal(t1.tlm_range(0, 3, v), before)
    t1.close()
    assert np.all(np.isfinite(t2.tlm_range(0, 3, v)))
    t2.close()


@pytest.mark.gpu
def test_step_range_validation(sdv):
    from paper_2401_15758_b200 import api

    n = 64
    prob = api.Problem(1, n, 1e-3, 1e-4, 2, 5, 0.1, 0.05, np.array([0, 8]), np.zeros((2, 2)), np.full((2, 2), 1e-4),
                       np.zeros(n))
    tr = prob.linearize(np.sin(np.arange(n)))
    with pytest.raises(ValueError):
        tr.tlm_range(5, 2, np.ones(n))
    with pytest.raises(ValueError):
        tr.adj_range(0, 11, np.ones(n))
    with pytest.raises(ValueError):
        tr.state_at(11)


def test_reference_format_artifacts(tmp_path):
    """CSV schemas of proj/src/harness.cpp:620-692 (headers, %.17g, CRLF)."""
    import numpy as np

    from paper_2401_15758_b200 import artifacts

    class P:
        n = 8
        obs_indices = np.array([1, 5])
        obs_values = np.array([[0.1, 0.2], [1.0 / 3.0, -2.5]])

    log = np.zeros((2, 16))
    log[0, :] = [0, 10.5, 2.0, 1.0, 7, 1, 1, 1, 12, 3.5, np.nan, 2, 9, 10, 30, 30]
    log[1, :] = [1, 1.25, 0.5, 0.5, 5, 2, 1, 0, 12, np.nan, 1.5, 4, 15, 17, 30, 30]
    res = {"log": log, "summary": np.array([1.0, 0.25, 12, 1, 0])}
    artifacts.write_run(str(tmp_path), "exp", P, res, mode=1, method=0, rank=12)
    obs = open(tmp_path / "observations.csv", "rb").read().decode()
    assert obs.startswith("time_index,component,state_index,value\r\n1,0,1,0.10000000000000001\r\n")
    it = open(tmp_path / "iterations.csv", "rb").read().decode().split("\r\n")
    assert it[0] == ("k,cost,grad_inf_norm,step_size,pcg_iterations,pcg_converged,line_search_trials,"
                     "sketch_recomputed,final_rank,kappa_sk,kappa_re,offline_tlm,offline_adj,fwd,tlm,adj")
    assert it[1] == "0,10.5,2,1,7,true,1,true,12,3.5,nan,30,30,2,9,10"
    sm = open(tmp_path / "summary.csv", "rb").read().decode().split("\r\n")
    assert sm[1] == "exp,gn,SketchPrec,RandSVD,12,8,true,2,12,30,30,4,15,17,1,0.125,ok"

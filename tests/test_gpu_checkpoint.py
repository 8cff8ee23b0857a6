"""Checkpointed trajectories (DynamicalModel::linearize's checkpoint_stride,
proj/include/sketchdav/model.hpp:36-40; the reference's checkpointed Burgers
trajectory, proj/src/burgers.cpp:114-191): states stored every `stride`
steps, one segment of RK stage inputs recomputed at a time inside the sweeps.

The recompute runs the same kernels on the same inputs as the full-store
linearize, so every result must be BITWISE equal to the full-store
trajectory's: state_at (on and between checkpoints), tlm_range / adj_range
across segment boundaries, misfit blocks and Gram blocks (the graph-replayed
small-block path, two-lane fused blocks), for periodic Burgers, the
reference's Dirichlet RK3 Burgers and the periodic BVE (128^2 and 512^2).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _trajs(api, prob, x0, stride):
    full = prob.linearize(x0, policy=api.STORE_FULL)
    ck = prob.linearize(x0, checkpoint_stride=stride, policy=api.STORE_CHECKPOINT)
    fi, ci = full.info(), ck.info()
    assert fi["stride"] == 0 and fi["segments"] == 1
    assert ci["stride"] == min(stride, prob.total_steps)
    assert ci["segments"] == -(-prob.total_steps // ci["stride"])
    if ci["stride"] * 3 <= prob.total_steps:
        assert ci["bytes"] < fi["bytes"]
    return full, ck


def _check_pair(prob, full, ck, stride, blocks, seed=5):
    from paper_2401_15758_b200 import api

    T = prob.total_steps
    steps = sorted({0, T, min(T, stride), min(T, 2 * stride), max(0, stride - 1), min(T, stride + 1), T // 2, T - 1})
    for st in steps:
        assert np.array_equal(ck.state_at(st), full.state_at(st)), f"state_at({st})"
    rng = np.random.default_rng(seed)
    # sub-ranges crossing segment boundaries (and one inside a segment)
    for a, b in [(0, T), (1, min(T, 2 * stride + 1)), (min(T, stride), T), (max(0, stride - 1), min(T, stride))]:
        if a >= b:
            continue
        dx = rng.standard_normal((2, prob.n))
        assert np.array_equal(ck.tlm_range(a, b, dx), full.tlm_range(a, b, dx)), ("tlm", a, b)
        assert np.array_equal(ck.adj_range(a, b, dx), full.adj_range(a, b, dx)), ("adj", a, b)
    for s in blocks:
        V = api.gaussian_matrix(prob.n, s, 7 + s)
        assert np.array_equal(ck.misfit_apply(V), full.misfit_apply(V)), ("misfit", s)
        W = rng.standard_normal((s, prob.m))
        assert np.array_equal(ck.misfit_adjoint(W), full.misfit_adjoint(W)), ("adjoint", s)
        ref = full.gram(V)
        for rep in range(3):  # first use, graph capture, graph replay (s <= 8)
            assert np.array_equal(ck.gram(V), ref), ("gram", s, rep)


@pytest.mark.parametrize("stride", [7, 20, 1000])
def test_checkpoint_burgers_periodic(oracle, sdv, stride):
    from paper_2401_15758_b200 import api
    from test_gpu_parity import pair

    osc, prob = pair(oracle, 0)
    full, ck = _trajs(api, prob, osc.background, stride)
    _check_pair(prob, full, ck, min(stride, prob.total_steps), blocks=[1, 3])


def test_checkpoint_burgers_dirichlet(oracle, sdv):
    """The reference's own Burgers (paper Exp 1.1 preset) with the stride its gn_solve passes,
    steps_per_interval (proj/src/fourdvar.cpp:182), and a ragged stride."""
    from paper_2401_15758_b200 import api
    from test_gpu_dirichlet import ALPHA, BETA, DT, N, NT, NU, SPI

    osc = oracle.Scenario(100)
    prob = api.Problem(api.MODEL_BURGERS_DIRICHLET, N, NU, DT, NT, SPI, 0.0, 0.0, osc.indices, osc.values,
                       osc.variances, osc.background, prior_kind=api.PRIOR_LAPLACIAN, prior_alpha=ALPHA,
                       prior_beta=BETA)
    for stride in (SPI, 333):
        full, ck = _trajs(api, prob, osc.background, stride)
        _check_pair(prob, full, ck, stride, blocks=[2])


@pytest.mark.parametrize("cfg,steps,spi,stride,blocks", [
    (2, 40, 20, 7, [1, 2, 40]),  # 128^2: small-block path (graph replay) and a two-lane fused block (20 + 20)
    (3, 8, 4, 3, [1, 10]),       # 512^2: the hot grid, two fused lanes of 5
])
def test_checkpoint_bve(oracle, sdv, cfg, steps, spi, stride, blocks):
    from paper_2401_15758_b200 import api
    from test_gpu_parity import pair

    osc, prob = pair(oracle, cfg, steps, spi)
    full, ck = _trajs(api, prob, osc.background, stride)
    before = sdv.path_counts()
    _check_pair(prob, full, ck, stride, blocks)
    took = sdv.path_delta(before)
    assert took.get("bve_stage_fused", 0) > 0, took


def test_checkpoint_matches_oracle_and_rejects_bad_stride(oracle, sdv):
    """A checkpointed C2 trajectory's Gram block against the oracle (1e-10), and the argument errors
    (std::invalid_argument <-> ValueError)."""
    from paper_2401_15758_b200 import api
    from test_gpu_parity import pair, rel

    osc, prob = pair(oracle, 2, 20, 10)
    ck = prob.linearize(osc.background, checkpoint_stride=6, policy=api.STORE_CHECKPOINT)
    otr = osc.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, 2, 9)
    HVg = ck.gram(V)
    HVo = otr.gram(V, workers=2)
    for j in range(2):
        assert rel(HVg[j], HVo[j]) <= 1e-10
    with pytest.raises(ValueError):
        prob.linearize(osc.background, checkpoint_stride=0, policy=api.STORE_CHECKPOINT)
    with pytest.raises(ValueError):
        prob.linearize(osc.background, checkpoint_stride=4, policy=7)
    # auto policy on a trajectory that fits HBM: every stage stored
    assert prob.linearize(osc.background, checkpoint_stride=4).info()["stride"] == 0

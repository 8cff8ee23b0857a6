"""GPU first-iterate study (reference first_iterate_study,
proj/src/harness.cpp:529-609) for preset burgers_1_2, against the oracle's
burgers_1_1 scenario (same generation, harness.cpp:432-527): the product-side
scenario arrays, the materialised misfit operator A, and the study's
conditioning numbers recomputed from the oracle's own A and sketches."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def setup(oracle, sdv):
    from paper_2401_15758_b200 import studies

    osc = oracle.Scenario(100)
    prob, truth0, _ = studies.reference_burgers_scenario()
    return osc, prob, studies


def test_reference_scenario_matches_oracle(setup):
    osc, prob, _ = setup
    assert np.array_equal(prob.obs_indices, osc.indices)
    assert rel(prob.obs_values.reshape(-1), np.asarray(osc.values).reshape(-1)) <= 1e-12
    assert rel(prob.background, osc.background) <= 1e-12


def test_materialised_operator_and_study(setup, oracle, tmp_path):
    osc, prob, studies = setup
    otr = osc.linearize(osc.background)
    Ao = otr.misfit_adjoint(np.eye(osc.m), workers=16)
    ho = Ao.T @ Ao
    fi = studies.first_iterate_study(prob, ranks=(5, 15), seeds=2)
    gtr = prob.linearize(prob.background)
    A = gtr.misfit_adjoint(np.eye(prob.m))
    assert rel(A, Ao) <= 1e-10
    w = np.clip(np.linalg.eigvalsh(ho)[::-1], 0.0, None)
    assert abs(fi["kappa_ih"] - (1 + w[0]) / (1 + w[-1])) <= 1e-8 * fi["kappa_ih"]
    gi = studies.gamma_inv_sqrt_1d(osc.n, 0.5, 500.0)
    g = gi @ (np.eye(osc.n) + ho) @ gi
    wg = np.linalg.eigvalsh(0.5 * (g + g.T))
    assert abs(fi["kappa_gn_hessian"] - wg.max() / wg.min()) <= 1e-6 * fi["kappa_gn_hessian"]
    # rows: 3 methods x 2 ranks x 2 seeds + Lanczos x 2 ranks
    assert len(fi["rows"]) == 3 * 2 * 2 + 2
    for r in fi["rows"]:
        assert r["kappa_precond"] >= 1.0 - 1e-12
        assert 0 < r["pcg_iterations"] <= fi["pcg_prec_gamma"] + 1
    # RandSVD seed 0 at rank 15 against the oracle's own sketch on its own H
    from paper_2401_15758_b200 import api

    seed = api.mix_seed(2, studies.K_SCAN_STREAM + 0 * 65536 + 15 * 64 + 0)
    eo, bo, _ = otr.sketch(api.RANDSVD, 15, seed, workers=8)
    ko = studies.split_precond_condition(ho, bo, eo)
    row = next(r for r in fi["rows"] if r["method"] == "RandSVD" and r["rank"] == 15 and r["seed_index"] == 0)
    assert abs(row["kappa_precond"] - ko) <= 1e-6 * ko
    # the larger sketch conditions better
    k5 = next(r for r in fi["rows"] if r["method"] == "RandSVD" and r["rank"] == 5 and r["seed_index"] == 0)
    assert row["kappa_precond"] < k5["kappa_precond"]
    studies.write_first_iterate_artifacts(str(tmp_path), fi)
    lines = open(os.path.join(tmp_path, "first_iterate.csv"), newline="").read().split("\r\n")
    assert lines[0] == "method,rank,seed_index,kappa_precond,pcg_iterations"
    assert lines[1].startswith("PrecGamma,0,0,")
    assert open(os.path.join(tmp_path, "summary.csv")).readline().startswith("experiment,study,n,nu,kappa_ih")

"""GPU parity of the fused Poisson path (stage kernels with tile-local
y-recurrences + the tile-carry pass, bve_carry): the C3 hot path.

A block takes the fused path when its 8-row tiles make >= 128 stage CTAs,
(n/8) * s >= 128 (bve_stage_fill, measured on B200: tools/small_block.py):
blocks of >= 2 / 4 / 8 / 16 vectors at 512^2 / 256^2 / 128^2 / 64^2. It runs as
two concurrent sweep lanes of ceil(s/2) and floor(s/2) vectors once each lane
keeps >= 128 CTAs, i.e. from twice those widths (engine.cu split_lanes). Every
case below ASSERTS the kernel path it took through the per-variant launch
counters (sdv_path_counts). The
references are the column-pass path (SDV_NO_FUSE=1 SDV_NO_LITE=1: unfused
8-row stage kernels + col_solve_kernel, also asserted) and the CPU oracle.
Tolerances as test_gpu_parity (1e-10 relative for Hessian products and the
dot test, 1e-8 for sketch eigenvalues).
"""
import os

import numpy as np
import pytest

from test_gpu_parity import eig_rel, pair, rel

pytestmark = pytest.mark.gpu

# smallest block width that takes the fused path (one lane), per grid size; two lanes from twice that
FUSED_MIN = {64: 16, 128: 8, 256: 4, 512: 2}

# (config, steps, spi, s): the minimum fused widths (one lane, two lanes), odd and wider widths
CASES = [(3, 8, 4, 2), (3, 8, 4, 5), (3, 16, 8, 10), (3, 8, 4, 13), (2, 20, 10, 8), (2, 40, -1, 38), (2, 20, 10, 41),
         (4, 20, 10, 4), (4, 40, -1, 20), (4, 20, 10, 23)]


def _env(column_path):
    for k in ("SDV_NO_FUSE", "SDV_NO_LITE"):
        if column_path:
            os.environ[k] = "1"
        else:
            os.environ.pop(k, None)


def run_paths(sdv, fn, column_path):
    """fn() under the fused (default) or column-pass path; returns (result, path deltas) and asserts the path."""
    _env(column_path)
    try:
        before = sdv.path_counts()
        out = fn()
        took = sdv.path_delta(before)
    finally:
        _env(False)
    if column_path:
        assert fused_launches(took) == 0 and took["bve_stage_lite"] == 0 and took["bve_carry"] == 0, took
        # column pass: recurrence solver, or the 1-column FFT kernel when its CTAs would not fill the SMs
        assert took["bve_stage_plain"] > 0 and took["bve_col_solve"] + took["bve_col_fft"] > 0, took
    else:
        assert fused_launches(took) > 0 and took["bve_carry"] > 0, took
        assert took["bve_stage_lite"] == 0 and took["bve_stage_plain"] == 0, took
    return out, took


def fused_launches(took):
    """Fused-path stage launches (stage_kernel<N, TLM/ADJ, 8, stage, fused>)."""
    return took.get("bve_stage_fused", 0)


def test_fused_min_width_table(sdv):
    """The widths above are the boundary: one vector fewer leaves the block off the fused path, twice the
    width runs two fused lanes."""
    from paper_2401_15758_b200 import api, scenario

    for n, s in FUSED_MIN.items():
        spec = scenario.ConfigSpec(**{**scenario.CONFIGS[2].__dict__, "name": f"bve-{n}", "n": n, "steps": 2,
                                      "spi": 1, "dt": 0.01 * 128 / n})
        sc = scenario.build(spec)
        tr = sc.problem.linearize(sc.problem.background)
        for width, fused_lanes in ((2 * s, 2), (2 * s - 1, 1), (s, 1), (s - 1, 0)):
            V = api.gaussian_matrix(sc.problem.n, width, 3)
            before = sdv.path_counts()
            tr.misfit_apply(V)
            d = sdv.path_delta(before)
            # TLM over 2 RK4 steps: 8 stage launches per lane
            assert fused_launches(d) == 8 * fused_lanes, (n, width, d)


@pytest.mark.parametrize("cfg,steps,spi,s", CASES)
def test_fused_gram_matches_column_path_and_oracle(oracle, sdv, cfg, steps, spi, s):
    osc, prob = pair(oracle, cfg, steps, spi)
    assert s >= FUSED_MIN[osc_n(osc)]
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, s, 31)
    W = oracle.gaussian_matrix(osc.m, s, 32)
    (HV, Y, Z), _ = run_paths(sdv, lambda: (gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)), False)
    (HV0, Y0, Z0), _ = run_paths(sdv, lambda: (gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)), True)
    for j in range(s):
        assert rel(HV[j], HV0[j]) <= 1e-12, ("HV vs column path", j)
        assert rel(Y[j], Y0[j]) <= 1e-12, ("Y vs column path", j)
        assert rel(Z[j], Z0[j]) <= 1e-12, ("Z vs column path", j)
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])
    # oracle on the first and last column of each lane (1e-10 relative)
    a = (s + 1) // 2
    cols = [0, a - 1, a, s - 1]
    Yo = otr.misfit_apply(V[cols], workers=len(cols))
    HVo = otr.misfit_adjoint(Yo, workers=len(cols))
    Zo = otr.misfit_adjoint(W[cols], workers=len(cols))
    for i, j in enumerate(cols):
        assert rel(Y[j], Yo[i]) <= 1e-10, ("Y vs oracle", j)
        assert rel(HV[j], HVo[i]) <= 1e-10, ("HV vs oracle", j)
        assert rel(Z[j], Zo[i]) <= 1e-10, ("Z vs oracle", j)


def osc_n(osc):
    return int(round(np.sqrt(osc.n)))


def test_c3_bench_width_parity(oracle, sdv):
    """C3 at the benchmarked block width s = 110 (the sweep bench.py times: L2-resident sub-blocks, CUDA-graph
    replays), on an 8-step window (2 observation intervals): the first and last column of each lane vs the
    oracle <= 1e-10 for A V, A^T (A V) and A^T W, and the dot test on every column."""
    osc, prob = pair(oracle, 3, 8, 4)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    s = 110
    V = oracle.gaussian_matrix(osc.n, s, 71)
    W = oracle.gaussian_matrix(osc.m, s, 72)
    (HV, Y, Z), took = run_paths(sdv, lambda: (gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)), False)
    # swept as 14 L2-resident sub-blocks of 8 / 7 vectors (two lanes of 4 / 3-4 each); the launch counters see the
    # plain and the captured pass of each graph (replays add to the kernel count only)
    assert prob.sub_blocks(s) == 14 and fused_launches(took) > 0, took
    for j in range(s):
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j]), j
    cols = [0, 7, 8, 55, 103, 109]  # sub-block edges and interior
    Yo = otr.misfit_apply(V[cols], workers=4)
    HVo = otr.misfit_adjoint(Yo, workers=4)
    Zo = otr.misfit_adjoint(W[cols], workers=4)
    for i, j in enumerate(cols):
        assert rel(Y[j], Yo[i]) <= 1e-10, ("Y", j)
        assert rel(HV[j], HVo[i]) <= 1e-10, ("HV", j)
        assert rel(Z[j], Zo[i]) <= 1e-10, ("Z", j)


def test_c3_randsvd_k100_eigenvalues(oracle, sdv):
    """C3's own sketch, RandSVD with k = 100, p = 10 (one block of l = 110 TLM + 110 ADJ sweeps on the fused
    path) on a 4-step window, seeded as gn_solve's first iteration (mix_seed(2, kIterSketchStream)):
    eigenvalues within 1e-8 relative of the oracle's, orthonormal basis, identical apply counts
    (proj/src/sketch.cpp:142-160)."""
    osc, prob = pair(oracle, 3, 4, 2)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    seed = oracle.mix_seed(2, 0x736b6574636800)
    (eg, bg, cg), _ = run_paths(sdv, lambda: gtr.sketch(0, 110, seed), False)
    eo, bo, co = otr.sketch(0, 110, seed, workers=max(2, os.cpu_count() or 2))
    assert tuple(cg) == tuple(co) == (110, 110, 110)
    assert eig_rel(eg, eo) <= 1e-8
    # the leading eigenvalues (the ones a k = 100 preconditioner keeps) individually
    assert np.all(np.abs(eg[:100] - eo[:100]) <= 1e-8 * np.abs(eo[:100]) + 1e-12 * eo[0])
    assert np.linalg.norm(bg @ bg.T - np.eye(110)) <= 1e-8


def test_fused_sub_range_tlm_adj(oracle, sdv):
    """tlm_range/adj_range over sub-ranges on a fused-width block (C3 grid)."""
    osc, prob = pair(oracle, 3, 8, 4)
    otr = osc.linearize(osc.background)
    gtr = prob.linearize(osc.background)
    X = oracle.gaussian_matrix(osc.n, 12, 5)
    for b, e in [(0, 8), (3, 7), (5, 6)]:
        (Tg, Ag), _ = run_paths(sdv, lambda: (gtr.tlm_range(b, e, X), gtr.adj_range(b, e, X)), False)
        for j in (0, 5, 6, 11):
            assert rel(Tg[j], otr.tlm_range(b, e, X[j])) <= 1e-10, (b, e, j)
            assert rel(Ag[j], otr.adj_range(b, e, X[j])) <= 1e-10, (b, e, j)


def _grid_problem(n, steps, spi):
    from paper_2401_15758_b200 import scenario

    spec = scenario.ConfigSpec(**{**scenario.CONFIGS[2].__dict__, "name": f"bve-{n}", "n": n, "steps": steps,
                                  "spi": spi, "dt": 0.01 * 128 / n})
    sc = scenario.build(spec)
    return sc.problem, sc.problem.linearize(sc.problem.background)


@pytest.mark.parametrize("n,s", [(64, 74), (64, 80), (128, 38), (128, 41), (256, 20), (256, 23), (512, 10),
                                 (512, 13)])
def test_fused_vs_column_path_other_grids(sdv, n, s):
    """Fused path on grids without an oracle case (64^2) and on odd block widths
    (two unequal sweep lanes): Gram products equal the column-pass path to 1e-12
    and the misfit pair passes the dot test."""
    from paper_2401_15758_b200 import api

    prob, tr = _grid_problem(n, 8, 4)
    V = api.gaussian_matrix(prob.n, s, 51)
    W = api.gaussian_matrix(prob.m, s, 52)
    (HV, Y, Z), _ = run_paths(sdv, lambda: (tr.gram(V), tr.misfit_apply(V), tr.misfit_adjoint(W)), False)
    HV0, _ = run_paths(sdv, lambda: tr.gram(V), True)
    for j in range(s):
        assert rel(HV[j], HV0[j]) <= 1e-12, j
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * np.linalg.norm(V[j]) * np.linalg.norm(W[j])


@pytest.mark.parametrize("n,s", [(64, 74), (256, 20), (512, 10)])
def test_fused_sweeps_bitwise_deterministic(sdv, n, s):
    """Repeated fused-path Gram sweeps are bitwise identical (no shared-memory
    races in the in-place FFTs / per-team barriers, deterministic reductions)."""
    from paper_2401_15758_b200 import api

    prob, tr = _grid_problem(n, 4, 2)
    V = api.gaussian_matrix(prob.n, s, 61)
    first, _ = run_paths(sdv, lambda: tr.gram(V), False)
    for _ in range(3):
        assert np.array_equal(tr.gram(V), first)


def test_l2_resident_sub_blocks_bitwise(oracle, sdv):
    """A wide 512^2 block is swept as L2-resident sub-blocks (Problem::sub_blocks: 8 vectors each, CUDA-graph
    replays on staging buffers). Gram products, misfit applies and adjoints of a 19-wide block (sub-blocks of
    7 + 6 + 6: plain launches, graph capture, replay) equal the whole-block sweep (block_group forces it) to
    roundoff -- the first stage's column pass of a 3-4 vector lane is the y-FFT kernel, of a 9-10 vector lane the
    recurrence solver: the same operator, different rounding -- are bitwise reproducible across replays, and match
    the oracle on the sub-block edges to 1e-10."""
    osc, prob = pair(oracle, 3, 8, 4)
    _, whole = pair(oracle, 3, 8, 4, block_group=32)
    assert (prob.sub_blocks(110), prob.sub_blocks(32), prob.sub_blocks(19), prob.sub_blocks(16),
            prob.sub_blocks(15)) == (14, 4, 3, 2, 0)
    assert whole.sub_blocks(110) == 0
    _, c4 = pair(oracle, 4, 8, 4)
    assert c4.sub_blocks(100) == 0  # 256^2: the resident width (33) exceeds the graph-replay width
    s = 19
    gtr, wtr = prob.linearize(osc.background), whole.linearize(osc.background)
    V = oracle.gaussian_matrix(osc.n, s, 71)
    W = oracle.gaussian_matrix(osc.m, s, 72)
    before = sdv.path_counts()
    HV, Y, Z = gtr.gram(V), gtr.misfit_apply(V), gtr.misfit_adjoint(W)
    took = sdv.path_delta(before)
    assert took["bve_stage_fused"] > 0 and took["bve_stage_lite"] == 0 and took["bve_stage_plain"] == 0, took
    HVw, Yw, Zw = wtr.gram(V), wtr.misfit_apply(V), wtr.misfit_adjoint(W)
    for j in range(s):
        assert rel(HV[j], HVw[j]) <= 1e-13 and rel(Y[j], Yw[j]) <= 1e-13 and rel(Z[j], Zw[j]) <= 1e-13, j
    # replays of the captured graphs
    assert np.array_equal(HV, gtr.gram(V)) and np.array_equal(Y, gtr.misfit_apply(V))
    cols = [0, 6, 7, 12, 13, 18]
    otr = osc.linearize(osc.background)
    Yo = otr.misfit_apply(V[cols], workers=len(cols))
    HVo = otr.misfit_adjoint(Yo, workers=len(cols))
    for i, j in enumerate(cols):
        assert rel(Y[j], Yo[i]) <= 1e-10 and rel(HV[j], HVo[i]) <= 1e-10, j


@pytest.mark.parametrize("cfg,s", [(3, 16), (4, 10)])
def test_full_window_properties_at_baseline_size(sdv, cfg, s):
    """BASELINE.json's full sizes (C3: 512^2, 800 RK4 steps, swept as L2-resident sub-blocks; C4: 256^2, 400
    steps, its adaptive sketch's block of 10), where the oracle takes minutes per column: size-independent
    properties instead -- the dot test <A v, w> = <v, A^T w> on every column, linearity of the block sweep
    in its columns, H = A^T A symmetric and positive (v_i^T H v_j = v_j^T H v_i, v^T H v = |A v|^2), and
    bitwise reproducibility. (tools/full_window_parity.py runs the oracle itself on a few columns;
    profiles/r2_parity.md has its result.)"""
    from paper_2401_15758_b200 import api, scenario

    sc = scenario.build(cfg)
    prob = sc.problem
    tr = prob.linearize(prob.background)
    V = api.gaussian_matrix(prob.n, s, 81)
    W = api.gaussian_matrix(prob.m, s, 82)
    V[2] = 0.5 * V[0] - 2.0 * V[1]  # a column that is a combination of two others
    Y, Z, HV = tr.misfit_apply(V), tr.misfit_adjoint(W), tr.gram(V)
    nv, nw = np.linalg.norm(V, axis=1), np.linalg.norm(W, axis=1)
    for j in range(s):
        assert abs(Y[j] @ W[j] - V[j] @ Z[j]) <= 1e-10 * nv[j] * nw[j], j
        assert abs(V[j] @ HV[j] - Y[j] @ Y[j]) <= 1e-10 * (Y[j] @ Y[j]), j
    assert rel(Y[2], 0.5 * Y[0] - 2.0 * Y[1]) <= 1e-11
    assert rel(HV[2], 0.5 * HV[0] - 2.0 * HV[1]) <= 1e-11
    G = V @ HV.T
    assert np.max(np.abs(G - G.T)) <= 1e-10 * np.max(np.abs(G))
    assert np.array_equal(tr.gram(V), HV)

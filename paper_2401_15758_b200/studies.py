"""First-iterate conditioning study on the GPU engine: the reference's
first_iterate_study (/root/reference/proj/src/harness.cpp:529-609) for its
Burgers preset burgers_1_2 (harness.cpp:226-251), with the reference-format
CSV artifacts (harness.cpp:694-736).

The study linearises at the background, materialises the misfit operator A
by rows (m adjoint products, one block sweep on the device), forms H = A^T A,
and reports the spectrum of H, kappa(I + H), the condition number of the full
GN Hessian Gamma^{-1/2}(I + H)Gamma^{-1/2}, the unpreconditioned PCG count,
and for every (method, rank, seed) the split-preconditioned condition number
kappa((I+Hhat)^{-1/2}(I+H)(I+Hhat)^{-1/2}) (proj/src/analysis.cpp:92-120)
and the PCG count with the Woodbury preconditioner. Sketches (RandSVD,
Nystrom, SingleView, Lanczos) and PCG run on the device through the model
operator; the reference applies them to the materialised dense A and H, the
same operator up to rounding. The dense n x n algebra (n = 399) is host
numpy, as the reference's is host Eigen.
"""
import math
import os

import numpy as np

from . import api

K_BACKGROUND_STREAM = 2  # harness.cpp:33-37
K_OBS_STREAM = 100
K_SCAN_STREAM = 0x66690000
METHODS = {"RandSVD": api.RANDSVD, "Nystrom": api.NYSTROM, "SingleView": api.SINGLEVIEW, "Lanczos": api.LANCZOS}


def reference_burgers_scenario(n=399, nu=0.1, dt=2.5e-5, n_t=20, spi=400, alpha=0.5, beta=500.0, obs_var=0.01,
                               master=2, block_group=0):
    """Scenario of presets burgers_1_1 / burgers_1_2 (harness.cpp:226-251;
    generation harness.cpp:432-527): Dirichlet RK3-TVD Burgers on n interior
    points, truth sin(pi x), 15 equispaced sensors, obs at the end of each of
    n_t intervals of spi steps, Laplacian prior (alpha I - beta Lap)^{-2},
    background = truth + Gamma^{1/2} xi. Returns (problem, truth0, truth_states)."""
    truth0 = np.sin(np.pi * np.arange(1, n + 1) / (n + 1))
    idx = np.array([int(math.floor(j * (n + 1) / 16.0 + 0.5)) - 1 for j in range(1, 16)], np.int64)
    prior = dict(prior_kind=api.PRIOR_LAPLACIAN, prior_alpha=alpha, prior_beta=beta)
    shell = api.Problem(api.MODEL_BURGERS_DIRICHLET, n, nu, dt, n_t, spi, 0.0, 0.0, np.zeros(0, np.int64),
                        np.zeros(0), np.zeros(0), truth0, **prior)
    states = [truth0]
    x = truth0
    for _ in range(n_t):
        x = shell.forward(x, spi)
        states.append(x)
    values = np.empty((n_t, idx.size))
    for i in range(n_t):
        noise = api.gaussian_vector(idx.size, api.mix_seed(master, K_OBS_STREAM + i))
        values[i] = states[i + 1][idx] + math.sqrt(obs_var) * noise
    background = truth0 + shell.prior_sqrt(api.gaussian_vector(n, api.mix_seed(master, K_BACKGROUND_STREAM)))[0]
    variances = np.full((n_t, idx.size), obs_var)
    prob = api.Problem(api.MODEL_BURGERS_DIRICHLET, n, nu, dt, n_t, spi, 0.0, 0.0, idx, values, variances, background,
                       block_group=block_group, **prior)
    return prob, truth0, states


def gamma_inv_sqrt_1d(n, alpha, beta, stencil_scale=1.0):
    """Dense Gamma^{-1/2} = alpha I + beta s (-Lap_Dirichlet) (proj/src/prior.cpp:64-69)."""
    b = beta * stencil_scale
    return (np.diag(np.full(n, alpha + 2.0 * b)) + np.diag(np.full(n - 1, -b), 1) + np.diag(np.full(n - 1, -b), -1))


def split_precond_condition(h, basis, eig):
    """kappa_2 of (I+Hhat)^{-1/2}(I+H)(I+Hhat)^{-1/2}, Hhat = V diag(eig) V^T
    (proj/src/analysis.cpp:92-120)."""
    n = h.shape[0]
    middle = np.eye(n) + h
    if len(eig):
        V = np.asarray(basis).T  # n x l
        d = 1.0 / np.sqrt(1.0 + np.asarray(eig)) - 1.0
        c = middle @ V
        vc = V.T @ c
        middle = middle + (V * d) @ c.T + (c * d) @ V.T + (V * d) @ vc @ (V * d).T
    w = np.linalg.eigvalsh(0.5 * (middle + middle.T))
    return float(w.max() / w.min())


def first_iterate_study(prob, ranks=(5, 10, 15, 20, 25), methods=("RandSVD", "Nystrom", "SingleView", "Lanczos"),
                        seeds=5, pcg_tol=1e-9, pcg_max_iter=10000, master=2, alpha=0.5, beta=500.0, pcg=True):
    """first_iterate_study (harness.cpp:529-609) at the problem's background."""
    tr = prob.linearize(prob.background)
    _, ctrl_grad, _ = prob.evaluate(prob.background)  # x-space: Gamma^{1/2} g
    A = tr.misfit_adjoint(np.eye(prob.m))  # rows of A (materialize_by_rows, harness.cpp:208-217)
    h = A.T @ A
    n = h.shape[0]
    spectrum = np.clip(np.linalg.eigvalsh(h)[::-1], 0.0, None)
    out = {"h_spectrum": spectrum, "kappa_ih": float((1.0 + spectrum[0]) / (1.0 + spectrum[-1])), "rows": []}
    gi = gamma_inv_sqrt_1d(n, alpha, beta)
    gn = gi @ (np.eye(n) + h) @ gi
    w = np.linalg.eigvalsh(0.5 * (gn + gn.T))
    out["kappa_gn_hessian"] = float(w.max() / w.min())
    rhs = -ctrl_grad
    out["pcg_prec_gamma"] = tr.pcg_solve(rhs, tol=pcg_tol, max_iter=pcg_max_iter)[1] if pcg else 0
    for mi, name in enumerate(methods):
        method = METHODS[name]
        for rank in ranks:
            n_seeds = 1 if method == api.LANCZOS else seeds
            for s in range(n_seeds):
                seed = api.mix_seed(master, K_SCAN_STREAM + mi * 65536 + rank * 64 + s)
                if method == api.LANCZOS:
                    eig, basis, _ = tr.lanczos(rank, rhs)
                else:
                    eig, basis, _ = tr.sketch(method, rank, seed, rank2=2 * rank + 1)
                row = {"method": name, "rank": rank, "seed_index": s,
                       "kappa_precond": split_precond_condition(h, basis, eig), "pcg_iterations": 0}
                if pcg:
                    row["pcg_iterations"] = tr.pcg_solve(rhs, basis, eig, tol=pcg_tol, max_iter=pcg_max_iter)[1]
                out["rows"].append(row)
    return out


def _fmt(v):
    from .artifacts import fmt

    return fmt(v)


def write_first_iterate_artifacts(out_dir, fi, experiment="burgers_1_2", n=399, nu=0.1):
    """first_iterate.csv, spectrum.csv, summary.csv (harness.cpp:694-736)."""
    os.makedirs(out_dir, exist_ok=True)
    lines = ["method,rank,seed_index,kappa_precond,pcg_iterations",
             f"PrecGamma,0,0,{_fmt(fi['kappa_ih'])},{fi['pcg_prec_gamma']}"]
    lines += [f"{r['method']},{r['rank']},{r['seed_index']},{_fmt(r['kappa_precond'])},{r['pcg_iterations']}"
              for r in fi["rows"]]
    with open(os.path.join(out_dir, "first_iterate.csv"), "w", newline="") as f:
        f.write("\r\n".join(lines) + "\r\n")
    spec = ["index,eigenvalue"] + [f"{i + 1},{_fmt(v)}" for i, v in enumerate(fi["h_spectrum"])]
    with open(os.path.join(out_dir, "spectrum.csv"), "w", newline="") as f:
        f.write("\r\n".join(spec) + "\r\n")
    summ = ["experiment,study,n,nu,kappa_ih,kappa_gn_hessian,pcg_prec_gamma,status",
            f"{experiment},first_iterate,{n},{_fmt(nu)},{_fmt(fi['kappa_ih'])},{_fmt(fi['kappa_gn_hessian'])},"
            f"{fi['pcg_prec_gamma']},ok"]
    with open(os.path.join(out_dir, "summary.csv"), "w", newline="") as f:
        f.write("\r\n".join(summ) + "\r\n")


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser(description="first-iterate study of preset burgers_1_2 on the GPU")
    ap.add_argument("--out", default="runs/burgers_1_2")
    ap.add_argument("--seeds", type=int, default=5)
    args = ap.parse_args()
    api.init(0)
    prob, _, _ = reference_burgers_scenario()
    fi = first_iterate_study(prob, seeds=args.seeds)
    write_first_iterate_artifacts(args.out, fi)
    print(f"kappa(I+H) {fi['kappa_ih']:.6g}, kappa(GN Hessian) {fi['kappa_gn_hessian']:.6g}, "
          f"PCG (Prec_Gamma) {fi['pcg_prec_gamma']}, {len(fi['rows'])} sketch rows -> {args.out}")

"""Reference-format CSV artifacts of a GN run (schemas of
proj/src/harness.cpp:620-740), so GPU runs diff against the reference's own
artifacts: observations.csv, iterations.csv, summary.csv.

Doubles are written as ``%.17g`` (format_csv_double, harness.cpp:184-188),
booleans as true/false (bool_str, :180), lines end in CRLF.
"""
import math
import os

from .api import MODES

MODE_NAMES = {v: k for k, v in MODES.items()}
METHOD_NAMES = {0: "RandSVD", 1: "Nystrom", 2: "SingleView", 3: "Lanczos"}


def fmt(v):
    """format_csv_double: printf("%.17g")."""
    v = float(v)
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def _b(x):
    return "true" if bool(x) else "false"


def _write(path, lines):
    with open(path, "wb") as f:
        f.write("".join(line + "\r\n" for line in lines).encode())


def write_observations_csv(out_dir, indices, values):
    """harness.cpp:620-632. values: [n_t][n_obs] (time-major)."""
    lines = ["time_index,component,state_index,value"]
    for i, row in enumerate(values):
        for k, idx in enumerate(indices):
            lines.append(f"{i + 1},{k},{int(idx)},{fmt(row[k])}")
    _write(os.path.join(out_dir, "observations.csv"), lines)


def write_iterations_csv(out_dir, result):
    """harness.cpp:634-654. result: Problem.gn_solve() dict (log rows of 16)."""
    lines = ["k,cost,grad_inf_norm,step_size,pcg_iterations,pcg_converged,line_search_trials,sketch_recomputed,"
             "final_rank,kappa_sk,kappa_re,offline_tlm,offline_adj,fwd,tlm,adj"]
    for r in result["log"]:
        lines.append(",".join([str(int(r[0])), fmt(r[1]), fmt(r[2]), fmt(r[3]), str(int(r[4])), _b(r[6]),
                               str(int(r[5])), _b(r[7]), str(int(r[8])), fmt(r[9]), fmt(r[10]), str(int(r[14])),
                               str(int(r[15])), str(int(r[11])), str(int(r[12])), str(int(r[13]))]))
    _write(os.path.join(out_dir, "iterations.csv"), lines)


def write_summary_csv(out_dir, experiment, study, mode, method, rank, state_dim, result, status="ok"):
    """harness.cpp:671-692."""
    log = result["log"]
    s = result["summary"]  # final_cost, final_grad_inf_norm, total_pcg, converged, line_search_failed
    g0 = float(log[0][2]) if len(log) else 0.0
    last = log[-1] if len(log) else [0.0] * 16
    mode = MODE_NAMES.get(mode, mode) if not isinstance(mode, str) else mode
    lines = ["experiment,study,mode,method,rank,state_dim,converged,gn_iterations,total_pcg,offline_tlm,offline_adj,"
             "fwd,tlm,adj,final_cost,final_grad_rel,status",
             ",".join([experiment, study, mode, METHOD_NAMES.get(method, str(method)), str(int(rank)),
                       str(int(state_dim)), _b(s[3]), str(len(log)), str(int(s[2])), str(int(last[14])),
                       str(int(last[15])), str(int(last[11])), str(int(last[12])), str(int(last[13])), fmt(s[0]),
                       fmt(s[1] / g0 if g0 > 0.0 else 0.0), status])]
    _write(os.path.join(out_dir, "summary.csv"), lines)


def write_run(out_dir, experiment, problem, result, mode, method, rank, study="gn"):
    """observations.csv + iterations.csv + summary.csv of one gn_solve result."""
    os.makedirs(out_dir, exist_ok=True)
    write_observations_csv(out_dir, problem.obs_indices, problem.obs_values)
    write_iterations_csv(out_dir, result)
    write_summary_csv(out_dir, experiment, study, mode, method, rank, problem.n, result)

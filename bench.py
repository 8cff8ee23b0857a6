#!/usr/bin/env python
"""Benchmark: batched prior-preconditioned GN Hessian-vector products (TLM+ADJ).

One step = one block of s Hessian products (H V, V n x s) through the
device-resident sweep engine (the sketch block of the config). Default
workload: BASELINE.json configs[3] (2-D barotropic vorticity 512^2, 800 RK4
steps, s = k+p = 110), the configuration the north-star roofline target is
stated on.

Multi-GPU (torchrun): sketch columns are independent HVPs, so every rank runs
its own block of s columns against its own copy of the (deterministic) base
trajectory — weak scaling, no data-path collective; torch.distributed is used
only for the barrier and the max-over-ranks timing.

--impl reference: the reference's CPU path timed on the host cores. The
reference itself cannot be built (Eigen3 absent), so this is the C++ oracle
port of it (oracle/), all host threads, bounded sample extrapolated to HVP/s.
"""
import argparse
import json
import os

# CPU timings (cpu_baseline, the --impl reference arm, the GN CPU baseline) use
# the oracle's -O3 FMA build (oracle/Makefile ALTFLAGS); parity tests use the
# primary build the golden fixtures were generated with.
os.environ.setdefault("ORACLE_BUILD", "alt")
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian-vector products/s (TLM+ADJ)"
UNIT = "HVP/s"
K_ITER_SKETCH_STREAM = 0x736B6574636800  # proj/src/fourdvar.cpp:16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--s", type=int, default=0, help="block width (default: the config's sketch size k+p)")
    ap.add_argument("--group", type=int, default=0, help="BVE sweep group size (0 = auto, L2-resident)")
    ap.add_argument("--sweep", default="auto",
                    help="extra block widths to report, e.g. 1,8,32; 'auto' = 1,8,32 for config 3 at N=1 "
                         "(BASELINE.json configs[3] asks for the s in {1, 8, 32, 110} sweep), 'none' = off")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gn", default="auto",
                    help="also time full GN solves (the metric's second half) for these configs, e.g. 0,1,2,4, "
                         "'all', or 'none'; 'auto' = 0,1,2 at N=1 (C3/C4 take 1-3 min each), none under torchrun")
    ap.add_argument("--window", type=int, default=0,
                    help="profiling only (ncu launch lists): shorten the model window to this many RK4 steps "
                         "(2 observation intervals); the reported line then names the window in config")
    return ap.parse_args()


def gn_solve_timing(cfg, method=None):
    """Wall time of a full gn_solve (device-resident: FWD/evaluate, sketch, PCG,
    More-Thuente) on BASELINE config `cfg`, with its counters. `method`
    overrides the config's sketch (C4 compares Nystrom and SingleView)."""
    from paper_2401_15758_b200 import api, scenario

    sc = scenario.build(cfg)
    sc.problem.synchronize()
    kw = sc.spec.gn_kwargs()
    if method is not None:
        kw["method"] = method
    t0 = time.perf_counter()
    r = sc.problem.gn_solve(**kw)
    dt = time.perf_counter() - t0
    log = r["log"]
    last = log[-1] if len(log) else [0] * 16
    import numpy as np

    err_a = float(np.linalg.norm(r["analysis"] - sc.truth0) / np.linalg.norm(sc.truth0))
    err_b = float(np.linalg.norm(sc.problem.background - sc.truth0) / np.linalg.norm(sc.truth0))
    names = {api.RANDSVD: "randsvd", api.NYSTROM: "nystrom", api.SINGLEVIEW: "singleview"}
    cnt = {"fwd": int(last[11]), "tlm": int(last[12]), "adj": int(last[13]),
           "offline_tlm": int(last[14]), "offline_adj": int(last[15])}
    return {"config": sc.spec.name, "method": names.get(kw["method"], str(kw["method"])), "seconds": dt,
            "gn_iterations": int(len(log)), "total_pcg": int(r["summary"][2]), "counters": cnt,
            # model applications including sketch construction (BASELINE configs[4] compares these)
            "tlm_plus_adj_total": cnt["tlm"] + cnt["adj"] + cnt["offline_tlm"] + cnt["offline_adj"],
            "final_cost": float(r["summary"][0]), "rel_error_analysis": err_a, "rel_error_background": err_b}


def cpu_sweep_seconds(cfg, budget_s=3.0):
    """One-core seconds of one full-window single-vector sweep (TLM or ADJ) of
    the oracle port on config `cfg`, from a timed short window (TLM + ADJ over
    k steps on one thread, scaled by steps / k / 2)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    from paper_2401_15758_b200 import scenario

    spec = scenario.CONFIGS[cfg]
    v = O.gaussian_matrix(spec.dim, 1, 5)[0]

    def timed(k):
        osc = O.Scenario(cfg, steps=k, spi=k)
        tr = osc.linearize(osc.background)
        t0 = time.perf_counter()
        tr.adj_range(0, k, tr.tlm_range(0, k, v))
        return time.perf_counter() - t0

    k = 1
    dt = timed(k)
    k = max(1, min(spec.steps, int(round(budget_s / max(dt, 1e-4)))))
    dt = timed(k)
    return dt / 2.0 * spec.steps / k, k


def cpu_gn_baseline(run, cfg, method=None):
    """the CPU GN solve time beside the GPU one. C0/C1: the
    oracle port's own gn_solve, timed (all host threads for the sketch's column
    fan-out, serial PCG, as the reference's apply_columns / pcg_solve). C2-C4
    (tens of minutes to hours on the CPU): the port's one-core sweep time times
    the GPU run's own sweep counters (serial: fwd + online tlm + adj; sketch:
    offline tlm + adj over all threads), labelled as extrapolated."""
    cores = os.cpu_count() or 1
    if cfg in (0, 1):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_lib as O

        from paper_2401_15758_b200 import api, scenario

        kw = scenario.CONFIGS[cfg].gn_kwargs()
        if method is not None:
            kw["method"] = method
        kw["mode"] = api.MODES[kw["mode"]] if isinstance(kw["mode"], str) else kw["mode"]
        osc = O.Scenario(cfg)
        t0 = time.perf_counter()
        r = osc.gn_solve(workers=cores, **kw)
        dt = time.perf_counter() - t0
        return {"seconds": dt, "kind": "measured", "cores": cores, "total_pcg": int(r["summary"][2]),
                "build": "oracle port, ALTFLAGS (-O3 -march=x86-64-v3 -ffp-contract=fast)"}
    c = run["counters"]
    t1, k = cpu_sweep_seconds(cfg)
    serial = c["fwd"] + c["tlm"] + c["adj"]
    fan = c["offline_tlm"] + c["offline_adj"]
    return {"seconds": t1 * (serial + fan / cores), "kind": "extrapolated", "cores": cores,
            "one_core_sweep_s": t1, "sample": f"1 vector, TLM+ADJ over {k} RK4 steps, one core",
            "model": "one-core sweep time x (fwd + online tlm + adj + (offline tlm + adj) / cores) of this GPU run",
            "build": "oracle port, ALTFLAGS (-O3 -march=x86-64-v3 -ffp-contract=fast)"}


# ------------------------------------------------------------------ dist ----
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def local_device(local):
    """GPU of a local rank: one per rank; with fewer visible GPUs than ranks
    (a functional run on a 1-GPU box) ranks share them round-robin."""
    import torch

    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    return local % n if n > 0 else local


def dist_init(world, backend=None):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist

    if backend is None:
        # NCCL needs one GPU per rank; with fewer GPUs than ranks (functional
        # runs) the barrier and the max-over-ranks timing go through gloo
        ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
        backend = "nccl" if ngpu >= world else "gloo"
    if torch.cuda.is_available():
        torch.cuda.set_device(local_device(int(os.environ.get("LOCAL_RANK", "0"))))
    dist.init_process_group(backend=backend)
    return dist


def dist_barrier(dist):
    if dist is not None:
        dist.barrier()


def dist_max(dist, x):
    """Max over ranks (timings are max-reduced, never wall-clock)."""
    if dist is None:
        return x
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_seed(rank):
    """Per-rank sketch block seed (rank 0 = the reference's first GN sketch seed)."""
    from paper_2401_15758_b200 import api

    return api.mix_seed(2, K_ITER_SKETCH_STREAM) + rank


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- roofline -----
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def group_size(dim, requested):
    """Mirror of Problem::group(): vectors per L2-resident BVE sweep group."""
    if requested > 0:
        return requested
    return max(1, int(4e9 / (6.0 * 8.0 * dim)))


def algorithmic_bytes_per_hvp(n_grid_points, stages, s):
    """B_HVP = 2 S (16 N) + 2 B_traj / s, B_traj = 8 N S."""
    return 2.0 * stages * 16.0 * n_grid_points + 2.0 * (8.0 * n_grid_points * stages) / s


# --------------------------------------------------------- CPU baseline -----
def cpu_reference_sample(cfg, budget_s=10.0):
    """Oracle port of the reference path on all host threads; bounded sample.

    Each thread owns one vector and runs TLM then ADJ over a short window of the
    config's grid/physics (the reference's apply_columns std::thread fan-out,
    proj/src/sketch.cpp:116-140); HVP/s is extrapolated by the step ratio.
    """
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import concurrent.futures as cf

    import numpy as np
    import oracle_lib as O

    from paper_2401_15758_b200 import scenario

    spec = scenario.CONFIGS[cfg]
    cores = os.cpu_count() or 1
    V = O.gaussian_matrix(spec.dim, cores, 5)

    def timed(k):
        osc = O.Scenario(cfg, steps=k, spi=k)
        tr = osc.linearize(osc.background)

        def one(j):
            y = tr.tlm_range(0, k, V[j])
            return tr.adj_range(0, k, y)

        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(cores) as ex:
            list(ex.map(one, range(cores)))
        return time.perf_counter() - t0

    # calibrate the window so the timed sample is ~budget_s of wall time
    k = 1
    dt = timed(k)
    k = max(1, min(spec.steps, int(round(k * budget_s / max(dt, 1e-3)))))
    dt = timed(k)
    hvp_equiv = cores * k / spec.steps
    return {"value": hvp_equiv / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"{cores} vectors x (TLM+ADJ over {k} of {spec.steps} RK4 steps) on the {spec.name} grid, "
                       f"{dt:.1f} s wall, extrapolated by steps; oracle C++ port (reference unbuildable: Eigen3 absent)"),
            "seconds": dt}


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2401_15758_b200 import scenario

    spec = scenario.CONFIGS[args.config]
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_reference_sample(args.config))
    timed = vals[args.warmup:]
    value = statistics.median(v["value"] for v in timed)
    cb = dict(timed[-1])
    cb["value"] = value
    cb.pop("seconds", None)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * (args.s or spec.rank) / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            # the same config block as our arm (sweep group resolved the same way)
            "config": config_block(spec, args.s or spec.rank,
                                   min(args.s or spec.rank, group_size(spec.dim, args.group)) if spec.model == 2
                                   else args.s or spec.rank, args.group),
            "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def sub_block_plan(spec, s, group_arg=0):
    """(n_sub, width) of the L2-resident sub-blocks engine.cu sweeps an s-wide BVE block as
    (Problem::sub_blocks: 6.4 fields of RK workspace per vector, 112 MB budget, graph-replay width <= 8)."""
    from paper_2401_15758_b200 import api

    if spec.model != api.MODEL_BVE or group_arg > 0 or os.environ.get("SDV_NO_SUBBLOCK"):
        return 0, s
    cap = int(112e6 / (6.4 * 8.0 * spec.dim))
    if cap < 2 or cap > 8 or s < 2 * cap:
        return 0, s
    nb = -(-s // cap)
    return nb, -(-s // nb)


def config_block(spec, s, group, group_arg=0):
    # bytes one block sweep streams: the stored base trajectory (BVE: omega and
    # psi per RK4 stage; Burgers: the stage inputs) + the block's RK workspace
    from paper_2401_15758_b200 import api

    bve = spec.model == api.MODEL_BVE
    field = 8.0 * spec.dim
    base = (2 if bve else 1) * 4 * spec.steps * field
    work = s * (6 if bve else 2) * field
    l2 = 126e6
    nb, wsub = sub_block_plan(spec, s, group_arg)
    if nb:
        note = (f"inputs larger than L2: the {s * field / 1e6:.3g} MB block and the {base / 1e9:.3g} GB base trajectory "
                f"(streamed from HBM once per sub-block sweep); the block is swept as {nb} sub-blocks of <= {wsub} "
                f"vectors whose {wsub * 6.4 * field / 1e6:.3g} MB RK workspace is deliberately L2-resident (L2 126 MB)")
    else:
        note = (f"inputs larger than L2: {base / 1e9:.3g} GB base trajectory + {work / 1e9:.3g} GB block workspace "
                f"streamed per sweep (L2 126 MB)" if base + work > l2 else
                f"on-chip problem: {(base + work) / 1e6:.3g} MB per sweep fits the 126 MB L2")
    return {"workload": f"{spec.name}: block of s={s} GN Hessian products (TLM+ADJ), BASELINE.json configs",
            "model": spec.name, "grid": spec.n, "rk4_steps": spec.steps, "block_s": s,
            "global_batch": s, "seq_len": spec.steps, "parallelism": "sketch-column sharding (weak)",
            "sweep_group": group, "sub_blocks": nb, "l2": note}


# ------------------------------------------------------------------ ours ----
def run_ours(args, world, rank, local):
    import numpy as np

    import paper_2401_15758_b200 as sdv
    from paper_2401_15758_b200 import api, scenario

    dist = dist_init(world)
    sdv.init(local_device(local))
    spec = scenario.CONFIGS[args.config]
    if args.window:
        spec = scenario.with_window(spec, steps=args.window, spi=max(1, args.window // 2))
    s = args.s or spec.rank
    sc = scenario.build(spec, block_group=args.group)
    prob = sc.problem
    tr = prob.linearize(prob.background)
    n = prob.n
    stages = 4 * prob.total_steps
    ngrid = n
    V = api.gaussian_matrix(n, s, rank_seed(rank))
    dV = api.DeviceBuffer(V.nbytes)
    dV.upload(V)
    dHV = api.DeviceBuffer(V.nbytes)
    for _ in range(args.warmup):
        tr.gram_dev(dV.ptr.value, s, dHV.ptr.value)
    prob.synchronize()
    dist_barrier(dist)

    clk = ClockSampler(local)
    clk.start()
    e0, e1 = api.Event(), api.Event()
    l0 = sdv.launch_count()
    e0.record(prob)
    for _ in range(args.steps):
        tr.gram_dev(dV.ptr.value, s, dHV.ptr.value)
    e1.record(prob)
    ms = e0.elapsed_ms(e1)
    launches = sdv.launch_count() - l0
    clocks = clk.stop()
    dist_barrier(dist)
    ms_max = dist_max(dist, ms)
    value = world * s * args.steps / (ms_max / 1000.0)

    # End-to-end through the public host-buffer API: pinned H2D of V, D2H of H V.
    e2e = None
    if not args.no_e2e:
        pin_in = api.PinnedBuffer((s, n))
        pin_out = api.PinnedBuffer((s, n))
        pin_in.array[...] = V
        tr.gram_host(pin_in.array, pin_out.array)
        dist_barrier(dist)
        f0, f1 = api.Event(), api.Event()
        f0.record(prob)
        for _ in range(args.steps):
            tr.gram_host(pin_in.array, pin_out.array)
        f1.record(prob)
        ems = dist_max(dist, f0.elapsed_ms(f1))
        e2e = {"value": world * s * args.steps / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(V.nbytes), "d2h_bytes_per_step": int(V.nbytes)}
        ok = np.allclose(pin_out.array, dHV.download((s, n)), rtol=0, atol=1e-12 * np.abs(pin_out.array).max())
        if not ok:
            raise RuntimeError("e2e result differs from the device-resident result")
        pin_in.free()
        pin_out.free()

    # Roofline of the dominant kernel (the fused RK4 stage kernel), timed live
    # with CUDA events on the library stream.
    hbm, peak_src = peaks()
    probe_stages = 64
    ms_stage, ms_col = tr.probe_stage_kernels(s, probe_stages)
    probe = {"tlm_stage_ms": ms_stage, "tlm_col_ms": ms_col}
    if spec.model == api.MODEL_BVE:
        g = min(s, group_size(n, args.group))
        ms_adj, ms_carry_adj = tr.probe_adj_stage_kernels(s, probe_stages)
        probe.update(adj_stage_ms=ms_adj, adj_carry_ms=ms_carry_adj)
        # per stage launch: read+write the g tangent fields (16 N each) + read
        # the two base stage fields (omega_b, psi_b) once for the group
        alg_bytes = g * 16.0 * ngrid + 2 * 8.0 * ngrid
        dur = 0.5 * (ms_stage + ms_adj)  # the sweeps run as many ADJ stage launches as TLM ones
        kname = ("bve stage_kernel TLM + ADJ (mean), fused Poisson path (y-solved spectra from tile carries, "
                 "in-place inverse x-FFT, Arakawa stencils + RK4 / adjoint-RK4 update, forward x-FFT, tile-local "
                 f"y-recurrences); probe: one launch of g = {g} vectors per stage, the kernel filling the GPU for "
                 "12 waves" + (f" (the sweep itself runs {prob.sub_blocks(s)} L2-resident sub-blocks of <= 8 vectors, "
                               "each as two concurrent lanes on two streams, replayed as CUDA graphs)"
                               if prob.sub_blocks(s) else " (the sweep runs the block as two concurrent lanes of g/2)"))
    else:
        g = s
        k = max(1, min(prob.total_steps, probe_stages // 4))
        # tangent fields stay on-chip for the whole sweep: compulsory traffic is
        # the state in/out per vector + the base stage inputs read once
        alg_bytes = g * 16.0 * ngrid + 4 * k * 8.0 * ngrid
        dur = ms_stage
        kname = f"burgers_tlm_kernel (persistent, {k} steps)"
    achieved = alg_bytes / (dur / 1000.0) / 1e9
    b_hvp = algorithmic_bytes_per_hvp(ngrid, stages, s)
    step_achieved = value / world * b_hvp / 1e9
    # measured DRAM bytes of this kernel per launch (ncu --set full capture in
    # profiles/ncu_traffic.json, per vector x the probe's group), when profiled
    traffic = None
    fp64 = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if spec.model == api.MODEL_BVE and os.path.exists(tf):
        tj = json.load(open(tf))
        t, ta = tj.get("bve_stage_kernel_tlm", {}), tj.get("bve_stage_kernel_adj", {})
        if t.get("grid") == spec.n and ta.get("grid") == spec.n:
            traffic = 0.5 * (t["dram_bytes_per_vector"] + ta["dram_bytes_per_vector"]) * g
            if "fp64_pipe_pct" in t and "fp64_pipe_pct" in ta:
                fp64 = 0.5 * (t["fp64_pipe_pct"] + ta["fp64_pipe_pct"])
    # the same kernel as the sweep launches it (4-vector lanes of an L2-resident
    # sub-block): measured DRAM bytes per vector-stage, when profiled
    traffic_sweep = None
    if spec.model == api.MODEL_BVE and os.path.exists(tf) and prob.sub_blocks(s):
        tsb = json.load(open(tf)).get("bve_stage_kernel_adj_subblock", {})
        if tsb.get("grid") == spec.n:
            traffic_sweep = {"dram_bytes_per_vector_stage": tsb["dram_bytes_per_vector"],
                             "vectors_per_launch": tsb["vectors_per_launch"], "source": tsb["source"]}
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic, "traffic_sweep_shape": traffic_sweep,
            # measured DRAM bytes (ncu) over the live launch time: how close the
            # kernel's actual data movement runs to the HBM peak
            "traffic_GBs": (traffic / (dur / 1000.0) / 1e9) if traffic else None,
            "traffic_source": "ncu --set full capture (profiles/ncu_traffic.json), per vector x g" if traffic else None,
            # FP64 pipe utilisation of the same capture (the north star's co-bound)
            "fp64_pipe_pct": fp64,
            "kernel": kname, "kernel_ms": dur, "col_kernel_ms": ms_col, "probe": probe,
            "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
            "step_model": {"B_HVP_bytes": b_hvp, "achieved_GBs": step_achieved, "frac": step_achieved / hbm,
                           "note": "SURVEY.md 8(d) streaming model: HVP/s x B_HVP per GPU"}}

    sweep = {}
    sw = args.sweep
    if sw == "auto":
        sw = "1,8,32" if args.config == 3 and world == 1 and not args.window else "none"
    if sw and sw != "none":
        for sv in [int(x) for x in sw.split(",") if x]:
            Vs = api.gaussian_matrix(n, sv, rank_seed(rank))
            dVs = api.DeviceBuffer(Vs.nbytes)
            dVs.upload(Vs)
            dHs = api.DeviceBuffer(Vs.nbytes)
            for _ in range(3):  # small blocks: CUDA-graph capture happens on an early call; time the replay
                tr.gram_dev(dVs.ptr.value, sv, dHs.ptr.value)
            a, b = api.Event(), api.Event()
            a.record(prob)
            tr.gram_dev(dVs.ptr.value, sv, dHs.ptr.value)
            b.record(prob)
            t = a.elapsed_ms(b)
            sweep[str(sv)] = {"hvp_per_s": sv / (t / 1000.0), "ms": t,
                              "frac_step_model": sv / (t / 1000.0) * algorithmic_bytes_per_hvp(ngrid, stages, sv)
                              / 1e9 / hbm}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(args.config)
            cpu.pop("seconds", None)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_block(spec, s, min(s, group_size(n, args.group)) if spec.model == 2 else s,
                                       args.group),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": launches}
        if sweep:
            line["block_sweep"] = sweep
        gn = args.gn
        if gn == "auto":
            # every config's GN solve (C4: its adaptive Nystrom arm; the SingleView arm, ~9 min, under 'all')
            gn = "0,1,2,3,4" if world == 1 and not args.window else "none"
        if gn and gn != "none":
            cfgs = [0, 1, 2, 3, 4] if gn == "all" else [int(x) for x in gn.split(",") if x]
            runs = []
            for c in cfgs:
                runs.append(gn_solve_timing(c))
                if c == 4 and args.gn == "all":  # BASELINE configs[4]: SingleView vs Nystrom on total products
                    runs.append(gn_solve_timing(4, method=api.SINGLEVIEW))
            if not args.no_cpu_baseline:
                for r in runs:
                    try:
                        meth = {"randsvd": api.RANDSVD, "nystrom": api.NYSTROM, "singleview": api.SINGLEVIEW}
                        cfg_i = [sp.name for sp in scenario.CONFIGS].index(r["config"])
                        r["cpu_baseline"] = cpu_gn_baseline(r, cfg_i, meth.get(r["method"]))
                    except Exception as e:  # reported, not fatal
                        r["cpu_baseline"] = {"seconds": None, "kind": f"failed: {e}"}
            line["gn_solve"] = runs
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()

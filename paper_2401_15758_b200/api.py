"""Python host mirror of the reference's hot-path interfaces over the C-ABI.

Names and argument meaning follow /root/reference/proj/include/sketchdav:
  Problem            <- AssimilationProblem + DynamicalModel + PriorCovariance
  Problem.linearize  <- DynamicalModel::linearize          (model.hpp:36-40)
  Trajectory         <- LinearizedTrajectory (state_at, tlm_range, adj_range)
  MisfitOperator     <- MisfitOperator::apply/adjoint_apply (fourdvar.hpp:75-89)
                        batched over column blocks (apply_columns, sketch.hpp:54-58)
  Problem.evaluate   <- evaluate                            (fourdvar.cpp:92-132)
  woodbury_apply, pcg_solve, sketches, gn_solve             (linalg/sketch/fourdvar)
Errors map to ValueError (std::invalid_argument) and SdvError (std::runtime_error).
Blocks are numpy arrays of shape (s, n) (row-major == column-major n x s).
"""
from __future__ import annotations

import ctypes as C
import sys

import numpy as np

from ._lib import D, GNConfigC, I32, I64, ProblemDesc, check, lib

MODEL_BURGERS, MODEL_BVE, MODEL_BURGERS_DIRICHLET, MODEL_BVE_DIRICHLET = 1, 2, 3, 4
PRIOR_FOURIER, PRIOR_LAPLACIAN = 0, 1
RANDSVD, NYSTROM, SINGLEVIEW, LANCZOS = 0, 1, 2, 3
# linearize storage policies (sdv.h SDV_STORE_*)
STORE_AUTO, STORE_FULL, STORE_CHECKPOINT = 0, 1, 2
MODES = {"SketchSolv": 0, "SketchPrec": 1, "SketchPrecA": 2, "PrecGamma": 3, "PrecLanczos": 4, "PrecALanczos": 5}


def _p(a):
    return None if a is None else a.ctypes.data_as(D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def init(device=0):
    check(lib().sdv_device_init(device))


def launch_count():
    return int(lib().sdv_launch_count())


def path_counts():
    """Launch counts per sweep-kernel variant ({"bve_stage_fused": k, ...}),
    process-wide: which kernel path the calls so far took (sdv_path_counts)."""
    L = lib()
    n = L.sdv_path_counts(None, 0)
    buf = (C.c_uint64 * n)()
    L.sdv_path_counts(buf, n)
    return {L.sdv_path_name(i).decode(): int(buf[i]) for i in range(n)}


def path_delta(before):
    """Per-variant launches since a path_counts() snapshot."""
    now = path_counts()
    return {k: now[k] - before.get(k, 0) for k in now}


def mix_seed(seed, stream):
    return int(lib().sdv_mix_seed(seed, stream))


def gaussian_matrix(n, l, seed):
    """n x l standard normal block as an (l, n) array (column-major n x l)."""
    out = np.empty((l, n))
    check(lib().sdv_gaussian_matrix(n, l, seed, _p(out)))
    return out


def gaussian_vector(n, seed):
    return gaussian_matrix(n, 1, seed)[0]


class Problem:
    """Device-resident AssimilationProblem.

    model 1/2: periodic Burgers / BVE with the Fourier-diagonal prior
    (prior_sigma, prior_length; control-variable background term).
    model 3: the reference's Dirichlet RK3 Burgers with the Laplacian prior
    (prior_kind=1, prior_alpha, prior_beta; x-space background term as
    proj/src/fourdvar.cpp:92-132).
    model 4: the reference's Dirichlet BVE (n = nx columns, ny rows, reynolds,
    rossby; proj/src/bve.cpp) with the 2-D Laplacian prior.
    """

    def __init__(self, model, n, nu, dt, n_t, steps_per_interval, prior_sigma, prior_length, obs_indices, obs_values,
                 obs_variances, background, block_group=0, prior_kind=0, prior_alpha=0.0, prior_beta=0.0, ny=0,
                 reynolds=0.0, rossby=0.0):
        self.desc = ProblemDesc(model, n, nu, dt, n_t, steps_per_interval, prior_sigma, prior_length, block_group,
                                prior_kind, prior_alpha, prior_beta, ny, reynolds, rossby)
        idx = np.ascontiguousarray(obs_indices, dtype=np.int64)
        vals = _f64(obs_values)
        var = _f64(obs_variances)
        bg = _f64(background)
        self._h = C.c_void_p()
        check(lib().sdv_problem_create(C.byref(self.desc), idx.size, idx.ctypes.data_as(I64), _p(vals), _p(var),
                                       _p(bg), C.byref(self._h)))
        dims = np.zeros(6, np.int64)
        check(lib().sdv_problem_dims(self._h, dims.ctypes.data_as(I64)))
        self.n, self.m, self.n_obs, self.n_t, self.spi, self.total_steps = (int(x) for x in dims)
        self.background = bg.copy()
        self.obs_indices = idx.copy()
        self.obs_values = vals.reshape(self.n_t, self.n_obs).copy()
        self.obs_variances = var.reshape(self.n_t, self.n_obs).copy()

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().sdv_problem_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        # at interpreter shutdown the CUDA runtime may already be tearing down
        # (its calls can block): leave the handle to process exit
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x0, steps):
        out = np.empty(self.n)
        check(lib().sdv_forward(self._h, _p(_f64(x0)), steps, _p(out)))
        return out

    def linearize(self, x0, checkpoint_stride=None, policy=None):
        """DynamicalModel::linearize (model.hpp:36-40). With no stride: every
        RK stage stored when it fits HBM (else checkpoints every
        steps_per_interval steps). policy: STORE_AUTO / STORE_FULL /
        STORE_CHECKPOINT (sdv.h)."""
        t = C.c_void_p()
        if checkpoint_stride is None and policy is None:
            check(lib().sdv_linearize(self._h, _p(_f64(x0)), C.byref(t)))
        else:
            stride = self.spi if checkpoint_stride is None else int(checkpoint_stride)
            pol = STORE_AUTO if policy is None else int(policy)
            check(lib().sdv_linearize_ex(self._h, _p(_f64(x0)), stride, pol, C.byref(t)))
        return Trajectory(self, t)

    def linearize_dev(self, x0_dev, checkpoint_stride=None, policy=None):
        t = C.c_void_p()
        if checkpoint_stride is None and policy is None:
            check(lib().sdv_linearize_dev(self._h, C.c_void_p(x0_dev), C.byref(t)))
        else:
            stride = self.spi if checkpoint_stride is None else int(checkpoint_stride)
            pol = STORE_AUTO if policy is None else int(policy)
            check(lib().sdv_linearize_ex_dev(self._h, C.c_void_p(x0_dev), stride, pol, C.byref(t)))
        return Trajectory(self, t)

    def prior_sqrt(self, V):
        V = _f64(np.atleast_2d(V))
        out = np.empty_like(V)
        check(lib().sdv_prior_sqrt_block(self._h, _p(V), V.shape[0], _p(out)))
        return out

    def evaluate(self, x0, z=None):
        """(cost, ctrl_grad, lambda0) in the control-variable form."""
        cost = C.c_double()
        g = np.empty(self.n)
        lam = np.empty(self.n)
        check(lib().sdv_evaluate(self._h, _p(_f64(x0)), _p(None if z is None else _f64(z)), C.byref(cost), _p(g),
                                 _p(lam)))
        return cost.value, g, lam

    def woodbury_apply(self, basis, eig, V):
        """basis: (l, n) rows = basis vectors; V: (s, n)."""
        basis = _f64(np.atleast_2d(basis))
        V = _f64(np.atleast_2d(V))
        out = np.empty_like(V)
        check(lib().sdv_woodbury_apply(self._h, basis.shape[0], _p(basis), _p(_f64(eig)), _p(V), V.shape[0],
                                       _p(out)))
        return out

    def thin_qr(self, Y):
        """Device Householder QR of an (n, l) matrix. Returns q (n, l), r (l, l), n_deficient."""
        n, l = Y.shape
        yt = _f64(np.asarray(Y).T)
        q = np.empty((l, n))
        r = np.empty((l, l))
        nd = C.c_int()
        check(lib().sdv_thin_qr(self._h, n, l, _p(yt), _p(q), _p(r), C.byref(nd)))
        return q.T, r.T, nd.value

    def gn_solve(self, mode="SketchPrec", method=RANDSVD, rank=10, rank2=-1, growth=5, max_rank=-1,
                 eps_sketch=1.5, eps_reuse=10.0, seed=0, grad_tol=1e-6, pcg_tol=1e-9, max_gn_iters=50,
                 pcg_max_iter=10000, max_eig=256):
        cfg = GNConfigC(MODES[mode] if isinstance(mode, str) else mode, method, rank, rank2, growth, max_rank,
                        eps_sketch, eps_reuse, seed, grad_tol, pcg_tol, max_gn_iters, pcg_max_iter)
        analysis = np.empty(self.n)
        log = np.zeros((64, 16))
        n_it = C.c_int()
        summary = np.zeros(5)
        eig0 = np.full(max_eig, np.nan)
        check(lib().sdv_gn_solve(self._h, C.byref(cfg), _p(analysis), _p(log), 64, C.byref(n_it), _p(summary),
                                 _p(eig0), max_eig))
        return dict(analysis=analysis, log=log[:n_it.value], summary=summary, eig0=eig0[~np.isnan(eig0)])

    def synchronize(self):
        check(lib().sdv_synchronize(self._h))

    def sub_blocks(self, s):
        """L2-resident sub-blocks an s-wide block is swept as (0 = as one block)."""
        n = C.c_int(0)
        check(lib().sdv_sub_blocks(self._h, int(s), C.byref(n)))
        return n.value


class Trajectory:
    """Frozen device linearization (LinearizedTrajectory) + its MisfitOperator."""

    def __init__(self, problem, handle):
        self.problem = problem
        self._h = handle

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().sdv_traj_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        # at interpreter shutdown the CUDA runtime may already be tearing down
        # (its calls can block): leave the handle to process exit
        if sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass

    def total_steps(self):
        return self.problem.total_steps

    def info(self):
        """{steps, stride (0 = every stage stored), segments, bytes}"""
        v = (C.c_int64 * 4)()
        check(lib().sdv_traj_info(self._h, v))
        return {"steps": v[0], "stride": v[1], "segments": v[2], "bytes": v[3]}

    def state_at(self, step):
        out = np.empty(self.problem.n)
        check(lib().sdv_traj_state_at(self._h, step, _p(out)))
        return out

    def tlm_range(self, begin, end, dx):
        dx = _f64(np.atleast_2d(dx))
        out = np.empty_like(dx)
        check(lib().sdv_tlm_range(self._h, begin, end, _p(dx), dx.shape[0], _p(out)))
        return out

    def adj_range(self, begin, end, lam):
        lam = _f64(np.atleast_2d(lam))
        out = np.empty_like(lam)
        check(lib().sdv_adj_range(self._h, begin, end, _p(lam), lam.shape[0], _p(out)))
        return out

    # MisfitOperator (apply_columns batched)
    def misfit_apply(self, V):
        V = _f64(np.atleast_2d(V))
        out = np.empty((V.shape[0], self.problem.m))
        check(lib().sdv_misfit_apply_block(self._h, _p(V), V.shape[0], _p(out)))
        return out

    def misfit_adjoint(self, W):
        W = _f64(np.atleast_2d(W))
        out = np.empty((W.shape[0], self.problem.n))
        check(lib().sdv_misfit_adjoint_block(self._h, _p(W), W.shape[0], _p(out)))
        return out

    def gram(self, V):
        V = _f64(np.atleast_2d(V))
        out = np.empty_like(V)
        check(lib().sdv_gram_apply_block(self._h, _p(V), V.shape[0], _p(out)))
        return out

    def gram_dev(self, v_dev, s, out_dev):
        check(lib().sdv_gram_apply_block_dev(self._h, C.c_void_p(v_dev), s, C.c_void_p(out_dev)))

    def gram_host(self, V, out):
        """Public host-buffer entry (e2e path): V, out are (s, n) float64 arrays (pinned or not)."""
        check(lib().sdv_gram_apply_block(self._h, V.ctypes.data_as(D), V.shape[0], out.ctypes.data_as(D)))

    def probe_stage_kernels(self, s, stages):
        a, b = C.c_float(), C.c_float()
        check(lib().sdv_probe_stage_kernels(self._h, s, stages, C.byref(a), C.byref(b)))
        return a.value, b.value

    def probe_adj_stage_kernels(self, s, stages):
        a, b = C.c_float(), C.c_float()
        check(lib().sdv_probe_adj_stage_kernels(self._h, s, stages, C.byref(a), C.byref(b)))
        return a.value, b.value

    def sketch(self, method, rank, seed, rank2=-1, want_basis=True):
        eig = np.empty(rank)
        basis = np.empty((rank, self.problem.n)) if want_basis else None
        counts = np.zeros(3, np.int64)
        check(lib().sdv_sketch(self._h, method, rank, rank2, seed, _p(eig), _p(basis), counts.ctypes.data_as(I64)))
        k = int(counts[2])
        return eig[:k], (basis[:k] if basis is not None else None), counts

    def lanczos(self, rank, start):
        """lanczos_sketch(h, rank, start) (proj/src/sketch.cpp:292-389) from a given start vector."""
        eig = np.empty(rank)
        basis = np.empty((rank, self.problem.n))
        counts = np.zeros(3, np.int64)
        check(lib().sdv_lanczos_sketch(self._h, rank, _p(_f64(start)), _p(eig), _p(basis),
                                       counts.ctypes.data_as(I64)))
        k = int(counts[2])
        return eig[:k], basis[:k], counts

    def sketch_adaptive(self, method, rank, growth, max_rank, seed, rank2=-1, eps_sketch=1.5):
        """adaptive_{randsvd,nystrom,singleview} (proj/src/sketch.cpp:402-564).

        Returns (eig, basis, counts = [tlm, adj, final_rank, probes, tolerance_met], kappa history)."""
        eig = np.empty(max_rank)
        basis = np.empty((max_rank, self.problem.n))
        counts = np.zeros(5, np.int64)
        kappa = np.full(64, np.nan)
        check(lib().sdv_sketch_adaptive(self._h, method, rank, growth, max_rank, rank2, eps_sketch, seed, _p(eig),
                                        _p(basis), counts.ctypes.data_as(I64), _p(kappa), kappa.size))
        k = int(counts[2])
        return eig[:k], basis[:k], counts, kappa[~np.isnan(kappa)]

    def cond_estimate(self, basis, eig, seed):
        """cond_estimate (proj/src/sketch.cpp:391-400) of (I + H)(I + H_hat)^-1."""
        basis = _f64(np.atleast_2d(basis))
        out = C.c_double()
        check(lib().sdv_cond_estimate(self._h, basis.shape[0], _p(basis), _p(_f64(eig)), seed, C.byref(out)))
        return out.value

    def pcg_solve(self, rhs, basis=None, eig=None, tol=1e-9, max_iter=10000):
        l = 0 if basis is None else np.atleast_2d(basis).shape[0]
        x = np.empty(self.problem.n)
        info = np.zeros(2, np.int32)
        check(lib().sdv_pcg_solve(self._h, _p(_f64(rhs)), l, _p(None if basis is None else _f64(basis)),
                                  _p(None if eig is None else _f64(eig)), tol, max_iter, _p(x),
                                  info.ctypes.data_as(I32)))
        return x, int(info[0]), bool(info[1])


class Event:
    """CUDA event recorded on a problem's stream (device timing)."""

    def __init__(self):
        self.h = C.c_void_p()
        check(lib().sdv_event_create(C.byref(self.h)))

    def record(self, problem):
        check(lib().sdv_event_record(problem.handle, self.h))

    def elapsed_ms(self, end):
        ms = C.c_float()
        check(lib().sdv_event_elapsed_ms(self.h, end.h, C.byref(ms)))
        return ms.value

    def __del__(self):
        if sys.is_finalizing():
            return
        try:
            lib().sdv_event_destroy(self.h)
        except Exception:
            pass


class DeviceBuffer:
    """Raw device allocation (for device-resident benchmark inputs)."""

    def __init__(self, nbytes):
        self.ptr = C.c_void_p()
        self.nbytes = nbytes
        check(lib().sdv_dev_alloc(nbytes, C.byref(self.ptr)))

    def upload(self, arr):
        a = np.ascontiguousarray(arr)
        check(lib().sdv_memcpy_htod(self.ptr, a.ctypes.data_as(C.c_void_p), a.nbytes))

    def download(self, shape, dtype=np.float64):
        out = np.empty(shape, dtype)
        check(lib().sdv_memcpy_dtoh(out.ctypes.data_as(C.c_void_p), self.ptr, out.nbytes))
        return out

    def free(self):
        if self.ptr:
            lib().sdv_dev_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        if sys.is_finalizing():
            return
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host buffer viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float64):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.ptr = C.c_void_p()
        check(lib().sdv_host_alloc(nbytes, C.byref(self.ptr)))
        buf = (C.c_char * nbytes).from_address(self.ptr.value)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self):
        if self.ptr:
            self.array = None
            lib().sdv_host_free(self.ptr)
            self.ptr = C.c_void_p()

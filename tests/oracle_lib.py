"""ctypes binding of the CPU oracle (oracle/_build/libsdv_oracle.so).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg as the checker. The product
(paper_2401_15758_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# ORACLE_BUILD=alt selects the second build (oracle/Makefile ALTFLAGS: -O3
# -march=native -ffp-contract=fast): same algorithm, different rounding.
LIB_PATH = os.path.join(ROOT, "oracle", "_build",
                        "libsdv_oracle_alt.so" if os.environ.get("ORACLE_BUILD") == "alt" else "libsdv_oracle.so")

_lib = None

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)


def build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_mix_seed.restype = C.c_uint64
        _lib.oracle_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.oracle_gaussian_matrix.argtypes = [C.c_int64, C.c_int64, C.c_uint64, D]
        _lib.oracle_gn_solve.argtypes = [C.c_int, I64, D, C.c_uint64, D, D, C.c_int, C.POINTER(C.c_int), D, D,
                                         C.c_int]
        _lib.oracle_sketch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, D, D, I64]
        _lib.oracle_sketch_adaptive.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.c_double, C.c_uint64, C.c_int, D, D, I64, D, C.c_int]
        _lib.oracle_cond_estimate.argtypes = [C.c_int, C.c_int, C.c_int64, D, D, C.c_uint64, D]
        _lib.oracle_sketch_dense.argtypes = [C.c_int64, C.c_int64, D, C.c_int, C.c_int, C.c_int, C.c_uint64, D, D]
        _lib.oracle_bve_fixture.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                            C.c_uint64, D]
        _lib.oracle_pcg_dense.argtypes = [C.c_int64, D, D, D, C.c_double, C.c_int, D, C.POINTER(C.c_int),
                                          C.POINTER(C.c_int)]
    return _lib


def _p(a):
    return a.ctypes.data_as(D) if a is not None else None


def _chk(rc):
    if rc < 0:
        msg = lib().oracle_last_error().decode()
        if rc == -22:
            raise ValueError(msg)
        raise RuntimeError(msg)
    return rc


def mix_seed(seed, stream):
    return lib().oracle_mix_seed(seed, stream)


def gaussian_matrix(n, l, seed):
    out = np.empty((l, n))  # column-major n x l == row-major l x n
    _chk(lib().oracle_gaussian_matrix(n, l, seed, _p(out)))
    return out


class Scenario:
    """Oracle scenario for BASELINE config 0..4 (or 100 = burgers_1_1)."""

    def __init__(self, cfg, steps=-1, spi=-1):
        self.cfg = cfg
        self.h = _chk(lib().oracle_scenario_create_ex(cfg, steps, spi))
        info = np.zeros(4, np.int64)
        _chk(lib().oracle_scenario_info(self.h, info.ctypes.data_as(I64)))
        self.n, self.n_obs, self.n_t, self.spi = (int(x) for x in info)
        self.m = self.n_obs * self.n_t
        self.background = np.empty(self.n)
        self.truth0 = np.empty(self.n)
        self.indices = np.empty(self.n_obs, np.int64)
        self.values = np.empty((self.n_t, self.n_obs))
        self.variances = np.empty((self.n_t, self.n_obs))
        _chk(lib().oracle_scenario_arrays(self.h, _p(self.background), _p(self.truth0),
                                          self.indices.ctypes.data_as(I64), _p(self.values), _p(self.variances)))

    def prior_sqrt(self, v):
        out = np.empty(self.n)
        _chk(lib().oracle_prior_sqrt(self.h, _p(np.ascontiguousarray(v, np.float64)), _p(out)))
        return out

    def forward(self, x0, steps):
        out = np.empty(self.n)
        _chk(lib().oracle_forward(self.h, _p(np.ascontiguousarray(x0, np.float64)), steps, _p(out)))
        return out

    def linearize(self, x0):
        return Trajectory(self, _chk(lib().oracle_linearize(self.h, _p(np.ascontiguousarray(x0, np.float64)))))

    def evaluate(self, x0, z=None):
        cost = C.c_double()
        g = np.empty(self.n)
        lam = np.empty(self.n)
        innov = np.empty(self.m)
        zz = None if z is None else np.ascontiguousarray(z, np.float64)
        _chk(lib().oracle_evaluate(self.h, _p(np.ascontiguousarray(x0, np.float64)), _p(zz), C.byref(cost),
                                   _p(g), _p(lam), _p(innov)))
        return cost.value, g, lam, innov

    def gn_solve(self, mode=-1, method=-1, rank=-1, rank2=-1, growth=-1, max_rank=-1, max_gn_iters=-1,
                 pcg_max_iter=-1, workers=1, grad_tol=-1.0, pcg_tol=-1.0, eps_sketch=-1.0, eps_reuse=-1.0,
                 seed=None, max_eig=256):
        params = np.array([mode, method, rank, rank2, growth, max_rank, max_gn_iters, pcg_max_iter, workers],
                          np.int64)
        dparams = np.array([grad_tol, pcg_tol, eps_sketch, eps_reuse])
        analysis = np.empty(self.n)
        log = np.zeros((64, 16))
        n_it = C.c_int()
        summary = np.zeros(5)
        eig0 = np.full(max_eig, np.nan)
        _chk(lib().oracle_gn_solve(self.h, params.ctypes.data_as(I64), _p(dparams),
                                   C.c_uint64(0xFFFFFFFFFFFFFFFF if seed is None else seed), _p(analysis),
                                   _p(log), 64, C.byref(n_it), _p(summary), _p(eig0), max_eig))
        return dict(analysis=analysis, log=log[:n_it.value], summary=summary, eig0=eig0[~np.isnan(eig0)])

    def __del__(self):
        try:
            lib().oracle_scenario_destroy(self.h)
        except Exception:
            pass


class Trajectory:
    def __init__(self, sc, h):
        self.sc, self.h = sc, h

    def tlm_range(self, b, e, dx):
        out = np.empty(self.sc.n)
        _chk(lib().oracle_tlm_range(self.sc.h, self.h, b, e, _p(np.ascontiguousarray(dx, np.float64)), _p(out)))
        return out

    def adj_range(self, b, e, lam):
        out = np.empty(self.sc.n)
        _chk(lib().oracle_adj_range(self.sc.h, self.h, b, e, _p(np.ascontiguousarray(lam, np.float64)), _p(out)))
        return out

    def state_at(self, step):
        out = np.empty(self.sc.n)
        _chk(lib().oracle_state_at(self.sc.h, self.h, step, _p(out)))
        return out

    def misfit_apply(self, V, workers=1):
        """V: (s, n) row-major == column-major n x s. Returns (s, m)."""
        V = np.ascontiguousarray(V, np.float64)
        out = np.empty((V.shape[0], self.sc.m))
        _chk(lib().oracle_misfit_apply_block(self.sc.h, self.h, _p(V), V.shape[0], _p(out), workers))
        return out

    def misfit_adjoint(self, W, workers=1):
        W = np.ascontiguousarray(W, np.float64)
        out = np.empty((W.shape[0], self.sc.n))
        _chk(lib().oracle_misfit_adjoint_block(self.sc.h, self.h, _p(W), W.shape[0], _p(out), workers))
        return out

    def gram(self, V, workers=1):
        V = np.ascontiguousarray(V, np.float64)
        out = np.empty((V.shape[0], self.sc.n))
        _chk(lib().oracle_gram_block(self.sc.h, self.h, _p(V), V.shape[0], _p(out), workers))
        return out

    def sketch(self, method, rank, seed, rank2=-1, workers=1):
        eig = np.empty(rank)
        basis = np.empty((rank, self.sc.n))
        counts = np.zeros(3, np.int64)
        _chk(lib().oracle_sketch(self.sc.h, self.h, method, rank, rank2, seed, workers, _p(eig), _p(basis),
                                 counts.ctypes.data_as(I64)))
        return eig, basis, counts

    def sketch_adaptive(self, method, rank, growth, max_rank, seed, rank2=-1, eps=1.5, workers=1):
        eig = np.empty(max_rank)
        basis = np.empty((max_rank, self.sc.n))
        counts = np.zeros(5, np.int64)
        kappa = np.full(64, np.nan)
        _chk(lib().oracle_sketch_adaptive(self.sc.h, self.h, method, rank, growth, max_rank, rank2, eps, seed,
                                          workers, _p(eig), _p(basis), counts.ctypes.data_as(I64), _p(kappa), 64))
        k = int(counts[2])
        return eig[:k], basis[:k], counts, kappa[~np.isnan(kappa)]

    def cond_estimate(self, basis, eig, seed):
        basis = np.ascontiguousarray(np.atleast_2d(basis), np.float64)
        out = C.c_double()
        _chk(lib().oracle_cond_estimate(self.sc.h, self.h, basis.shape[0], _p(basis),
                                        _p(np.ascontiguousarray(eig, np.float64)), seed, C.byref(out)))
        return out.value

    def __del__(self):
        try:
            lib().oracle_traj_destroy(self.h)
        except Exception:
            pass


def thin_qr(y):
    """y: (n, l) numpy array. Returns q (n, l), r (l, l), number of deficient columns."""
    n, l = y.shape
    yc = np.asfortranarray(y)
    q = np.empty((l, n))
    r = np.empty((l, l))
    nd = C.c_int64()
    _chk(lib().oracle_thin_qr(n, l, _p(np.ascontiguousarray(yc.T)), _p(q), _p(r), C.byref(nd)))
    return q.T, r.T, nd.value


def thin_svd(a):
    r, c = a.shape
    k = min(r, c)
    u = np.empty((k, r))
    s = np.empty(k)
    v = np.empty((k, c))
    _chk(lib().oracle_thin_svd(r, c, _p(np.ascontiguousarray(a.T)), _p(u), _p(s), _p(v)))
    return u.T, s, v.T


def woodbury(basis, lam, v):
    """basis: (n, l)."""
    n, l = basis.shape
    out = np.empty(n)
    _chk(lib().oracle_woodbury(n, l, _p(np.ascontiguousarray(basis.T)), _p(np.ascontiguousarray(lam, float)),
                               _p(np.ascontiguousarray(v, float)), _p(out)))
    return out


def pcg_dense(a, rhs, minv=None, tol=1e-10, max_iter=1000):
    n = a.shape[0]
    x = np.empty(n)
    it = C.c_int()
    conv = C.c_int()
    mi = None if minv is None else np.ascontiguousarray(minv.T)
    _chk(lib().oracle_pcg_dense(n, _p(np.ascontiguousarray(a.T)), _p(np.ascontiguousarray(rhs, float)), _p(mi),
                                tol, max_iter, _p(x), C.byref(it), C.byref(conv)))
    return x, it.value, bool(conv.value)


def sketch_dense(a, method, rank, seed, rank2=-1):
    """Sketch of H = A^T A for dense A (m, n)."""
    m, n = a.shape
    eig = np.empty(rank)
    basis = np.empty((rank, n))
    _chk(lib().oracle_sketch_dense(m, n, _p(np.ascontiguousarray(a.T)), method, rank, rank2, seed, _p(eig),
                                   _p(basis)))
    return eig, basis.T


def bve_fixture(nx, ny, re, ro, dt, steps, seed):
    out = np.empty(nx * ny)
    _chk(lib().oracle_bve_fixture(nx, ny, re, ro, dt, steps, seed, _p(out)))
    return out


def bve_op(n, op, a, b=None):
    out = np.empty(n * n)
    bb = None if b is None else np.ascontiguousarray(b, np.float64)
    _chk(lib().oracle_bve_op(n, op, _p(np.ascontiguousarray(a, np.float64)), _p(bb), _p(out)))
    return out

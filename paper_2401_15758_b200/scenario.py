"""Synthetic twin-experiment inputs for the five BASELINE.json configs.

Product-side generator (no oracle involvement): the truth, observations and
background follow the reference harness conventions
(/root/reference/proj/src/harness.cpp:432-527; seeds per SURVEY.md Appendix C):
  truth      Burgers: sin(2 pi x) + 0.5 sin(4 pi x); BVE: Gaussian random field
             with vorticity power ∝ k^4 exp(-(k/4)^2) from gaussian_vector(n^2, mix_seed(0, 7)), rms 1
  background truth + B^{1/2} gaussian_vector(n, mix_seed(0, 2))
  obs noise  sigma_o * gaussian_vector(n_obs, mix_seed(1, 100 + i)), observed at the END of interval i
The model integrations (truth trajectory, B^{1/2}) run on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import api

MODES = api.MODES


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    model: int
    n: int
    nu: float
    dt: float
    steps: int
    spi: int
    obs_stride: int
    corr_len: float
    sigma_b: float
    sigma_o: float
    mode: str
    method: int
    rank: int
    growth: int
    max_rank: int
    gn_iters: int
    pcg_tol: float

    @property
    def n_t(self):
        return self.steps // self.spi

    @property
    def dim(self):
        return self.n if self.model == api.MODEL_BURGERS else self.n * self.n

    def gn_kwargs(self):
        kw = dict(mode=self.mode, method=self.method, rank=self.rank, growth=self.growth, max_rank=self.max_rank,
                  eps_sketch=1.5, eps_reuse=10.0, seed=2, grad_tol=1e-12, pcg_tol=self.pcg_tol,
                  max_gn_iters=self.gn_iters)
        if self.max_rank > 0:
            kw["rank2"] = 2 * self.max_rank + 1
        return kw


CONFIGS = [
    ConfigSpec("C0-burgers-256", api.MODEL_BURGERS, 256, 0.005, 1e-3, 100, 10, 4, 0.05, 0.1, 0.01, "SketchPrec",
               api.RANDSVD, 30, 10, -1, 5, 1e-6),
    ConfigSpec("C1-burgers-4096", api.MODEL_BURGERS, 4096, 1e-4, 1e-4, 1000, 50, 8, 0.02, 0.1, 0.01, "SketchPrec",
               api.RANDSVD, 60, 10, -1, 5, 1e-8),
    ConfigSpec("C2-bve-128", api.MODEL_BVE, 128, 1e-4, 0.01, 200, 20, 4, 0.3, 0.2, 0.05, "SketchPrec", api.NYSTROM,
               50, 10, -1, 5, 1e-6),
    ConfigSpec("C3-bve-512", api.MODEL_BVE, 512, 1e-4, 0.0025, 800, 80, 8, 0.3, 0.2, 0.05, "SketchPrec",
               api.RANDSVD, 110, 10, -1, 3, 1e-6),
    ConfigSpec("C4-bve-256-adaptive", api.MODEL_BVE, 256, 1e-4, 0.005, 400, 20, 4, 0.3, 0.2, 0.05, "SketchPrecA",
               api.NYSTROM, 10, 10, 100, 8, 1e-6),
]


def grf_truth(n, seed):
    w = api.gaussian_vector(n * n, seed).reshape(n, n)  # [j][i], x fastest
    k = np.fft.fftfreq(n, 1.0 / n)
    kk = np.sqrt(k[None, :] ** 2 + k[:, None] ** 2)
    p = kk ** 4 * np.exp(-(kk / 4.0) ** 2)
    f = np.fft.ifft2(np.fft.fft2(w) * np.sqrt(p)).real.reshape(-1)
    f -= f.mean()
    return f / np.sqrt(np.mean(f * f))


def obs_indices(spec):
    if spec.model == api.MODEL_BURGERS:
        return np.arange(0, spec.n, spec.obs_stride, dtype=np.int64)
    g = np.arange(0, spec.n, spec.obs_stride, dtype=np.int64)
    return (g[None, :] + spec.n * g[:, None]).reshape(-1)


@dataclass
class Scenario:
    spec: ConfigSpec
    problem: api.Problem
    truth0: np.ndarray
    truth_states: list


def build(cfg, block_group=0, steps=None):
    """Build config `cfg` (index or ConfigSpec). `steps` truncates the window (tests)."""
    spec = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if steps is not None:
        spec = ConfigSpec(**{**spec.__dict__, "steps": steps})
    n, dim, n_t = spec.n, spec.dim, spec.n_t
    if spec.model == api.MODEL_BURGERS:
        x = np.arange(n) / n
        truth0 = np.sin(2 * np.pi * x) + 0.5 * np.sin(4 * np.pi * x)
    else:
        truth0 = grf_truth(n, api.mix_seed(0, 7))
    idx = obs_indices(spec)
    n_obs = idx.size
    common = (spec.model, n, spec.nu, spec.dt, n_t, spec.spi, spec.sigma_b, spec.corr_len)
    shell = api.Problem(*common, np.zeros(0, np.int64), np.zeros(0), np.zeros(0), truth0, block_group=block_group)
    states = [truth0]
    x = truth0
    for _ in range(n_t):
        x = shell.forward(x, spec.spi)
        states.append(x)
    background = truth0 + shell.prior_sqrt(api.gaussian_vector(dim, api.mix_seed(0, 2)))[0]
    shell.close()
    values = np.empty((n_t, n_obs))
    for i in range(n_t):
        noise = api.gaussian_vector(n_obs, api.mix_seed(1, 100 + i))
        values[i] = states[i + 1][idx] + spec.sigma_o * noise
    variances = np.full((n_t, n_obs), spec.sigma_o ** 2)
    prob = api.Problem(*common, idx, values, variances, background, block_group=block_group)
    return Scenario(spec, prob, truth0, states)


def with_window(spec, steps=None, spi=None):
    """Same grid/physics with a shorter window (parity cases at full grid size)."""
    upd = {}
    if spi is not None and spi > 0:
        upd["spi"] = spi
    if steps is not None and steps > 0:
        upd["steps"] = steps
    return ConfigSpec(**{**spec.__dict__, **upd}) if upd else spec


def from_arrays(spec, indices, values, variances, background, block_group=0, steps=None, spi=None):
    """Problem for `spec` from explicit arrays (e.g. the oracle's scenario)."""
    spec = with_window(spec, steps, spi)
    return api.Problem(spec.model, spec.n, spec.nu, spec.dt, spec.n_t, spec.spi, spec.sigma_b, spec.corr_len,
                       indices, values, variances, background, block_group=block_group)

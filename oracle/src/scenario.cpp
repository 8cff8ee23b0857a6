// CPU ORACLE (test infrastructure only): scenario generation for the five
// BASELINE.json configs and the reference's burgers_1_1 preset / BVE truth
// fixture. Seed/stream conventions follow proj/src/harness.cpp:33-37,
// :432-527, :735-755 and SURVEY.md Appendix C.
#include "oracle.hpp"

#include <algorithm>

namespace oracle {

namespace {
constexpr uint64_t kBackgroundStream = 2;  // proj/src/harness.cpp:33
constexpr uint64_t kSpinupStream = 7;      // proj/src/harness.cpp:34
constexpr uint64_t kSolverSketchStream = 42;
constexpr uint64_t kObsStream = 100;

struct CfgSpec {
  bool bve;
  int n;
  double nu, dt;
  int steps, spi, stride;
  double corr_len, sigma_b, sigma_o;
  SolveMode mode;
  SketchMethod method;
  int rank, growth, max_rank, gn_iters;
  double pcg_tol;
};

const CfgSpec kSpecs[5] = {
    // C0: Burgers n=256
    {false, 256, 0.005, 1e-3, 100, 10, 4, 0.05, 0.1, 0.01, SolveMode::SketchPrec, SketchMethod::RandSVD, 30, 10, -1,
     5, 1e-6},
    // C1: Burgers n=4096
    {false, 4096, 1e-4, 1e-4, 1000, 50, 8, 0.02, 0.1, 0.01, SolveMode::SketchPrec, SketchMethod::RandSVD, 60, 10, -1,
     5, 1e-8},
    // C2: BVE 128^2
    {true, 128, 1e-4, 0.01, 200, 20, 4, 0.3, 0.2, 0.05, SolveMode::SketchPrec, SketchMethod::Nystrom, 50, 10, -1, 5,
     1e-6},
    // C3: BVE 512^2
    {true, 512, 1e-4, 0.0025, 800, 80, 8, 0.3, 0.2, 0.05, SolveMode::SketchPrec, SketchMethod::RandSVD, 110, 10, -1,
     3, 1e-6},
    // C4: BVE 256^2 adaptive (start 10, +10 per pass, capped at 100)
    {true, 256, 1e-4, 0.005, 400, 20, 4, 0.3, 0.2, 0.05, SolveMode::SketchPrecA, SketchMethod::Nystrom, 10, 10, 100,
     8, 1e-6},
};
}  // namespace

// Gaussian random field, isotropic vorticity power spectrum ∝ k^4 exp(-(k/4)^2)
// (random phases from a seeded white-noise field), rms normalised to 1.
Vec periodic_grf_truth(int n, uint64_t seed) {
  const size_t nn = static_cast<size_t>(n) * n;
  const Vec w = gaussian_vector(static_cast<int64_t>(nn), seed);
  std::vector<cplx> z(nn);
  for (size_t i = 0; i < nn; ++i) z[i] = cplx(w[i], 0.0);
  fft2_inplace(z, n, n, false);
  auto kk = [n](int k) { return k <= n / 2 ? k : k - n; };
  for (int ky = 0; ky < n; ++ky)
    for (int kx = 0; kx < n; ++kx) {
      const double k = std::sqrt(static_cast<double>(kk(kx) * kk(kx) + kk(ky) * kk(ky)));
      const double p = k * k * k * k * std::exp(-(k / 4.0) * (k / 4.0));
      z[kx + static_cast<size_t>(n) * ky] *= std::sqrt(p);
    }
  fft2_inplace(z, n, n, true);
  Vec o(nn);
  double mean = 0.0;
  for (size_t i = 0; i < nn; ++i) mean += (o[i] = z[i].real());
  mean /= static_cast<double>(nn);
  double ss = 0.0;
  for (size_t i = 0; i < nn; ++i) {
    o[i] -= mean;
    ss += o[i] * o[i];
  }
  const double rms = std::sqrt(ss / static_cast<double>(nn));
  for (auto& v : o) v /= rms;
  return o;
}

Scenario make_config(int id, int steps_override, int spi_override) {
  if (id < 0 || id > 4) throw std::invalid_argument("make_config: config id must be 0..4");
  CfgSpec c = kSpecs[id];
  if (spi_override > 0) c.spi = spi_override;
  if (steps_override > 0) {
    if (steps_override % c.spi) throw std::invalid_argument("make_config: steps must be a multiple of spi");
    c.steps = steps_override;
  }
  Scenario sc;
  sc.name = "config" + std::to_string(id);
  AssimilationProblem& p = sc.problem;
  const int n_t = c.steps / c.spi;
  std::vector<int64_t> idx;
  if (!c.bve) {
    p.model = std::make_shared<PeriodicBurgers>(c.n, c.nu, c.dt);
    p.prior = std::make_shared<FourierPrior>(c.n, 1, c.sigma_b, c.corr_len);
    sc.truth0.resize(static_cast<size_t>(c.n));
    for (int i = 0; i < c.n; ++i) {
      const double x = static_cast<double>(i) / c.n;
      sc.truth0[i] = std::sin(2.0 * M_PI * x) + 0.5 * std::sin(4.0 * M_PI * x);
    }
    for (int i = 0; i < c.n; i += c.stride) idx.push_back(i);
  } else {
    p.model = std::make_shared<PeriodicBVE>(c.n, c.nu, c.dt);
    p.prior = std::make_shared<FourierPrior>(c.n, 2, c.sigma_b, c.corr_len);
    sc.truth0 = periodic_grf_truth(c.n, mix_seed(0, kSpinupStream));
    for (int j = 0; j < c.n; j += c.stride)
      for (int i = 0; i < c.n; i += c.stride) idx.push_back(i + static_cast<int64_t>(c.n) * j);
  }
  sc.truth_states.push_back(sc.truth0);
  Vec x = sc.truth0;
  for (int i = 1; i <= n_t; ++i) {
    x = p.model->forward(x, c.spi);
    sc.truth_states.push_back(x);
  }
  const int64_t no = static_cast<int64_t>(idx.size());
  p.obs.indices = idx;
  p.obs.values = Mat(no, n_t);
  p.obs.variances = Mat(no, n_t);
  for (auto& v : p.obs.variances.a) v = c.sigma_o * c.sigma_o;
  for (int i = 0; i < n_t; ++i) {
    const Vec noise = gaussian_vector(no, mix_seed(1, kObsStream + static_cast<uint64_t>(i)));
    for (int64_t k = 0; k < no; ++k) p.obs.values(k, i) = sc.truth_states[i + 1][idx[k]] + c.sigma_o * noise[k];
  }
  p.background = p.prior->sample_background(sc.truth0, mix_seed(0, kBackgroundStream));
  p.n_t = n_t;
  p.steps_per_interval = c.spi;
  p.validate();

  GNConfig& g = sc.gn;
  g.mode = c.mode;
  g.sketch.method = c.method;
  g.sketch.rank = c.rank;
  g.sketch.growth = c.growth;
  g.sketch.max_rank = c.max_rank;
  if (c.max_rank > 0) g.sketch.rank2 = 2 * c.max_rank + 1;
  g.sketch.eps_sketch = 1.5;
  g.sketch.eps_reuse = 10.0;
  g.sketch.seed = 2;
  g.grad_tol = 1e-12;
  g.pcg_tol = c.pcg_tol;
  g.max_gn_iters = c.gn_iters;
  return sc;
}

// Preset burgers_1_1 (proj/src/harness.cpp:226-248, :432-527, :753-755).
Scenario make_reference_burgers_1_1() {
  Scenario sc;
  sc.name = "burgers_1_1";
  const uint64_t master = 2;
  const int n = 399, n_t = 20, spi = 400;
  AssimilationProblem& p = sc.problem;
  p.model = std::make_shared<DirichletBurgers>(n, 0.1, 2.5e-5);
  p.prior = LaplacianPrior::make_1d(n, 0.5, 500.0, 1.0);
  sc.truth0.resize(n);
  for (int i = 0; i < n; ++i) sc.truth0[i] = std::sin(M_PI * (i + 1) / (n + 1));
  std::vector<int64_t> idx;
  for (int j = 1; j <= 15; ++j) idx.push_back(static_cast<int64_t>(std::llround(j * (n + 1) / 16.0)) - 1);
  sc.truth_states.push_back(sc.truth0);
  Vec x = sc.truth0;
  for (int i = 1; i <= n_t; ++i) {
    x = p.model->forward(x, spi);
    sc.truth_states.push_back(x);
  }
  p.obs.indices = idx;
  p.obs.values = Mat(15, n_t);
  p.obs.variances = Mat(15, n_t);
  for (auto& v : p.obs.variances.a) v = 0.01;
  for (int i = 0; i < n_t; ++i) {
    const Vec noise = gaussian_vector(15, mix_seed(master, kObsStream + static_cast<uint64_t>(i)));
    for (int k = 0; k < 15; ++k) p.obs.values(k, i) = sc.truth_states[i + 1][idx[k]] + std::sqrt(0.01) * noise[k];
  }
  p.background = p.prior->sample_background(sc.truth0, mix_seed(master, kBackgroundStream));
  p.n_t = n_t;
  p.steps_per_interval = spi;
  p.validate();
  sc.gn.mode = SolveMode::SketchPrec;
  sc.gn.sketch.method = SketchMethod::RandSVD;
  sc.gn.sketch.rank = 15;
  sc.gn.sketch.growth = 5;
  sc.gn.max_gn_iters = 20;
  sc.gn.sketch.seed = mix_seed(master, kSolverSketchStream);
  return sc;
}

// Preset bve_2 (proj/src/harness.cpp:285-309, scenario generation :432-527):
// 64 x 129 Dirichlet BVE (RK3-TVD, Re 200, Ro 0.0016), dt 0.001225 split into
// spi = 4 inner steps, n_t = 8, 16 x 16 sensor grid (:85-103), obs variance
// 361, prior (alpha I - beta Lap*)^{-2} with alpha 0, beta 0.06 and unscaled
// stencil, truth = the spun-up fixture field (600 steps, mix_seed(1234, 7)).
Scenario make_reference_bve_2() {
  Scenario sc;
  sc.name = "bve_2";
  const uint64_t master = 1234;
  const int nx = 64, ny = 129, n_t = 8, spi = 4;
  const double re = 200.0, ro = 0.0016, dt = 0.001225 / spi, var = 361.0;
  AssimilationProblem& p = sc.problem;
  p.model = std::make_shared<DirichletBVE>(nx, ny, re, ro, dt);
  p.prior = LaplacianPrior::make_2d(nx, ny, 0.0, 0.06);
  sc.truth0 = bve_truth_fixture_regen(nx, ny, re, ro, dt, 600, mix_seed(master, kSpinupStream));
  std::vector<int64_t> idx;
  for (int l = 1; l <= 16; ++l) {
    const long long iy = std::llround(l * (ny + 1) / 17.0);
    for (int k = 1; k <= 16; ++k) {
      const long long ix = std::llround(k * (nx + 1) / 17.0);
      idx.push_back((ix - 1) + static_cast<long long>(nx) * (iy - 1));
    }
  }
  sc.truth_states.push_back(sc.truth0);
  Vec x = sc.truth0;
  for (int i = 1; i <= n_t; ++i) {
    x = p.model->forward(x, spi);
    sc.truth_states.push_back(x);
  }
  const int64_t no = static_cast<int64_t>(idx.size());
  p.obs.indices = idx;
  p.obs.values = Mat(no, n_t);
  p.obs.variances = Mat(no, n_t);
  for (auto& v : p.obs.variances.a) v = var;
  for (int i = 0; i < n_t; ++i) {
    const Vec noise = gaussian_vector(no, mix_seed(master, kObsStream + static_cast<uint64_t>(i)));
    for (int64_t k = 0; k < no; ++k)
      p.obs.values(k, i) = sc.truth_states[i + 1][idx[k]] + std::sqrt(var) * noise[k];
  }
  p.background = p.prior->sample_background(sc.truth0, mix_seed(master, kBackgroundStream));
  p.n_t = n_t;
  p.steps_per_interval = spi;
  p.validate();
  sc.gn.mode = SolveMode::SketchPrec;
  sc.gn.sketch.method = SketchMethod::RandSVD;
  sc.gn.sketch.rank = 192;
  sc.gn.sketch.growth = 64;
  sc.gn.sketch.eps_sketch = 1.5;
  sc.gn.sketch.eps_reuse = 50.0;
  sc.gn.max_gn_iters = 4;
  sc.gn.pcg_max_iter = 4000;
  sc.gn.sketch.seed = mix_seed(master, kSolverSketchStream);
  return sc;
}

// proj/src/harness.cpp:119-170: seeded smooth field, scaled to max 50, spun up.
Vec bve_truth_fixture_regen(int nx, int ny, double re, double ro, double dt, int steps, uint64_t seed) {
  const DirichletBVE model(nx, ny, re, ro, dt);
  const auto smooth = LaplacianPrior::make_2d(nx, ny, 0.0, 0.06);
  Vec f = smooth->apply_sqrt(gaussian_vector(model.dim(), seed));
  const double mx = std::max(1e-12, norm_inf(f));
  for (auto& v : f) v *= 50.0 / mx;
  return model.forward(f, steps);
}

}  // namespace oracle

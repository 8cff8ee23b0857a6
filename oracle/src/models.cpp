// CPU ORACLE (test infrastructure only): dynamical models and priors.
//  * PeriodicBurgers / PeriodicBVE: the BASELINE.json config discretisations,
//    written as new implementations of the reference interfaces
//    (proj/include/sketchdav/model.hpp:14-41) following the reference's
//    stage-by-stage discrete TLM/ADJ pattern (proj/src/burgers.cpp:218-236,
//    proj/src/bve.cpp:184-211), extended to RK4.
//  * DirichletBurgers / DirichletBVE / Tridiagonal1D / DirichletSolver2D /
//    LaplacianPrior: faithful restatements of proj/src/{burgers,bve,dirichlet,
//    prior}.cpp used to pin the oracle to the reference fixture and bands.
#include "oracle.hpp"

#include <algorithm>
#include <array>

namespace oracle {

// =========================================================== periodic Burgers
PeriodicBurgers::PeriodicBurgers(int n, double nu, double dt) : n_(n), nu_(nu), dt_(dt) {
  if (n < 3 || nu < 0.0 || dt <= 0.0) throw std::invalid_argument("PeriodicBurgers: invalid parameters");
}

namespace {
inline int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
}  // namespace

// f(u) = -u D1 u + nu D2 u (advective form, as proj/src/burgers.cpp:56-61).
Vec PeriodicBurgers::rhs(const Vec& u) const {
  const double c1 = 0.5 * n_, c2 = static_cast<double>(n_) * n_;
  Vec f(n_);
  for (int i = 0; i < n_; ++i) {
    const double l = u[wrap(i - 1, n_)], r = u[wrap(i + 1, n_)];
    f[i] = -u[i] * (r - l) * c1 + nu_ * (l - 2.0 * u[i] + r) * c2;
  }
  return f;
}
// J(u) d = -d D1u - u D1d + nu D2 d (proj/src/burgers.cpp:63-72).
Vec PeriodicBurgers::rhs_jacobian(const Vec& u, const Vec& d) const {
  const double c1 = 0.5 * n_, c2 = static_cast<double>(n_) * n_;
  Vec f(n_);
  for (int i = 0; i < n_; ++i) {
    const int im = wrap(i - 1, n_), ip = wrap(i + 1, n_);
    const double du = (u[ip] - u[im]) * c1, dd = (d[ip] - d[im]) * c1;
    f[i] = -d[i] * du - u[i] * dd + nu_ * (d[im] - 2.0 * d[i] + d[ip]) * c2;
  }
  return f;
}
// J(u)^T lam = -lam D1u + D1(u lam) + nu D2 lam; periodic D1^T = -D1
// (proj/src/burgers.cpp:74-86).
Vec PeriodicBurgers::rhs_jacobian_adjoint(const Vec& u, const Vec& lam) const {
  const double c1 = 0.5 * n_, c2 = static_cast<double>(n_) * n_;
  Vec f(n_);
  for (int i = 0; i < n_; ++i) {
    const int im = wrap(i - 1, n_), ip = wrap(i + 1, n_);
    const double du = (u[ip] - u[im]) * c1;
    const double dul = (u[ip] * lam[ip] - u[im] * lam[im]) * c1;
    f[i] = -lam[i] * du + dul + nu_ * (lam[im] - 2.0 * lam[i] + lam[ip]) * c2;
  }
  return f;
}
// Classical RK4.
Vec PeriodicBurgers::step(const Vec& u) const {
  const double dt = dt_;
  const Vec k1 = rhs(u);
  const Vec k2 = rhs(axpby(1.0, u, 0.5 * dt, k1));
  const Vec k3 = rhs(axpby(1.0, u, 0.5 * dt, k2));
  const Vec k4 = rhs(axpby(1.0, u, dt, k3));
  Vec o(n_);
  for (int i = 0; i < n_; ++i) o[i] = u[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  return o;
}
Vec PeriodicBurgers::forward(const Vec& x0, int steps) const {
  if (static_cast<int>(x0.size()) != n_) throw std::invalid_argument("PeriodicBurgers::forward: size mismatch");
  Vec u = x0;
  for (int k = 0; k < steps; ++k) {
    u = step(u);
    if (!all_finite(u))
      throw std::runtime_error("PeriodicBurgers::forward: non-finite state at step " + std::to_string(k + 1));
  }
  return u;
}

namespace {
// RK4 discrete TLM/ADJ over stored stage inputs.
template <class Jac, class JacT>
Vec rk4_tlm_step(const std::array<const Vec*, 4>& st, const Vec& d, double dt, const Jac& jac) {
  const size_t n = d.size();
  const Vec k1 = jac(*st[0], d);
  const Vec k2 = jac(*st[1], axpby(1.0, d, 0.5 * dt, k1));
  const Vec k3 = jac(*st[2], axpby(1.0, d, 0.5 * dt, k2));
  const Vec k4 = jac(*st[3], axpby(1.0, d, dt, k3));
  Vec o(n);
  for (size_t i = 0; i < n; ++i) o[i] = d[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  (void)sizeof(JacT);
  return o;
}
template <class JacT>
Vec rk4_adj_step(const std::array<const Vec*, 4>& st, const Vec& lam, double dt, const JacT& jt) {
  const size_t n = lam.size();
  const Vec m4 = jt(*st[3], scaled(dt / 6.0, lam));
  const Vec m3 = jt(*st[2], axpby(dt / 3.0, lam, dt, m4));
  const Vec m2 = jt(*st[1], axpby(dt / 3.0, lam, 0.5 * dt, m3));
  const Vec m1 = jt(*st[0], axpby(dt / 6.0, lam, 0.5 * dt, m2));
  Vec o(n);
  for (size_t i = 0; i < n; ++i) o[i] = lam[i] + m1[i] + m2[i] + m3[i] + m4[i];
  return o;
}

class PeriodicBurgersTrajectory final : public LinearizedTrajectory {
 public:
  PeriodicBurgersTrajectory(const PeriodicBurgers& m, const Vec& x0, int steps)
      : m_(m), steps_(steps), stages_(static_cast<size_t>(steps) * 4) {
    const double dt = m.inner_dt();
    Vec u = x0;
    for (int k = 0; k < steps; ++k) {
      stages_[4 * k] = u;
      const Vec k1 = m.rhs(u);
      stages_[4 * k + 1] = axpby(1.0, u, 0.5 * dt, k1);
      const Vec k2 = m.rhs(stages_[4 * k + 1]);
      stages_[4 * k + 2] = axpby(1.0, u, 0.5 * dt, k2);
      const Vec k3 = m.rhs(stages_[4 * k + 2]);
      stages_[4 * k + 3] = axpby(1.0, u, dt, k3);
      const Vec k4 = m.rhs(stages_[4 * k + 3]);
      Vec o(u.size());
      for (size_t i = 0; i < u.size(); ++i) o[i] = u[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
      u = std::move(o);
      if (!all_finite(u))
        throw std::runtime_error("PeriodicBurgers::linearize: non-finite state at step " + std::to_string(k + 1));
    }
    final_ = u;
  }
  int total_steps() const override { return steps_; }
  Vec state_at(int step) const override {
    if (step < 0 || step > steps_) throw std::invalid_argument("trajectory: step out of range");
    return step == steps_ ? final_ : stages_[4 * step];
  }
  Vec tlm_range(int b, int e, const Vec& dx) const override {
    check(b, e);
    Vec d = dx;
    auto jac = [&](const Vec& u, const Vec& x) { return m_.rhs_jacobian(u, x); };
    for (int k = b; k < e; ++k) d = rk4_tlm_step<decltype(jac), int>(st(k), d, m_.inner_dt(), jac);
    return d;
  }
  Vec adj_range(int b, int e, const Vec& lambda) const override {
    check(b, e);
    Vec l = lambda;
    auto jt = [&](const Vec& u, const Vec& x) { return m_.rhs_jacobian_adjoint(u, x); };
    for (int k = e - 1; k >= b; --k) l = rk4_adj_step(st(k), l, m_.inner_dt(), jt);
    return l;
  }
  const Vec& stage(int k, int s) const { return stages_[4 * k + s]; }

 private:
  std::array<const Vec*, 4> st(int k) const {
    return {&stages_[4 * k], &stages_[4 * k + 1], &stages_[4 * k + 2], &stages_[4 * k + 3]};
  }
  void check(int b, int e) const {
    if (b < 0 || e > steps_ || b > e) throw std::invalid_argument("trajectory: step range out of bounds");
  }
  const PeriodicBurgers m_;
  int steps_;
  std::vector<Vec> stages_;
  Vec final_;
};
}  // namespace

std::shared_ptr<const LinearizedTrajectory> PeriodicBurgers::linearize(const Vec& x0, int steps, int) const {
  if (static_cast<int>(x0.size()) != n_) throw std::invalid_argument("PeriodicBurgers::linearize: size mismatch");
  return std::make_shared<PeriodicBurgersTrajectory>(*this, x0, steps);
}

// =============================================================== periodic BVE
PeriodicBVE::PeriodicBVE(int n, double nu, double dt) : n_(n), nu_(nu), dt_(dt) {
  if (n < 4 || (n & (n - 1)) || nu < 0.0 || dt <= 0.0)
    throw std::invalid_argument("PeriodicBVE: invalid parameters (n must be a power of two)");
  const double h = 2.0 * M_PI / n;
  inv_symbol_.assign(static_cast<size_t>(n) * n, 0.0);
  for (int ky = 0; ky < n; ++ky)
    for (int kx = 0; kx < n; ++kx) {
      const double sx = std::sin(M_PI * kx / n), sy = std::sin(M_PI * ky / n);
      const double mu = 4.0 / (h * h) * (sx * sx + sy * sy);
      inv_symbol_[kx + static_cast<size_t>(n) * ky] =
          (kx == 0 && ky == 0) ? 0.0 : 1.0 / (mu * static_cast<double>(n) * n);
    }
}

// psi = (-Lap5)^{-1} w with psi_hat(0) = 0 (SURVEY.md Appendix A "Poisson").
Vec PeriodicBVE::poisson(const Vec& w) const {
  const size_t nn = static_cast<size_t>(n_) * n_;
  std::vector<cplx> z(nn);
  for (size_t i = 0; i < nn; ++i) z[i] = cplx(w[i], 0.0);
  fft2_inplace(z, n_, n_, false);
  for (size_t i = 0; i < nn; ++i) z[i] *= inv_symbol_[i];
  fft2_inplace(z, n_, n_, true);
  Vec o(nn);
  for (size_t i = 0; i < nn; ++i) o[i] = z[i].real();
  return o;
}

// Arakawa (1966) Jacobian J(a,b) ~ a_x b_y - a_y b_x = (J++ + J+x + Jx+)/3.
Vec PeriodicBVE::arakawa(const Vec& a, const Vec& b) const {
  const int n = n_;
  const double h = 2.0 * M_PI / n;
  const double s = 1.0 / (12.0 * h * h);
  Vec o(static_cast<size_t>(n) * n);
  auto A = [&](int i, int j) { return a[wrap(i, n) + static_cast<size_t>(n) * wrap(j, n)]; };
  auto B = [&](int i, int j) { return b[wrap(i, n) + static_cast<size_t>(n) * wrap(j, n)]; };
  par_for(n, [&](int64_t j0, int64_t j1) {
  for (int j = static_cast<int>(j0); j < j1; ++j)
    for (int i = 0; i < n; ++i) {
      const double jpp = (A(i + 1, j) - A(i - 1, j)) * (B(i, j + 1) - B(i, j - 1)) -
                         (A(i, j + 1) - A(i, j - 1)) * (B(i + 1, j) - B(i - 1, j));
      const double jpx = A(i + 1, j) * (B(i + 1, j + 1) - B(i + 1, j - 1)) -
                         A(i - 1, j) * (B(i - 1, j + 1) - B(i - 1, j - 1)) -
                         A(i, j + 1) * (B(i + 1, j + 1) - B(i - 1, j + 1)) +
                         A(i, j - 1) * (B(i + 1, j - 1) - B(i - 1, j - 1));
      const double jxp = B(i, j + 1) * (A(i + 1, j + 1) - A(i - 1, j + 1)) -
                         B(i, j - 1) * (A(i + 1, j - 1) - A(i - 1, j - 1)) -
                         B(i + 1, j) * (A(i + 1, j + 1) - A(i + 1, j - 1)) +
                         B(i - 1, j) * (A(i - 1, j + 1) - A(i - 1, j - 1));
      o[i + static_cast<size_t>(n) * j] = (jpp + jpx + jxp) * s;
    }
  });
  return o;
}

Vec PeriodicBVE::laplacian(const Vec& f) const {
  const int n = n_;
  const double h = 2.0 * M_PI / n, c = 1.0 / (h * h);
  Vec o(static_cast<size_t>(n) * n);
  par_for(n, [&](int64_t j0, int64_t j1) {
  for (int j = static_cast<int>(j0); j < j1; ++j)
    for (int i = 0; i < n; ++i) {
      const size_t id = i + static_cast<size_t>(n) * j;
      o[id] = (f[wrap(i + 1, n) + static_cast<size_t>(n) * j] + f[wrap(i - 1, n) + static_cast<size_t>(n) * j] +
               f[i + static_cast<size_t>(n) * wrap(j + 1, n)] + f[i + static_cast<size_t>(n) * wrap(j - 1, n)] -
               4.0 * f[id]) * c;
    }
  });
  return o;
}

// w_t = J(psi, w) + nu Lap w,  -Lap psi = w  (reference sign convention
// w_t + (psi_y w_x - psi_x w_y) = ..., proj/include/sketchdav/bve.hpp:10-20).
Vec PeriodicBVE::rhs(const Vec& w) const {
  const Vec psi = poisson(w);
  const Vec j = arakawa(psi, w);
  const Vec l = laplacian(w);
  Vec o(w.size());
  for (size_t i = 0; i < w.size(); ++i) o[i] = j[i] + nu_ * l[i];
  return o;
}

Vec PeriodicBVE::step(const Vec& u) const {
  const double dt = dt_;
  const Vec k1 = rhs(u);
  const Vec k2 = rhs(axpby(1.0, u, 0.5 * dt, k1));
  const Vec k3 = rhs(axpby(1.0, u, 0.5 * dt, k2));
  const Vec k4 = rhs(axpby(1.0, u, dt, k3));
  Vec o(u.size());
  for (size_t i = 0; i < u.size(); ++i) o[i] = u[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  return o;
}

Vec PeriodicBVE::forward(const Vec& x0, int steps) const {
  if (static_cast<int64_t>(x0.size()) != dim()) throw std::invalid_argument("PeriodicBVE::forward: size mismatch");
  Vec u = x0;
  for (int k = 0; k < steps; ++k) {
    u = step(u);
    if (!all_finite(u))
      throw std::runtime_error("PeriodicBVE::forward: non-finite state at step " + std::to_string(k + 1));
  }
  return u;
}

namespace {
// Stores each step's initial state; stage inputs (w_s, psi_s) are recomputed
// per step on demand (bitwise identical to the forward integration) so the
// oracle's memory stays at one field per step.
class PeriodicBVETrajectory final : public LinearizedTrajectory {
 public:
  PeriodicBVETrajectory(const PeriodicBVE& m, const Vec& x0, int steps) : m_(m), steps_(steps) {
    states_.reserve(static_cast<size_t>(steps) + 1);
    states_.push_back(x0);
    Vec u = x0;
    for (int k = 0; k < steps; ++k) {
      u = m_.step(u);
      if (!all_finite(u))
        throw std::runtime_error("PeriodicBVE::linearize: non-finite state at step " + std::to_string(k + 1));
      states_.push_back(u);
    }
    const double bytes = 8.0 * static_cast<double>(steps) * 8.0 * static_cast<double>(x0.size());
    if (bytes <= 4e9) {
      cache_w_.resize(static_cast<size_t>(steps) * 4);
      cache_p_.resize(static_cast<size_t>(steps) * 4);
      std::array<Vec, 4> w, psi;
      for (int k = 0; k < steps; ++k) {
        compute_stages(k, w, psi);
        for (int s = 0; s < 4; ++s) {
          cache_w_[4 * k + s] = std::move(w[s]);
          cache_p_[4 * k + s] = std::move(psi[s]);
        }
      }
    }
  }
  int total_steps() const override { return steps_; }
  Vec state_at(int step) const override {
    if (step < 0 || step > steps_) throw std::invalid_argument("trajectory: step out of range");
    return states_[step];
  }
  // Stage inputs of step k: w_s and psi_s = P w_s, s = 0..3 (cached when the
  // whole stage store fits in 4 GB, otherwise recomputed per step).
  void stages(int k, std::array<Vec, 4>& w, std::array<Vec, 4>& psi) const {
    if (!cache_w_.empty()) {
      for (int s = 0; s < 4; ++s) {
        w[s] = cache_w_[4 * k + s];
        psi[s] = cache_p_[4 * k + s];
      }
      return;
    }
    compute_stages(k, w, psi);
  }
  void compute_stages(int k, std::array<Vec, 4>& w, std::array<Vec, 4>& psi) const {
    const double dt = m_.inner_dt();
    const Vec& u = states_[k];
    w[0] = u;
    for (int s = 0; s < 4; ++s) {
      psi[s] = m_.poisson(w[s]);
      if (s == 3) break;
      const Vec j = m_.arakawa(psi[s], w[s]);
      const Vec l = m_.laplacian(w[s]);
      Vec kk(u.size());
      for (size_t i = 0; i < u.size(); ++i) kk[i] = j[i] + m_.nu() * l[i];
      w[s + 1] = axpby(1.0, u, s == 2 ? dt : 0.5 * dt, kk);
    }
  }
  Vec tlm_range(int b, int e, const Vec& dx) const override {
    check(b, e);
    Vec d = dx;
    std::array<Vec, 4> w, psi;
    for (int k = b; k < e; ++k) {
      stages(k, w, psi);
      int s = 0;
      auto jac = [&](const Vec&, const Vec& x) {
        const Vec a = m_.arakawa(psi[s], x);
        const Vec bb = m_.arakawa(m_.poisson(x), w[s]);
        const Vec l = m_.laplacian(x);
        Vec o(x.size());
        for (size_t i = 0; i < x.size(); ++i) o[i] = a[i] + bb[i] + m_.nu() * l[i];
        ++s;
        return o;
      };
      std::array<const Vec*, 4> st{&w[0], &w[1], &w[2], &w[3]};
      d = rk4_tlm_step<decltype(jac), int>(st, d, m_.inner_dt(), jac);
    }
    return d;
  }
  Vec adj_range(int b, int e, const Vec& lambda) const override {
    check(b, e);
    Vec l = lambda;
    std::array<Vec, 4> w, psi;
    for (int k = e - 1; k >= b; --k) {
      stages(k, w, psi);
      // J_s^T a = -J(psi_s, a) - P J(a, w_s) + nu Lap a.
      auto jt = [&](const Vec& ws, const Vec& a) {
        const int s = static_cast<int>(&ws - &w[0]);
        const Vec t1 = m_.arakawa(psi[s], a);
        const Vec t2 = m_.poisson(m_.arakawa(a, w[s]));
        const Vec lp = m_.laplacian(a);
        Vec o(a.size());
        for (size_t i = 0; i < a.size(); ++i) o[i] = -t1[i] - t2[i] + m_.nu() * lp[i];
        return o;
      };
      std::array<const Vec*, 4> st{&w[0], &w[1], &w[2], &w[3]};
      l = rk4_adj_step(st, l, m_.inner_dt(), jt);
    }
    return l;
  }

 private:
  void check(int b, int e) const {
    if (b < 0 || e > steps_ || b > e) throw std::invalid_argument("trajectory: step range out of bounds");
  }
  const PeriodicBVE m_;
  int steps_;
  std::vector<Vec> states_;
  std::vector<Vec> cache_w_, cache_p_;
};
}  // namespace

std::shared_ptr<const LinearizedTrajectory> PeriodicBVE::linearize(const Vec& x0, int steps, int) const {
  if (static_cast<int64_t>(x0.size()) != dim()) throw std::invalid_argument("PeriodicBVE::linearize: size mismatch");
  return std::make_shared<PeriodicBVETrajectory>(*this, x0, steps);
}

// ================================================= reference Dirichlet models
// proj/src/dirichlet.cpp:19-47
Vec neg_laplacian_1d(const Vec& u) {
  const int64_t n = static_cast<int64_t>(u.size());
  Vec o(u.size());
  for (int64_t i = 0; i < n; ++i) {
    const double l = i > 0 ? u[i - 1] : 0.0, r = i + 1 < n ? u[i + 1] : 0.0;
    o[i] = 2.0 * u[i] - l - r;
  }
  return o;
}
Vec neg_laplacian_2d(const Vec& u, int nx, int ny, double sx, double sy) {
  if (static_cast<int64_t>(u.size()) != static_cast<int64_t>(nx) * ny)
    throw std::invalid_argument("neg_laplacian_2d: size mismatch");
  Vec o(u.size());
  for (int j = 0; j < ny; ++j) {
    const int base = j * nx;
    for (int i = 0; i < nx; ++i) {
      const double c = u[base + i];
      const double w = i > 0 ? u[base + i - 1] : 0.0;
      const double e = i + 1 < nx ? u[base + i + 1] : 0.0;
      const double s = j > 0 ? u[base + i - nx] : 0.0;
      const double nn = j + 1 < ny ? u[base + i + nx] : 0.0;
      o[base + i] = sx * (2.0 * c - w - e) + sy * (2.0 * c - s - nn);
    }
  }
  return o;
}

// proj/src/dirichlet.cpp:82-155 (dense sine-matrix path).
DirichletSolver2D::DirichletSolver2D(int nx, int ny, double a, double bx, double by)
    : nx_(nx), ny_(ny), sx_(nx, nx), sy_(ny, ny), inv_eig_(nx, ny) {
  auto mu = [](int k, int n) { return 2.0 - 2.0 * std::cos(static_cast<double>(k) * M_PI / (n + 1.0)); };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const double lam = a + bx * mu(i + 1, nx) + by * mu(j + 1, ny);
      if (!(lam > 0.0)) throw std::invalid_argument("DirichletSolver2D: operator is not positive definite");
      inv_eig_(i, j) = 1.0 / lam;
    }
  auto fill = [](Mat& s, int n) {
    const double nr = std::sqrt(2.0 / (n + 1));
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) s(i, k) = nr * std::sin((i + 1.0) * (k + 1.0) * M_PI / (n + 1));
  };
  fill(sx_, nx);
  fill(sy_, ny);
}
Vec DirichletSolver2D::solve(const Vec& rhs) const {
  if (static_cast<int64_t>(rhs.size()) != static_cast<int64_t>(nx_) * ny_)
    throw std::invalid_argument("DirichletSolver2D::solve: size mismatch");
  Mat f(nx_, ny_);
  f.a = rhs;
  Mat hat = matmul(matmul(sx_, f), sy_);
  for (size_t i = 0; i < hat.a.size(); ++i) hat.a[i] *= inv_eig_.a[i];
  return matmul(matmul(sx_, hat), sy_).a;
}

// proj/src/dirichlet.cpp:157-187
Tridiagonal1D::Tridiagonal1D(int n, double diag, double off) : n_(n), off_(off), pivot_(static_cast<size_t>(n)) {
  if (n < 1) throw std::invalid_argument("Tridiagonal1D: n must be >= 1");
  double d = diag;
  for (int i = 0; i < n; ++i) {
    if (!(d > 0.0)) throw std::runtime_error("Tridiagonal1D: factorization failed");
    pivot_[i] = d;
    d = diag - off * off / d;
  }
}
Vec Tridiagonal1D::solve(const Vec& rhs) const {
  if (static_cast<int>(rhs.size()) != n_) throw std::invalid_argument("Tridiagonal1D::solve: size mismatch");
  Vec y(n_), x(n_);
  y[0] = rhs[0];
  for (int i = 1; i < n_; ++i) y[i] = rhs[i] - off_ / pivot_[i - 1] * y[i - 1];
  x[n_ - 1] = y[n_ - 1] / pivot_[n_ - 1];
  for (int i = n_ - 2; i >= 0; --i) x[i] = (y[i] - off_ * x[i + 1]) / pivot_[i];
  return x;
}

// ---- Dirichlet Burgers, RK3-TVD (proj/src/burgers.cpp) ----
DirichletBurgers::DirichletBurgers(int n, double nu, double dt) : n_(n), nu_(nu), dt_(dt) {
  if (n < 1 || nu < 0.0 || dt <= 0.0) throw std::invalid_argument("BurgersModel: invalid parameters");
}
namespace {
void d1z(const Vec& u, double c, Vec& o) {
  const int64_t n = static_cast<int64_t>(u.size());
  for (int64_t i = 0; i < n; ++i) o[i] = ((i + 1 < n ? u[i + 1] : 0.0) - (i > 0 ? u[i - 1] : 0.0)) * c;
}
void d2z(const Vec& u, double c, Vec& o) {
  const int64_t n = static_cast<int64_t>(u.size());
  for (int64_t i = 0; i < n; ++i) o[i] = ((i > 0 ? u[i - 1] : 0.0) - 2.0 * u[i] + (i + 1 < n ? u[i + 1] : 0.0)) * c;
}
}  // namespace
Vec DirichletBurgers::rhs(const Vec& u) const {
  Vec a(n_), b(n_), o(n_);
  d1z(u, 0.5 * (n_ + 1), a);
  d2z(u, static_cast<double>(n_ + 1) * (n_ + 1), b);
  for (int i = 0; i < n_; ++i) o[i] = -u[i] * a[i] + nu_ * b[i];
  return o;
}
Vec DirichletBurgers::rhs_jacobian(const Vec& u, const Vec& d) const {
  Vec a(n_), b(n_), o(n_);
  d1z(u, 0.5 * (n_ + 1), a);
  for (int i = 0; i < n_; ++i) o[i] = -d[i] * a[i];
  d1z(d, 0.5 * (n_ + 1), a);
  for (int i = 0; i < n_; ++i) o[i] -= u[i] * a[i];
  d2z(d, static_cast<double>(n_ + 1) * (n_ + 1), b);
  for (int i = 0; i < n_; ++i) o[i] += nu_ * b[i];
  return o;
}
Vec DirichletBurgers::rhs_jacobian_adjoint(const Vec& u, const Vec& lam) const {
  Vec a(n_), b(n_), o(n_);
  d1z(u, 0.5 * (n_ + 1), a);
  for (int i = 0; i < n_; ++i) o[i] = -lam[i] * a[i];
  for (int i = 0; i < n_; ++i) b[i] = u[i] * lam[i];
  d1z(b, 0.5 * (n_ + 1), a);
  for (int i = 0; i < n_; ++i) o[i] += a[i];
  d2z(lam, static_cast<double>(n_ + 1) * (n_ + 1), b);
  for (int i = 0; i < n_; ++i) o[i] += nu_ * b[i];
  return o;
}
Vec DirichletBurgers::step(const Vec& u) const {
  const Vec r0 = rhs(u);
  Vec u1(n_), u2(n_), o(n_);
  for (int i = 0; i < n_; ++i) u1[i] = u[i] + dt_ * r0[i];
  const Vec r1 = rhs(u1);
  for (int i = 0; i < n_; ++i) u2[i] = 0.75 * u[i] + 0.25 * (u1[i] + dt_ * r1[i]);
  const Vec r2 = rhs(u2);
  for (int i = 0; i < n_; ++i) o[i] = u[i] / 3.0 + (2.0 / 3.0) * (u2[i] + dt_ * r2[i]);
  return o;
}
Vec DirichletBurgers::forward(const Vec& x0, int steps) const {
  Vec u = x0;
  for (int k = 0; k < steps; ++k) {
    u = step(u);
    if (!all_finite(u))
      throw std::runtime_error("BurgersModel::forward: non-finite state at step " + std::to_string(k + 1) +
                               " (time step too large for stability)");
  }
  return u;
}
namespace {
class DirichletBurgersTrajectory final : public LinearizedTrajectory {
 public:
  DirichletBurgersTrajectory(const DirichletBurgers& m, const Vec& x0, int steps) : m_(m), steps_(steps) {
    states_.push_back(x0);
    Vec u = x0;
    for (int k = 0; k < steps; ++k) {
      u = m_.step(u);
      if (!all_finite(u))
        throw std::runtime_error("BurgersModel::linearize: non-finite state at step " + std::to_string(k + 1));
      states_.push_back(u);
    }
  }
  int total_steps() const override { return steps_; }
  Vec state_at(int s) const override { return states_.at(static_cast<size_t>(s)); }
  void stages(const Vec& u, Vec& u1, Vec& u2) const {
    const double dt = m_.inner_dt();
    const Vec r0 = m_.rhs(u);
    u1.resize(u.size());
    u2.resize(u.size());
    for (size_t i = 0; i < u.size(); ++i) u1[i] = u[i] + dt * r0[i];
    const Vec r1 = m_.rhs(u1);
    for (size_t i = 0; i < u.size(); ++i) u2[i] = 0.75 * u[i] + 0.25 * (u1[i] + dt * r1[i]);
  }
  // proj/src/burgers.cpp:218-225
  Vec tlm_range(int b, int e, const Vec& dx) const override {
    check(b, e);
    const double dt = m_.inner_dt();
    Vec d = dx, u1, u2;
    for (int k = b; k < e; ++k) {
      const Vec& u = states_[k];
      stages(u, u1, u2);
      const Vec j0 = m_.rhs_jacobian(u, d);
      Vec d1(d.size()), d2(d.size()), o(d.size());
      for (size_t i = 0; i < d.size(); ++i) d1[i] = d[i] + dt * j0[i];
      const Vec j1 = m_.rhs_jacobian(u1, d1);
      for (size_t i = 0; i < d.size(); ++i) d2[i] = 0.75 * d[i] + 0.25 * (d1[i] + dt * j1[i]);
      const Vec j2 = m_.rhs_jacobian(u2, d2);
      for (size_t i = 0; i < d.size(); ++i) o[i] = d[i] / 3.0 + (2.0 / 3.0) * (d2[i] + dt * j2[i]);
      d = std::move(o);
    }
    return d;
  }
  // proj/src/burgers.cpp:227-236
  Vec adj_range(int b, int e, const Vec& lambda) const override {
    check(b, e);
    const double dt = m_.inner_dt();
    Vec lam = lambda, u1, u2;
    for (int k = e - 1; k >= b; --k) {
      const Vec& u = states_[k];
      stages(u, u1, u2);
      const Vec a2 = m_.rhs_jacobian_adjoint(u2, lam);
      Vec t2(lam.size()), t1(lam.size()), o(lam.size());
      for (size_t i = 0; i < lam.size(); ++i) t2[i] = (2.0 / 3.0) * (lam[i] + dt * a2[i]);
      const Vec a1 = m_.rhs_jacobian_adjoint(u1, t2);
      for (size_t i = 0; i < lam.size(); ++i) t1[i] = 0.25 * (t2[i] + dt * a1[i]);
      const Vec a0 = m_.rhs_jacobian_adjoint(u, t1);
      for (size_t i = 0; i < lam.size(); ++i) o[i] = lam[i] / 3.0 + 0.75 * t2[i] + t1[i] + dt * a0[i];
      lam = std::move(o);
    }
    return lam;
  }

 private:
  void check(int b, int e) const {
    if (b < 0 || e > steps_ || b > e) throw std::invalid_argument("BurgersTrajectory: step range out of bounds");
  }
  const DirichletBurgers m_;
  int steps_;
  std::vector<Vec> states_;
};
}  // namespace
std::shared_ptr<const LinearizedTrajectory> DirichletBurgers::linearize(const Vec& x0, int steps, int) const {
  return std::make_shared<DirichletBurgersTrajectory>(*this, x0, steps);
}

// ---- Dirichlet BVE, RK3-TVD (proj/src/bve.cpp) ----
DirichletBVE::DirichletBVE(int nx, int ny, double re, double ro, double dt)
    : nx_(nx), ny_(ny), re_(re), ro_(ro), dt_(dt) {
  if (nx < 3 || ny < 3 || re <= 0.0 || ro <= 0.0 || dt <= 0.0)
    throw std::invalid_argument("BVEModel: invalid parameters");
  forcing_.resize(static_cast<size_t>(nx) * ny);
  for (int j = 0; j < ny; ++j) {
    const double y = -1.0 + (j + 1) * dy();
    const double f = std::sin(M_PI * y);
    for (int i = 0; i < nx; ++i) forcing_[i + static_cast<size_t>(nx) * j] = f;
  }
  poisson_ = std::make_shared<DirichletSolver2D>(nx, ny, 0.0, 1.0 / (dx() * dx()), 1.0 / (dy() * dy()));
}
Vec DirichletBVE::d_x(const Vec& f) const {
  Vec o(f.size());
  const double c = 0.5 * (nx_ + 1);
  for (int j = 0; j < ny_; ++j) {
    const size_t base = static_cast<size_t>(j) * nx_;
    for (int i = 0; i < nx_; ++i) {
      const double w = i > 0 ? f[base + i - 1] : 0.0, e = i + 1 < nx_ ? f[base + i + 1] : 0.0;
      o[base + i] = (e - w) * c;
    }
  }
  return o;
}
Vec DirichletBVE::d_y(const Vec& f) const {
  Vec o(f.size());
  const double c = 0.25 * (ny_ + 1);
  for (int j = 0; j < ny_; ++j) {
    const size_t base = static_cast<size_t>(j) * nx_;
    for (int i = 0; i < nx_; ++i) {
      const double s = j > 0 ? f[base + i - nx_] : 0.0, n = j + 1 < ny_ ? f[base + i + nx_] : 0.0;
      o[base + i] = (n - s) * c;
    }
  }
  return o;
}
Vec DirichletBVE::laplacian(const Vec& f) const {
  return scaled(-1.0, neg_laplacian_2d(f, nx_, ny_, 1.0 / (dx() * dx()), 1.0 / (dy() * dy())));
}
Vec DirichletBVE::rhs(const Vec& w) const {
  const Vec psi = poisson_solve(w);
  const Vec ox = d_x(w), oy = d_y(w), px = d_x(psi), py = d_y(psi);
  const Vec lap = laplacian(w);
  Vec o(w.size());
  for (size_t i = 0; i < w.size(); ++i) {
    o[i] = -(py[i] * ox[i] - px[i] * oy[i]);
    o[i] += (1.0 / ro_) * (px[i] + forcing_[i]);
    o[i] += (1.0 / re_) * lap[i];
  }
  return o;
}
Vec DirichletBVE::step(const Vec& w) const {
  const Vec r0 = rhs(w);
  Vec o1(w.size()), o2(w.size()), o(w.size());
  for (size_t i = 0; i < w.size(); ++i) o1[i] = w[i] + dt_ * r0[i];
  const Vec r1 = rhs(o1);
  for (size_t i = 0; i < w.size(); ++i) o2[i] = 0.75 * w[i] + 0.25 * (o1[i] + dt_ * r1[i]);
  const Vec r2 = rhs(o2);
  for (size_t i = 0; i < w.size(); ++i) o[i] = w[i] / 3.0 + (2.0 / 3.0) * (o2[i] + dt_ * r2[i]);
  return o;
}
Vec DirichletBVE::forward(const Vec& x0, int steps) const {
  Vec u = x0;
  for (int k = 0; k < steps; ++k) {
    u = step(u);
    if (!all_finite(u))
      throw std::runtime_error("BVEModel::forward: non-finite state at step " + std::to_string(k + 1) +
                               " (time step too large for stability)");
  }
  return u;
}
namespace {
struct StageFields {
  Vec ox, oy, px, py;
};
class DirichletBVETrajectory final : public LinearizedTrajectory {
 public:
  DirichletBVETrajectory(const DirichletBVE& m, const Vec& x0, int steps) : m_(m), steps_(steps) {
    states_.push_back(x0);
    stages_.resize(static_cast<size_t>(steps));
    Vec u = x0;
    const double dt = m.inner_dt();
    for (int k = 0; k < steps; ++k) {
      const Vec t0 = tendency(u, stages_[k][0]);
      Vec u1(u.size()), u2(u.size()), o(u.size());
      for (size_t i = 0; i < u.size(); ++i) u1[i] = u[i] + dt * t0[i];
      const Vec t1 = tendency(u1, stages_[k][1]);
      for (size_t i = 0; i < u.size(); ++i) u2[i] = 0.75 * u[i] + 0.25 * (u1[i] + dt * t1[i]);
      const Vec t2 = tendency(u2, stages_[k][2]);
      for (size_t i = 0; i < u.size(); ++i) o[i] = u[i] / 3.0 + (2.0 / 3.0) * (u2[i] + dt * t2[i]);
      u = std::move(o);
      if (!all_finite(u))
        throw std::runtime_error("BVEModel::linearize: non-finite state at step " + std::to_string(k + 1));
      states_.push_back(u);
    }
  }
  int total_steps() const override { return steps_; }
  Vec state_at(int s) const override { return states_.at(static_cast<size_t>(s)); }
  Vec tlm_range(int b, int e, const Vec& dx) const override {
    const double dt = m_.inner_dt();
    Vec d = dx;
    for (int k = b; k < e; ++k) {
      const Vec j0 = jac(stages_[k][0], d);
      Vec d1(d.size()), d2(d.size()), o(d.size());
      for (size_t i = 0; i < d.size(); ++i) d1[i] = d[i] + dt * j0[i];
      const Vec j1 = jac(stages_[k][1], d1);
      for (size_t i = 0; i < d.size(); ++i) d2[i] = 0.75 * d[i] + 0.25 * (d1[i] + dt * j1[i]);
      const Vec j2 = jac(stages_[k][2], d2);
      for (size_t i = 0; i < d.size(); ++i) o[i] = d[i] / 3.0 + (2.0 / 3.0) * (d2[i] + dt * j2[i]);
      d = std::move(o);
    }
    return d;
  }
  Vec adj_range(int b, int e, const Vec& lambda) const override {
    const double dt = m_.inner_dt();
    Vec lam = lambda;
    for (int k = e - 1; k >= b; --k) {
      const Vec a2 = jac_adj(stages_[k][2], lam);
      Vec t2(lam.size()), t1(lam.size()), o(lam.size());
      for (size_t i = 0; i < lam.size(); ++i) t2[i] = (2.0 / 3.0) * (lam[i] + dt * a2[i]);
      const Vec a1 = jac_adj(stages_[k][1], t2);
      for (size_t i = 0; i < lam.size(); ++i) t1[i] = 0.25 * (t2[i] + dt * a1[i]);
      const Vec a0 = jac_adj(stages_[k][0], t1);
      for (size_t i = 0; i < lam.size(); ++i) o[i] = lam[i] / 3.0 + 0.75 * t2[i] + t1[i] + dt * a0[i];
      lam = std::move(o);
    }
    return lam;
  }

 private:
  Vec tendency(const Vec& w, StageFields& f) const {
    const Vec psi = m_.poisson_solve(w);
    f.ox = m_.d_x(w);
    f.oy = m_.d_y(w);
    f.px = m_.d_x(psi);
    f.py = m_.d_y(psi);
    const Vec lap = m_.laplacian(w);
    Vec o(w.size());
    for (size_t i = 0; i < w.size(); ++i) {
      o[i] = -(f.py[i] * f.ox[i] - f.px[i] * f.oy[i]);
      o[i] += (1.0 / m_.ro()) * (f.px[i] + m_.forcing()[i]);
      o[i] += (1.0 / m_.re()) * lap[i];
    }
    return o;
  }
  // proj/src/bve.cpp:184-197
  Vec jac(const StageFields& f, const Vec& d) const {
    const Vec dpsi = m_.poisson_solve(d);
    const Vec dx = m_.d_x(d), dy = m_.d_y(d), dpx = m_.d_x(dpsi), dpy = m_.d_y(dpsi);
    const Vec lap = m_.laplacian(d);
    Vec o(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
      o[i] = -(dpy[i] * f.ox[i] + f.py[i] * dx[i] - dpx[i] * f.oy[i] - f.px[i] * dy[i]);
      o[i] += (1.0 / m_.ro()) * dpx[i];
      o[i] += (1.0 / m_.re()) * lap[i];
    }
    return o;
  }
  // proj/src/bve.cpp:199-211
  Vec jac_adj(const StageFields& f, const Vec& lam) const {
    const size_t n = lam.size();
    Vec t(n);
    for (size_t i = 0; i < n; ++i) t[i] = f.py[i] * lam[i];
    Vec out = m_.d_x(t);
    for (size_t i = 0; i < n; ++i) t[i] = f.px[i] * lam[i];
    const Vec a = m_.d_y(t);
    for (size_t i = 0; i < n; ++i) out[i] -= a[i];
    for (size_t i = 0; i < n; ++i) t[i] = f.ox[i] * lam[i];
    Vec vp = m_.d_y(t);
    for (size_t i = 0; i < n; ++i) t[i] = f.oy[i] * lam[i];
    const Vec b = m_.d_x(t);
    const Vec c = m_.d_x(lam);
    for (size_t i = 0; i < n; ++i) vp[i] = vp[i] - b[i] - (1.0 / m_.ro()) * c[i];
    const Vec ps = m_.poisson_solve(vp);
    const Vec lap = m_.laplacian(lam);
    for (size_t i = 0; i < n; ++i) out[i] += ps[i] + (1.0 / m_.re()) * lap[i];
    return out;
  }
  const DirichletBVE m_;
  int steps_;
  std::vector<Vec> states_;
  std::vector<std::array<StageFields, 3>> stages_;
};
}  // namespace
std::shared_ptr<const LinearizedTrajectory> DirichletBVE::linearize(const Vec& x0, int steps, int) const {
  return std::make_shared<DirichletBVETrajectory>(*this, x0, steps);
}

// ===================================================================== priors
Vec Prior::sample_background(const Vec& truth, uint64_t seed) const {
  if (static_cast<int64_t>(truth.size()) != dim()) throw std::invalid_argument("PriorCovariance: size mismatch");
  const Vec s = apply_sqrt(gaussian_vector(dim(), seed));
  return axpby(1.0, truth, 1.0, s);
}

// proj/src/prior.cpp:9-69
std::shared_ptr<LaplacianPrior> LaplacianPrior::make_1d(int n, double alpha, double beta, double scale) {
  if (n < 1) throw std::invalid_argument("PriorCovariance: n must be >= 1");
  if (alpha < 0.0 || beta < 0.0 || (alpha == 0.0 && beta == 0.0))
    throw std::invalid_argument("PriorCovariance: need alpha, beta >= 0 with alpha + beta > 0");
  auto p = std::make_shared<LaplacianPrior>();
  p->dim_ = n;
  p->nx_ = n;
  p->alpha_ = alpha;
  p->beta_ = beta;
  p->sx_ = scale;
  const double b = beta * scale;
  p->s1_ = std::make_shared<Tridiagonal1D>(n, alpha + 2.0 * b, -b);
  return p;
}
std::shared_ptr<LaplacianPrior> LaplacianPrior::make_2d(int nx, int ny, double alpha, double beta, double sx,
                                                        double sy) {
  if (alpha < 0.0 || beta < 0.0 || (alpha == 0.0 && beta == 0.0))
    throw std::invalid_argument("PriorCovariance: need alpha, beta >= 0 with alpha + beta > 0");
  auto p = std::make_shared<LaplacianPrior>();
  p->dim_ = static_cast<int64_t>(nx) * ny;
  p->nx_ = nx;
  p->ny_ = ny;
  p->alpha_ = alpha;
  p->beta_ = beta;
  p->sx_ = sx;
  p->sy_ = sy;
  p->s2_ = std::make_shared<DirichletSolver2D>(nx, ny, alpha, beta * sx, beta * sy);
  return p;
}
Vec LaplacianPrior::apply_inv_sqrt(const Vec& v) const {
  if (static_cast<int64_t>(v.size()) != dim_) throw std::invalid_argument("PriorCovariance: size mismatch");
  if (ny_ == 0) return axpby(alpha_, v, beta_ * sx_, neg_laplacian_1d(v));
  return axpby(alpha_, v, 1.0, neg_laplacian_2d(v, nx_, ny_, beta_ * sx_, beta_ * sy_));
}
Vec LaplacianPrior::apply_sqrt(const Vec& v) const {
  if (static_cast<int64_t>(v.size()) != dim_) throw std::invalid_argument("PriorCovariance: size mismatch");
  return ny_ == 0 ? s1_->solve(v) : s2_->solve(v);
}

FourierPrior::FourierPrior(int n, int dims, double sigma, double length) : n_(n), dims_(dims) {
  if (n < 2 || (n & (n - 1)) || (dims != 1 && dims != 2) || !(sigma > 0) || !(length > 0))
    throw std::invalid_argument("FourierPrior: invalid parameters");
  const size_t nn = dims == 1 ? static_cast<size_t>(n) : static_cast<size_t>(n) * n;
  Vec c(nn);
  double sum = 0.0;
  auto kk = [n](int k) { return k <= n / 2 ? k : k - n; };
  for (size_t idx = 0; idx < nn; ++idx) {
    double e;
    if (dims == 1) {
      const double k = kk(static_cast<int>(idx));
      e = std::exp(-0.5 * (2.0 * M_PI * k * length) * (2.0 * M_PI * k * length));
    } else {
      const double kx = kk(static_cast<int>(idx % n)), ky = kk(static_cast<int>(idx / n));
      e = std::exp(-0.5 * (kx * kx + ky * ky) * length * length);
    }
    c[idx] = e;
    sum += e;
  }
  sym_.resize(nn);
  for (size_t idx = 0; idx < nn; ++idx) {
    const double chat = c[idx] * static_cast<double>(nn) / sum;  // (1/N) sum chat = c(0) = 1
    sym_[idx] = sigma * std::sqrt(chat) / static_cast<double>(nn);
  }
}
Vec FourierPrior::apply_sqrt(const Vec& v) const {
  if (static_cast<int64_t>(v.size()) != dim()) throw std::invalid_argument("PriorCovariance: size mismatch");
  std::vector<cplx> z(v.size());
  for (size_t i = 0; i < v.size(); ++i) z[i] = cplx(v[i], 0.0);
  if (dims_ == 1) fft_inplace(z, false); else fft2_inplace(z, n_, n_, false);
  for (size_t i = 0; i < v.size(); ++i) z[i] *= sym_[i];
  if (dims_ == 1) fft_inplace(z, true); else fft2_inplace(z, n_, n_, true);
  Vec o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = z[i].real();
  return o;
}

}  // namespace oracle

// Device-resident problem, base trajectory and batched Hessian-product sweeps.
//
// Reference correspondence (/root/reference/proj):
//   Problem::linearize      <- DynamicalModel::linearize (include/sketchdav/model.hpp:36-40),
//                              BurgersTrajectory/BVETrajectory ctors (src/burgers.cpp:114-138, src/bve.cpp:103-127)
//   Problem::tlm / adj      <- LinearizedTrajectory::tlm_range / adj_range (src/burgers.cpp:152-191,
//                              src/bve.cpp:138-161), batched over s vectors
//   Problem::misfit_apply   <- MisfitOperator::apply (src/fourdvar.cpp:145-160)
//   Problem::misfit_adjoint <- MisfitOperator::adjoint_apply (src/fourdvar.cpp:162-176)
//   Problem::gram_apply     <- GramMap::apply (include/sketchdav/linalg.hpp:72-74)
//   Problem::evaluate       <- evaluate (src/fourdvar.cpp:92-132), control-variable background term
//   Problem::prior_sqrt     <- PriorCovariance::apply_sqrt (src/prior.cpp:64-69), Fourier-diagonal B
#include <algorithm>
#include <cmath>
#include <map>
#include <cstdlib>
#include <mutex>

#include "engine.hpp"
#include "fft.cuh"

namespace sdv {

// ------------------------------------------------------------ twiddles ------
const double2* twiddle_table(int n) {
  static std::mutex mu;
  static std::map<int, double2*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  const int cnt = std::max(1, fft_twiddle_count(n));
  std::vector<double2> h(static_cast<size_t>(cnt), make_double2(1.0, 0.0));
  fft_build_twiddles(n, h.data(), [](double ang) { return make_double2(std::cos(ang), std::sin(ang)); });
  double2* d = nullptr;
  SDV_CUDA(cudaMalloc(&d, sizeof(double2) * cnt));
  SDV_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * cnt, cudaMemcpyHostToDevice));
  cache[n] = d;
  return d;
}

namespace {

__global__ void innovation_kernel(const double* __restrict__ f, const long long* __restrict__ idx, int n_obs,
                                  const double* __restrict__ values, const double* __restrict__ rinv,
                                  double* __restrict__ innov, double* __restrict__ winnov) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_obs) return;
  const double d = f[idx[k]] - values[k];
  innov[k] = d;
  winnov[k] = d * rinv[k];
}

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// Fourier symbols, computed exactly as the oracle's FourierPrior /
// PeriodicBVE (identical expression order, so the tables agree bitwise).
std::vector<double> fourier_b_full(int n, int dims, double sigma, double len) {
  const size_t nn = dims == 1 ? static_cast<size_t>(n) : static_cast<size_t>(n) * n;
  std::vector<double> c(nn), sym(nn);
  double sum = 0.0;
  auto kk = [n](int k) { return k <= n / 2 ? k : k - n; };
  for (size_t idx = 0; idx < nn; ++idx) {
    double e;
    if (dims == 1) {
      const double k = kk(static_cast<int>(idx));
      e = std::exp(-0.5 * (2.0 * M_PI * k * len) * (2.0 * M_PI * k * len));
    } else {
      const double kx = kk(static_cast<int>(idx % n)), ky = kk(static_cast<int>(idx / n));
      e = std::exp(-0.5 * (kx * kx + ky * ky) * len * len);
    }
    c[idx] = e;
    sum += e;
  }
  for (size_t idx = 0; idx < nn; ++idx) {
    const double chat = c[idx] * static_cast<double>(nn) / sum;
    sym[idx] = sigma * std::sqrt(chat) / static_cast<double>(nn);
  }
  return sym;
}

}  // namespace

// ------------------------------------------------------------- problem ------
Problem::Problem(const ProblemDesc& d, long long n_obs, const long long* idx, const double* values,
                 const double* variances, const double* background)
    : d_(d), n_obs_(n_obs) {
  if (d.model != kModelBurgers && d.model != kModelBVE && d.model != kModelBurgers3 && d.model != kModelBVE3)
    throw std::invalid_argument("problem: unknown model kind");
  if (d.model == kModelBurgers3) {
    if (d.n < 3 || d.n > 4096) throw std::invalid_argument("problem: Dirichlet Burgers needs 3 <= n <= 4096");
    if (d.prior_kind != kPriorLaplacian)
      throw std::invalid_argument("problem: the Dirichlet Burgers model takes the Laplacian prior");
  } else if (d.model == kModelBVE3) {
    // proj/src/bve.cpp:12-26 (BVEModel ctor)
    if (d.n < 3 || d.ny < 3 || !(d.reynolds > 0.0) || !(d.rossby > 0.0) || d.n > 1024 || d.ny > 1024)
      throw std::invalid_argument("BVEModel: invalid parameters (need 3 <= nx, ny <= 1024, Re, Ro > 0)");
    if (d.prior_kind != kPriorLaplacian)
      throw std::invalid_argument("problem: the Dirichlet BVE model takes the Laplacian prior");
  } else {
    if (!is_pow2(d.n) || d.n < 32 || (d.model == kModelBurgers && d.n > 4096) || (d.model == kModelBVE && d.n > 512))
      throw std::invalid_argument("problem: n must be a power of two (Burgers 32..4096, BVE 32..512)");
    if (d.prior_kind != kPriorFourier)
      throw std::invalid_argument("problem: periodic models take the Fourier-diagonal prior");
  }
  if (!(d.nu >= 0.0) || !(d.dt > 0.0)) throw std::invalid_argument("problem: need nu >= 0 and dt > 0");
  if (d.n_t < 1 || d.spi < 1) throw std::invalid_argument("AssimilationProblem: need n_t >= 1 and steps_per_interval >= 1");
  if (d.prior_kind == kPriorFourier && (!(d.prior_sigma > 0.0) || !(d.prior_length > 0.0)))
    throw std::invalid_argument("problem: prior sigma/length must be positive");
  if (d.prior_kind == kPriorLaplacian &&
      (d.prior_alpha < 0.0 || d.prior_beta < 0.0 || (d.prior_alpha == 0.0 && d.prior_beta == 0.0)))
    throw std::invalid_argument("PriorCovariance: need alpha, beta >= 0 with alpha + beta > 0");
  dim_ = d.model == kModelBVE ? static_cast<long long>(d.n) * d.n
                              : (d.model == kModelBVE3 ? static_cast<long long>(d.n) * d.ny : d.n);
  if (n_obs < 0 || n_obs > dim_) throw std::invalid_argument("AssimilationProblem: n_obs > n");
  long long prev = -1;
  for (long long k = 0; k < n_obs; ++k) {
    if (idx[k] <= prev || idx[k] >= dim_)
      throw std::invalid_argument(
          "AssimilationProblem: observation indices must be strictly increasing and in range");
    prev = idx[k];
  }
  const long long m = n_obs * d.n_t;
  std::vector<double> rs(static_cast<size_t>(m)), ri(static_cast<size_t>(m));
  for (long long i = 0; i < m; ++i) {
    if (!(variances[i] > 0.0)) throw std::invalid_argument("AssimilationProblem: observation variances must be positive");
    rs[i] = 1.0 / std::sqrt(variances[i]);
    ri[i] = 1.0 / variances[i];
  }
  SDV_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  // Zero observations (a model-only problem) still gets 1-element buffers.
  const long long zero_idx = 0;
  const double zero = 0.0;
  idx_.upload(n_obs > 0 ? idx : &zero_idx, static_cast<size_t>(std::max<long long>(n_obs, 1)), st_);
  values_.upload(m > 0 ? values : &zero, static_cast<size_t>(std::max<long long>(m, 1)), st_);
  rinv_sqrt_.upload(m > 0 ? rs.data() : &zero, static_cast<size_t>(std::max<long long>(m, 1)), st_);
  rinv_.upload(m > 0 ? ri.data() : &zero, static_cast<size_t>(std::max<long long>(m, 1)), st_);
  background_.upload(background, static_cast<size_t>(dim_), st_);
  const int n = d.n;
  if (d.model == kModelBVE && n_obs > 0 && n % 8 == 0 && std::is_sorted(idx, idx + n_obs)) {
    // observations per 8-row tile for the gather fused into the TLM stage kernel
    const int q = n / 8;
    std::vector<int> tile(static_cast<size_t>(q) + 1);
    for (int t = 0; t <= q; ++t)
      tile[t] = static_cast<int>(std::lower_bound(idx, idx + n_obs, static_cast<long long>(t) * 8 * n) - idx);
    obs_tile_.upload(tile.data(), tile.size(), st_);
  }
  if (d.model == kModelBVE3) {
    // proj/src/bve.cpp:12-26: dx = 1/(nx+1) on [0,1], dy = 2/(ny+1) on [-1,1]
    const double dx = 1.0 / (n + 1), dy = 2.0 / (d.ny + 1);
    b3_.nx = n;
    b3_.ny = d.ny;
    b3_.cx = 0.5 * (n + 1);
    b3_.cy = 0.25 * (d.ny + 1);
    b3_.lx = 1.0 / (dx * dx);
    b3_.ly = 1.0 / (dy * dy);
    b3_.inv_ro = 1.0 / d.rossby;
    b3_.inv_re = 1.0 / d.reynolds;
    b3_.dt = d.dt;
    std::vector<double> f(static_cast<size_t>(d.ny));
    for (int j = 0; j < d.ny; ++j) f[j] = std::sin(M_PI * (-1.0 + (j + 1) * dy));
    forcing_.upload(f.data(), f.size(), st_);
    b3_.forcing = forcing_.get();
    poisson3_ = std::make_unique<DstSolver>(n, d.ny, 0.0, b3_.lx, b3_.ly, st_);
    // Gamma^{1/2} = (alpha I + beta (-Lap*))^{-1}, unscaled stencil (proj/src/prior.cpp:32-51)
    prior3_ = std::make_unique<DstSolver>(n, d.ny, d.prior_alpha, d.prior_beta, d.prior_beta, st_);
    lap_b_ = d.prior_beta;
  } else if (d.prior_kind == kPriorLaplacian) {
    // Tridiagonal1D(n, alpha + 2b, -b) pivots (proj/src/dirichlet.cpp:157-170,
    // proj/src/prior.cpp:9-30 with stencil scale 1).
    lap_b_ = d.prior_beta;
    const double diag = d.prior_alpha + 2.0 * lap_b_, off = -lap_b_;
    std::vector<double> piv(static_cast<size_t>(n));
    double dd = diag;
    for (int i = 0; i < n; ++i) {
      if (!(dd > 0.0)) throw std::runtime_error("Tridiagonal1D: factorization failed");
      piv[i] = dd;
      dd = diag - off * off / dd;
    }
    pivot_.upload(piv.data(), piv.size(), st_);
  } else if (d.model == kModelBurgers) {
    const std::vector<double> sb = fourier_b_full(n, 1, d.prior_sigma, d.prior_length);
    sym_b_.upload(sb.data(), sb.size(), st_);
  } else {
    const std::vector<double> full = fourier_b_full(n, 2, d.prior_sigma, d.prior_length);
    std::vector<double> sb(static_cast<size_t>(n / 2 + 1) * n), sp(sb.size());
    const double h = 2.0 * M_PI / n;
    for (int kx = 0; kx <= n / 2; ++kx)
      for (int ky = 0; ky < n; ++ky) {
        sb[static_cast<size_t>(kx) * n + ky] = full[kx + static_cast<size_t>(n) * ky];
        const double sx = std::sin(M_PI * kx / n), sy = std::sin(M_PI * ky / n);
        const double mu = 4.0 / (h * h) * (sx * sx + sy * sy);
        sp[static_cast<size_t>(kx) * n + ky] = (kx == 0 && ky == 0) ? 0.0 : 1.0 / (mu * static_cast<double>(n) * n);
      }
    sym_b_.upload(sb.data(), sb.size(), st_);
    sym_p_.upload(sp.data(), sp.size(), st_);
    // recurrence constants per kx (see col_solve_kernel): d = 2 + 4 s^2,
    // rho = 1 / (1 + 2 s^2 + 2 s sqrt(1 + s^2)) (the root < 1 of rho + 1/rho = d)
    std::vector<double> tab(static_cast<size_t>(n / 2) * 4, 0.0);
    for (int kx = 1; kx < n / 2; ++kx) {
      const double sx = std::sin(M_PI * kx / n);
      const double rho = 1.0 / (1.0 + 2.0 * sx * sx + 2.0 * sx * std::sqrt(1.0 + sx * sx));
      tab[4 * kx + 0] = rho;
      tab[4 * kx + 1] = std::pow(rho, n / 32);
      tab[4 * kx + 2] = 1.0 / (1.0 - std::pow(rho, n));
      tab[4 * kx + 3] = h * h * rho / n;
    }
    // entry 0 (kx = 0 is not a recurrence column): the packed column's
    // constants for the carry pass (col0_warp_solve): x-mode N/2 (d = 6,
    // rho = 3 - 2 sqrt 2) and the h^2/N scale of the singular x-mode 0
    {
      const double rho = 3.0 - 2.0 * std::sqrt(2.0);
      tab[0] = rho;
      tab[1] = h * h / n;
      tab[2] = 1.0 / (1.0 - std::pow(rho, n));
      tab[3] = h * h * rho / n;
    }
    solve_tab_.upload(tab.data(), tab.size(), st_);
  }
  SDV_CUDA(cudaStreamSynchronize(st_));
}

void Problem::poisson_col(double2* s, int nvec, cudaStream_t st) const {
  static const bool fft = std::getenv("SDV_COL_FFT") != nullptr;
  if (fft) {
    bve_col(d_.n, s, sym_p_.get(), nvec, st);
    count_launch();
  } else {
    bve_col_solve(d_.n, s, reinterpret_cast<const double4*>(solve_tab_.get()), sym_p_.get(), nvec, st);
    count_launch();
  }
}

bool Problem::fused(int nvec) const { return d_.model == kModelBVE && bve_fused_ok(d_.n, nvec); }

long long fused_stride(int n) { return static_cast<long long>(n / 8) * (n / 2); }

void Problem::poisson_carry(double2* s, long long woff, int nvec, cudaStream_t st) const {
  const long long fs = fused_stride(d_.n);
  bve_carry(d_.n, s, lsum_.get() + woff * fs, carc_.get() + woff * fs, care_.get() + woff * fs,
            reinterpret_cast<const double4*>(solve_tab_.get()), sym_p_.get(), nvec, st);
  count_launch();
}

void Problem::set_fused(StageArgs& a, long long woff) const {
  const long long fs = fused_stride(d_.n);
  a.car_c = carc_.get() + woff * fs;
  a.car_e = care_.get() + woff * fs;
  a.lsum = lsum_.get() + woff * fs;
  a.stab = reinterpret_cast<const double4*>(solve_tab_.get());
}

int Problem::group() const {
  if (d_.model != kModelBVE) return 1 << 30;
  if (d_.block_group > 0) return d_.block_group;
  // Whole block per launch (measured on B200: per-vector stage time is flat
  // or falls with the group size, and L2 residency of small groups did not
  // pay — the stage kernels are issue/latency bound, not bandwidth bound),
  // capped so the sweep workspace (~6 fields per vector) stays under ~4 GB.
  const double per = 6.0 * 8.0 * static_cast<double>(dim_);
  return std::max(1, static_cast<int>(4e9 / per));
}

void Problem::ensure_work(int nvec) const {
  if (d_.model != kModelBVE) return;
  const int g = std::min(nvec, group());
  if (g <= work_nvec_) return;
  const size_t f = static_cast<size_t>(g) * dim_;
  wa_.alloc(f);
  wx0_.alloc(f);
  wx1_.alloc(f);
  ws0_.alloc(static_cast<size_t>(g) * d_.n * (d_.n / 2));
  ws1_.alloc(static_cast<size_t>(g) * d_.n * (d_.n / 2));
  const size_t fs = static_cast<size_t>(g) * (d_.n / 8) * (d_.n / 2);
  lsum_.alloc(fs);
  carc_.alloc(fs);
  care_.alloc(fs);
  work_nvec_ = g;
}

const double* Trajectory::state_at(int step) const {
  if (step < 0 || step > steps) throw std::invalid_argument("trajectory: step out of range");
  if (step == steps) return final.get();
  if (!checkpointed()) return w.get() + static_cast<long long>(step) * stages * prob->dim();
  // checkpoint mode (proj/src/burgers.cpp:142-150): the floor checkpoint,
  // integrated forward to `step` when it is not one itself
  const int j = step / stride;
  const double* c = ckpt.get() + static_cast<long long>(j) * prob->dim();
  if (step == j * stride) return c;
  scratch.ensure(static_cast<size_t>(prob->dim()));
  prob->forward(c, step - j * stride, scratch.get());
  return scratch.get();
}

namespace {
BurgersArgs burgers_args(const ProblemDesc& d) {
  BurgersArgs a;
  a.n = d.n;
  a.dt = d.dt;
  a.nu = d.nu;
  // periodic: dx = 1/n; Dirichlet: dx = 1/(n+1) (proj/src/burgers.cpp:57-58)
  const int m = d.model == kModelBurgers3 ? d.n + 1 : d.n;
  a.c1 = 0.5 * m;
  a.c2 = static_cast<double>(m) * m;
  a.spi = d.spi;
  return a;
}
StageArgs bve_args(const ProblemDesc& d) {
  StageArgs a;
  const double h = 2.0 * M_PI / d.n;
  a.dt = d.dt;
  a.nu = d.nu;
  a.inv12h2 = 1.0 / (12.0 * h * h);
  a.invh2 = 1.0 / (h * h);
  a.tw = twiddle_table(d.n);
  return a;
}
}  // namespace

void Problem::forward(const double* d_x0, int steps, double* d_out) const {
  if (d_.model == kModelBurgers3) {
    burgers3_fwd(burgers_args(d_), d_x0, nullptr, d_out, steps, st_);
    count_launch();
    return;
  }
  if (d_.model == kModelBurgers) {
    burgers_fwd(burgers_args(d_), d_x0, nullptr, d_out, steps, st_);
    count_launch();
    return;
  }
  if (d_.model == kModelBVE3) {
    // RK3-TVD (proj/src/bve.cpp:84-101): stage s solves psi_s = P(w_s), then
    // w_{s+1} = combination(u, w_s, rhs(w_s, psi_s))
    bve3_work(1);
    double* u = b3w_[0].get();
    SDV_CUDA(cudaMemcpyAsync(u, d_x0, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    double* ws[3] = {u, b3w_[1].get(), b3w_[2].get()};
    double* ps = b3w_[3].get();
    for (int k = 0; k < steps; ++k)
      for (int s = 0; s < 3; ++s) {
        poisson3_->solve(ws[s], ps, 1);
        bve3_nl_stage(b3_, s, u, ws[s], ps, s < 2 ? ws[s + 1] : b3w_[4].get(), 1, st_);
        count_launch(2);  // DST scale + stage (the 4 GEMMs are cuBLAS)
        if (s == 2) SDV_CUDA(cudaMemcpyAsync(u, b3w_[4].get(), sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
      }
    SDV_CUDA(cudaMemcpyAsync(d_out, u, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    return;
  }
  ensure_work(1);
  if (d_out != d_x0) SDV_CUDA(cudaMemcpyAsync(d_out, d_x0, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
  bve_nl(d_out, steps, nullptr, nullptr, NlWork{wx0_.get(), wx1_.get(), wa_.get(), ws0_.get(), ws1_.get()});
}

// Periodic BVE NL forward (RK4 stages of NL-mode stage_kernel, column Poisson
// pass), u in/out; stores every stage input / streamfunction when store_w is
// set ([steps][4][dim] from store_w / store_p).
void Problem::bve_nl(double* u, int steps, double* store_w, double* store_p, const NlWork& wk) const {
  const int n = d_.n;
  double2* s_cur = wk.s0;
  double2* s_nxt = wk.s1;
  bve_row_fwd(n, u, s_cur, 1, st_);
  count_launch();
  double* xb[2] = {wk.x0, wk.x1};
  for (int k = 0; k < steps; ++k)
    for (int s = 0; s < 4; ++s) {
      poisson_col(s_cur, 1, st_);
      StageArgs a = bve_args(d_);
      a.stage = s;
      a.s_in = s_cur;
      a.s_out = s_nxt;
      a.x_in = s == 0 ? u : xb[(s - 1) & 1];
      a.x_out = s < 3 ? xb[s & 1] : nullptr;
      a.d = u;
      a.acc = wk.acc;
      if (store_w) {
        a.store_w = store_w + (static_cast<long long>(k) * 4 + s) * dim_;
        a.store_p = store_p + (static_cast<long long>(k) * 4 + s) * dim_;
      }
      bve_stage(n, kModeNl, a, 1, st_);
      count_launch();
      std::swap(s_cur, s_nxt);
    }
}

std::unique_ptr<Trajectory> Problem::linearize(const double* d_x0, int stride, int policy) const {
  if (policy != kStoreAuto && policy != kStoreFull && policy != kStoreCheckpoint)
    throw std::invalid_argument("linearize: unknown storage policy");
  if (policy == kStoreCheckpoint && stride < 1) throw std::invalid_argument("linearize: checkpoint stride must be >= 1");
  auto tr = std::make_unique<Trajectory>();
  tr->prob = this;
  tr->steps = total_steps();
  tr->stages = (d_.model == kModelBurgers3 || d_.model == kModelBVE3) ? 3 : 4;
  const int fields = (d_.model == kModelBVE || d_.model == kModelBVE3) ? 2 : 1;
  // The reference BVE stores every stage whatever the stride
  // (proj/src/bve.cpp:221-225); the Dirichlet BVE here does the same.
  if (d_.model != kModelBVE3 && tr->steps > 1) {
    if (policy == kStoreAuto) {
      size_t free_b = 0, total_b = 0;
      SDV_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const double full = 8.0 * fields * tr->stages * static_cast<double>(dim_) * tr->steps;
      if (full > 0.75 * static_cast<double>(free_b)) {
        // largest segment that leaves half the free memory to the sweeps
        const double seg_step = 8.0 * fields * tr->stages * static_cast<double>(dim_);
        const int fit = static_cast<int>(std::max(1.0, 0.5 * static_cast<double>(free_b) / seg_step - 1.0));
        tr->stride = std::min(tr->steps, std::max(1, stride > 0 ? std::min(stride, fit) : fit));
      }
    } else if (policy == kStoreCheckpoint) {
      tr->stride = std::min(stride, tr->steps);
    }
    if (tr->stride >= tr->steps && policy != kStoreCheckpoint) tr->stride = 0;
  }
  if (tr->checkpointed()) {
    linearize_ckpt(*tr, d_x0);
    return tr;
  }
  const long long st_elems = static_cast<long long>(tr->steps) * tr->stages * dim_;
  tr->w.alloc(static_cast<size_t>(st_elems));
  tr->final.alloc(static_cast<size_t>(dim_));
  if (d_.model == kModelBVE3) {
    // stored per stage: w_s (stage input) and psi_s = P(w_s); the reference's
    // StageFields ox, oy, px, py are their derivatives (proj/src/bve.cpp:171-182),
    // recomputed in the TLM/ADJ kernels
    tr->p.alloc(static_cast<size_t>(st_elems));
    bve3_work(1);
    double* u = tr->final.get();
    SDV_CUDA(cudaMemcpyAsync(u, d_x0, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    for (int k = 0; k < tr->steps; ++k) {
      double* wk = tr->w.get() + static_cast<long long>(k) * 3 * dim_;
      double* pk = tr->p.get() + static_cast<long long>(k) * 3 * dim_;
      SDV_CUDA(cudaMemcpyAsync(wk, u, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
      for (int s = 0; s < 3; ++s) {
        poisson3_->solve(wk + s * dim_, pk + s * dim_, 1);
        bve3_nl_stage(b3_, s, wk, wk + s * dim_, pk + s * dim_, s < 2 ? wk + (s + 1) * dim_ : u, 1, st_);
        count_launch(2);  // DST scale + stage (the 4 GEMMs are cuBLAS)
      }
    }
  } else if (d_.model == kModelBurgers3) {
    burgers3_fwd(burgers_args(d_), d_x0, tr->w.get(), tr->final.get(), tr->steps, st_);
    count_launch();
  } else if (d_.model == kModelBurgers) {
    burgers_fwd(burgers_args(d_), d_x0, tr->w.get(), tr->final.get(), tr->steps, st_);
    count_launch();
  } else {
    tr->p.alloc(static_cast<size_t>(st_elems));
    ensure_work(1);
    double* u = tr->final.get();
    SDV_CUDA(cudaMemcpyAsync(u, d_x0, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    bve_nl(u, tr->steps, tr->w.get(), tr->p.get(), NlWork{wx0_.get(), wx1_.get(), wa_.get(), ws0_.get(), ws1_.get()});
  }
  check_final(*tr);
  return tr;
}

// Non-finite check on the final state (reference throws on NaN/Inf,
// proj/src/burgers.cpp:128-131, proj/src/bve.cpp:120-124).
void Problem::check_final(const Trajectory& tr) const {
  DevBuf<double> r(1);
  dev_dot(tr.final.get(), tr.final.get(), dim_, r.get(), st_);
  double nn = 0.0;
  SDV_CUDA(cudaMemcpyAsync(&nn, r.get(), sizeof(double), cudaMemcpyDeviceToHost, st_));
  SDV_CUDA(cudaStreamSynchronize(st_));
  if (!std::isfinite(nn))
    throw std::runtime_error("linearize: non-finite state (time step too large for stability)");
}

// Checkpoint-mode linearize (proj/src/burgers.cpp:114-138): the states at
// multiples of the stride, one segment buffer of stage inputs (left holding
// the last segment).
void Problem::linearize_ckpt(Trajectory& tr, const double* d_x0) const {
  const int nseg = tr.segments();
  const long long seg_elems = static_cast<long long>(tr.stride) * tr.stages * dim_;
  tr.w.alloc(static_cast<size_t>(seg_elems));
  if (d_.model == kModelBVE) tr.p.alloc(static_cast<size_t>(seg_elems));
  tr.ckpt.alloc(static_cast<size_t>(nseg) * dim_);
  tr.final.alloc(static_cast<size_t>(dim_));
  SDV_CUDA(cudaMemcpyAsync(tr.ckpt.get(), d_x0, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
  for (int j = 0; j < nseg; ++j) {
    tr.seg = -1;
    fill_segment(tr, j);
    // the segment's end state: the next checkpoint, or the final state
    double* nxt = j + 1 < nseg ? tr.ckpt.get() + static_cast<long long>(j + 1) * dim_ : tr.final.get();
    const double* end = d_.model == kModelBVE ? tr.ru.get() : tr.scratch.get();
    SDV_CUDA(cudaMemcpyAsync(nxt, end, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
  }
  check_final(tr);
}

// Recompute segment j's stage inputs from its checkpoint into tr.w / tr.p; the
// segment's end state is left in tr.ru (BVE) / tr.scratch (Burgers).
void Problem::fill_segment(const Trajectory& tr, int j) const {
  const int k0 = j * tr.stride, len = std::min(tr.stride, tr.steps - k0);
  const double* c = tr.ckpt.get() + static_cast<long long>(j) * dim_;
  if (d_.model == kModelBVE) {
    const size_t f = static_cast<size_t>(dim_), sp = static_cast<size_t>(d_.n) * (d_.n / 2);
    tr.ru.ensure(f);
    tr.rx0.ensure(f);
    tr.rx1.ensure(f);
    tr.racc.ensure(f);
    tr.rs0.ensure(sp);
    tr.rs1.ensure(sp);
    SDV_CUDA(cudaMemcpyAsync(tr.ru.get(), c, sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    bve_nl(tr.ru.get(), len, tr.w.get(), tr.p.get(), NlWork{tr.rx0.get(), tr.rx1.get(), tr.racc.get(), tr.rs0.get(), tr.rs1.get()});
  } else {
    tr.scratch.ensure(static_cast<size_t>(dim_));
    if (d_.model == kModelBurgers3) burgers3_fwd(burgers_args(d_), c, tr.w.get(), tr.scratch.get(), len, st_);
    else burgers_fwd(burgers_args(d_), c, tr.w.get(), tr.scratch.get(), len, st_);
    count_launch();
  }
  tr.seg = j;
}

void Problem::hold_segment(const Trajectory& tr, int k) const {
  if (!tr.checkpointed()) return;
  const int j = k / tr.stride;
  if (j != tr.seg) fill_segment(tr, j);
}

void Problem::prior_sqrt(const double* in, double* out, int nvec) const {
  if (d_.model == kModelBVE3) {
    prior3_->solve(in, out, nvec);  // DirichletSolver2D(nx, ny, alpha, beta, beta)
    count_launch();
    return;
  }
  if (d_.prior_kind == kPriorLaplacian) {
    // Gamma^{1/2} = (alpha I - beta Lap*)^{-1}: tridiagonal solve per vector
    thomas_solve(d_.n, -lap_b_, pivot_.get(), in, out, nvec, st_);
    count_launch();
    return;
  }
  if (d_.model == kModelBurgers) {
    spectral1d(d_.n, in, out, sym_b_.get(), nvec, st_);
    count_launch();
    return;
  }
  ensure_work(nvec);
  const int g = std::min(nvec, group());
  for (int v0 = 0; v0 < nvec; v0 += g) {
    const int gn = std::min(g, nvec - v0);
    bve_row_fwd(d_.n, in + v0 * dim_, ws0_.get(), gn, st_);
    bve_col(d_.n, ws0_.get(), sym_b_.get(), gn, st_);
    bve_row_inv(d_.n, ws0_.get(), out + v0 * dim_, gn, st_);
    count_launch(3);
  }
}

void Problem::tlm(const Trajectory& tr, double* state, int nvec, int k0, int k1, double* y, const double* w) const {
  if (k0 < 0 || k1 > tr.steps || k0 > k1) throw std::invalid_argument("trajectory: step range out of bounds");
  if (y && k0 != 0) throw std::invalid_argument("tlm: observation gathers need k0 == 0");
  if (nvec <= 0 || k0 == k1) return;
  if (d_.model == kModelBVE3) return bve3_tlm(tr, state, nvec, k0, k1, y, w);
  if (d_.model == kModelBurgers || d_.model == kModelBurgers3) {
    BurgersArgs a = burgers_args(d_);
    a.base = tr.w.get();
    a.k0 = k0;
    a.k1 = k1;
    a.idx = idx_.get();
    a.n_obs = static_cast<int>(n_obs_);
    a.w = w;
    a.y = y;
    a.m = m();
    // checkpoint mode: one launch per segment, in step order
    const int step = tr.checkpointed() ? tr.stride : k1 - k0;
    if (tr.checkpointed()) tr.seg = -1;
    for (int ka = tr.checkpointed() ? (k0 / step) * step : k0; ka < k1; ka += step) {
      a.k0 = std::max(k0, ka);
      a.k1 = std::min(k1, ka + step);
      hold_segment(tr, a.k0);
      a.base = tr.w.get();
      a.base_k0 = tr.held_k0();
      if (d_.model == kModelBurgers3)
        burgers3_tlm(a, state, nvec, st_);
      else
        burgers_tlm(a, state, nvec, st_);
      count_launch();
      count_path(kPathBurgers);
    }
    return;
  }
  ensure_work(nvec);
  if (tr.checkpointed()) tr.seg = -1;  // each sweep recomputes what it reads (graph replays stay valid)
  const int n = d_.n, g = std::min(nvec, group());
  const long long sdim = static_cast<long long>(n) * (n / 2);
  for (int v0 = 0; v0 < nvec; v0 += g) {
    const int gn = std::min(g, nvec - v0);
    std::vector<Lane> lanes = split_lanes(v0, gn);
    for (auto& L : lanes) {
      L.s_cur = ws0_.get() + L.woff * sdim;
      L.s_nxt = ws1_.get() + L.woff * sdim;
      bve_row_fwd(n, state + L.v0 * dim_, L.s_cur, L.cnt, L.st);
      count_launch();
    }
    bool first = true;
    for (int k = k0; k < k1; ++k) {
      if (tr.checkpointed() && k / tr.stride != tr.seg) {
        // the lanes finish the held segment before it is overwritten
        join_lanes(lanes);
        hold_segment(tr, k);
        refork_lanes(lanes);
      }
      for (int s = 0; s < 4; ++s) {
        // interleave the lanes' launches so their kernels co-reside on SMs;
        // fused lanes: the first stage reads column-solved spectra, later
        // stages the tile-local values + carries
        for (auto& L : lanes) {
          if (L.fz && !first) poisson_carry(L.s_cur, L.woff, L.cnt, L.st);
          else poisson_col(L.s_cur, L.cnt, L.st);
        }
        for (auto& L : lanes) {
          const bool fz = L.fz;
          double* dst = state + L.v0 * dim_;
          double* xb[2] = {wx0_.get() + L.woff * dim_, wx1_.get() + L.woff * dim_};
          StageArgs a = bve_args(d_);
          a.stage = s;
          a.s_in = L.s_cur;
          a.s_out = L.s_nxt;
          a.x_in = s == 0 ? dst : xb[(s - 1) & 1];
          a.x_out = s < 3 ? xb[s & 1] : nullptr;
          a.d = dst;
          a.acc = wa_.get() + L.woff * dim_;
          a.base_w = tr.base_w(k, s, dim_);
          a.base_p = tr.base_p(k, s, dim_);
          if (fz) {
            set_fused(a, L.woff);
            if (first) a.flags |= kFlagRawIn;
            if (s == 3 && y && (k + 1) % d_.spi == 0 && obs_tile_.get() && !L.lite) {
              const int iv = (k + 1) / d_.spi - 1;
              a.obs_idx = idx_.get();
              a.obs_w = w + static_cast<long long>(iv) * n_obs_;
              a.obs_y = y + L.v0 * m() + static_cast<long long>(iv) * n_obs_;
              a.obs_tile = obs_tile_.get();
              a.obs_m = m();
            }
          }
          if (L.lite) {
            set_fused(a, L.woff);
            a.flags |= kFlagRawIn | kFlagNoRecur;
            bve_stage_lite(n, kModeTlm, a, L.cnt, L.st);
          } else {
            bve_stage(n, kModeTlm, a, L.cnt, L.st, fz);
          }
          count_launch();
          std::swap(L.s_cur, L.s_nxt);
        }
        first = false;
      }
      if (y && (k + 1) % d_.spi == 0) {
        const int iv = (k + 1) / d_.spi - 1;
        for (auto& L : lanes) {
          if (L.fz && !L.lite && obs_tile_.get()) continue;  // gathered inside the stage-3 launch
          gather_obs(state + L.v0 * dim_, dim_, idx_.get(), static_cast<int>(n_obs_),
                     w + static_cast<long long>(iv) * n_obs_, y + L.v0 * m() + static_cast<long long>(iv) * n_obs_,
                     m(), L.cnt, L.st);
          count_launch();
        }
      }
    }
    join_lanes(lanes);
  }
}

std::vector<Problem::Lane> Problem::split_lanes(int v0, int gn) const {
  // Concurrent lanes (streams) per group: two by default when it holds >= 2
  // vectors (SDV_LANES=k for k lanes, SDV_ONE_LANE for one), near-equal widths.
  std::vector<Lane> lanes;
  static const int nl_env = [] {
    if (std::getenv("SDV_ONE_LANE")) return 1;
    const char* e = std::getenv("SDV_LANES");
    return e ? std::max(1, std::min(8, std::atoi(e))) : 2;
  }();
  int nl = std::min(nl_env, gn);
  // fused BVE blocks: every lane keeps at least bve_stage_fill() stage CTAs
  // (narrow blocks run as one fused lane rather than two small-block lanes)
  if (fused(gn)) nl = std::min(nl, std::max(1, (d_.n / 8) * gn / bve_stage_fill()));
  if (nl <= 1) {
    lanes.push_back(Lane{v0, gn, 0, st_});
    lanes.back().fz = fused(gn);
    lanes.back().lite = !lanes.back().fz && d_.model == kModelBVE && bve_lite_ok(d_.n, gn);
    return lanes;
  }
  while (static_cast<int>(lane_st_.size()) < nl - 1) {
    cudaStream_t s2;
    cudaEvent_t e2;
    SDV_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    SDV_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    lane_st_.push_back(s2);
    lane_ev_.push_back(e2);
  }
  if (!ev_fork_) SDV_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  SDV_CUDA(cudaEventRecord(ev_fork_, st_));
  int off = 0;
  for (int i = 0; i < nl; ++i) {
    const int cnt = gn / nl + (i < gn % nl ? 1 : 0);
    cudaStream_t st = i == 0 ? st_ : lane_st_[i - 1];
    if (i > 0) SDV_CUDA(cudaStreamWaitEvent(st, ev_fork_, 0));
    lanes.push_back(Lane{v0 + off, cnt, off, st});
    off += cnt;
  }
  for (auto& L : lanes) {
    L.fz = fused(L.cnt);
    L.lite = !L.fz && d_.model == kModelBVE && bve_lite_ok(d_.n, L.cnt);
  }
  return lanes;
}

void Problem::refork_lanes(const std::vector<Lane>& lanes) const {
  if (lanes.size() < 2) return;
  SDV_CUDA(cudaEventRecord(ev_fork_, st_));
  for (size_t i = 1; i < lanes.size(); ++i) SDV_CUDA(cudaStreamWaitEvent(lanes[i].st, ev_fork_, 0));
}

void Problem::join_lanes(const std::vector<Lane>& lanes) const {
  for (size_t i = 1; i < lanes.size(); ++i) {
    SDV_CUDA(cudaEventRecord(lane_ev_[i - 1], lanes[i].st));
    SDV_CUDA(cudaStreamWaitEvent(st_, lane_ev_[i - 1], 0));
  }
}

void Problem::adj(const Trajectory& tr, double* state, int nvec, int k0, int k1, const double* y,
                  const double* w) const {
  if (k0 < 0 || k1 > tr.steps || k0 > k1) throw std::invalid_argument("trajectory: step range out of bounds");
  if (nvec <= 0 || k0 == k1) return;
  if (d_.model == kModelBVE3) return bve3_adj(tr, state, nvec, k0, k1, y, w);
  if (d_.model == kModelBurgers || d_.model == kModelBurgers3) {
    BurgersArgs a = burgers_args(d_);
    a.base = tr.w.get();
    a.k0 = k0;
    a.k1 = k1;
    a.idx = idx_.get();
    a.n_obs = static_cast<int>(n_obs_);
    a.w = w;
    a.y = const_cast<double*>(y);
    a.m = m();
    // checkpoint mode: one launch per segment, in reverse step order
    if (!tr.checkpointed()) {
      if (d_.model == kModelBurgers3)
        burgers3_adj(a, state, nvec, st_);
      else
        burgers_adj(a, state, nvec, st_);
      count_launch();
      count_path(kPathBurgers);
      return;
    }
    tr.seg = -1;
    for (int kb = ((k1 - 1) / tr.stride) * tr.stride; kb + tr.stride > k0 && kb >= 0; kb -= tr.stride) {
      a.k0 = std::max(k0, kb);
      a.k1 = std::min(k1, kb + tr.stride);
      hold_segment(tr, a.k0);
      a.base = tr.w.get();
      a.base_k0 = tr.held_k0();
      if (d_.model == kModelBurgers3)
        burgers3_adj(a, state, nvec, st_);
      else
        burgers_adj(a, state, nvec, st_);
      count_launch();
      count_path(kPathBurgers);
    }
    return;
  }
  ensure_work(nvec);
  if (tr.checkpointed()) tr.seg = -1;  // each sweep recomputes what it reads (graph replays stay valid)
  const int n = d_.n, g = std::min(nvec, group());
  const long long sdim = static_cast<long long>(n) * (n / 2);
  for (int v0 = 0; v0 < nvec; v0 += g) {
    const int gn = std::min(g, nvec - v0);
    std::vector<Lane> lanes = split_lanes(v0, gn);
    for (auto& L : lanes) {
      L.s_cur = ws0_.get() + L.woff * sdim;
      L.s_nxt = ws1_.get() + L.woff * sdim;
    }
    int qi = 0;
    bool first = true;
    for (int k = k1 - 1; k >= k0; --k) {
      if (tr.checkpointed() && k / tr.stride != tr.seg) {
        join_lanes(lanes);
        hold_segment(tr, k);
        refork_lanes(lanes);
      }
      if (y && (k + 1) % d_.spi == 0) {
        const int iv = (k + 1) / d_.spi - 1;
        for (auto& L : lanes) {
          double* lam = state + L.v0 * dim_;
          double* acc = wa_.get() + L.woff * dim_;
          scatter_obs(first ? lam : acc, dim_, idx_.get(), static_cast<int>(n_obs_),
                      w + static_cast<long long>(iv) * n_obs_, y + L.v0 * m() + static_cast<long long>(iv) * n_obs_,
                      m(), L.cnt, L.st);
          count_launch();
        }
      }
      for (int s = 3; s >= 0; --s) {
        const bool has_prev = !first;
        if (has_prev)
          for (auto& L : lanes) {
            if (L.fz) poisson_carry(L.s_cur, L.woff, L.cnt, L.st);
            else poisson_col(L.s_cur, L.cnt, L.st);
          }
        for (auto& L : lanes) {
          const bool fz = L.fz;
          StageArgs a = bve_args(d_);
          a.stage = s;
          a.flags = has_prev ? kFlagHasPrev : 0;
          a.s_in = L.s_cur;
          a.s_out = L.s_nxt;
          a.d = state + L.v0 * dim_;
          a.acc = wa_.get() + L.woff * dim_;
          a.q_in = (qi ? wx1_.get() : wx0_.get()) + L.woff * dim_;
          a.q_out = (qi ? wx0_.get() : wx1_.get()) + L.woff * dim_;
          a.base_w = tr.base_w(k, s, dim_);
          a.base_p = tr.base_p(k, s, dim_);
          if (fz) set_fused(a, L.woff);
          if (L.lite) {
            set_fused(a, L.woff);
            a.flags |= kFlagRawIn | kFlagNoRecur;
            bve_stage_lite(n, kModeAdj, a, L.cnt, L.st);
          } else {
            bve_stage(n, kModeAdj, a, L.cnt, L.st, fz);
          }
          count_launch();
          std::swap(L.s_cur, L.s_nxt);
        }
        qi ^= 1;
        first = false;
      }
    }
    for (auto& L : lanes) {
      const bool fz = L.fz;
      if (fz) poisson_carry(L.s_cur, L.woff, L.cnt, L.st);
      else poisson_col(L.s_cur, L.cnt, L.st);
      StageArgs a = bve_args(d_);
      a.flags = kFlagHasPrev | kFlagFinish;
      a.s_in = L.s_cur;
      a.d = state + L.v0 * dim_;
      a.acc = wa_.get() + L.woff * dim_;
      a.q_in = (qi ? wx1_.get() : wx0_.get()) + L.woff * dim_;
      if (fz) set_fused(a, L.woff);
      if (L.lite) {
        set_fused(a, L.woff);
        a.flags |= kFlagRawIn | kFlagNoRecur;
        bve_stage_lite(n, kModeAdj, a, L.cnt, L.st);
      } else {
        bve_stage(n, kModeAdj, a, L.cnt, L.st, fz);
      }
      count_launch();
    }
    join_lanes(lanes);
  }
}

// ADJ counterpart of probe_stage_kernels (BVE only): `stages` adjoint RK
// stages of one s-vector launch (reverse stage order, has_prev after the
// first), with the carry / column pass timed separately. The inputs are the
// probe's own workspaces; only the timing is meaningful.
void Problem::probe_adj_stage_kernels(const Trajectory& tr, int s, int stages, float* ms_stage, float* ms_col) const {
  if (s < 1 || stages < 1) throw std::invalid_argument("probe: need s >= 1 and stages >= 1");
  if (d_.model != kModelBVE) throw std::invalid_argument("probe: the ADJ stage probe covers the periodic BVE model");
  cudaEvent_t ev[3];
  for (auto& e : ev) SDV_CUDA(cudaEventCreate(&e));
  s = std::min(s, group());
  wstate_.ensure(static_cast<size_t>(s) * dim_);
  ensure_work(s);
  for (int v = 0; v < s; ++v)
    SDV_CUDA(cudaMemcpyAsync(wstate_.get() + v * dim_, tr.w.get(), sizeof(double) * dim_, cudaMemcpyDeviceToDevice,
                             st_));
  const int n = d_.n;
  const bool fz = fused(s);
  double2* s_cur = ws0_.get();
  double2* s_nxt = ws1_.get();
  bve_row_fwd(n, wstate_.get(), s_cur, s, st_);
  SDV_CUDA(cudaMemcpyAsync(wx0_.get(), wstate_.get(), sizeof(double) * dim_ * s, cudaMemcpyDeviceToDevice, st_));
  double tot_stage = 0.0, tot_col = 0.0;
  int qi = 0;
  for (int q = 0; q < stages; ++q) {
    const int k = tr.held_steps() - 1 - (q / 4) % tr.held_steps(), sg = 3 - q % 4;
    const bool has_prev = q > 0;
    SDV_CUDA(cudaEventRecord(ev[0], st_));
    if (has_prev) {
      if (fz) poisson_carry(s_cur, 0, s, st_);
      else poisson_col(s_cur, s, st_);
    }
    SDV_CUDA(cudaEventRecord(ev[1], st_));
    StageArgs a = bve_args(d_);
    a.stage = sg;
    a.flags = has_prev ? kFlagHasPrev : 0;
    a.s_in = s_cur;
    a.s_out = s_nxt;
    a.d = wstate_.get();
    a.acc = wa_.get();
    a.q_in = qi ? wx1_.get() : wx0_.get();
    a.q_out = qi ? wx0_.get() : wx1_.get();
    a.base_w = tr.w.get() + (static_cast<long long>(k) * 4 + sg) * dim_;
    a.base_p = tr.p.get() + (static_cast<long long>(k) * 4 + sg) * dim_;
    if (fz) set_fused(a, 0);
    bve_stage(n, kModeAdj, a, s, st_, fz);
    SDV_CUDA(cudaEventRecord(ev[2], st_));
    SDV_CUDA(cudaEventSynchronize(ev[2]));
    float m1 = 0, m2 = 0;
    SDV_CUDA(cudaEventElapsedTime(&m1, ev[0], ev[1]));
    SDV_CUDA(cudaEventElapsedTime(&m2, ev[1], ev[2]));
    tot_col += m1;
    tot_stage += m2;
    std::swap(s_cur, s_nxt);
    qi ^= 1;
  }
  *ms_stage = static_cast<float>(tot_stage / stages);
  *ms_col = static_cast<float>(tot_col / std::max(1, stages - 1));
  for (auto& e : ev) SDV_CUDA(cudaEventDestroy(e));
}

void Problem::probe_stage_kernels(const Trajectory& tr, int s, int stages, float* ms_stage, float* ms_col) const {
  if (s < 1 || stages < 1) throw std::invalid_argument("probe: need s >= 1 and stages >= 1");
  if (d_.model == kModelBVE3) throw std::invalid_argument("probe: the stage-kernel probe covers the BASELINE models");
  cudaEvent_t ev[3];
  for (auto& e : ev) SDV_CUDA(cudaEventCreate(&e));
  wstate_.ensure(static_cast<size_t>(s) * dim_);
  for (int v = 0; v < s; ++v)
    SDV_CUDA(cudaMemcpyAsync(wstate_.get() + v * dim_, tr.w.get(), sizeof(double) * dim_, cudaMemcpyDeviceToDevice,
                             st_));
  double tot_stage = 0.0, tot_col = 0.0;
  if (d_.model == kModelBurgers || d_.model == kModelBurgers3) {
    const int steps = std::max(1, std::min(tr.held_steps(), stages / tr.stages));
    BurgersArgs a = burgers_args(d_);
    a.base = tr.w.get();
    a.k0 = 0;
    a.k1 = steps;
    SDV_CUDA(cudaEventRecord(ev[0], st_));
    if (d_.model == kModelBurgers3)
      burgers3_tlm(a, wstate_.get(), s, st_);
    else
      burgers_tlm(a, wstate_.get(), s, st_);
    SDV_CUDA(cudaEventRecord(ev[1], st_));
    SDV_CUDA(cudaEventSynchronize(ev[1]));
    float ms = 0;
    SDV_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    *ms_stage = ms;
    *ms_col = 0.0f;
  } else {
    s = std::min(s, group());  // one launch covers one sweep group
    ensure_work(s);
    const int n = d_.n;
    double* dst = wstate_.get();
    double* xb[2] = {wx0_.get(), wx1_.get()};
    double2* s_cur = ws0_.get();
    double2* s_nxt = ws1_.get();
    bve_row_fwd(n, dst, s_cur, s, st_);
    const bool fz = fused(s);
    for (int q = 0; q < stages; ++q) {
      const int k = (q / 4) % tr.held_steps(), sg = q % 4;
      SDV_CUDA(cudaEventRecord(ev[0], st_));
      if (fz && q > 0) poisson_carry(s_cur, 0, s, st_);
      else poisson_col(s_cur, s, st_);
      SDV_CUDA(cudaEventRecord(ev[1], st_));
      StageArgs a = bve_args(d_);
      a.stage = sg;
      // SDV_PROBE_FLAGS (timing experiments): skip phases, see kFlagSkip*.
      if (const char* e = std::getenv("SDV_PROBE_FLAGS")) a.flags = std::atoi(e);
      a.s_in = s_cur;
      a.s_out = s_nxt;
      a.x_in = sg == 0 ? dst : xb[(sg - 1) & 1];
      a.x_out = sg < 3 ? xb[sg & 1] : nullptr;
      a.d = dst;
      a.acc = wa_.get();
      a.base_w = tr.w.get() + (static_cast<long long>(k) * 4 + sg) * dim_;
      a.base_p = tr.p.get() + (static_cast<long long>(k) * 4 + sg) * dim_;
      if (fz) {
        set_fused(a, 0);
        if (q == 0) a.flags |= kFlagRawIn;
      }
      bve_stage(n, kModeTlm, a, s, st_, fz);
      SDV_CUDA(cudaEventRecord(ev[2], st_));
      SDV_CUDA(cudaEventSynchronize(ev[2]));
      float m1 = 0, m2 = 0;
      SDV_CUDA(cudaEventElapsedTime(&m1, ev[0], ev[1]));
      SDV_CUDA(cudaEventElapsedTime(&m2, ev[1], ev[2]));
      tot_col += m1;
      tot_stage += m2;
      std::swap(s_cur, s_nxt);
    }
    *ms_stage = static_cast<float>(tot_stage / stages);
    *ms_col = static_cast<float>(tot_col / stages);
  }
  for (auto& e : ev) SDV_CUDA(cudaEventDestroy(e));
}

// L2-resident sub-blocks. A BVE block whose RK workspace (d, acc, X0, X1, two
// row-spectra buffers, tile carries: ~6.4 fields per vector) does not fit the
// 126 MB L2 is swept as consecutive sub-blocks that do (512^2: 8 vectors x
// 13.4 MB), each through the whole window as one CUDA-graph replay on fixed
// staging buffers, so HBM carries only the base trajectory (re-read once per
// sub-block: 14 x 13.4 GB for s = 110, ~2% of the sweep time). Measured on
// B200 (profiles/r2_small_blocks.md): 8-vector graph-replayed sub-blocks run at
// 39.0 HVP/s against 36.6 for the 110-wide block. Widths differ by at most
// one (110 = 12 x 8 + 2 x 7: two graphs). Returns the sub-block count (0 = sweep
// the block whole).
int Problem::sub_blocks(int s) const {
  static const bool off = std::getenv("SDV_NO_SUBBLOCK") != nullptr;
  if (off || d_.model != kModelBVE || d_.block_group > 0) return 0;
  const double per = 6.4 * 8.0 * static_cast<double>(dim_);
  const int cap = static_cast<int>(112e6 / per);  // vectors whose workspace stays in L2
  // grids whose resident width exceeds the graph-replay width (<= 256^2) keep
  // the whole-block sweep: their blocks fit L2 or nearly so
  if (cap < 2 || cap > graph_max() || s < 2 * cap) return 0;
  return (s + cap - 1) / cap;
}

int Problem::graph_max() {
  static const int g = [] {
    const char* e = std::getenv("SDV_GRAPH_MAX");
    return e ? std::atoi(e) : 8;
  }();
  return g;
}

// run() for every sub-block [off, off + w) of an s-wide block: `in` (s x
// in_dim) is staged into sub_in_, run(sub_in_, w, sub_out_) produces w x
// out_dim, copied to `out`.
template <class F>
void Problem::for_sub_blocks(int nb, const double* in, long long in_dim, double* out, long long out_dim, int s,
                             F&& run) const {
  const int base = s / nb, rem = s % nb;
  const int wmax = base + (rem ? 1 : 0);
  sub_in_.ensure(static_cast<size_t>(wmax) * in_dim);
  sub_out_.ensure(static_cast<size_t>(wmax) * out_dim);
  int off = 0;
  for (int b = 0; b < nb; ++b) {
    const int w = base + (b < rem ? 1 : 0);
    SDV_CUDA(cudaMemcpyAsync(sub_in_.get(), in + static_cast<long long>(off) * in_dim, sizeof(double) * w * in_dim,
                             cudaMemcpyDeviceToDevice, st_));
    run(sub_in_.get(), w, sub_out_.get());
    SDV_CUDA(cudaMemcpyAsync(out + static_cast<long long>(off) * out_dim, sub_out_.get(), sizeof(double) * w * out_dim,
                             cudaMemcpyDeviceToDevice, st_));
    off += w;
  }
}

void Problem::misfit_apply_whole(const Trajectory& tr, const double* v, int s, double* y) const {
  wstate_.ensure(static_cast<size_t>(s) * dim_);
  prior_sqrt(v, wstate_.get(), s);
  tlm(tr, wstate_.get(), s, 0, total_steps(), y, rinv_sqrt_.get());
}

void Problem::misfit_adjoint_whole(const Trajectory& tr, const double* w, int s, double* z) const {
  wstate_.ensure(static_cast<size_t>(s) * dim_);
  dev_fill(static_cast<long long>(s) * dim_, 0.0, wstate_.get(), st_);
  adj(tr, wstate_.get(), s, 0, total_steps(), w, rinv_sqrt_.get());
  prior_sqrt(wstate_.get(), z, s);
}

void Problem::misfit_apply(const Trajectory& tr, const double* v, int s, double* y) const {
  const int nb = sub_blocks(s);
  if (nb == 0) return misfit_apply_whole(tr, v, s, y);
  for_sub_blocks(nb, v, dim_, y, m(), s, [&](const double* vi, int w, double* yo) {
    wstate_.ensure(static_cast<size_t>(w) * dim_);
    ensure_work(w);
    graph_cached(kOpApply, tr, vi, yo, w, [&] { misfit_apply_whole(tr, vi, w, yo); });
  });
}

void Problem::misfit_adjoint(const Trajectory& tr, const double* w, int s, double* z) const {
  const int nb = sub_blocks(s);
  if (nb == 0) return misfit_adjoint_whole(tr, w, s, z);
  for_sub_blocks(nb, w, m(), z, dim_, s, [&](const double* wi, int wd, double* zo) {
    wstate_.ensure(static_cast<size_t>(wd) * dim_);
    ensure_work(wd);
    graph_cached(kOpAdjoint, tr, wi, zo, wd, [&] { misfit_adjoint_whole(tr, wi, wd, zo); });
  });
}

void Problem::gram_apply(const Trajectory& tr, const double* v, int s, double* hv) const {
  const int nb = sub_blocks(s);
  if (nb > 0) {
    for_sub_blocks(nb, v, dim_, hv, dim_, s,
                   [&](const double* vi, int w, double* ho) { gram_apply(tr, vi, w, ho); });
    return;
  }
  wy_.ensure(static_cast<size_t>(s) * m());
  wstate_.ensure(static_cast<size_t>(s) * dim_);
  ensure_work(s);
  auto run = [&] {
    misfit_apply_whole(tr, v, s, wy_.get());
    misfit_adjoint_whole(tr, wy_.get(), s, hv);
  };
  // Small blocks are launch-latency bound (thousands of short kernels per
  // sweep): capture the sweep once as a CUDA graph and replay it.
  if (s > graph_max()) return run();
  graph_cached(kOpGram, tr, v, hv, s, run);
}

// Replays `run` (a sweep on this problem's stream whose launches depend only
// on the key) as a CUDA graph: the first use runs plain launches (lazy
// initialisation happens there), the second captures and instantiates, later
// ones replay. The key is the operation and every pointer the captured
// launches bake in.
template <class F>
void Problem::graph_cached(int op, const Trajectory& tr, const double* in, double* out, int s, F&& run) const {
  if (std::getenv("SDV_NO_GRAPHS")) return run();
  const std::vector<const void*> key = {reinterpret_cast<const void*>(static_cast<intptr_t>(op)),
                                        &tr,         tr.w.get(),    tr.p.get(),   in,         out,
                                        wy_.get(),   wstate_.get(), wa_.get(),    wx0_.get(), wx1_.get(),
                                        ws0_.get(),  ws1_.get(),    reinterpret_cast<const void*>(static_cast<intptr_t>(s)),
                                        // the sweep structure the launches follow
                                        reinterpret_cast<const void*>(static_cast<intptr_t>(tr.steps)),
                                        reinterpret_cast<const void*>(static_cast<intptr_t>(tr.stride))};
  GraphEntry* hit = nullptr;
  for (auto& g : graphs_)
    if (g.key == key) hit = &g;
  if (hit && hit->exec) {
    SDV_CUDA(cudaGraphLaunch(hit->exec, st_));
    count_launch(hit->nodes);
    return;
  }
  if (!hit) {  // first use: plain launches (lazy initialisation happens here)
    if (graphs_.size() >= 8) {
      if (graphs_.front().exec) cudaGraphExecDestroy(graphs_.front().exec);
      graphs_.erase(graphs_.begin());
    }
    graphs_.push_back(GraphEntry{key, nullptr, 0});
    run();
    return;
  }
  cudaGraph_t graph = nullptr;
  const unsigned long long before = t_launches;
  SDV_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
  try {
    run();
  } catch (...) {
    cudaStreamEndCapture(st_, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  SDV_CUDA(cudaStreamEndCapture(st_, &graph));
  hit->nodes = t_launches - before;  // kernels per replay (recorded, not launched)
  g_launches.fetch_sub(hit->nodes, std::memory_order_relaxed);
  t_launches = before;
  SDV_CUDA(cudaGraphInstantiate(&hit->exec, graph, 0));
  SDV_CUDA(cudaGraphDestroy(graph));
  SDV_CUDA(cudaGraphLaunch(hit->exec, st_));
  count_launch(hit->nodes);
}

void Problem::clear_graphs() const {
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
}

Problem::~Problem() {
  clear_graphs();
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  for (auto e : lane_ev_) cudaEventDestroy(e);
  for (auto s2 : lane_st_) {
    release_stream_work(s2);
    cudaStreamDestroy(s2);
  }
  if (st_) {
    release_stream_work(st_);
    cudaStreamDestroy(st_);
  }
}

// --------------------------------------------- reference BVE (kModelBVE3) --
void Problem::bve3_work(int nvec) const {
  for (auto& b : b3w_) b.ensure(static_cast<size_t>(nvec) * dim_);
}

// LinearizedTrajectory::tlm_range of proj/src/bve.cpp:138-148 for a block:
// per step d1 = d + dt J0 d, d2 = 0.75 d + 0.25 (d1 + dt J1 d1),
// d' = d/3 + 2/3 (d2 + dt J2 d2), each J_s d needing psi' = P(d_s).
void Problem::bve3_tlm(const Trajectory& tr, double* state, int nvec, int k0, int k1, double* y,
                       const double* w) const {
  bve3_work(nvec);
  double* st[3] = {state, b3w_[0].get(), b3w_[1].get()};
  double* dp = b3w_[2].get();
  for (int k = k0; k < k1; ++k) {
    const double* wk = tr.w.get() + static_cast<long long>(k) * 3 * dim_;
    const double* pk = tr.p.get() + static_cast<long long>(k) * 3 * dim_;
    for (int s = 0; s < 3; ++s) {
      poisson3_->solve(st[s], dp, nvec);
      // stage 2 writes d' in place over d (point-wise read of d only)
      bve3_tlm_stage(b3_, s, state, st[s], dp, wk + s * dim_, pk + s * dim_, s < 2 ? st[s + 1] : state, nvec, st_);
      count_launch(2);  // DST scale + stage (the GEMMs are cuBLAS)
    }
    if (y && (k + 1) % d_.spi == 0) {
      const int iv = (k + 1) / d_.spi - 1;
      gather_obs(state, dim_, idx_.get(), static_cast<int>(n_obs_), w + static_cast<long long>(iv) * n_obs_,
                 y + static_cast<long long>(iv) * n_obs_, m(), nvec, st_);
      count_launch();
    }
  }
}

// adj_range of proj/src/bve.cpp:150-161 for a block: per step (reverse)
// t2 = 2/3 (lam + dt J2^T lam), t1 = 0.25 (t2 + dt J1^T t2),
// lam' = lam/3 + 0.75 t2 + t1 + dt J0^T t1, J^T (:199-211) with one Poisson
// solve of its vp part; observation scatters at interval ends first.
void Problem::bve3_adj(const Trajectory& tr, double* state, int nvec, int k0, int k1, const double* y,
                       const double* w) const {
  bve3_work(nvec);
  double* t2 = b3w_[0].get();
  double* t1 = b3w_[1].get();
  double* vp = b3w_[2].get();
  for (int k = k1 - 1; k >= k0; --k) {
    if (y && (k + 1) % d_.spi == 0) {
      const int iv = (k + 1) / d_.spi - 1;
      scatter_obs(state, dim_, idx_.get(), static_cast<int>(n_obs_), w + static_cast<long long>(iv) * n_obs_,
                  y + static_cast<long long>(iv) * n_obs_, m(), nvec, st_);
      count_launch();
    }
    const double* wk = tr.w.get() + static_cast<long long>(k) * 3 * dim_;
    const double* pk = tr.p.get() + static_cast<long long>(k) * 3 * dim_;
    const double* L[3] = {t1, t2, state};  // argument of J_s^T
    double* out[3] = {state, t1, t2};      // stage 0 writes lam' in place (point-wise read of lam only)
    for (int s = 2; s >= 0; --s) {
      bve3_adj_vp(b3_, L[s], wk + s * dim_, vp, nvec, st_);
      poisson3_->solve(vp, vp, nvec);
      bve3_adj_stage(b3_, s, L[s], vp, pk + s * dim_, state, t2, out[s], nvec, st_);
      count_launch(3);  // vp, DST scale, stage (the GEMMs are cuBLAS)
    }
  }
}

void Problem::prior_inv_sqrt(const double* in, double* out, int nvec) const {
  if (d_.prior_kind != kPriorLaplacian) throw std::invalid_argument("prior_inv_sqrt: only the Laplacian prior has one");
  if (d_.model == kModelBVE3) {
    lap2_inv_sqrt(d_.n, d_.ny, d_.prior_alpha, d_.prior_beta, in, out, nvec, st_);
    count_launch();
    return;
  }
  lap_inv_sqrt(d_.n, d_.prior_alpha, lap_b_, in, out, nvec, st_);
  count_launch();
}

double Problem::evaluate(const Trajectory& tr, const double* d_z, double* d_ctrl_grad, double* d_lambda0,
                         double* d_grad_x) const {
  const long long mm = m();
  DevBuf<double> innov(static_cast<size_t>(std::max<long long>(mm, 1))), winnov(innov.size()), sc(2),
      lam(static_cast<size_t>(dim_));
  // x-space background term (proj/src/fourdvar.cpp:101-104): dxb = x0 - xb,
  // ib = Gamma^{-1} dxb, cost_b = dxb . ib / 2.
  DevBuf<double> dxb, ib;
  if (xspace()) {
    dxb.alloc(static_cast<size_t>(dim_));
    ib.alloc(static_cast<size_t>(dim_));
    SDV_CUDA(cudaMemcpyAsync(dxb.get(), tr.state_at(0), sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    dev_axpby(dim_, -1.0, background_.get(), 1.0, dxb.get(), st_);
    prior_inv_sqrt(dxb.get(), lam.get(), 1);
    prior_inv_sqrt(lam.get(), ib.get(), 1);
  }
  for (int i = 1; i <= d_.n_t; ++i) {
    const long long o = static_cast<long long>(i - 1) * n_obs_;
    if (n_obs_ > 0) {
      innovation_kernel<<<ceil_div(n_obs_, 256), 256, 0, st_>>>(tr.state_at(i * d_.spi), idx_.get(),
                                                                static_cast<int>(n_obs_), values_.get() + o,
                                                                rinv_.get() + o, innov.get() + o, winnov.get() + o);
      count_launch();
      SDV_LAUNCH_CHECK();
    }
  }
  dev_dot(innov.get(), winnov.get(), mm, sc.get(), st_);
  if (xspace()) dev_dot(dxb.get(), ib.get(), dim_, sc.get() + 1, st_);
  else if (d_z) dev_dot(d_z, d_z, dim_, sc.get() + 1, st_);
  else dev_fill(1, 0.0, sc.get() + 1, st_);
  dev_fill(dim_, 0.0, lam.get(), st_);
  adj(tr, lam.get(), 1, 0, total_steps(), innov.get(), rinv_.get());
  if (d_lambda0) SDV_CUDA(cudaMemcpyAsync(d_lambda0, lam.get(), sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
  if (xspace()) {
    // g = Gamma^{-1}(x0 - xb) + lambda0; ctrl_grad = Gamma^{1/2} g
    dev_axpby(dim_, 1.0, lam.get(), 1.0, ib.get(), st_);
    if (d_grad_x) SDV_CUDA(cudaMemcpyAsync(d_grad_x, ib.get(), sizeof(double) * dim_, cudaMemcpyDeviceToDevice, st_));
    if (d_ctrl_grad) prior_sqrt(ib.get(), d_ctrl_grad, 1);
  } else if (d_ctrl_grad) {
    prior_sqrt(lam.get(), d_ctrl_grad, 1);
    if (d_z) dev_axpby(dim_, 1.0, d_z, 1.0, d_ctrl_grad, st_);
  }
  double h[2];
  SDV_CUDA(cudaMemcpyAsync(h, sc.get(), sizeof(h), cudaMemcpyDeviceToHost, st_));
  SDV_CUDA(cudaStreamSynchronize(st_));
  return 0.5 * h[1] + 0.5 * h[0];
}

}  // namespace sdv

// CPU ORACLE — test infrastructure only. Never linked, imported or executed by
// the product path (paper_2401_15758_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it.
//
// A C++ restatement of the reference sketchdav library (/root/reference/proj),
// Eigen-free, following it function by function (file:line cited at each
// definition), plus the BASELINE.json config discretisations (periodic RK4
// Burgers, periodic RK4 Arakawa BVE, Fourier-diagonal Gaussian B) written as new
// implementations of the reference's DynamicalModel / LinearizedTrajectory /
// prior interfaces.
#pragma once

#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;
using cplx = std::complex<double>;

// Column-major dense matrix (Eigen::MatrixXd stand-in).
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int64_t rows, int64_t cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return a[static_cast<size_t>(i + j * r)]; }
  double operator()(int64_t i, int64_t j) const { return a[static_cast<size_t>(i + j * r)]; }
  double* col(int64_t j) { return a.data() + j * r; }
  const double* col(int64_t j) const { return a.data() + j * r; }
  Vec colv(int64_t j) const { return Vec(col(j), col(j) + r); }
  void set_col(int64_t j, const Vec& v) { std::copy(v.begin(), v.end(), col(j)); }
  static Mat identity(int64_t n, int64_t m);
};

// ---- vector helpers --------------------------------------------------------
double dot(const Vec& a, const Vec& b);
double norm2(const Vec& a);
double norm_inf(const Vec& a);
Vec axpby(double a, const Vec& x, double b, const Vec& y);  // a x + b y
Vec scaled(double a, const Vec& x);
bool all_finite(const Vec& v);

Mat matmul(const Mat& a, const Mat& b);        // a b
Mat matmul_tn(const Mat& a, const Mat& b);     // a^T b
Mat transpose(const Mat& a);
Vec matvec(const Mat& a, const Vec& x);
Vec matvec_t(const Mat& a, const Vec& x);
Mat append_columns(const Mat& a, const Mat& b);
Mat left_cols(const Mat& a, int64_t k);

// ---- rng (proj/src/rng.cpp) -------------------------------------------------
uint64_t mix_seed(uint64_t seed, uint64_t stream);
Mat gaussian_matrix(int64_t n, int64_t l, uint64_t seed);
Vec gaussian_vector(int64_t n, uint64_t seed);

// ---- dense linear algebra (proj/src/linalg.cpp) ----------------------------
struct ThinQR {
  Mat q, r;
  std::vector<int64_t> deficient_columns;
};
ThinQR thin_qr(const Mat& y);
struct ThinSVD {
  Mat u;
  Vec s;
  Mat v;
};
ThinSVD thin_svd(const Mat& a);
Mat pseudo_inverse(const Mat& a, int* truncated = nullptr);
Mat cholesky_lower(const Mat& spd);
double spectral_norm(const Mat& a);
// Symmetric eigen-decomposition (cyclic Jacobi); eigenvalues ascending.
void sym_eig(const Mat& a, Vec& evals, Mat& evecs);
// Lower-triangular solve L X = B.
Mat lower_solve(const Mat& l, const Mat& b);

// ---- intra-operator threading (speed only; results are bitwise identical) --
// par_for(n, f) calls f(b, e) on a static partition of [0, n) over
// ORACLE_THREADS threads (default 1 = serial). Every output element is computed
// by exactly the same arithmetic whichever thread owns it, and reductions stay
// serial, so threading never changes a bit. Serial inside apply_columns
// workers (no nested oversubscription) and when the pool is busy.
void par_for(int64_t n, const std::function<void(int64_t, int64_t)>& f);
void set_no_par(bool v);  // this thread: run par_for serially

// ---- FFT (radix-2, power-of-two lengths) -----------------------------------
void fft_inplace(std::vector<cplx>& x, bool inverse);  // unnormalised
void fft2_inplace(std::vector<cplx>& x, int nx, int ny, bool inverse);

// ---- LinearMap (proj/include/sketchdav/linalg.hpp:17-99) -------------------
class LinearMap {
 public:
  virtual ~LinearMap() = default;
  virtual int64_t rows() const = 0;
  virtual int64_t cols() const = 0;
  virtual Vec apply(const Vec& x) const = 0;
  virtual Vec adjoint_apply(const Vec& y) const = 0;
};

class DenseMap final : public LinearMap {
 public:
  explicit DenseMap(Mat a) : a_(std::move(a)) {}
  int64_t rows() const override { return a_.r; }
  int64_t cols() const override { return a_.c; }
  Vec apply(const Vec& x) const override { return matvec(a_, x); }
  Vec adjoint_apply(const Vec& y) const override { return matvec_t(a_, y); }
  const Mat& matrix() const { return a_; }

 private:
  Mat a_;
};

class FunctionMap final : public LinearMap {
 public:
  using Fn = std::function<Vec(const Vec&)>;
  FunctionMap(int64_t r, int64_t c, Fn ap, Fn adj = {})
      : r_(r), c_(c), ap_(std::move(ap)), adj_(std::move(adj)) {}
  int64_t rows() const override { return r_; }
  int64_t cols() const override { return c_; }
  Vec apply(const Vec& x) const override { return ap_(x); }
  Vec adjoint_apply(const Vec& y) const override { return adj_ ? adj_(y) : ap_(y); }

 private:
  int64_t r_, c_;
  Fn ap_, adj_;
};

class GramMap final : public LinearMap {
 public:
  explicit GramMap(const LinearMap& a) : a_(a) {}
  int64_t rows() const override { return a_.cols(); }
  int64_t cols() const override { return a_.cols(); }
  Vec apply(const Vec& x) const override { return a_.adjoint_apply(a_.apply(x)); }
  Vec adjoint_apply(const Vec& y) const override { return apply(y); }

 private:
  const LinearMap& a_;
};

class CountingMap final : public LinearMap {
 public:
  explicit CountingMap(const LinearMap& inner) : inner_(inner) {}
  int64_t rows() const override { return inner_.rows(); }
  int64_t cols() const override { return inner_.cols(); }
  Vec apply(const Vec& x) const override;
  Vec adjoint_apply(const Vec& y) const override;
  long applies() const;
  long adjoint_applies() const;

 private:
  const LinearMap& inner_;
  mutable std::atomic<long> applies_{0}, adjoint_applies_{0};
};

struct LowRankEVD {
  Mat basis;
  Vec eigenvalues;
  int64_t dim() const { return basis.r; }
  int64_t rank() const { return basis.c; }
  static LowRankEVD zero(int64_t n) { return LowRankEVD{Mat(n, 0), Vec()}; }
};

Vec woodbury_apply(const LowRankEVD& evd, const Vec& v);

struct PCGReport {
  Vec solution;
  int iterations = 0;
  std::vector<double> relative_residuals;
  bool converged = false;
};
using Preconditioner = std::function<Vec(const Vec&)>;
PCGReport pcg_solve(const LinearMap& op, const Vec& rhs, const Preconditioner& precond,
                    double tol, int max_iter);

// ---- models (proj/include/sketchdav/model.hpp:14-41) -----------------------
class LinearizedTrajectory {
 public:
  virtual ~LinearizedTrajectory() = default;
  virtual int total_steps() const = 0;
  virtual Vec state_at(int step) const = 0;
  virtual Vec tlm_range(int begin, int end, const Vec& dx) const = 0;
  virtual Vec adj_range(int begin, int end, const Vec& lambda) const = 0;
};

class DynamicalModel {
 public:
  virtual ~DynamicalModel() = default;
  virtual int64_t dim() const = 0;
  virtual double inner_dt() const = 0;
  virtual Vec forward(const Vec& x0, int steps) const = 0;
  virtual std::shared_ptr<const LinearizedTrajectory> linearize(const Vec& x0, int steps,
                                                                int stride) const = 0;
};

// 1-D viscous Burgers, periodic [0,1), dx = 1/n, centred advective form, RK4.
class PeriodicBurgers final : public DynamicalModel {
 public:
  PeriodicBurgers(int n, double nu, double dt);
  int64_t dim() const override { return n_; }
  double inner_dt() const override { return dt_; }
  int n() const { return n_; }
  double nu() const { return nu_; }
  Vec rhs(const Vec& u) const;
  Vec rhs_jacobian(const Vec& u, const Vec& d) const;
  Vec rhs_jacobian_adjoint(const Vec& u, const Vec& lam) const;
  Vec step(const Vec& u) const;
  Vec forward(const Vec& x0, int steps) const override;
  std::shared_ptr<const LinearizedTrajectory> linearize(const Vec& x0, int steps,
                                                        int stride) const override;

 private:
  int n_;
  double nu_, dt_;
};

// 2-D barotropic vorticity, periodic [0,2pi)^2, n x n, Arakawa Jacobian,
// 5-point Laplacian viscosity, spectral (5-point symbol) Poisson psi = (-Lap)^-1 w,
// RK4. Index i + n*j (x fastest).
class PeriodicBVE final : public DynamicalModel {
 public:
  PeriodicBVE(int n, double nu, double dt);
  int64_t dim() const override { return static_cast<int64_t>(n_) * n_; }
  double inner_dt() const override { return dt_; }
  int n() const { return n_; }
  double nu() const { return nu_; }
  double h() const { return 2.0 * M_PI / n_; }
  Vec poisson(const Vec& w) const;            // psi with -Lap5 psi = w, mean(psi)=0
  Vec arakawa(const Vec& a, const Vec& b) const;  // J(a,b) ~ a_x b_y - a_y b_x
  Vec laplacian(const Vec& f) const;          // 5-point
  Vec rhs(const Vec& w) const;
  Vec step(const Vec& w) const;
  Vec forward(const Vec& x0, int steps) const override;
  std::shared_ptr<const LinearizedTrajectory> linearize(const Vec& x0, int steps,
                                                        int stride) const override;

 private:
  int n_;
  double nu_, dt_;
  Vec inv_symbol_;  // 1/(n^2 mu(k)) on the full n x n spectrum, 0 at k=0
};

// Reference-faithful Dirichlet models (proj/src/burgers.cpp, proj/src/bve.cpp),
// RK3-TVD, used to pin the oracle against the reference's own fixture/bands.
class DirichletBurgers final : public DynamicalModel {
 public:
  DirichletBurgers(int n, double nu, double dt);
  int64_t dim() const override { return n_; }
  double inner_dt() const override { return dt_; }
  Vec rhs(const Vec& u) const;
  Vec rhs_jacobian(const Vec& u, const Vec& d) const;
  Vec rhs_jacobian_adjoint(const Vec& u, const Vec& lam) const;
  Vec step(const Vec& u) const;
  Vec forward(const Vec& x0, int steps) const override;
  std::shared_ptr<const LinearizedTrajectory> linearize(const Vec& x0, int steps,
                                                        int stride) const override;

 private:
  int n_;
  double nu_, dt_;
};

class DirichletSolver2D {
 public:
  DirichletSolver2D(int nx, int ny, double a, double bx, double by);
  Vec solve(const Vec& rhs) const;

 private:
  int nx_, ny_;
  Mat sx_, sy_;   // orthonormal DST-I matrices
  Mat inv_eig_;   // nx x ny
};

class Tridiagonal1D {
 public:
  Tridiagonal1D(int n, double diag, double off);
  Vec solve(const Vec& rhs) const;

 private:
  int n_;
  double off_;
  Vec pivot_;
};

Vec neg_laplacian_1d(const Vec& u);
Vec neg_laplacian_2d(const Vec& u, int nx, int ny, double sx, double sy);

class DirichletBVE final : public DynamicalModel {
 public:
  DirichletBVE(int nx, int ny, double re, double ro, double dt);
  int64_t dim() const override { return static_cast<int64_t>(nx_) * ny_; }
  double inner_dt() const override { return dt_; }
  double dx() const { return 1.0 / (nx_ + 1); }
  double dy() const { return 2.0 / (ny_ + 1); }
  Vec poisson_solve(const Vec& w) const { return poisson_->solve(w); }
  Vec d_x(const Vec& f) const;
  Vec d_y(const Vec& f) const;
  Vec laplacian(const Vec& f) const;
  Vec rhs(const Vec& w) const;
  Vec step(const Vec& w) const;
  Vec forward(const Vec& x0, int steps) const override;
  std::shared_ptr<const LinearizedTrajectory> linearize(const Vec& x0, int steps,
                                                        int stride) const override;
  int nx() const { return nx_; }
  int ny() const { return ny_; }
  double re() const { return re_; }
  double ro() const { return ro_; }
  const Vec& forcing() const { return forcing_; }

 private:
  int nx_, ny_;
  double re_, ro_, dt_;
  Vec forcing_;
  std::shared_ptr<DirichletSolver2D> poisson_;
};

// ---- priors (proj/include/sketchdav/prior.hpp) ------------------------------
// Common interface. has_inverse() selects the reference's x-space background
// term (Gamma^{-1} stencil); otherwise the control-variable form (Appendix B.3).
class Prior {
 public:
  virtual ~Prior() = default;
  virtual int64_t dim() const = 0;
  virtual Vec apply_sqrt(const Vec& v) const = 0;
  virtual bool has_inverse() const { return false; }
  virtual Vec apply_inv(const Vec& v) const {
    (void)v;
    throw std::logic_error("prior has no usable inverse (control-variable form)");
  }
  Vec sample_background(const Vec& truth, uint64_t seed) const;
};

// Gamma = (alpha I - beta Lap*)^{-2}, Dirichlet (proj/src/prior.cpp).
class LaplacianPrior final : public Prior {
 public:
  static std::shared_ptr<LaplacianPrior> make_1d(int n, double alpha, double beta, double scale = 1.0);
  static std::shared_ptr<LaplacianPrior> make_2d(int nx, int ny, double alpha, double beta,
                                                 double sx = 1.0, double sy = 1.0);
  int64_t dim() const override { return dim_; }
  Vec apply_sqrt(const Vec& v) const override;
  Vec apply_inv_sqrt(const Vec& v) const;
  bool has_inverse() const override { return true; }
  Vec apply_inv(const Vec& v) const override { return apply_inv_sqrt(apply_inv_sqrt(v)); }

 private:
  int64_t dim_ = 0;
  int nx_ = 0, ny_ = 0;
  double alpha_ = 0, beta_ = 0, sx_ = 1, sy_ = 1;
  std::shared_ptr<Tridiagonal1D> s1_;
  std::shared_ptr<DirichletSolver2D> s2_;
};

// B = sigma^2 C, C periodic Gaussian correlation; Fourier diagonal.
// 1-D: unit period, chat(k) ∝ exp(-(2 pi k L)^2/2); 2-D: 2pi period,
// chat(k) ∝ exp(-(|k| L)^2/2); normalised so c(0) = 1.
class FourierPrior final : public Prior {
 public:
  FourierPrior(int n, int dims, double sigma, double length);
  int64_t dim() const override { return dims_ == 1 ? n_ : static_cast<int64_t>(n_) * n_; }
  Vec apply_sqrt(const Vec& v) const override;
  const Vec& sqrt_symbol() const { return sym_; }  // includes 1/N, full spectrum

 private:
  int n_, dims_;
  Vec sym_;
};

// ---- 4D-Var (proj/src/fourdvar.cpp) ----------------------------------------
struct Observations {
  std::vector<int64_t> indices;
  Mat values;     // n_obs x n_t
  Mat variances;  // n_obs x n_t
};

struct AssimilationProblem {
  std::shared_ptr<const DynamicalModel> model;
  std::shared_ptr<const Prior> prior;
  Vec background;
  Observations obs;
  int n_t = 0;
  int steps_per_interval = 0;
  int64_t state_dim() const { return static_cast<int64_t>(background.size()); }
  int64_t n_obs() const { return obs.values.r; }
  int64_t misfit_dim() const { return obs.values.r * n_t; }
  int total_steps() const { return n_t * steps_per_interval; }
  void validate() const;
};

struct Counters {
  long fwd = 0, tlm = 0, adj = 0, offline_tlm = 0, offline_adj = 0;
};

// Control-variable form: x0 = xb + B^{1/2} z; for priors with an inverse the
// reference x-space form is used and z is unused.
struct Evaluation {
  double cost = 0.0;
  Vec gradient;        // x-space gradient (x-space form) — unused in control form
  Vec ctrl_gradient;   // Gamma^{1/2} g = z + Gamma^{1/2} lambda
  Vec lambda0;         // adjoint at t=0 (= sum_i M_i^T O^T R^-1 innov_i)
  std::shared_ptr<const LinearizedTrajectory> trajectory;
  std::vector<Vec> interval_states;
  Vec innovations;     // n_t x n_obs, time-major
};

Evaluation evaluate(const AssimilationProblem& p, const Vec& x0, const Vec* z, Counters* c);

class MisfitOperator final : public LinearMap {
 public:
  MisfitOperator(const AssimilationProblem& p, std::shared_ptr<const LinearizedTrajectory> traj);
  int64_t rows() const override { return p_.misfit_dim(); }
  int64_t cols() const override { return p_.state_dim(); }
  Vec apply(const Vec& v) const override;
  Vec adjoint_apply(const Vec& w) const override;

 private:
  const AssimilationProblem& p_;
  std::shared_ptr<const LinearizedTrajectory> traj_;
  Mat inv_sqrt_r_;
};

// ---- sketch (proj/src/sketch.cpp) ------------------------------------------
enum class SketchMethod { RandSVD, Nystrom, SingleView, Lanczos };
struct SketchConfig {
  SketchMethod method = SketchMethod::RandSVD;
  int rank = 10, rank2 = -1, growth = 5, growth2 = -1;
  double eps_sketch = 1.5, eps_reuse = 10.0;
  uint64_t seed = 0;
  int max_rank = -1;
  int workers = 1;
  int resolved_rank2() const { return rank2 > 0 ? rank2 : 2 * rank + 1; }
  void validate(int64_t m, int64_t n) const;
};
struct SketchReport {
  LowRankEVD evd;
  long tlm_applies = 0, adj_applies = 0;
  int final_rank = 0;
  std::vector<double> kappa_history;
  bool tolerance_met = true;
  int probe_applies = 0;
  Mat range_factor;
};
Mat apply_columns(const LinearMap& op, const Mat& x, bool adjoint, int workers = 1);
SketchReport randsvd_sketch(const LinearMap& a, int rank, uint64_t seed, int workers = 1);
LowRankEVD nystrom_assemble(const Mat& omega, const Mat& y);
SketchReport nystrom_sketch(const LinearMap& h, int rank, uint64_t seed, int workers = 1);
SketchReport singleview_sketch(const LinearMap& a, int rank1, int rank2, uint64_t seed,
                               int workers = 1);
SketchReport lanczos_sketch(const LinearMap& h, int rank, const Vec& start);
double cond_estimate(const LinearMap& h, const LowRankEVD& evd, uint64_t seed);
SketchReport adaptive_randsvd(const LinearMap& a, const SketchConfig& cfg, const LinearMap& h_probe);
SketchReport adaptive_nystrom(const LinearMap& h, const SketchConfig& cfg,
                              const LinearMap* h_probe = nullptr);
SketchReport adaptive_singleview(const LinearMap& a, const SketchConfig& cfg,
                                 const LinearMap& h_probe);
SketchReport adaptive_lanczos(const LinearMap& h, const SketchConfig& cfg, const Vec& start,
                              const LinearMap* h_probe = nullptr);
uint64_t probe_seed(uint64_t seed, int pass);
uint64_t growth_seed(uint64_t seed, int pass);
uint64_t psi_seed(uint64_t seed);

// ---- line search (proj/src/linesearch.cpp) ---------------------------------
struct LineSearchConfig {
  double sufficient_decrease = 1e-4, curvature = 0.9, step_tol = 1e-12;
  double step_min = 1e-20, step_max = 1e20;
  int max_trials = 20;
};
struct LineSearchResult {
  double step = 1.0, f = 0.0, dphi = 0.0;
  int trials = 0;
  bool ok = false;
};
LineSearchResult more_thuente_search(const std::function<std::pair<double, double>(double)>& phi,
                                     double f0, double dphi0, double initial_step,
                                     const LineSearchConfig& cfg);

// ---- Gauss-Newton (proj/src/fourdvar.cpp:213-422) --------------------------
enum class SolveMode { SketchSolv, SketchPrec, SketchPrecA, PrecGamma, PrecLanczos, PrecALanczos };
struct GNConfig {
  SolveMode mode = SolveMode::SketchPrec;
  SketchConfig sketch;
  double grad_tol = 1e-6, pcg_tol = 1e-9;
  int max_gn_iters = 50, pcg_max_iter = 10000;
  LineSearchConfig line_search;
};
struct GNIterationLog {
  int k = 0;
  double cost = 0, grad_inf_norm = 0, step_size = 0;
  int pcg_iterations = 0, line_search_trials = 0;
  bool pcg_converged = true, sketch_recomputed = false;
  int final_rank = 0;
  double kappa_sk = NAN, kappa_re = NAN;
  std::vector<double> eigenvalues;  // sketch eigenvalues when recomputed
  Counters totals;
};
struct GNResult {
  Vec analysis;
  std::vector<GNIterationLog> iterations;
  Counters counters;
  bool converged = false, line_search_failed = false;
  double final_cost = 0, final_grad_inf_norm = 0;
  long total_pcg = 0;
};
GNResult gn_solve(const AssimilationProblem& p, const GNConfig& cfg);

// ---- scenarios (BASELINE.json configs + reference presets) ------------------
struct Scenario {
  AssimilationProblem problem;
  Vec truth0;
  std::vector<Vec> truth_states;
  GNConfig gn;
  std::string name;
};
// cfg_id 0..4 = BASELINE.json configs; extra ids for reference presets.
Scenario make_config(int cfg_id, int steps_override = -1, int spi_override = -1);
Scenario make_reference_burgers_1_1();  // preset burgers_1_1 (Dirichlet RK3)
Scenario make_reference_bve_2();        // preset bve_2 (Dirichlet BVE, RK3)
Vec bve_truth_fixture_regen(int nx, int ny, double re, double ro, double dt, int steps,
                            uint64_t seed);
Vec periodic_grf_truth(int n, uint64_t seed);  // spectrum ∝ k^4 exp(-(k/4)^2), rms 1

}  // namespace oracle

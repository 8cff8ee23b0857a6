// Device-resident sketch / preconditioner / PCG / Gauss-Newton layer.
// Mirrors /root/reference/proj/include/sketchdav/{linalg,sketch,fourdvar,
// linesearch}.hpp with the tall n x l work on the GPU and only the l x l
// projected problems on the host.
#pragma once

#include <map>
#include <optional>

#include "engine.hpp"
#include "hostla.hpp"

namespace sdv {

// LowRankEVD (proj/include/sketchdav/linalg.hpp:103-113) with a device basis.
struct DeviceEVD {
  long long n = 0;
  int l = 0;
  DevBuf<double> basis;         // n x l
  std::vector<double> eig;      // l
  DevBuf<double> coef, scratch; // lambda/(1+lambda), l-vector scratch
  void set_eig(const std::vector<double>& e, cudaStream_t st);
  void upload(long long n_, int l_, const double* basis_host, const double* eig_host, cudaStream_t st);
};

// EVD of G^T G from its tall factor Wt = G^T (n x l, overwritten by its QR
// factor): the RandSVD / Nystrom tail (proj/src/sketch.cpp:27-33, :191-197).
DeviceEVD evd_from_tall(DevBuf<double>& wt, long long n, int l, double shift, bool floor0, cudaStream_t st);
// Stabilised Nystrom assembly from Omega and Y = H Omega (n x l each, device;
// proj/src/sketch.cpp:162-200).
DeviceEVD nystrom_assemble(const double* omega, const double* y, long long n, int l, cudaStream_t st);

// out = (I + V diag(lambda) V^T)^{-1} v (proj/src/linalg.cpp:32-50).
void woodbury_apply(const DeviceEVD& e, const double* v, double* out, long long n, cudaStream_t st);

// CountingMap(MisfitOperator) over a frozen trajectory (proj/src/linalg.cpp:14-30).
class MisfitOp {
 public:
  MisfitOp(const Problem& p, const Trajectory& t) : p_(p), t_(t) {}
  long long n() const { return p_.dim(); }
  long long m() const { return p_.m(); }
  cudaStream_t stream() const { return p_.stream(); }
  void apply(const double* v, int s, double* y) {
    p_.misfit_apply(t_, v, s, y);
    applies += s;
  }
  void adjoint(const double* w, int s, double* z) {
    p_.misfit_adjoint(t_, w, s, z);
    adjoint_applies += s;
  }
  void gram(const double* v, int s, double* hv) {
    p_.gram_apply(t_, v, s, hv);
    applies += s;
    adjoint_applies += s;
  }
  const Problem& problem() const { return p_; }
  long applies = 0, adjoint_applies = 0;

 private:
  const Problem& p_;
  const Trajectory& t_;
};

struct SketchCfg {
  int method = 0, rank = 10, rank2 = -1, growth = 5, max_rank = -1;
  double eps_sketch = 1.5, eps_reuse = 10.0;
  uint64_t seed = 0;
  int resolved_rank2() const { return rank2 > 0 ? rank2 : 2 * rank + 1; }
  void validate(long long m, long long n) const;
};

struct SketchResult {
  DeviceEVD evd;
  long tlm = 0, adj = 0;
  int final_rank = 0;
  std::vector<double> kappa;
  bool tolerance_met = true;
  int probes = 0;
};

// Fixed-size sketches (proj/src/sketch.cpp:142-287, :405-414).
SketchResult sketch(MisfitOp& op, int method, int rank, int rank2, uint64_t seed);
SketchResult randsvd_sketch(MisfitOp& a, int rank, uint64_t seed);
SketchResult nystrom_sketch(MisfitOp& h, int rank, uint64_t seed);
SketchResult singleview_sketch(MisfitOp& a, int rank1, int rank2, uint64_t seed);
SketchResult lanczos_sketch(MisfitOp& h, int rank, const double* start_dev);
double cond_estimate(MisfitOp& h, const DeviceEVD& e, uint64_t seed);
// Adaptive variants (proj/src/sketch.cpp:402-602).
SketchResult adaptive_randsvd(MisfitOp& a, const SketchCfg& cfg, MisfitOp& probe);
SketchResult adaptive_nystrom(MisfitOp& h, const SketchCfg& cfg, MisfitOp& probe);
SketchResult adaptive_singleview(MisfitOp& a, const SketchCfg& cfg, MisfitOp& probe);
SketchResult adaptive_lanczos(MisfitOp& h, const SketchCfg& cfg, const double* start_dev, MisfitOp& probe);

struct PCGResult {
  int iterations = 0;
  bool converged = false;
  std::vector<double> relres;
};
// (I + H) x = b, zero initial guess, optional Woodbury preconditioner.
PCGResult pcg_solve(MisfitOp& h, const double* b, const DeviceEVD* pre, double tol, int max_iter, double* x);

struct GNConfig {
  int mode = 1, method = 0, rank = 10, rank2 = -1, growth = 5, max_rank = -1;
  double eps_sketch = 1.5, eps_reuse = 10.0;
  uint64_t seed = 0;
  double grad_tol = 1e-6, pcg_tol = 1e-9;
  int max_gn_iters = 50, pcg_max_iter = 10000;
};
struct GNIter {
  double rec[16];
};
struct GNResult {
  std::vector<double> analysis;
  std::vector<GNIter> iterations;
  std::vector<double> eig0;
  double final_cost = 0, final_grad_inf_norm = 0;
  long total_pcg = 0;
  bool converged = false, line_search_failed = false;
};
GNResult gn_solve(const Problem& p, const GNConfig& cfg);

}  // namespace sdv

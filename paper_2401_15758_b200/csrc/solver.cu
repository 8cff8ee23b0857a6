// Device-resident sketches, Woodbury preconditioner, PCG and the Gauss-Newton
// driver. Reference: /root/reference/proj/src/{sketch,linalg,fourdvar,
// linesearch}.cpp (file:line at each function). The n x l contractions
// (Householder QR, Gram, tall x small products, row triangular solves) run on
// the device; the l x l SVD / Cholesky / pseudo-inverse on the host.
#include <future>
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <iostream>
#include <tuple>

#include "solver.hpp"

namespace sdv {

namespace {
constexpr uint64_t kPsiStream = 0x707369;               // proj/src/sketch.cpp:18
constexpr uint64_t kGrowStream = 0x67726f77;            // proj/src/sketch.cpp:19
constexpr uint64_t kProbeStream = 0x70726f6265;         // proj/src/sketch.cpp:20
constexpr uint64_t kIterSketchStream = 0x736b6574636800;  // proj/src/fourdvar.cpp:16
constexpr uint64_t kReuseStream = 0x7265757365;           // proj/src/fourdvar.cpp:17

void warn(const std::string& m) { std::cerr << "[sdv] warning: " << m << "\n"; }

__global__ void mul_elem_kernel(int l, const double* __restrict__ c, double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < l) x[i] *= c[i];
}

double host_dot(const double* a, const double* b, long long n, cudaStream_t st) {
  DevBuf<double>& r = stream_work(st).dot;
  r.ensure(1);
  dev_dot(a, b, n, r.get(), st);
  double h = 0;
  SDV_CUDA(cudaMemcpyAsync(&h, r.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  SDV_CUDA(cudaStreamSynchronize(st));
  return h;
}
double host_norm(const double* a, long long n, cudaStream_t st) { return std::sqrt(host_dot(a, a, n, st)); }

DevBuf<double> to_dev(const std::vector<double>& h, cudaStream_t st) {
  DevBuf<double> d;
  d.upload(h.data(), h.size(), st);
  return d;
}
DevBuf<double> to_dev(const HMat& h, cudaStream_t st) { return to_dev(h.a, st); }
HMat small_from_dev(const double* d, int r, int c, cudaStream_t st) {
  HMat h(r, c);
  SDV_CUDA(cudaMemcpyAsync(h.a.data(), d, sizeof(double) * h.a.size(), cudaMemcpyDeviceToHost, st));
  SDV_CUDA(cudaStreamSynchronize(st));
  return h;
}
// C (k x l) = A^T B on the device, returned on the host.
HMat gram_tn(long long n, int k, int l, const double* a, const double* b, cudaStream_t st) {
  DevBuf<double> c(static_cast<size_t>(k) * l);
  dev_gemm_tn(n, k, l, a, b, c.get(), st);
  return small_from_dev(c.get(), k, l, st);
}
// out (n x l) = A (n x k) * B (host k x l)
void tall_times_small(long long n, int k, const double* a, const HMat& b, double* out, cudaStream_t st,
                      double alpha = 1.0, double beta = 0.0) {
  DevBuf<double> db = to_dev(b, st);
  dev_gemm_nn_small(n, k, b.c, alpha, a, db.get(), beta, out, st);
}
void copy_dev(double* dst, const double* src, long long n, cudaStream_t st) {
  SDV_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
}

}  // namespace

// EVD of G^T G from a tall factor Wt (= G^T, n x l): Wt = Q R, R = U S V^T
// => basis = Q U, eigenvalues = S^2 - shift (floored at 0 when shift > 0).
// proj/src/sketch.cpp:27-33 (and the Nystrom tail, :191-197).
DeviceEVD evd_from_tall(DevBuf<double>& wt, long long n, int l, double shift, bool floor0, cudaStream_t st) {
  HMat r(l, l), u, v;
  std::vector<double> s;
  dev_thin_qr(n, l, wt.get(), r.a.data(), st);
  hsvd_square(r, u, s, v);
  DeviceEVD e;
  e.n = n;
  e.l = l;
  e.basis.alloc(static_cast<size_t>(n) * l);
  tall_times_small(n, l, wt.get(), u, e.basis.get(), st);
  std::vector<double> ev(static_cast<size_t>(l));
  for (int i = 0; i < l; ++i) ev[i] = floor0 ? std::max(0.0, s[i] * s[i] - shift) : s[i] * s[i];
  e.set_eig(ev, st);
  return e;
}

namespace {
std::vector<double> col_norms(const double* y, long long n, int l, cudaStream_t st) {
  DevBuf<double> d(static_cast<size_t>(l));
  dev_coldots(y, n, y, n, n, l, d.get(), st);
  std::vector<double> h(static_cast<size_t>(l));
  SDV_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(double) * l, cudaMemcpyDeviceToHost, st));
  SDV_CUDA(cudaStreamSynchronize(st));
  for (auto& x : h) x = std::sqrt(x);
  return h;
}
// Y -= Q (Q^T Y), repeated once under the Kahan-Parlett test (proj/src/sketch.cpp:38-52).
void orthogonalize_block(double* y, int ly, const double* q, int lq, long long n, cudaStream_t st) {
  if (lq == 0 || ly == 0) return;
  const std::vector<double> pre = col_norms(y, n, ly, st);
  auto pass = [&] {
    DevBuf<double> c(static_cast<size_t>(lq) * ly);
    dev_gemm_tn(n, lq, ly, q, y, c.get(), st);
    dev_gemm_nn_small(n, lq, ly, -1.0, q, c.get(), 1.0, y, st);
  };
  pass();
  const std::vector<double> post = col_norms(y, n, ly, st);
  for (int j = 0; j < ly; ++j)
    if (post[j] < 0.70710678118654752 * pre[j]) {
      pass();
      break;
    }
}

// The host RNG (bit-exact mt19937_64 + Box-Muller, proj/src/rng.cpp:9-48) needs
// ~1.2 s for C3's 262144 x 110 test block, during which the GPU would idle.
// gn_solve therefore has the NEXT iteration's block generated on a worker
// thread while the GPU runs the current iteration's PCG; gaussian_dev picks
// it up when (n, l, seed) match and generates inline otherwise.
struct GaussPrefetch {
  long long n = 0, l = 0;
  uint64_t seed = 0;
  std::future<std::vector<double>> fut;
  void start(long long n_, long long l_, uint64_t seed_) {
    n = n_;
    l = l_;
    seed = seed_;
    fut = std::async(std::launch::async, [n_, l_, seed_] { return gaussian_matrix(n_, l_, seed_); });
  }
};
thread_local GaussPrefetch* tl_gauss = nullptr;

DevBuf<double> gaussian_dev(long long n, long long l, uint64_t seed, cudaStream_t st) {
  if (tl_gauss && tl_gauss->fut.valid() && tl_gauss->n == n && tl_gauss->l == l && tl_gauss->seed == seed)
    return to_dev(tl_gauss->fut.get(), st);
  return to_dev(gaussian_matrix(n, l, seed), st);
}
DevBuf<double> append_dev(const DevBuf<double>& a, long long la, const double* b, long long lb, long long n,
                          cudaStream_t st) {
  DevBuf<double> o(static_cast<size_t>(n * (la + lb)));
  if (la) copy_dev(o.get(), a.get(), n * la, st);
  copy_dev(o.get() + n * la, b, n * lb, st);
  return o;
}
}  // namespace

// ------------------------------------------------------------- Woodbury -----
void DeviceEVD::set_eig(const std::vector<double>& e, cudaStream_t st) {
  eig = e;
  std::vector<double> c(e.size());
  for (size_t i = 0; i < e.size(); ++i) c[i] = e[i] / (1.0 + e[i]);
  coef.upload(c.data(), std::max<size_t>(c.size(), 1), st);
  scratch.ensure(std::max<size_t>(c.size(), 1));
}
void DeviceEVD::upload(long long n_, int l_, const double* basis_host, const double* eig_host, cudaStream_t st) {
  n = n_;
  l = l_;
  for (int i = 0; i < l_; ++i)
    if (!std::isfinite(eig_host[i])) throw std::invalid_argument("woodbury_apply: non-finite input");
  if (l_ > 0) basis.upload(basis_host, static_cast<size_t>(n_) * l_, st);
  set_eig(std::vector<double>(eig_host, eig_host + l_), st);
}

// proj/src/linalg.cpp:32-50: v - V diag(l/(1+l)) V^T v.
void woodbury_apply(const DeviceEVD& e, const double* v, double* out, long long n, cudaStream_t st) {
  if (e.l > 0 && e.n != n) throw std::invalid_argument("woodbury_apply: dimension mismatch");
  if (out != v) copy_dev(out, v, n, st);
  if (e.l == 0) return;
  double* c = const_cast<double*>(e.scratch.get());
  dev_gemm_tn(n, e.l, 1, e.basis.get(), v, c, st);
  mul_elem_kernel<<<ceil_div(e.l, 128), 128, 0, st>>>(e.l, e.coef.get(), c);
  count_launch();
  dev_gemm_nn_small(n, e.l, 1, -1.0, e.basis.get(), c, 1.0, out, st);
}

void SketchCfg::validate(long long m, long long n) const {
  const long long cap = max_rank > 0 ? max_rank : std::min(m, n);
  if (rank < 1 || rank > cap) throw std::invalid_argument("SketchConfig: need 1 <= rank <= max_rank");
  if (cap > std::min(m, n)) throw std::invalid_argument("SketchConfig: max_rank exceeds min(m, n)");
  if (method == 2 && resolved_rank2() < rank) throw std::invalid_argument("SketchConfig: need rank2 >= rank");
  if (!(eps_sketch >= 1.0)) throw std::invalid_argument("SketchConfig: need eps_sketch >= 1");
  if (!(eps_reuse > eps_sketch)) throw std::invalid_argument("SketchConfig: need eps_reuse > eps_sketch");
  if (growth < 1) throw std::invalid_argument("SketchConfig: need growth >= 1");
}

// ------------------------------------------------------------- sketches -----
// Algorithm 1, proj/src/sketch.cpp:142-160.
SketchResult randsvd_sketch(MisfitOp& a, int rank, uint64_t seed) {
  const long long m = a.m(), n = a.n();
  if (rank < 1 || rank > std::min(m, n)) throw std::invalid_argument("randsvd_sketch: need 1 <= rank <= min(m, n)");
  cudaStream_t st = a.stream();
  DevBuf<double> omega = gaussian_dev(n, rank, seed, st);
  DevBuf<double> y(static_cast<size_t>(m) * rank), wt(static_cast<size_t>(n) * rank);
  a.apply(omega.get(), rank, y.get());
  std::vector<double> r(static_cast<size_t>(rank) * rank);
  dev_thin_qr(m, rank, y.get(), r.data(), st);
  a.adjoint(y.get(), rank, wt.get());
  SketchResult res;
  res.evd = evd_from_tall(wt, n, rank, 0.0, false, st);
  res.tlm = rank;
  res.adj = rank;
  res.final_rank = rank;
  return res;
}

// Stabilised Nystrom assembly (proj/src/sketch.cpp:162-200).
DeviceEVD nystrom_assemble(const double* omega, const double* y, long long n, int l, cudaStream_t st) {
  DevBuf<double> tmp(static_cast<size_t>(n) * l);
  copy_dev(tmp.get(), y, n * l, st);
  HMat ry(l, l), u, v;
  std::vector<double> s;
  dev_thin_qr(n, l, tmp.get(), ry.a.data(), st);
  hsvd_square(ry, u, s, v);
  const double ynorm = s.empty() ? 0.0 : s[0];
  if (ynorm == 0.0) {
    DeviceEVD e;
    e.n = n;
    e.l = l;
    e.basis.alloc(static_cast<size_t>(n) * l);
    copy_dev(e.basis.get(), omega, n * l, st);
    std::vector<double> r(static_cast<size_t>(l) * l);
    dev_thin_qr(n, l, e.basis.get(), r.data(), st);
    e.set_eig(std::vector<double>(static_cast<size_t>(l), 0.0), st);
    return e;
  }
  double nu = std::sqrt(static_cast<double>(n)) * DBL_EPSILON * ynorm;
  for (int attempt = 0; attempt < 2; ++attempt) {
    DevBuf<double> ys(static_cast<size_t>(n) * l);
    copy_dev(ys.get(), y, n * l, st);
    dev_axpby(n * l, nu, omega, 1.0, ys.get(), st);
    const HMat c = gram_tn(n, l, l, omega, ys.get(), st);
    HMat cs(l, l);
    for (int j = 0; j < l; ++j)
      for (int i = 0; i < l; ++i) cs(i, j) = 0.5 * (c(i, j) + c(j, i));
    HMat lower;
    try {
      lower = hcholesky(cs);
    } catch (const std::runtime_error&) {
      if (attempt == 0) {
        nu *= 10.0;
        continue;
      }
      throw std::runtime_error(
          "nystrom_assemble: Cholesky failed even with a 10x shift; a larger stabilization shift is required");
    }
    // W^T = Ys L^{-T}: row-wise forward substitution (same arithmetic as L^{-1} Ys^T).
    DevBuf<double> dl = to_dev(lower, st);
    DevBuf<double> wt(static_cast<size_t>(n) * l);
    dev_trsm_rows_lower(n, l, dl.get(), ys.get(), wt.get(), st);
    return evd_from_tall(wt, n, l, nu, true, st);
  }
  throw std::logic_error("nystrom_assemble: unreachable");
}

// proj/src/sketch.cpp:202-220 (h = GramMap, one H-apply = 1 TLM + 1 ADJ).
SketchResult nystrom_sketch(MisfitOp& h, int rank, uint64_t seed) {
  const long long n = h.n();
  if (rank < 1 || rank > n) throw std::invalid_argument("nystrom_sketch: need 1 <= rank <= n");
  cudaStream_t st = h.stream();
  DevBuf<double> omega = gaussian_dev(n, rank, seed, st);
  DevBuf<double> y(static_cast<size_t>(n) * rank);
  h.gram(omega.get(), rank, y.get());
  SketchResult res;
  res.evd = nystrom_assemble(omega.get(), y.get(), n, rank, st);
  res.tlm = rank;
  res.adj = rank;
  res.final_rank = rank;
  return res;
}

namespace {
struct SVState {
  DevBuf<double> psi, z, q_y;  // m x l2, n x l2, m x l1
  int l1 = 0, l2 = 0;
  HMat q_m, r_m;  // l2 x l1, l1 x l1
};
// proj/src/sketch.cpp:230-248
DeviceEVD singleview_evd(const SVState& s, long long n, cudaStream_t st) {
  int trunc = 0;
  const HMat rp = hpinv(s.r_m, &trunc);
  if (trunc > 0)
    warn("singleview: rank-deficient R_M, pseudoinverse truncated " + std::to_string(trunc) + " singular value(s)");
  DevBuf<double> zq(static_cast<size_t>(n) * s.l1), wt(static_cast<size_t>(n) * s.l1);
  tall_times_small(n, s.l2, s.z.get(), s.q_m, zq.get(), st);
  tall_times_small(n, s.l1, zq.get(), hmat_t(rp), wt.get(), st);
  return evd_from_tall(wt, n, s.l1, 0.0, false, st);
}
// proj/src/sketch.cpp:250-276
SVState singleview_init(MisfitOp& a, int r1, int r2, uint64_t seed, long* tlm, long* adj) {
  const long long m = a.m(), n = a.n();
  if (r1 < 1 || r1 > std::min(m, n)) throw std::invalid_argument("singleview_sketch: need 1 <= rank1 <= min(m, n)");
  if (r2 < r1) throw std::invalid_argument("singleview_sketch: need rank2 >= rank1");
  cudaStream_t st = a.stream();
  SVState s;
  s.l1 = r1;
  s.l2 = r2;
  DevBuf<double> omega = gaussian_dev(n, r1, seed, st);
  s.psi = gaussian_dev(m, r2, mix_seed(seed, kPsiStream), st);
  s.q_y.alloc(static_cast<size_t>(m) * r1);
  s.z.alloc(static_cast<size_t>(n) * r2);
  a.apply(omega.get(), r1, s.q_y.get());
  a.adjoint(s.psi.get(), r2, s.z.get());
  *tlm += r1;
  *adj += r2;
  std::vector<double> r(static_cast<size_t>(r1) * r1);
  dev_thin_qr(m, r1, s.q_y.get(), r.data(), st);
  const HMat mm = gram_tn(m, r2, r1, s.psi.get(), s.q_y.get(), st);
  hqr(mm, s.q_m, s.r_m);
  return s;
}
}  // namespace

SketchResult singleview_sketch(MisfitOp& a, int rank1, int rank2, uint64_t seed) {
  SketchResult res;
  SVState s = singleview_init(a, rank1, rank2, seed, &res.tlm, &res.adj);
  res.evd = singleview_evd(s, a.n(), a.stream());
  res.final_rank = rank1;
  return res;
}

namespace {
// Lanczos with full reorthogonalisation (proj/src/sketch.cpp:292-389).
struct Lanczos {
  DevBuf<double> v;  // n x cap
  int cap = 0;
  std::vector<double> alpha, beta;
  int k = 0;
  bool exhausted = false;
  double scale = 0.0;
};
Lanczos lanczos_start(MisfitOp& h, const double* start, int cap) {
  cudaStream_t st = h.stream();
  const long long n = h.n();
  const double nn = host_norm(start, n, st);
  if (nn == 0.0) throw std::invalid_argument("lanczos: start vector must be nonzero");
  Lanczos f;
  f.cap = cap + 1;
  f.v.alloc(static_cast<size_t>(n) * f.cap);
  dev_axpby(n, 1.0 / nn, start, 0.0, f.v.get(), st);
  return f;
}
void lanczos_extend(MisfitOp& h, Lanczos& f, int target, long* applies) {
  cudaStream_t st = h.stream();
  const long long n = h.n();
  target = static_cast<int>(std::min<long long>(target, n));
  DevBuf<double> w(static_cast<size_t>(n)), c(static_cast<size_t>(f.cap));
  while (f.k < target && !f.exhausted) {
    const int k = f.k;
    double* vk = f.v.get() + static_cast<long long>(k) * n;
    h.gram(vk, 1, w.get());
    ++*applies;
    const double ak = host_dot(vk, w.get(), n, st);
    f.alpha.push_back(ak);
    dev_axpby(n, -ak, vk, 1.0, w.get(), st);
    if (k > 0) dev_axpby(n, -f.beta[k - 1], vk - n, 1.0, w.get(), st);
    const double pre = host_norm(w.get(), n, st);
    dev_gemm_tn(n, k + 1, 1, f.v.get(), w.get(), c.get(), st);
    dev_gemm_nn_small(n, k + 1, 1, -1.0, f.v.get(), c.get(), 1.0, w.get(), st);
    if (host_norm(w.get(), n, st) < 0.70710678118654752 * pre) {
      dev_gemm_tn(n, k + 1, 1, f.v.get(), w.get(), c.get(), st);
      dev_gemm_nn_small(n, k + 1, 1, -1.0, f.v.get(), c.get(), 1.0, w.get(), st);
    }
    f.scale = std::max(f.scale, std::abs(ak));
    const double bk = host_norm(w.get(), n, st);
    f.k = k + 1;
    if (bk <= 1e3 * DBL_EPSILON * std::max(f.scale, 1.0)) {
      f.exhausted = true;
      break;
    }
    f.beta.push_back(bk);
    f.scale = std::max(f.scale, bk);
    if (f.k >= f.cap) throw std::logic_error("lanczos: capacity exceeded");
    dev_axpby(n, 1.0 / bk, w.get(), 0.0, f.v.get() + static_cast<long long>(k + 1) * n, st);
  }
}
DeviceEVD lanczos_ritz(const Lanczos& f, long long n, cudaStream_t st) {
  const int k = f.k;
  HMat t(k, k), vec;
  for (int i = 0; i < k; ++i) {
    t(i, i) = f.alpha[i];
    if (i + 1 < k) t(i, i + 1) = t(i + 1, i) = f.beta[i];
  }
  std::vector<double> w;
  hsym_eig(t, w, vec);
  HMat rev(k, k);
  std::vector<double> ev(static_cast<size_t>(k));
  for (int i = 0; i < k; ++i) {
    ev[i] = std::max(0.0, w[k - 1 - i]);
    for (int r = 0; r < k; ++r) rev(r, i) = vec(r, k - 1 - i);
  }
  DeviceEVD e;
  e.n = n;
  e.l = k;
  e.basis.alloc(static_cast<size_t>(n) * std::max(k, 1));
  if (k > 0) tall_times_small(n, k, f.v.get(), rev, e.basis.get(), st);
  e.set_eig(ev, st);
  return e;
}
}  // namespace

SketchResult lanczos_sketch(MisfitOp& h, int rank, const double* start) {
  Lanczos f = lanczos_start(h, start, rank);
  SketchResult res;
  lanczos_extend(h, f, rank, &res.tlm);
  res.adj = res.tlm;
  res.evd = lanczos_ritz(f, h.n(), h.stream());
  res.final_rank = f.k;
  return res;
}

SketchResult sketch(MisfitOp& op, int method, int rank, int rank2, uint64_t seed) {
  switch (method) {
    case 0: return randsvd_sketch(op, rank, seed);
    case 1: return nystrom_sketch(op, rank, seed);
    case 2: return singleview_sketch(op, rank, rank2 > 0 ? rank2 : 2 * rank + 1, seed);
    case 3: {
      DevBuf<double> st = gaussian_dev(op.n(), 1, seed, op.stream());
      return lanczos_sketch(op, rank, st.get());
    }
  }
  throw std::invalid_argument("unknown sketch method");
}

// proj/src/sketch.cpp:391-400
double cond_estimate(MisfitOp& h, const DeviceEVD& e, uint64_t seed) {
  const long long n = h.n();
  if (e.n != n) throw std::invalid_argument("cond_estimate: dimension mismatch");
  cudaStream_t st = h.stream();
  std::vector<double> v = gaussian_matrix(n, 1, seed);
  double ss = 0.0;
  for (double x : v) ss += x * x;
  const double nv = std::sqrt(ss);
  for (auto& x : v) x /= nv;
  DevBuf<double> dv = to_dev(v, st), u(static_cast<size_t>(n)), hu(static_cast<size_t>(n));
  woodbury_apply(e, dv.get(), u.get(), n, st);
  h.gram(u.get(), 1, hu.get());
  dev_axpby(n, 1.0, u.get(), 1.0, hu.get(), st);
  return host_norm(hu.get(), n, st);
}

// proj/src/sketch.cpp:402-446
SketchResult adaptive_randsvd(MisfitOp& a, const SketchCfg& cfg, MisfitOp& probe) {
  const long long m = a.m(), n = a.n();
  cfg.validate(m, n);
  const int cap = cfg.max_rank > 0 ? cfg.max_rank : static_cast<int>(std::min(m, n));
  cudaStream_t st = a.stream();
  SketchResult res;
  int l = std::min(cfg.rank, cap);
  DevBuf<double> omega = gaussian_dev(n, l, cfg.seed, st);
  DevBuf<double> q(static_cast<size_t>(m) * l), wt(static_cast<size_t>(n) * l);
  a.apply(omega.get(), l, q.get());
  std::vector<double> r(static_cast<size_t>(l) * l);
  dev_thin_qr(m, l, q.get(), r.data(), st);
  a.adjoint(q.get(), l, wt.get());
  res.tlm += l;
  res.adj += l;
  for (int pass = 0;; ++pass) {
    DevBuf<double> wcopy(static_cast<size_t>(n) * l);
    copy_dev(wcopy.get(), wt.get(), n * l, st);
    res.evd = evd_from_tall(wcopy, n, l, 0.0, false, st);
    const double kappa = cond_estimate(probe, res.evd, mix_seed(cfg.seed, kProbeStream + pass));
    ++res.probes;
    res.kappa.push_back(kappa);
    if (kappa <= cfg.eps_sketch) {
      res.tolerance_met = true;
      break;
    }
    if (l >= cap) {
      res.tolerance_met = false;
      warn("adaptive_randsvd: max_rank " + std::to_string(cap) + " reached");
      break;
    }
    const int lh = std::min(cfg.growth, cap - l);
    DevBuf<double> g = gaussian_dev(n, lh, mix_seed(cfg.seed, kGrowStream + pass), st);
    DevBuf<double> ynew(static_cast<size_t>(m) * lh), wnew(static_cast<size_t>(n) * lh);
    a.apply(g.get(), lh, ynew.get());
    orthogonalize_block(ynew.get(), lh, q.get(), l, m, st);
    std::vector<double> rr(static_cast<size_t>(lh) * lh);
    dev_thin_qr(m, lh, ynew.get(), rr.data(), st);
    a.adjoint(ynew.get(), lh, wnew.get());
    res.tlm += lh;
    res.adj += lh;
    q = append_dev(q, l, ynew.get(), lh, m, st);
    wt = append_dev(wt, l, wnew.get(), lh, n, st);
    l += lh;
  }
  res.final_rank = l;
  return res;
}

// proj/src/sketch.cpp:448-489
SketchResult adaptive_nystrom(MisfitOp& h, const SketchCfg& cfg, MisfitOp& probe) {
  const long long n = h.n();
  cfg.validate(n, n);
  const int cap = cfg.max_rank > 0 ? cfg.max_rank : static_cast<int>(n);
  cudaStream_t st = h.stream();
  SketchResult res;
  int l = std::min(cfg.rank, cap);
  DevBuf<double> omega = gaussian_dev(n, l, cfg.seed, st);
  DevBuf<double> y(static_cast<size_t>(n) * l);
  h.gram(omega.get(), l, y.get());
  res.tlm += l;
  res.adj += l;
  for (int pass = 0;; ++pass) {
    res.evd = nystrom_assemble(omega.get(), y.get(), n, l, st);
    const double kappa = cond_estimate(probe, res.evd, mix_seed(cfg.seed, kProbeStream + pass));
    ++res.probes;
    res.kappa.push_back(kappa);
    if (kappa <= cfg.eps_sketch) {
      res.tolerance_met = true;
      break;
    }
    if (l >= cap) {
      res.tolerance_met = false;
      warn("adaptive_nystrom: max_rank " + std::to_string(cap) + " reached");
      break;
    }
    const int lh = std::min(cfg.growth, cap - l);
    DevBuf<double> on = gaussian_dev(n, lh, mix_seed(cfg.seed, kGrowStream + pass), st);
    DevBuf<double> yn(static_cast<size_t>(n) * lh);
    h.gram(on.get(), lh, yn.get());
    res.tlm += lh;
    res.adj += lh;
    omega = append_dev(omega, l, on.get(), lh, n, st);
    y = append_dev(y, l, yn.get(), lh, n, st);
    l += lh;
  }
  res.final_rank = l;
  return res;
}

// proj/src/sketch.cpp:491-564
SketchResult adaptive_singleview(MisfitOp& a, const SketchCfg& cfg, MisfitOp& probe) {
  const long long m = a.m(), n = a.n();
  cfg.validate(m, n);
  const int l2 = cfg.resolved_rank2();
  const int cap = std::min(cfg.max_rank > 0 ? cfg.max_rank : static_cast<int>(std::min(m, n)), l2);
  cudaStream_t st = a.stream();
  SketchResult res;
  int l1 = std::min(cfg.rank, cap);
  SVState s = singleview_init(a, l1, l2, cfg.seed, &res.tlm, &res.adj);
  for (int pass = 0;; ++pass) {
    res.evd = singleview_evd(s, n, st);
    const double kappa = cond_estimate(probe, res.evd, mix_seed(cfg.seed, kProbeStream + pass));
    ++res.probes;
    res.kappa.push_back(kappa);
    if (kappa <= cfg.eps_sketch) {
      res.tolerance_met = true;
      break;
    }
    if (l1 >= cap) {
      res.tolerance_met = false;
      warn("adaptive_singleview: range rank limit " + std::to_string(cap) + " reached");
      break;
    }
    const int lh = std::min(cfg.growth, cap - l1);
    DevBuf<double> g = gaussian_dev(n, lh, mix_seed(cfg.seed, kGrowStream + pass), st);
    DevBuf<double> ynew(static_cast<size_t>(m) * lh);
    a.apply(g.get(), lh, ynew.get());
    res.tlm += lh;
    orthogonalize_block(ynew.get(), lh, s.q_y.get(), l1, m, st);
    std::vector<double> rr(static_cast<size_t>(lh) * lh);
    dev_thin_qr(m, lh, ynew.get(), rr.data(), st);
    // Column-append QR update of M = Psi^T [Q_Y Q_Y_new].
    const HMat pm = gram_tn(m, l2, lh, s.psi.get(), ynew.get(), st);
    HMat c = hmat_mul(hmat_t(s.q_m), pm);
    HMat pperp = pm;
    {
      const HMat qc = hmat_mul(s.q_m, c);
      for (size_t i = 0; i < pperp.a.size(); ++i) pperp.a[i] -= qc.a[i];
      const HMat c2 = hmat_mul(hmat_t(s.q_m), pperp);
      const HMat qc2 = hmat_mul(s.q_m, c2);
      for (size_t i = 0; i < pperp.a.size(); ++i) pperp.a[i] -= qc2.a[i];
      for (size_t i = 0; i < c.a.size(); ++i) c.a[i] += c2.a[i];
    }
    HMat pq, pr;
    hqr(pperp, pq, pr);
    s.q_y = append_dev(s.q_y, l1, ynew.get(), lh, m, st);
    HMat qm2(l2, l1 + lh);
    std::copy(s.q_m.a.begin(), s.q_m.a.end(), qm2.a.begin());
    std::copy(pq.a.begin(), pq.a.end(), qm2.a.begin() + s.q_m.a.size());
    s.q_m = qm2;
    HMat rn(l1 + lh, l1 + lh);
    for (int j = 0; j < l1; ++j)
      for (int i = 0; i < l1; ++i) rn(i, j) = s.r_m(i, j);
    for (int j = 0; j < lh; ++j)
      for (int i = 0; i < l1; ++i) rn(i, l1 + j) = c(i, j);
    for (int j = 0; j < lh; ++j)
      for (int i = 0; i < lh; ++i) rn(l1 + i, l1 + j) = pr(i, j);
    s.r_m = rn;
    l1 += lh;
    s.l1 = l1;
  }
  res.final_rank = l1;
  return res;
}

// proj/src/sketch.cpp:566-602
SketchResult adaptive_lanczos(MisfitOp& h, const SketchCfg& cfg, const double* start, MisfitOp& probe) {
  const long long n = h.n();
  cfg.validate(n, n);
  const int cap = cfg.max_rank > 0 ? cfg.max_rank : static_cast<int>(n);
  SketchResult res;
  Lanczos f = lanczos_start(h, start, cap);
  lanczos_extend(h, f, std::min(cfg.rank, cap), &res.tlm);
  for (int pass = 0;; ++pass) {
    res.evd = lanczos_ritz(f, n, h.stream());
    const double kappa = cond_estimate(probe, res.evd, mix_seed(cfg.seed, kProbeStream + pass));
    ++res.probes;
    res.kappa.push_back(kappa);
    if (kappa <= cfg.eps_sketch) {
      res.tolerance_met = true;
      break;
    }
    if (f.k >= cap || f.exhausted) {
      res.tolerance_met = false;
      warn("adaptive_lanczos: rank limit reached");
      break;
    }
    lanczos_extend(h, f, std::min(f.k + cfg.growth, cap), &res.tlm);
  }
  res.adj = res.tlm;
  res.final_rank = f.k;
  return res;
}

// ------------------------------------------------------------------ PCG -----
// proj/src/linalg.cpp:52-106 on (I + H).
PCGResult pcg_solve(MisfitOp& h, const double* b, const DeviceEVD* pre, double tol, int max_iter, double* x) {
  // proj/src/linalg.cpp:52-106. One host read per iteration: the fused
  // kernels leave <p, q>, <r, r> and <r, z> in a device scalar block and the
  // host applies the reference's checks in the reference's order.
  if (!(tol > 0.0)) throw std::invalid_argument("pcg_solve: tolerance must be positive");
  const long long n = h.n();
  cudaStream_t st = h.stream();
  PCGResult res;
  dev_fill(n, 0.0, x, st);
  const double rhs_norm = host_norm(b, n, st);
  if (rhs_norm == 0.0) {
    res.converged = true;
    return res;
  }
  DevBuf<double> r(static_cast<size_t>(n)), z(static_cast<size_t>(n)), p(static_cast<size_t>(n)),
      q(static_cast<size_t>(n)), sc(3);
  copy_dev(r.get(), b, n, st);
  // unpreconditioned: z = r (no copy; <r, z> = <r, r>)
  const double* zp = pre ? z.get() : r.get();
  if (pre) woodbury_apply(*pre, r.get(), z.get(), n, st);
  double rz = host_dot(r.get(), zp, n, st);
  if (rz <= 0.0) throw std::runtime_error("pcg_solve: preconditioner is not positive definite (<r, M^-1 r> <= 0)");
  copy_dev(p.get(), zp, n, st);
  double hs[3];
  for (int k = 1; k <= max_iter; ++k) {
    h.gram(p.get(), 1, q.get());
    dev_pcg_q(n, p.get(), q.get(), sc.get(), st);                                   // q = p + Hp, <p, q>
    dev_pcg_xr(n, rz, sc.get(), p.get(), q.get(), x, r.get(), sc.get() + 1, st);  // x, r updates, <r, r>
    if (pre) {
      woodbury_apply(*pre, r.get(), z.get(), n, st);
      dev_dot(r.get(), z.get(), n, sc.get() + 2, st);
    }
    SDV_CUDA(cudaMemcpyAsync(hs, sc.get(), sizeof(double) * (pre ? 3 : 2), cudaMemcpyDeviceToHost, st));
    SDV_CUDA(cudaStreamSynchronize(st));
    const double pq = hs[0];
    if (pq <= 0.0) throw std::runtime_error("pcg_solve: operator is not positive definite (<p, A p> <= 0)");
    const double relres = std::sqrt(hs[1]) / rhs_norm;
    res.relres.push_back(relres);
    res.iterations = k;
    if (relres <= tol) {
      res.converged = true;
      return res;
    }
    const double rzn = pre ? hs[2] : hs[1];
    if (rzn <= 0.0) throw std::runtime_error("pcg_solve: preconditioner is not positive definite (<r, M^-1 r> <= 0)");
    dev_axpby(n, 1.0, zp, rzn / rz, p.get(), st);
    rz = rzn;
  }
  return res;
}

// ---------------------------------------------------------- line search -----
namespace {
struct LSConfig {
  double ftol = 1e-4, gtol = 0.9, xtol = 1e-12, stpmin = 1e-20, stpmax = 1e20;
  int max_trials = 20;
};
struct LSResult {
  double step = 1.0, f = 0, g = 0;
  int trials = 0;
  bool ok = false;
};
struct Pt {
  double t, f, g;
};
// Safeguarded step of More & Thuente (MINPACK-2 dcstep), as used by
// proj/src/linesearch.cpp:13-117.
double mt_step(Pt& lo, Pt& hi, double t, double f, double g, bool& br, double tmin, double tmax) {
  const double sgnd = g * (lo.g / std::abs(lo.g));
  auto gamma_of = [](double theta, double d1, double d2) {
    const double s = std::max({std::abs(theta), std::abs(d1), std::abs(d2)});
    return s * std::sqrt((theta / s) * (theta / s) - (d1 / s) * (d2 / s));
  };
  double nt;
  if (f > lo.f) {
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    double gam = gamma_of(theta, lo.g, g);
    if (t < lo.t) gam = -gam;
    const double r = ((gam - lo.g) + theta) / (((gam - lo.g) + gam) + g);
    const double tc = lo.t + r * (t - lo.t);
    const double tq = lo.t + ((lo.g / ((lo.f - f) / (t - lo.t) + lo.g)) / 2.0) * (t - lo.t);
    nt = std::abs(tc - lo.t) < std::abs(tq - lo.t) ? tc : tc + (tq - tc) / 2.0;
    br = true;
  } else if (sgnd < 0.0) {
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    double gam = gamma_of(theta, lo.g, g);
    if (t > lo.t) gam = -gam;
    const double r = ((gam - g) + theta) / (((gam - g) + gam) + lo.g);
    const double tc = t + r * (lo.t - t);
    const double tq = t + (g / (g - lo.g)) * (lo.t - t);
    nt = std::abs(tc - t) > std::abs(tq - t) ? tc : tq;
    br = true;
  } else if (std::abs(g) < std::abs(lo.g)) {
    const double theta = 3.0 * (lo.f - f) / (t - lo.t) + lo.g + g;
    const double s = std::max({std::abs(theta), std::abs(lo.g), std::abs(g)});
    double gam = s * std::sqrt(std::max(0.0, (theta / s) * (theta / s) - (lo.g / s) * (g / s)));
    if (t > lo.t) gam = -gam;
    const double r = ((gam - g) + theta) / ((gam + (lo.g - g)) + gam);
    const double tc = (r < 0.0 && gam != 0.0) ? t + r * (lo.t - t) : (t > lo.t ? tmax : tmin);
    const double tq = t + (g / (g - lo.g)) * (lo.t - t);
    if (br) {
      nt = std::abs(tc - t) < std::abs(tq - t) ? tc : tq;
      nt = t > lo.t ? std::min(t + 0.66 * (hi.t - t), nt) : std::max(t + 0.66 * (hi.t - t), nt);
    } else {
      nt = std::abs(tc - t) > std::abs(tq - t) ? tc : tq;
      nt = std::clamp(nt, tmin, tmax);
    }
  } else {
    if (br) {
      const double theta = 3.0 * (f - hi.f) / (hi.t - t) + hi.g + g;
      double gam = gamma_of(theta, hi.g, g);
      if (t > hi.t) gam = -gam;
      const double r = ((gam - g) + theta) / (((gam - g) + gam) + hi.g);
      nt = t + r * (hi.t - t);
    } else {
      nt = t > lo.t ? tmax : tmin;
    }
  }
  if (f > lo.f) {
    hi = {t, f, g};
  } else {
    if (sgnd < 0.0) hi = lo;
    lo = {t, f, g};
  }
  return std::clamp(nt, tmin, tmax);
}
// proj/src/linesearch.cpp:121-214
template <class Phi>
LSResult more_thuente(Phi&& phi, double f0, double g0, double t0, const LSConfig& c) {
  if (!(g0 < 0.0)) throw std::invalid_argument("more_thuente_search: direction is not a descent direction");
  LSResult res;
  const double gtest = c.ftol * g0;
  bool br = false, stage1 = true;
  double width = c.stpmax - c.stpmin, width1 = 2.0 * width;
  Pt lo{0.0, f0, g0}, hi{0.0, f0, g0};
  double t = std::clamp(t0, c.stpmin, c.stpmax);
  double tmin = 0.0, tmax = t + 4.0 * t;
  while (res.trials < c.max_trials) {
    double f, g;
    std::tie(f, g) = phi(t);
    ++res.trials;
    const double ftest = f0 + t * gtest;
    if (stage1 && f <= ftest && g >= 0.0) stage1 = false;
    if (f <= ftest && std::abs(g) <= c.gtol * (-g0)) {
      res.ok = true;
      res.step = t;
      res.f = f;
      res.g = g;
      return res;
    }
    if ((br && (t <= tmin || t >= tmax)) || (br && tmax - tmin <= c.xtol * tmax) ||
        (t == c.stpmax && f <= ftest && g <= gtest) || (t == c.stpmin && (f > ftest || g >= gtest)))
      break;
    if (stage1 && f <= lo.f && f > ftest) {
      Pt lm{lo.t, lo.f - lo.t * gtest, lo.g - gtest}, hm{hi.t, hi.f - hi.t * gtest, hi.g - gtest};
      t = mt_step(lm, hm, t, f - t * gtest, g - gtest, br, tmin, tmax);
      lo = {lm.t, lm.f + lm.t * gtest, lm.g + gtest};
      hi = {hm.t, hm.f + hm.t * gtest, hm.g + gtest};
    } else {
      t = mt_step(lo, hi, t, f, g, br, tmin, tmax);
    }
    if (br) {
      if (std::abs(hi.t - lo.t) >= 0.66 * width1) t = lo.t + 0.5 * (hi.t - lo.t);
      width1 = width;
      width = std::abs(hi.t - lo.t);
      tmin = std::min(lo.t, hi.t);
      tmax = std::max(lo.t, hi.t);
    } else {
      tmin = t + 1.1 * (t - lo.t);
      tmax = t + 4.0 * (t - lo.t);
    }
    t = std::clamp(t, c.stpmin, c.stpmax);
    if ((br && (t <= tmin || t >= tmax)) || (br && tmax - tmin <= c.xtol * tmax)) t = lo.t;
  }
  res.ok = false;
  res.step = lo.t;
  res.f = lo.f;
  res.g = lo.g;
  return res;
}

struct Eval {
  double cost = 0;
  DevBuf<double> g;   // control-space gradient Gamma^{1/2} g
  DevBuf<double> gx;  // x-space gradient (Laplacian prior only)
  std::unique_ptr<Trajectory> traj;
  // the gradient the reference measures convergence on (fourdvar.cpp:131)
  const double* conv() const { return gx.size() ? gx.get() : g.get(); }
};
Eval evaluate_at(const Problem& p, const double* x, const double* z) {
  Eval e;
  // proj/src/fourdvar.cpp:182: linearize(x0, total_steps, steps_per_interval)
  e.traj = p.linearize(x, p.desc().spi, kStoreAuto);
  e.g.alloc(static_cast<size_t>(p.dim()));
  if (p.xspace()) e.gx.alloc(static_cast<size_t>(p.dim()));
  e.cost = p.evaluate(*e.traj, z, e.g.get(), nullptr, p.xspace() ? e.gx.get() : nullptr);
  return e;
}
double inf_norm(const double* d, long long n, cudaStream_t st) {
  std::vector<double> h(static_cast<size_t>(n));
  SDV_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  SDV_CUDA(cudaStreamSynchronize(st));
  double m = 0;
  for (double v : h) m = std::max(m, std::abs(v));
  return m;
}
}  // namespace

// ------------------------------------------------------------ Gauss-Newton --
// proj/src/fourdvar.cpp:213-422, control-variable background term.
GNResult gn_solve(const Problem& p, const GNConfig& cfg) {
  if (!(cfg.grad_tol > 0 && cfg.grad_tol < 1) || !(cfg.pcg_tol > 0 && cfg.pcg_tol < 1))
    throw std::invalid_argument("GNConfig: tolerances must lie in (0, 1)");
  if (cfg.max_gn_iters < 1) throw std::invalid_argument("GNConfig: max_gn_iters must be >= 1");
  const long long n = p.dim();
  cudaStream_t st = p.stream();
  const int mode = cfg.mode;
  GNResult result;
  long c_fwd = 0, c_tlm = 0, c_adj = 0, c_otlm = 0, c_oadj = 0;
  DevBuf<double> x(static_cast<size_t>(n)), z(static_cast<size_t>(n));
  copy_dev(x.get(), p.d_background(), n, st);
  dev_fill(n, 0.0, z.get(), st);
  Eval ev = evaluate_at(p, x.get(), z.get());
  ++c_fwd;
  ++c_adj;
  const bool xspace = p.xspace();
  const double g0 = inf_norm(ev.conv(), n, st);
  if (g0 == 0.0) {
    result.analysis.resize(static_cast<size_t>(n));
    x.download(result.analysis.data(), static_cast<size_t>(n), st);
    SDV_CUDA(cudaStreamSynchronize(st));
    result.converged = true;
    result.final_cost = ev.cost;
    return result;
  }
  std::optional<DeviceEVD> held;
  int held_rank = 0;
  const bool adaptive = mode == 2 || mode == 5;
  const bool lanczos = mode == 4 || mode == 5 || cfg.method == 3;
  SketchCfg sc0;
  sc0.method = cfg.method;
  sc0.rank = cfg.rank;
  sc0.rank2 = cfg.rank2;
  sc0.growth = cfg.growth;
  sc0.max_rank = cfg.max_rank;
  sc0.eps_sketch = cfg.eps_sketch;
  sc0.eps_reuse = cfg.eps_reuse;
  DevBuf<double> rhs(static_cast<size_t>(n)), dxt(static_cast<size_t>(n)), dx(static_cast<size_t>(n)),
      tx(static_cast<size_t>(n)), tz(static_cast<size_t>(n));
  GaussPrefetch gauss;
  struct GaussScope {
    explicit GaussScope(GaussPrefetch* g) { tl_gauss = g; }
    ~GaussScope() { tl_gauss = nullptr; }
  } gauss_scope(&gauss);
  for (int k = 0; k < cfg.max_gn_iters; ++k) {
    const double gnorm = inf_norm(ev.conv(), n, st);
    if (gnorm / g0 < cfg.grad_tol) {
      result.converged = true;
      break;
    }
    GNIter log{};
    std::fill(std::begin(log.rec), std::end(log.rec), 0.0);
    log.rec[0] = k;
    log.rec[1] = ev.cost;
    log.rec[2] = gnorm;
    log.rec[6] = 1;
    log.rec[9] = NAN;
    log.rec[10] = NAN;
    MisfitOp a_off(p, *ev.traj), a_on(p, *ev.traj);
    dev_axpby(n, -1.0, ev.g.get(), 0.0, rhs.get(), st);
    bool build = mode != 3;
    if (adaptive && held) {
      const double kre = cond_estimate(a_on, *held, mix_seed(cfg.seed, kReuseStream + k));
      log.rec[10] = kre;
      if (kre < cfg.eps_reuse) {
        build = false;
        log.rec[8] = held_rank;
      }
    }
    if (build && mode != 3) {
      SketchCfg sc = sc0;
      sc.seed = mix_seed(cfg.seed, kIterSketchStream + k);
      SketchResult rep;
      if (mode == 4 || (!adaptive && lanczos)) rep = lanczos_sketch(a_on, sc.rank, rhs.get());
      else if (mode == 5) rep = adaptive_lanczos(a_on, sc, rhs.get(), a_on);
      else if (adaptive) {
        switch (sc.method) {
          case 0: rep = adaptive_randsvd(a_off, sc, a_on); break;
          case 1: rep = adaptive_nystrom(a_off, sc, a_on); break;
          case 2: rep = adaptive_singleview(a_off, sc, a_on); break;
          default: rep = adaptive_lanczos(a_on, sc, rhs.get(), a_on); break;
        }
      } else {
        switch (sc.method) {
          case 0: rep = randsvd_sketch(a_off, sc.rank, sc.seed); break;
          case 1: rep = nystrom_sketch(a_off, sc.rank, sc.seed); break;
          case 2: rep = singleview_sketch(a_off, sc.rank, sc.resolved_rank2(), sc.seed); break;
          default: rep = lanczos_sketch(a_on, sc.rank, rhs.get()); break;
        }
      }
      if (result.eig0.empty()) result.eig0 = rep.evd.eig;
      held = std::move(rep.evd);
      held_rank = rep.final_rank;
      log.rec[7] = 1;
      log.rec[8] = rep.final_rank;
      if (!rep.kappa.empty()) log.rec[9] = rep.kappa.back();
      if (!rep.tolerance_met) warn("gn_solve: adaptive sketch hit its rank cap at GN iteration " + std::to_string(k));
    }
    // next iteration's Gaussian test block (the non-adaptive sketches draw
    // n x rank with seed mix_seed(seed, kIterSketchStream + k + 1)), generated
    // while the GPU solves this iteration's system; only when it is large
    if (mode != 3 && mode != 4 && mode != 5 && !adaptive && !lanczos && sc0.method >= 0 && sc0.method <= 2 &&
        k + 1 < cfg.max_gn_iters && static_cast<double>(n) * sc0.rank >= 4e6 && !std::getenv("SDV_NO_GAUSS_PREFETCH"))
      gauss.start(n, sc0.rank, mix_seed(cfg.seed, kIterSketchStream + k + 1));
    if (mode == 0) {
      woodbury_apply(*held, ev.g.get(), dxt.get(), n, st);
      dev_axpby(n, -1.0, dxt.get(), 0.0, dxt.get(), st);
    } else {
      const DeviceEVD* pre = mode == 3 ? nullptr : &*held;
      const PCGResult pcg = pcg_solve(a_on, rhs.get(), pre, cfg.pcg_tol, cfg.pcg_max_iter, dxt.get());
      if (!pcg.converged)
        warn("gn_solve: PCG did not reach tolerance at GN iteration " + std::to_string(k) +
             "; continuing with the best iterate");
      log.rec[4] = pcg.iterations;
      if (std::getenv("SDV_DEBUG_PCG")) {
        std::cerr << "[sdv pcg k=" << k << "]";
        for (size_t q = pcg.relres.size() > 6 ? pcg.relres.size() - 6 : 0; q < pcg.relres.size(); ++q)
          std::cerr << " " << pcg.relres[q];
        std::cerr << "\n";
      }
      log.rec[6] = pcg.converged;
      result.total_pcg += pcg.iterations;
    }
    p.prior_sqrt(dxt.get(), dx.get(), 1);
    c_otlm += a_off.applies;
    c_oadj += a_off.adjoint_applies;
    c_tlm += a_on.applies;
    c_adj += a_on.adjoint_applies;

    // directional derivative: x-space g . dx, or control-space g~ . dxt
    auto slope = [&](const Eval& e) {
      return xspace ? host_dot(e.gx.get(), dx.get(), n, st) : host_dot(e.g.get(), dxt.get(), n, st);
    };
    const double dphi0 = slope(ev);
    std::map<double, Eval> trials;
    auto eval_step = [&](double a) {
      copy_dev(tx.get(), x.get(), n, st);
      dev_axpby(n, a, dx.get(), 1.0, tx.get(), st);
      copy_dev(tz.get(), z.get(), n, st);
      dev_axpby(n, a, dxt.get(), 1.0, tz.get(), st);
      Eval e = evaluate_at(p, tx.get(), tz.get());
      ++c_fwd;
      ++c_adj;
      return e;
    };
    bool accepted = false;
    if (dphi0 < 0.0) {
      auto phi = [&](double a) {
        auto it = trials.find(a);
        if (it == trials.end()) it = trials.emplace(a, eval_step(a)).first;
        return std::make_pair(it->second.cost, slope(it->second));
      };
      const LSResult ls = more_thuente(phi, ev.cost, dphi0, 1.0, LSConfig{});
      log.rec[5] = ls.trials;
      if (ls.ok && ls.step > 0.0) {
        dev_axpby(n, ls.step, dx.get(), 1.0, x.get(), st);
        dev_axpby(n, ls.step, dxt.get(), 1.0, z.get(), st);
        ev = std::move(trials.at(ls.step));
        log.rec[3] = ls.step;
        accepted = true;
      }
    } else {
      warn("gn_solve: step is not a descent direction at GN iteration " + std::to_string(k));
    }
    if (!accepted) {
      auto it = trials.find(1.0);
      if (it == trials.end()) {
        it = trials.emplace(1.0, eval_step(1.0)).first;
        log.rec[5] += 1;
      }
      if (it->second.cost < ev.cost) {
        warn("gn_solve: line search failed at GN iteration " + std::to_string(k) + "; accepting the unit step");
        dev_axpby(n, 1.0, dx.get(), 1.0, x.get(), st);
        dev_axpby(n, 1.0, dxt.get(), 1.0, z.get(), st);
        ev = std::move(it->second);
        log.rec[3] = 1.0;
      } else {
        warn("gn_solve: line search failed and the unit step increases the cost; terminating at GN iteration " +
             std::to_string(k));
        result.line_search_failed = true;
        log.rec[11] = c_fwd;
        log.rec[12] = c_tlm;
        log.rec[13] = c_adj;
        log.rec[14] = c_otlm;
        log.rec[15] = c_oadj;
        result.iterations.push_back(log);
        break;
      }
    }
    log.rec[11] = c_fwd;
    log.rec[12] = c_tlm;
    log.rec[13] = c_adj;
    log.rec[14] = c_otlm;
    log.rec[15] = c_oadj;
    result.iterations.push_back(log);
  }
  const double gf = inf_norm(ev.conv(), n, st);
  if (!result.line_search_failed && !result.converged) result.converged = gf / g0 < cfg.grad_tol;
  result.analysis.resize(static_cast<size_t>(n));
  x.download(result.analysis.data(), static_cast<size_t>(n), st);
  SDV_CUDA(cudaStreamSynchronize(st));
  result.final_cost = ev.cost;
  result.final_grad_inf_norm = gf;
  return result;
}

}  // namespace sdv

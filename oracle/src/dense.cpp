// CPU ORACLE (test infrastructure only): vectors, rng, dense linear algebra,
// FFT, Woodbury and PCG. Restates /root/reference/proj/src/rng.cpp and
// /root/reference/proj/src/linalg.cpp without Eigen.
#include "oracle.hpp"

#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>

#include <algorithm>
#include <limits>
#include <numeric>
#include <map>
#include <mutex>
#include <random>

namespace oracle {

// ---------------------------------------------------------------- helpers ---
double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }
double norm_inf(const Vec& a) {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::abs(v));
  return m;
}
Vec axpby(double a, const Vec& x, double b, const Vec& y) {
  Vec o(x.size());
  for (size_t i = 0; i < x.size(); ++i) o[i] = a * x[i] + b * y[i];
  return o;
}
Vec scaled(double a, const Vec& x) {
  Vec o(x.size());
  for (size_t i = 0; i < x.size(); ++i) o[i] = a * x[i];
  return o;
}
bool all_finite(const Vec& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

Mat Mat::identity(int64_t n, int64_t m) {
  Mat o(n, m);
  for (int64_t i = 0; i < std::min(n, m); ++i) o(i, i) = 1.0;
  return o;
}
Mat matmul(const Mat& a, const Mat& b) {
  if (a.c != b.r) throw std::invalid_argument("matmul: shape");
  Mat o(a.r, b.c);
  for (int64_t j = 0; j < b.c; ++j)
    for (int64_t k = 0; k < a.c; ++k) {
      const double bkj = b(k, j);
      if (bkj == 0.0) continue;
      const double* ac = a.col(k);
      double* oc = o.col(j);
      for (int64_t i = 0; i < a.r; ++i) oc[i] += ac[i] * bkj;
    }
  return o;
}
Mat matmul_tn(const Mat& a, const Mat& b) {
  if (a.r != b.r) throw std::invalid_argument("matmul_tn: shape");
  Mat o(a.c, b.c);
  for (int64_t j = 0; j < b.c; ++j)
    for (int64_t i = 0; i < a.c; ++i) {
      const double* ac = a.col(i);
      const double* bc = b.col(j);
      double s = 0.0;
      for (int64_t k = 0; k < a.r; ++k) s += ac[k] * bc[k];
      o(i, j) = s;
    }
  return o;
}
Mat transpose(const Mat& a) {
  Mat o(a.c, a.r);
  for (int64_t j = 0; j < a.c; ++j)
    for (int64_t i = 0; i < a.r; ++i) o(j, i) = a(i, j);
  return o;
}
Vec matvec(const Mat& a, const Vec& x) {
  Vec o(static_cast<size_t>(a.r), 0.0);
  for (int64_t j = 0; j < a.c; ++j) {
    const double xj = x[j];
    const double* ac = a.col(j);
    for (int64_t i = 0; i < a.r; ++i) o[i] += ac[i] * xj;
  }
  return o;
}
Vec matvec_t(const Mat& a, const Vec& x) {
  Vec o(static_cast<size_t>(a.c), 0.0);
  for (int64_t j = 0; j < a.c; ++j) {
    const double* ac = a.col(j);
    double s = 0.0;
    for (int64_t i = 0; i < a.r; ++i) s += ac[i] * x[i];
    o[j] = s;
  }
  return o;
}
Mat append_columns(const Mat& a, const Mat& b) {
  const int64_t r = a.c > 0 ? a.r : b.r;
  Mat o(r, a.c + b.c);
  std::copy(a.a.begin(), a.a.end(), o.a.begin());
  std::copy(b.a.begin(), b.a.end(), o.a.begin() + a.a.size());
  return o;
}
Mat left_cols(const Mat& a, int64_t k) {
  Mat o(a.r, k);
  std::copy(a.a.begin(), a.a.begin() + a.r * k, o.a.begin());
  return o;
}

// -------------------------------------------------------------------- rng ---
// proj/src/rng.cpp:9-14
uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

namespace {
// proj/src/rng.cpp:16-30: mt19937_64 + Box-Muller, spare cached.
struct Sampler {
  std::mt19937_64 gen;
  double spare = 0.0;
  bool have = false;
  explicit Sampler(uint64_t s) : gen(s) {}
  double next() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = static_cast<double>((gen() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * M_PI * u2;
    spare = r * std::sin(t);
    have = true;
    return r * std::cos(t);
  }
};
}  // namespace

// proj/src/rng.cpp:32-44: column-major fill from ONE sampler.
Mat gaussian_matrix(int64_t n, int64_t l, uint64_t seed) {
  if (n < 1 || l < 1) throw std::invalid_argument("gaussian_matrix: dimensions must be >= 1");
  Sampler s(seed);
  Mat o(n, l);
  for (auto& v : o.a) v = s.next();
  return o;
}
Vec gaussian_vector(int64_t n, uint64_t seed) { return gaussian_matrix(n, 1, seed).a; }

// ----------------------------------------------------------------- linalg ---
// Householder thin QR with R(i,i) >= 0 (proj/src/linalg.cpp:108-134). The
// reflector follows Eigen's makeHouseholder convention (beta = -sign(c0)|x|).
ThinQR thin_qr(const Mat& y) {
  const int64_t n = y.r, l = y.c;
  if (n < l) throw std::invalid_argument("thin_qr: need rows >= cols");
  Mat a = y;
  std::vector<double> tau(static_cast<size_t>(l), 0.0);
  for (int64_t k = 0; k < l; ++k) {
    double* x = a.col(k) + k;
    const int64_t len = n - k;
    double tail = 0.0;
    for (int64_t i = 1; i < len; ++i) tail += x[i] * x[i];
    const double c0 = x[0];
    double beta, t;
    if (tail <= std::numeric_limits<double>::min()) {
      t = 0.0;
      beta = c0;
      for (int64_t i = 1; i < len; ++i) x[i] = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double inv = 1.0 / (c0 - beta);
      for (int64_t i = 1; i < len; ++i) x[i] *= inv;
      t = (beta - c0) / beta;
    }
    x[0] = beta;
    tau[k] = t;
    if (t != 0.0) {
      for (int64_t j = k + 1; j < l; ++j) {
        double* cj = a.col(j) + k;
        double s = cj[0];
        for (int64_t i = 1; i < len; ++i) s += x[i] * cj[i];
        s *= t;
        cj[0] -= s;
        for (int64_t i = 1; i < len; ++i) cj[i] -= s * x[i];
      }
    }
  }
  ThinQR out;
  out.r = Mat(l, l);
  for (int64_t j = 0; j < l; ++j)
    for (int64_t i = 0; i <= j; ++i) out.r(i, j) = a(i, j);
  out.q = Mat::identity(n, l);
  for (int64_t k = l - 1; k >= 0; --k) {
    if (tau[k] == 0.0) continue;
    const double* v = a.col(k) + k;
    const int64_t len = n - k;
    for (int64_t j = 0; j < l; ++j) {
      double* qj = out.q.col(j) + k;
      double s = qj[0];
      for (int64_t i = 1; i < len; ++i) s += v[i] * qj[i];
      s *= tau[k];
      qj[0] -= s;
      for (int64_t i = 1; i < len; ++i) qj[i] -= s * v[i];
    }
  }
  for (int64_t i = 0; i < l; ++i) {
    if (out.r(i, i) < 0.0) {
      for (int64_t j = 0; j < l; ++j) out.r(i, j) = -out.r(i, j);
      double* qi = out.q.col(i);
      for (int64_t k = 0; k < n; ++k) qi[k] = -qi[k];
    }
  }
  double dmax = 0.0;
  for (int64_t i = 0; i < l; ++i) dmax = std::max(dmax, std::abs(out.r(i, i)));
  const double tol = static_cast<double>(std::max(n, l)) * std::numeric_limits<double>::epsilon() * dmax;
  for (int64_t i = 0; i < l; ++i)
    if (std::abs(out.r(i, i)) <= tol) out.deficient_columns.push_back(i);
  return out;
}

namespace {
// One-sided (Hestenes) Jacobi SVD of a square k x k matrix: B = U S V^T.
void jacobi_svd_square(const Mat& b, Mat& u, Vec& s, Mat& v) {
  const int64_t k = b.c;
  u = b;
  v = Mat::identity(k, k);
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int64_t p = 0; p < k - 1; ++p)
      for (int64_t q = p + 1; q < k; ++q) {
        double al = 0, be = 0, ga = 0;
        const double* up = u.col(p);
        const double* uq = u.col(q);
        for (int64_t i = 0; i < u.r; ++i) {
          al += up[i] * up[i];
          be += uq[i] * uq[i];
          ga += up[i] * uq[i];
        }
        if (ga == 0.0 || std::abs(ga) <= eps * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        double* upw = u.col(p);
        double* uqw = u.col(q);
        for (int64_t i = 0; i < u.r; ++i) {
          const double x = upw[i], y = uqw[i];
          upw[i] = c * x - sn * y;
          uqw[i] = sn * x + c * y;
        }
        double* vp = v.col(p);
        double* vq = v.col(q);
        for (int64_t i = 0; i < k; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - sn * y;
          vq[i] = sn * x + c * y;
        }
      }
    if (!rotated) break;
  }
  s.assign(static_cast<size_t>(k), 0.0);
  for (int64_t j = 0; j < k; ++j) {
    double nn = 0;
    for (int64_t i = 0; i < u.r; ++i) nn += u(i, j) * u(i, j);
    s[j] = std::sqrt(nn);
  }
  std::vector<int64_t> ord(static_cast<size_t>(k));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b2) { return s[a] > s[b2]; });
  Mat u2(u.r, k), v2(k, k);
  Vec s2(static_cast<size_t>(k));
  for (int64_t j = 0; j < k; ++j) {
    s2[j] = s[ord[j]];
    for (int64_t i = 0; i < u.r; ++i) u2(i, j) = s2[j] > 0 ? u(i, ord[j]) / s2[j] : 0.0;
    for (int64_t i = 0; i < k; ++i) v2(i, j) = v(i, ord[j]);
  }
  // Complete left vectors of exactly-zero singular values to an orthonormal set.
  for (int64_t j = 0; j < k; ++j) {
    if (s2[j] > 0) continue;
    for (int64_t e = 0; e < u.r; ++e) {
      Vec c(static_cast<size_t>(u.r), 0.0);
      c[e] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t jj = 0; jj < k; ++jj) {
          if (jj == j || (s2[jj] == 0 && jj > j)) continue;
          double d = 0;
          for (int64_t i = 0; i < u.r; ++i) d += u2(i, jj) * c[i];
          for (int64_t i = 0; i < u.r; ++i) c[i] -= d * u2(i, jj);
        }
      const double nn = norm2(c);
      if (nn > 0.5) {
        for (int64_t i = 0; i < u.r; ++i) u2(i, j) = c[i] / nn;
        break;
      }
    }
  }
  u = u2;
  v = v2;
  s = s2;
}
}  // namespace

// Thin SVD (proj/src/linalg.cpp:136-139 uses Eigen BDCSVD); here QR + one-sided
// Jacobi on the square factor, which is accurate to roundoff in the same sense.
ThinSVD thin_svd(const Mat& a) {
  ThinSVD out;
  if (a.r == 0 || a.c == 0) {
    out.u = Mat(a.r, 0);
    out.v = Mat(a.c, 0);
    return out;
  }
  if (a.r >= a.c) {
    const ThinQR qr = thin_qr(a);
    Mat ur, vr;
    Vec s;
    jacobi_svd_square(qr.r, ur, s, vr);
    out.u = matmul(qr.q, ur);
    out.s = s;
    out.v = vr;
  } else {
    const ThinSVD t = thin_svd(transpose(a));
    out.u = t.v;
    out.s = t.s;
    out.v = t.u;
  }
  return out;
}

Mat pseudo_inverse(const Mat& a, int* truncated) {
  const ThinSVD svd = thin_svd(a);
  const double smax = svd.s.empty() ? 0.0 : svd.s[0];
  const double tol = static_cast<double>(std::max(a.r, a.c)) * std::numeric_limits<double>::epsilon() * smax;
  int dropped = 0;
  Mat vs = svd.v;
  for (size_t i = 0; i < svd.s.size(); ++i) {
    const double inv = svd.s[i] > tol ? 1.0 / svd.s[i] : 0.0;
    if (!(svd.s[i] > tol)) ++dropped;
    for (int64_t r = 0; r < vs.r; ++r) vs(r, static_cast<int64_t>(i)) *= inv;
  }
  if (truncated) *truncated = dropped;
  return matmul(vs, transpose(svd.u));
}

Mat cholesky_lower(const Mat& spd) {
  const int64_t n = spd.r;
  Mat l(n, n);
  for (int64_t j = 0; j < n; ++j) {
    double d = spd(j, j);
    for (int64_t k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (!(d > 0.0)) throw std::runtime_error("cholesky_lower: matrix is not positive definite");
    const double ljj = std::sqrt(d);
    l(j, j) = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = spd(i, j);
      for (int64_t k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / ljj;
    }
  }
  return l;
}

Mat lower_solve(const Mat& l, const Mat& b) {
  Mat x = b;
  for (int64_t c = 0; c < b.c; ++c) {
    double* xc = x.col(c);
    for (int64_t i = 0; i < l.r; ++i) {
      double s = xc[i];
      for (int64_t k = 0; k < i; ++k) s -= l(i, k) * xc[k];
      xc[i] = s / l(i, i);
    }
  }
  return x;
}

double spectral_norm(const Mat& a) {
  if (a.a.empty()) return 0.0;
  const ThinSVD s = thin_svd(a);
  return s.s[0];
}

void sym_eig(const Mat& a0, Vec& evals, Mat& evecs) {
  const int64_t n = a0.r;
  Mat a = a0;
  evecs = Mat::identity(n, n);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int64_t p = 0; p < n - 1; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double vkp = evecs(k, p), vkq = evecs(k, q);
          evecs(k, p) = c * vkp - s * vkq;
          evecs(k, q) = s * vkp + c * vkq;
        }
      }
  }
  std::vector<int64_t> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return a(x, x) < a(y, y); });
  Mat v2(n, n);
  evals.assign(static_cast<size_t>(n), 0.0);
  for (int64_t j = 0; j < n; ++j) {
    evals[j] = a(ord[j], ord[j]);
    for (int64_t i = 0; i < n; ++i) v2(i, j) = evecs(i, ord[j]);
  }
  evecs = v2;
}

// -------------------------------------------------------------------- FFT ---
namespace {
// Per-length twiddle tables exp(-2 pi i k / n), k < n/2 (thread-safe cache).
const std::vector<cplx>& twiddles(size_t n) {
  static std::mutex mu;
  static std::map<size_t, std::vector<cplx>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  std::vector<cplx> w(n / 2 + 1);
  for (size_t k = 0; k <= n / 2; ++k) {
    const double ang = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
    w[k] = cplx(std::cos(ang), std::sin(ang));
  }
  return cache.emplace(n, std::move(w)).first->second;
}
}  // namespace

// Iterative radix-2 Cooley-Tukey; explicit real arithmetic (no __muldc3).
void fft_inplace(std::vector<cplx>& xv, bool inverse) {
  const size_t n = xv.size();
  if (n == 0 || (n & (n - 1))) throw std::invalid_argument("fft: length must be a power of two");
  double* x = reinterpret_cast<double*>(xv.data());
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(x[2 * i], x[2 * j]);
      std::swap(x[2 * i + 1], x[2 * j + 1]);
    }
  }
  const std::vector<cplx>& tw = twiddles(n);
  const double sgn = inverse ? -1.0 : 1.0;
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len / 2, step = n / len;
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < half; ++k) {
        const double wr = tw[k * step].real(), wi = sgn * tw[k * step].imag();
        double* a = x + 2 * (i + k);
        double* b = x + 2 * (i + k + half);
        const double tr = wr * b[0] - wi * b[1], ti = wr * b[1] + wi * b[0];
        b[0] = a[0] - tr;
        b[1] = a[1] - ti;
        a[0] += tr;
        a[1] += ti;
      }
  }
}

void fft2_inplace(std::vector<cplx>& x, int nx, int ny, bool inverse) {
  par_for(ny, [&](int64_t j0, int64_t j1) {
    std::vector<cplx> row(static_cast<size_t>(nx));
    for (int64_t j = j0; j < j1; ++j) {
      std::copy(x.begin() + static_cast<size_t>(j) * nx, x.begin() + static_cast<size_t>(j + 1) * nx, row.begin());
      fft_inplace(row, inverse);
      std::copy(row.begin(), row.end(), x.begin() + static_cast<size_t>(j) * nx);
    }
  });
  par_for(nx, [&](int64_t i0, int64_t i1) {
    std::vector<cplx> col(static_cast<size_t>(ny));
    for (int64_t i = i0; i < i1; ++i) {
      for (int j = 0; j < ny; ++j) col[j] = x[i + static_cast<size_t>(nx) * j];
      fft_inplace(col, inverse);
      for (int j = 0; j < ny; ++j) x[i + static_cast<size_t>(nx) * j] = col[j];
    }
  });
}

// ------------------------------------------------------------ par_for pool --
namespace {
thread_local bool t_no_par = false;
struct Pool {
  // Workers spin briefly on the generation counter before sleeping, so a
  // parallel region costs ~1 us to dispatch (the oracle issues thousands).
  int nt = 1;
  std::vector<std::thread> th;
  std::mutex busy;  // one parallel region at a time
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<uint64_t> gen{0};
  std::atomic<int> pending{0};
  std::atomic<bool> stop{false};
  int64_t n = 0;
  const std::function<void(int64_t, int64_t)>* f = nullptr;
  Pool() {
    if (const char* e = std::getenv("ORACLE_THREADS")) nt = std::max(1, std::atoi(e));
    for (int t = 1; t < nt; ++t) th.emplace_back([this, t] { worker(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
      gen.fetch_add(1);
    }
    cv.notify_all();
    for (auto& x : th) x.join();
  }
  void chunk(int t) {
    const int64_t b = n * t / nt, e = n * (t + 1) / nt;
    if (b < e) (*f)(b, e);
  }
  void worker(int t) {
    t_no_par = true;
    uint64_t seen = 0;
    for (;;) {
      int spins = 0;
      while (gen.load(std::memory_order_acquire) == seen && ++spins < 20000) {
      }
      if (gen.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> l(mu);
        cv.wait(l, [&] { return gen.load() != seen; });
      }
      seen = gen.load(std::memory_order_acquire);
      if (stop) return;
      chunk(t);
      pending.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  void run(int64_t nn, const std::function<void(int64_t, int64_t)>& ff) {
    n = nn;
    f = &ff;
    pending.store(nt - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> l(mu);
      gen.fetch_add(1, std::memory_order_release);
    }
    cv.notify_all();
    chunk(0);
    while (pending.load(std::memory_order_acquire) != 0) {
    }
  }
};
Pool& pool() {
  static Pool p;
  return p;
}
}  // namespace

void set_no_par(bool v) { t_no_par = v; }

void par_for(int64_t n, const std::function<void(int64_t, int64_t)>& f) {
  if (n <= 0) return;
  if (t_no_par || n < 2) return f(0, n);
  Pool& p = pool();
  if (p.nt <= 1 || !p.busy.try_lock()) return f(0, n);
  std::lock_guard<std::mutex> l(p.busy, std::adopt_lock);
  p.run(n, f);
}

// ---------------------------------------------------- maps, Woodbury, PCG ---
Vec CountingMap::apply(const Vec& x) const {
  applies_.fetch_add(1, std::memory_order_relaxed);
  return inner_.apply(x);
}
Vec CountingMap::adjoint_apply(const Vec& y) const {
  adjoint_applies_.fetch_add(1, std::memory_order_relaxed);
  return inner_.adjoint_apply(y);
}
long CountingMap::applies() const { return applies_.load(); }
long CountingMap::adjoint_applies() const { return adjoint_applies_.load(); }

// proj/src/linalg.cpp:32-50
Vec woodbury_apply(const LowRankEVD& evd, const Vec& v) {
  if (evd.basis.r != static_cast<int64_t>(v.size()))
    throw std::invalid_argument("woodbury_apply: dimension mismatch");
  if (evd.basis.c != static_cast<int64_t>(evd.eigenvalues.size()))
    throw std::invalid_argument("woodbury_apply: basis/eigenvalue mismatch");
  if (!all_finite(v) || !all_finite(evd.eigenvalues) || !all_finite(evd.basis.a))
    throw std::invalid_argument("woodbury_apply: non-finite input");
  if (evd.rank() == 0) return v;
  Vec coeff = matvec_t(evd.basis, v);
  for (size_t i = 0; i < coeff.size(); ++i)
    coeff[i] *= evd.eigenvalues[i] / (1.0 + evd.eigenvalues[i]);
  const Vec corr = matvec(evd.basis, coeff);
  Vec out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i] - corr[i];
  return out;
}

// proj/src/linalg.cpp:52-106
PCGReport pcg_solve(const LinearMap& op, const Vec& rhs, const Preconditioner& precond, double tol,
                    int max_iter) {
  if (op.rows() != op.cols() || op.rows() != static_cast<int64_t>(rhs.size()))
    throw std::invalid_argument("pcg_solve: dimension mismatch");
  if (!(tol > 0.0)) throw std::invalid_argument("pcg_solve: tolerance must be positive");
  PCGReport rep;
  const double rhs_norm = norm2(rhs);
  rep.solution.assign(rhs.size(), 0.0);
  if (rhs_norm == 0.0) {
    rep.converged = true;
    return rep;
  }
  Vec r = rhs;
  Vec z = precond ? precond(r) : r;
  double rz = dot(r, z);
  if (rz <= 0.0)
    throw std::runtime_error("pcg_solve: preconditioner is not positive definite (<r, M^-1 r> <= 0)");
  Vec p = z;
  for (int k = 1; k <= max_iter; ++k) {
    const Vec q = op.apply(p);
    const double pq = dot(p, q);
    if (pq <= 0.0) throw std::runtime_error("pcg_solve: operator is not positive definite (<p, A p> <= 0)");
    const double alpha = rz / pq;
    for (size_t i = 0; i < r.size(); ++i) {
      rep.solution[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    const double relres = norm2(r) / rhs_norm;
    rep.relative_residuals.push_back(relres);
    rep.iterations = k;
    if (relres <= tol) {
      rep.converged = true;
      return rep;
    }
    z = precond ? precond(r) : r;
    const double rz_next = dot(r, z);
    if (rz_next <= 0.0)
      throw std::runtime_error("pcg_solve: preconditioner is not positive definite (<r, M^-1 r> <= 0)");
    const double beta = rz_next / rz;
    for (size_t i = 0; i < p.size(); ++i) p[i] = z[i] + beta * p[i];
    rz = rz_next;
  }
  return rep;
}

}  // namespace oracle

// Small dense host linear algebra + seeded Gaussian generator (see hostla.hpp).
#include "hostla.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>

namespace sdv {

HMat hmat_mul(const HMat& a, const HMat& b) {
  if (a.c != b.r) throw std::invalid_argument("hmat_mul: shape");
  HMat o(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k) {
      const double bk = b(k, j);
      for (int i = 0; i < a.r; ++i) o(i, j) += a(i, k) * bk;
    }
  return o;
}
HMat hmat_t(const HMat& a) {
  HMat o(a.c, a.r);
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i) o(j, i) = a(i, j);
  return o;
}

void hqr(const HMat& y, HMat& q, HMat& r) {
  const int n = y.r, l = y.c;
  if (n < l) throw std::invalid_argument("thin_qr: need rows >= cols");
  HMat a = y;
  std::vector<double> tau(static_cast<size_t>(l), 0.0);
  for (int k = 0; k < l; ++k) {
    double tail = 0.0;
    for (int i = k + 1; i < n; ++i) tail += a(i, k) * a(i, k);
    const double c0 = a(k, k);
    double beta, t;
    if (tail <= DBL_MIN) {
      t = 0.0;
      beta = c0;
      for (int i = k + 1; i < n; ++i) a(i, k) = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double inv = 1.0 / (c0 - beta);
      for (int i = k + 1; i < n; ++i) a(i, k) *= inv;
      t = (beta - c0) / beta;
    }
    a(k, k) = beta;
    tau[k] = t;
    if (t == 0.0) continue;
    for (int j = k + 1; j < l; ++j) {
      double s = a(k, j);
      for (int i = k + 1; i < n; ++i) s += a(i, k) * a(i, j);
      s *= t;
      a(k, j) -= s;
      for (int i = k + 1; i < n; ++i) a(i, j) -= s * a(i, k);
    }
  }
  r = HMat(l, l);
  for (int j = 0; j < l; ++j)
    for (int i = 0; i <= j; ++i) r(i, j) = a(i, j);
  q = HMat(n, l);
  for (int i = 0; i < l; ++i) q(i, i) = 1.0;
  for (int k = l - 1; k >= 0; --k) {
    if (tau[k] == 0.0) continue;
    for (int j = k; j < l; ++j) {
      double s = q(k, j);
      for (int i = k + 1; i < n; ++i) s += a(i, k) * q(i, j);
      s *= tau[k];
      q(k, j) -= s;
      for (int i = k + 1; i < n; ++i) q(i, j) -= s * a(i, k);
    }
  }
  for (int i = 0; i < l; ++i)
    if (r(i, i) < 0.0) {
      for (int j = 0; j < l; ++j) r(i, j) = -r(i, j);
      for (int k = 0; k < n; ++k) q(k, i) = -q(k, i);
    }
}

void hsvd_square(const HMat& b, HMat& u, std::vector<double>& s, HMat& v) {
  const int k = b.c;
  u = b;
  v = HMat(k, k);
  for (int i = 0; i < k; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < u.r; ++i) {
          al += u(i, p) * u(i, p);
          be += u(i, q) * u(i, q);
          ga += u(i, p) * u(i, q);
        }
        if (ga == 0.0 || std::abs(ga) <= DBL_EPSILON * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < u.r; ++i) {
          const double x = u(i, p), y = u(i, q);
          u(i, p) = c * x - sn * y;
          u(i, q) = sn * x + c * y;
        }
        for (int i = 0; i < k; ++i) {
          const double x = v(i, p), y = v(i, q);
          v(i, p) = c * x - sn * y;
          v(i, q) = sn * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> nrm(static_cast<size_t>(k));
  for (int j = 0; j < k; ++j) {
    double s2 = 0;
    for (int i = 0; i < u.r; ++i) s2 += u(i, j) * u(i, j);
    nrm[j] = std::sqrt(s2);
  }
  std::vector<int> ord(static_cast<size_t>(k));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
  HMat u2(u.r, k), v2(k, k);
  s.assign(static_cast<size_t>(k), 0.0);
  for (int j = 0; j < k; ++j) {
    s[j] = nrm[ord[j]];
    for (int i = 0; i < u.r; ++i) u2(i, j) = s[j] > 0 ? u(i, ord[j]) / s[j] : 0.0;
    for (int i = 0; i < k; ++i) v2(i, j) = v(i, ord[j]);
  }
  for (int j = 0; j < k; ++j) {  // complete exact-zero columns orthonormally
    if (s[j] > 0) continue;
    for (int e = 0; e < u.r; ++e) {
      std::vector<double> c(static_cast<size_t>(u.r), 0.0);
      c[e] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int jj = 0; jj < k; ++jj) {
          if (jj == j || (s[jj] == 0 && jj > j)) continue;
          double d = 0;
          for (int i = 0; i < u.r; ++i) d += u2(i, jj) * c[i];
          for (int i = 0; i < u.r; ++i) c[i] -= d * u2(i, jj);
        }
      double nn = 0;
      for (double x : c) nn += x * x;
      nn = std::sqrt(nn);
      if (nn > 0.5) {
        for (int i = 0; i < u.r; ++i) u2(i, j) = c[i] / nn;
        break;
      }
    }
  }
  u = u2;
  v = v2;
}

void hsvd(const HMat& a, HMat& u, std::vector<double>& s, HMat& v) {
  if (a.r >= a.c) {
    HMat q, r, ur;
    hqr(a, q, r);
    hsvd_square(r, ur, s, v);
    u = hmat_mul(q, ur);
  } else {
    HMat ut, vt;
    hsvd(hmat_t(a), ut, s, vt);
    u = vt;
    v = ut;
  }
}

HMat hcholesky(const HMat& spd) {
  const int n = spd.r;
  HMat l(n, n);
  for (int j = 0; j < n; ++j) {
    double d = spd(j, j);
    for (int k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (!(d > 0.0)) throw std::runtime_error("cholesky_lower: matrix is not positive definite");
    const double ljj = std::sqrt(d);
    l(j, j) = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = spd(i, j);
      for (int k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / ljj;
    }
  }
  return l;
}

HMat hpinv(const HMat& a, int* truncated) {
  HMat u, v;
  std::vector<double> s;
  hsvd(a, u, s, v);
  const double smax = s.empty() ? 0.0 : s[0];
  const double tol = static_cast<double>(std::max(a.r, a.c)) * DBL_EPSILON * smax;
  int dropped = 0;
  for (size_t i = 0; i < s.size(); ++i) {
    const double inv = s[i] > tol ? 1.0 / s[i] : 0.0;
    if (!(s[i] > tol)) ++dropped;
    for (int r = 0; r < v.r; ++r) v(r, static_cast<int>(i)) *= inv;
  }
  if (truncated) *truncated = dropped;
  return hmat_mul(v, hmat_t(u));
}

void hsym_eig(const HMat& a0, std::vector<double>& w, HMat& vec) {
  const int n = a0.r;
  HMat a = a0;
  vec = HMat(n, n);
  for (int i = 0; i < n; ++i) vec(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off == 0.0 || off <= 1e-32 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double th = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double x = a(k, p), y = a(k, q);
          a(k, p) = c * x - s * y;
          a(k, q) = s * x + c * y;
        }
        for (int k = 0; k < n; ++k) {
          const double x = a(p, k), y = a(q, k);
          a(p, k) = c * x - s * y;
          a(q, k) = s * x + c * y;
        }
        for (int k = 0; k < n; ++k) {
          const double x = vec(k, p), y = vec(k, q);
          vec(k, p) = c * x - s * y;
          vec(k, q) = s * x + c * y;
        }
      }
  }
  std::vector<int> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
  HMat v2(n, n);
  w.assign(static_cast<size_t>(n), 0.0);
  for (int j = 0; j < n; ++j) {
    w[j] = a(ord[j], ord[j]);
    for (int i = 0; i < n; ++i) v2(i, j) = vec(i, ord[j]);
  }
  vec = v2;
}

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

std::vector<double> gaussian_matrix(int64_t n, int64_t l, uint64_t seed) {
  if (n < 1 || l < 1) throw std::invalid_argument("gaussian_matrix: dimensions must be >= 1");
  std::mt19937_64 gen(seed);
  std::vector<double> o(static_cast<size_t>(n * l));
  bool have = false;
  double spare = 0.0;
  for (auto& v : o) {
    if (have) {
      have = false;
      v = spare;
      continue;
    }
    const double u1 = static_cast<double>((gen() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * M_PI * u2;
    spare = r * std::sin(t);
    have = true;
    v = r * std::cos(t);
  }
  return o;
}

}  // namespace sdv

// Small dense host linear algebra for the l x l projected problems of the
// sketches (l <= a few hundred): one-sided Jacobi SVD, Jacobi symmetric
// eigensolver, Cholesky, Householder QR, pseudo-inverse; and the seeded
// Gaussian generator (bit-exact with proj/src/rng.cpp:9-48: mt19937_64 +
// Box-Muller with cached spare, column-major fill from one sampler).
// The n x l (tall) work of the sketches runs on the device; only l x l
// matrices reach these routines.
#pragma once

#include <cstdint>
#include <vector>

namespace sdv {

struct HMat {
  int r = 0, c = 0;
  std::vector<double> a;  // column-major
  HMat() = default;
  HMat(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
};

HMat hmat_mul(const HMat& a, const HMat& b);
HMat hmat_t(const HMat& a);

// Square one-sided Jacobi SVD: b = u diag(s) v^T, s non-increasing.
void hsvd_square(const HMat& b, HMat& u, std::vector<double>& s, HMat& v);
// Thin SVD of any small matrix (QR + Jacobi).
void hsvd(const HMat& a, HMat& u, std::vector<double>& s, HMat& v);
// Householder thin QR with R(i,i) >= 0 (proj/src/linalg.cpp:108-134).
void hqr(const HMat& y, HMat& q, HMat& r);
// Lower Cholesky; throws std::runtime_error when not positive definite.
HMat hcholesky(const HMat& spd);
// Moore-Penrose inverse with the reference truncation max(r,c) eps s_max.
HMat hpinv(const HMat& a, int* truncated);
// Symmetric eigen-decomposition, eigenvalues ascending.
void hsym_eig(const HMat& a, std::vector<double>& w, HMat& v);

uint64_t mix_seed(uint64_t seed, uint64_t stream);
// n x l standard normal, column-major, one mt19937_64 stream.
std::vector<double> gaussian_matrix(int64_t n, int64_t l, uint64_t seed);

}  // namespace sdv

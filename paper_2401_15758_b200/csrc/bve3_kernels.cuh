// Host-side interface of the reference-BVE kernels (bve3_kernels.cu).
#pragma once

#include "common.cuh"

namespace sdv {

// Model constants, computed on the host exactly as proj/src/bve.cpp does.
struct Bve3Args {
  int nx = 0, ny = 0;
  double cx = 0, cy = 0;      // d_x, d_y scales: 0.5 (nx+1), 0.25 (ny+1)
  double lx = 0, ly = 0;      // Laplacian scales 1/dx^2, 1/dy^2
  double inv_ro = 0, inv_re = 0, dt = 0;
  const double* forcing = nullptr;  // [ny]: sin(pi y_j), y_j = -1 + (j+1) dy
};

// (a I + bx Lx + by Ly)^{-1} on the Dirichlet grid (proj/src/dirichlet.cpp:
// 82-155): the orthonormal sine transform in x (shared-memory matvec kernel)
// diagonalises Lx; per x-mode the system in y is tridiagonal and solved
// exactly (Thomas, tabulated multipliers). Hand-written kernels, no library.
class DstSolver {
 public:
  DstSolver(int nx, int ny, double a, double bx, double by, cudaStream_t st);
  ~DstSolver();
  DstSolver(const DstSolver&) = delete;
  DstSolver& operator=(const DstSolver&) = delete;
  void solve(const double* in, double* out, int nvec) const;  // in may alias out

 private:
  size_t sine_smem(int rows) const;
  int nx_, ny_;
  double off_;
  cudaStream_t st_;
  DevBuf<double> sx_, m_, c_;
  mutable DevBuf<double> tmp_;
};

void bve3_nl_stage(const Bve3Args& a, int stage, const double* u, const double* ws, const double* ps, double* out,
                   int nvec, cudaStream_t st);
void bve3_tlm_stage(const Bve3Args& a, int stage, const double* d, const double* ds, const double* dp,
                    const double* wb, const double* pb, double* out, int nvec, cudaStream_t st);
void bve3_adj_vp(const Bve3Args& a, const double* L, const double* wb, double* vp, int nvec, cudaStream_t st);
void bve3_adj_stage(const Bve3Args& a, int stage, const double* L, const double* ps, const double* pb,
                    const double* lam, const double* t2, double* out, int nvec, cudaStream_t st);
// Gamma^{-1/2} of the 2-D Laplacian prior: alpha v + b (4v - neighbours), unscaled stencil
void lap2_inv_sqrt(int nx, int ny, double alpha, double b, const double* in, double* out, int nvec, cudaStream_t st);

}  // namespace sdv

// Host-side launch interface of the Burgers sweep kernels (burgers_kernels.cu).
#pragma once

#include "common.cuh"

namespace sdv {

struct BurgersArgs {
  int n = 0;
  double dt = 0, nu = 0, c1 = 0, c2 = 0;  // c1 = 1/(2 dx), c2 = 1/dx^2
  const double* base = nullptr;           // [steps][4][n] stage inputs
  int k0 = 0, k1 = 0;                     // step range
  int base_k0 = 0;                        // step of base's first row block (checkpoint segments)
  // observation gather/scatter (enabled when y != nullptr)
  const long long* idx = nullptr;
  int n_obs = 0;
  const double* w = nullptr;  // [n_t][n_obs] weights
  double* y = nullptr;        // [nvec][m]
  long long m = 0;
  int spi = 1;
};

void burgers_fwd(const BurgersArgs& p, const double* x0, double* base, double* out, int steps, cudaStream_t st);
void burgers_tlm(const BurgersArgs& p, double* state, int nvec, cudaStream_t st);
void burgers_adj(const BurgersArgs& p, double* state, int nvec, cudaStream_t st);
void spectral1d(int n, const double* in, double* out, const double* sym, int nvec, cudaStream_t st);

// The reference's own Burgers discretisation (proj/src/burgers.cpp): n
// interior points of (0,1), homogeneous Dirichlet walls, dx = 1/(n+1),
// Shu-Osher RK3-TVD; base = [steps][3][n] stage inputs (u, u1, u2).
void burgers3_fwd(const BurgersArgs& p, const double* x0, double* base, double* out, int steps, cudaStream_t st);
void burgers3_tlm(const BurgersArgs& p, double* state, int nvec, cudaStream_t st);
void burgers3_adj(const BurgersArgs& p, double* state, int nvec, cudaStream_t st);
// Gamma^{1/2} of the 1-D (alpha I - beta Lap*)^{-2} prior: Thomas solve with
// the reference's cached pivots (proj/src/dirichlet.cpp:157-187), and
// Gamma^{-1/2} = alpha v + b (2v - v_l - v_r) (proj/src/prior.cpp:53-62).
void thomas_solve(int n, double off, const double* pivot, const double* in, double* out, int nvec, cudaStream_t st);
void lap_inv_sqrt(int n, double alpha, double b, const double* in, double* out, int nvec, cudaStream_t st);

}  // namespace sdv

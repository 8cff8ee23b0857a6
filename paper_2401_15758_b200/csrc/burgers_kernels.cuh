// Host-side launch interface of the Burgers sweep kernels (burgers_kernels.cu).
#pragma once

#include "common.cuh"

namespace sdv {

struct BurgersArgs {
  int n = 0;
  double dt = 0, nu = 0, c1 = 0, c2 = 0;  // c1 = 1/(2 dx), c2 = 1/dx^2
  const double* base = nullptr;           // [steps][4][n] stage inputs
  int k0 = 0, k1 = 0;                     // step range
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

}  // namespace sdv

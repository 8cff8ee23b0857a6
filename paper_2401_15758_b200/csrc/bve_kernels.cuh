// Host-side launch interface of the batched BVE stage kernels (bve_kernels.cu).
#pragma once

#include "common.cuh"

namespace sdv {

enum StageMode { kModeTlm = 0, kModeAdj = 1, kModeNl = 2 };
enum StageFlags {
  kFlagHasPrev = 1,
  kFlagFinish = 2,
  // timing experiments only (probe): skip a phase, results are garbage
  kFlagSkipInvFft = 16,
  kFlagSkipStencil = 32,
  kFlagSkipFwdFft = 64,
  kFlagNoPrefetch = 128  // A/B timing of the tile prefetches
};

// Arguments of one fused RK stage launch over a group of vectors.
//   TLM/NL: d = step-start state, acc = RK accumulator, x_in = stage input
//           (read with halo), x_out = next stage input (stages 0-2).
//   ADJ   : d = lambda' (state at the step end), acc = lambda accumulator,
//           q_in/q_out = non-Poisson part of the previous/current mu.
//   NL    : store_w/store_p receive the stage input and its streamfunction.
struct StageArgs {
  int stage = 0;
  int flags = 0;
  const double2* s_in = nullptr;
  double2* s_out = nullptr;
  const double* x_in = nullptr;
  double* x_out = nullptr;
  double* d = nullptr;
  double* acc = nullptr;
  const double* q_in = nullptr;
  double* q_out = nullptr;
  const double* base_w = nullptr;
  const double* base_p = nullptr;
  double* store_w = nullptr;
  double* store_p = nullptr;
  const double2* tw = nullptr;
  double dt = 0, nu = 0, inv12h2 = 0, invh2 = 0;
};

void bve_row_fwd(int n, const double* f, double2* s, int nvec, cudaStream_t st);
void bve_row_inv(int n, const double2* s, double* f, int nvec, cudaStream_t st);
void bve_col(int n, double2* s, const double* sym, int nvec, cudaStream_t st);
void bve_stage(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st);
// Poisson column pass by cyclic first-order recurrences (kx >= 1) + the FFT
// column kernel on the packed kx = 0 column; tab: [n/2] {rho, rho^(n/32),
// 1/(1-rho^n), h^2 rho/n}; sym: the Poisson spectral symbol (column 0 only).
void bve_col_solve(int n, double2* s, const double4* tab, const double* sym, int nvec, cudaStream_t st);

void gather_obs(const double* f, long long dim, const long long* idx, int n_obs, const double* w, double* y,
                long long m, int nvec, cudaStream_t st);
void scatter_obs(double* f, long long dim, const long long* idx, int n_obs, const double* w, const double* y,
                 long long m, int nvec, cudaStream_t st);

}  // namespace sdv

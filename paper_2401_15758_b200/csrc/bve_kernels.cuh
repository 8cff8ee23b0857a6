// Host-side launch interface of the batched BVE stage kernels (bve_kernels.cu).
#pragma once

#include "common.cuh"

namespace sdv {

enum StageMode { kModeTlm = 0, kModeAdj = 1, kModeNl = 2 };
enum StageFlags {
  kFlagHasPrev = 1,
  kFlagFinish = 2,
  // fused Poisson path: s_in already holds final spectra (first TLM stage,
  // solved by the column pass), no tile-carry correction on load
  kFlagRawIn = 4,
  // fused kernel used as a plain stage (small blocks): write the packed
  // spectra of the next Poisson input, no tile-local recurrences
  kFlagNoRecur = 8,
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
  // Fused Poisson path (bve_stage(..., fused = true)): s_in/s_out hold the
  // tile-local recurrence values H of the y-solve (see bve_carry); car_c /
  // car_e are the tile carries of s_in, lsum receives the tile end values of
  // s_out; stab = the recurrence table of bve_col_solve. [v][n/8][n/2] double2.
  const double2* car_c = nullptr;
  const double2* car_e = nullptr;
  double2* lsum = nullptr;
  const double4* stab = nullptr;
  // Observation gather fused into the fused TLM stage-3 launch at an
  // interval end (proj/src/fourdvar.cpp:145-160: y_i = R_i^{-1/2} O x_i):
  // obs_y[v * obs_m + o] = d[v][obs_idx[o]] * obs_w[o] for the observations
  // o in [obs_tile[q], obs_tile[q + 1]) of the CTA's 8-row tile q (indices
  // sorted). obs_y == nullptr: no gather.
  const long long* obs_idx = nullptr;
  const double* obs_w = nullptr;
  double* obs_y = nullptr;
  const int* obs_tile = nullptr;
  long long obs_m = 0;
  double dt = 0, nu = 0, inv12h2 = 0, invh2 = 0;
};

void bve_row_fwd(int n, const double* f, double2* s, int nvec, cudaStream_t st);
void bve_row_inv(int n, const double2* s, double* f, int nvec, cudaStream_t st);
void bve_col(int n, double2* s, const double* sym, int nvec, cudaStream_t st);
void bve_stage(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st, bool fused = false);
// Whether a stage launch over nvec vectors takes the fused Poisson path
// (8-row tiles; smaller blocks use 2-row tiles and the column pass).
bool bve_fused_ok(int n, int nvec);
int bve_stage_fill();  // 8-row stage CTAs per lane from which the fused path is taken
// Small blocks on grids >= 256^2: the fused stage kernel with 2-row tiles as a
// plain stage (in-place x-FFTs, stencil input staged up front), flags must
// include kFlagRawIn | kFlagNoRecur; the column pass stays.
bool bve_lite_ok(int n, int nvec);
void bve_stage_lite(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st);
// Tile carries of the fused Poisson path. The stage kernels leave, per
// 8-row tile q and x-mode kx >= 1, the zero-carry forward/backward recurrence
// values H (in s) and the forward end value L_q (in lsum); this pass scans the
// n/8 tiles of every column (cyclic affine scans) into the carries C_q (from
// the rows below) and E_q (from the rows above), so that the next stage
// reconstructs psi_hat = scale (H + alpha_o C_q + rho^(8-o) E_q) on load. The
// packed kx = 0 column is solved in place by the FFT column path.
void bve_carry(int n, double2* s, const double2* lsum, double2* car_c, double2* car_e, const double4* tab,
               const double* sym, int nvec, cudaStream_t st);
// Poisson column pass by cyclic first-order recurrences (kx >= 1) + the FFT
// column kernel on the packed kx = 0 column; tab: [n/2] {rho, rho^(n/32),
// 1/(1-rho^n), h^2 rho/n}; sym: the Poisson spectral symbol (column 0 only).
void bve_col_solve(int n, double2* s, const double4* tab, const double* sym, int nvec, cudaStream_t st);

void gather_obs(const double* f, long long dim, const long long* idx, int n_obs, const double* w, double* y,
                long long m, int nvec, cudaStream_t st);
void scatter_obs(double* f, long long dim, const long long* idx, int n_obs, const double* w, const double* y,
                 long long m, int nvec, cudaStream_t st);

}  // namespace sdv

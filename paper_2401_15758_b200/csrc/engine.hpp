// Host-side engine: the device-resident problem, base trajectory and the
// batched Hessian-product sweeps. Mirrors the reference interfaces
//   AssimilationProblem / DynamicalModel::linearize / LinearizedTrajectory
//   MisfitOperator::apply / adjoint_apply / GramMap
// (/root/reference/proj/include/sketchdav/{fourdvar,model,linalg}.hpp) with
// block (s-vector) device entry points.
#pragma once

#include <algorithm>
#include <memory>

#include "bve3_kernels.cuh"
#include "bve_kernels.cuh"
#include "burgers_kernels.cuh"
#include "linalg_kernels.cuh"

namespace sdv {

// kModelBurgers3 / kModelBVE3: the reference's own Dirichlet RK3-TVD Burgers
// and barotropic-vorticity models (F3).
enum ModelKind { kModelBurgers = 1, kModelBVE = 2, kModelBurgers3 = 3, kModelBVE3 = 4 };
// kPriorFourier: B = sigma^2 C, Fourier-diagonal Gaussian (control-variable
// background term). kPriorLaplacian: Gamma = (alpha I - beta Lap*)^{-2}
// (proj/src/prior.cpp), x-space background term as the reference.
enum PriorKind { kPriorFourier = 0, kPriorLaplacian = 1 };

struct ProblemDesc {
  int model = kModelBurgers;
  int n = 0;  // grid points per dimension
  double nu = 0, dt = 0;
  int n_t = 0, spi = 0;
  double prior_sigma = 0, prior_length = 0;
  int block_group = 0;  // vectors per BVE sweep group (0 = auto)
  int prior_kind = kPriorFourier;
  double prior_alpha = 0, prior_beta = 0;
  int ny = 0;                        // kModelBVE3: rows (n = nx columns)
  double reynolds = 0, rossby = 0;   // kModelBVE3
};

class Problem;

// Storage policy of linearize (DynamicalModel::linearize's checkpoint_stride,
// proj/include/sketchdav/model.hpp:36-40): kStoreAuto keeps every RK stage in
// HBM when that fits the device (the contract's "implementations may store
// more") and falls back to checkpoints otherwise; kStoreCheckpoint always
// stores states every `stride` steps and recomputes one segment of stage
// inputs at a time inside the sweeps (proj/src/burgers.cpp:114-191).
enum StorePolicy { kStoreAuto = 0, kStoreFull = 1, kStoreCheckpoint = 2 };

// Device-resident base trajectory (FWD sweep output).
struct Trajectory {
  const Problem* prob = nullptr;
  int steps = 0;
  int stages = 4;        // stored stage inputs per step (RK4: 4, RK3-TVD: 3)
  DevBuf<double> w;      // [steps][4][dim] stage inputs (checkpoint mode: one segment, [stride][4][dim])
  DevBuf<double> p;      // BVE: [steps][4][dim] stage streamfunctions (checkpoint mode: one segment)
  DevBuf<double> final;  // [dim]
  // Checkpoint mode (stride > 0): ckpt[j] = state at step j*stride; w/p hold
  // the stage inputs of segment `seg` (steps [seg*stride, min(steps, (seg+1)*stride))).
  int stride = 0;
  DevBuf<double> ckpt;                  // [segments][dim]
  mutable int seg = -1;                 // segment held in w/p (-1: none)
  mutable DevBuf<double> scratch;       // state_at between checkpoints
  mutable DevBuf<double> rx0, rx1, racc, ru;  // BVE segment recompute workspace
  mutable DevBuf<double2> rs0, rs1;
  bool checkpointed() const { return stride > 0; }
  int segments() const { return stride > 0 ? (steps + stride - 1) / stride : 1; }
  int held_steps() const { return stride > 0 ? std::min(stride, steps) : steps; }
  // first step of the stored stage inputs (0 in full mode)
  int held_k0() const { return stride > 0 ? seg * stride : 0; }
  size_t stored_bytes() const {
    return sizeof(double) * (w.size() + p.size() + final.size() + ckpt.size());
  }
  const double* state_at(int step) const;  // step in [0, steps]
  // stage inputs / streamfunctions of step k, stage s (k must be held)
  const double* base_w(int k, int s, long long dim) const {
    return w.get() + (static_cast<long long>(k - held_k0()) * stages + s) * dim;
  }
  const double* base_p(int k, int s, long long dim) const {
    return p.get() + (static_cast<long long>(k - held_k0()) * stages + s) * dim;
  }
};

class Problem {
 public:
  Problem(const ProblemDesc& d, long long n_obs, const long long* idx, const double* values, const double* variances,
          const double* background);
  const ProblemDesc& desc() const { return d_; }
  long long dim() const { return dim_; }
  long long n_obs() const { return n_obs_; }
  long long m() const { return n_obs_ * d_.n_t; }
  int total_steps() const { return d_.n_t * d_.spi; }
  cudaStream_t stream() const { return st_; }

  // FWD nonlinear sweep from device x0, storing every RK4 stage input (or,
  // under kStoreCheckpoint / an auto fallback, checkpoints every `stride` steps).
  std::unique_ptr<Trajectory> linearize(const double* d_x0, int stride = 0, int policy = kStoreAuto) const;
  // Checkpoint mode: make the segment holding step k resident in tr.w / tr.p
  // (recomputed from its checkpoint on the problem stream).
  void hold_segment(const Trajectory& tr, int k) const;
  // Nonlinear forward of `steps` steps (device in/out), no storage.
  void forward(const double* d_x0, int steps, double* d_out) const;

  // out = B^{1/2} in, nvec vectors (device).
  void prior_sqrt(const double* in, double* out, int nvec) const;
  // TLM over steps [k0,k1) on state (nvec x dim, in/out); gathers obs*w to y
  // ([nvec][m]) at interval ends when y != null (requires k0 == 0).
  void tlm(const Trajectory& tr, double* state, int nvec, int k0, int k1, double* y, const double* w) const;
  // ADJ over [k0,k1) backwards on state (in/out); scatters y*w at interval ends.
  void adj(const Trajectory& tr, double* state, int nvec, int k0, int k1, const double* y, const double* w) const;

  // Prior-preconditioned misfit operator A = [R^{-1/2} O M Gamma^{1/2}] blocks.
  void misfit_apply(const Trajectory& tr, const double* v, int s, double* y) const;
  void misfit_adjoint(const Trajectory& tr, const double* w, int s, double* z) const;
  void gram_apply(const Trajectory& tr, const double* v, int s, double* hv) const;
  // number of L2-resident sub-blocks an s-wide block is swept as (0 = whole)
  int sub_blocks(int s) const;

  // cost (host); ctrl_grad = Gamma^{1/2} g (control form: z + Gamma^{1/2} lambda0);
  // lambda0; x-space gradient g = Gamma^{-1}(x0 - xb) + lambda0 (Laplacian
  // prior only). Device outputs may be null.
  double evaluate(const Trajectory& tr, const double* d_z, double* d_ctrl_grad, double* d_lambda0,
                  double* d_grad_x = nullptr) const;
  bool xspace() const { return d_.prior_kind == kPriorLaplacian; }
  // Gamma^{-1/2} (Laplacian prior only).
  void prior_inv_sqrt(const double* in, double* out, int nvec) const;

  // Timing probe (bench roofline): mean duration of the fused stage kernel and
  // the column kernel over `stages` TLM stages on a group of s vectors. For
  // Burgers the persistent sweep kernel is timed instead (ms_col = 0).
  void probe_stage_kernels(const Trajectory& tr, int s, int stages, float* ms_stage, float* ms_col) const;
  void probe_adj_stage_kernels(const Trajectory& tr, int s, int stages, float* ms_stage, float* ms_col) const;

  const double* d_rinv_sqrt() const { return rinv_sqrt_.get(); }
  const double* d_rinv() const { return rinv_.get(); }
  const double* d_background() const { return background_.get(); }
  const long long* d_idx() const { return idx_.get(); }

 private:
  void ensure_work(int nvec) const;
  int group() const;
  ProblemDesc d_;
  long long dim_ = 0, n_obs_ = 0;
  cudaStream_t st_ = nullptr;
  DevBuf<long long> idx_;
  DevBuf<int> obs_tile_;  // BVE, sorted indices: first observation of each 8-row tile (fused gather)
  DevBuf<double> values_, rinv_sqrt_, rinv_, background_;
  DevBuf<double> sym_b_, sym_p_;
  DevBuf<double> solve_tab_;  // BVE: per-kx recurrence constants of the Poisson column solve
  // Poisson column pass on row spectra (recurrence solver; SDV_COL_FFT=1 selects
  // the y-FFT / multiply / inverse y-FFT kernel instead).
  void poisson_col(double2* s, int nvec, cudaStream_t st) const;
  // Fused Poisson path (bve_stage fused = true): tile carries of the spectra
  // in s for the lane's vectors (see bve_carry).
  void poisson_carry(double2* s, long long woff, int nvec, cudaStream_t st) const;
  bool fused(int nvec) const;
  void set_fused(StageArgs& a, long long woff) const;
  // kModelBVE3: model constants, forcing, Poisson and prior DST solvers, and
  // sweep workspace (5 fields per vector)
  Bve3Args b3_;
  DevBuf<double> forcing_;
  std::unique_ptr<DstSolver> poisson3_, prior3_;
  mutable DevBuf<double> b3w_[5];
  void bve3_work(int nvec) const;
  void bve3_tlm(const Trajectory& tr, double* state, int nvec, int k0, int k1, double* y, const double* w) const;
  void bve3_adj(const Trajectory& tr, double* state, int nvec, int k0, int k1, const double* y, const double* w) const;
  DevBuf<double> pivot_;  // Laplacian prior: Thomas pivots
  double lap_b_ = 0;      // beta * stencil scale
  double dt_ = 0;
  // sweep workspace (grown on demand)
  mutable DevBuf<double> wa_, wx0_, wx1_, wstate_, wy_, sub_in_, sub_out_;
  mutable DevBuf<double2> ws0_, ws1_;
  mutable DevBuf<double2> lsum_, carc_, care_;  // fused path: [g][n/8][n/2] tile sums / carries
  mutable int work_nvec_ = 0;
  // CUDA graphs of small-block Gram sweeps (PCG / probes replay the same
  // launch sequence on the same buffers every iteration).
  struct GraphEntry {
    std::vector<const void*> key;
    cudaGraphExec_t exec = nullptr;
    unsigned long long nodes = 0;
  };
  mutable std::vector<GraphEntry> graphs_;
  void clear_graphs() const;
  enum { kOpGram = 1, kOpApply = 2, kOpAdjoint = 3 };
  template <class F>
  void graph_cached(int op, const Trajectory& tr, const double* in, double* out, int s, F&& run) const;
  // L2-resident sub-blocks of a wide BVE block (engine.cu; sub_blocks is public)
  static int graph_max();
  template <class F>
  void for_sub_blocks(int nb, const double* in, long long in_dim, double* out, long long out_dim, int s, F&& run) const;
  void misfit_apply_whole(const Trajectory& tr, const double* v, int s, double* y) const;
  void misfit_adjoint_whole(const Trajectory& tr, const double* w, int s, double* z) const;
  // Concurrent lanes: a sweep group split over two streams so the stage and
  // column kernels of the two halves co-reside on the SMs.
  struct Lane {
    int v0 = 0, cnt = 0;   // vectors [v0, v0+cnt) of the caller's block
    long long woff = 0;    // vector offset inside the sweep workspace
    cudaStream_t st = nullptr;
    double2* s_cur = nullptr;
    double2* s_nxt = nullptr;
    bool fz = false;       // fused Poisson path (decided once per sweep)
    bool lite = false;     // small block: fused kernel as a plain stage (column pass kept)
  };
  std::vector<Lane> split_lanes(int v0, int gn) const;
  void join_lanes(const std::vector<Lane>& lanes) const;
  void refork_lanes(const std::vector<Lane>& lanes) const;
  // BVE NL forward of `steps` steps on u (in/out) with explicit workspace,
  // storing stage inputs / streamfunctions when store_w != null.
  struct NlWork {
    double *x0, *x1, *acc;
    double2 *s0, *s1;
  };
  void bve_nl(double* u, int steps, double* store_w, double* store_p, const NlWork& wk) const;
  void linearize_ckpt(Trajectory& tr, const double* d_x0) const;
  void fill_segment(const Trajectory& tr, int j) const;
  void check_final(const Trajectory& tr) const;
  mutable std::vector<cudaStream_t> lane_st_;  // lanes 1.. of a sweep group (lane 0 runs on st_)
  mutable std::vector<cudaEvent_t> lane_ev_;
  mutable cudaEvent_t ev_fork_ = nullptr;

 public:
  ~Problem();
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;
};

}  // namespace sdv

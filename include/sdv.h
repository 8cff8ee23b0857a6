/*
 * sdv.h — C-ABI of the B200-native SC-4DVAR Hessian-product engine
 * (libsdv_cuda.so, built from paper_2401_15758_b200/csrc/).
 *
 * The entry points replace, call for call, the reference's hot-path C++
 * interfaces in /root/reference/proj/include/sketchdav (file:line below).
 * Conventions:
 *   - every function returns 0 on success, SDV_EINVAL for shape/config errors
 *     (the reference's std::invalid_argument), SDV_ENUMERIC for numerical
 *     failures (std::runtime_error: non-finite state, PCG breakdown, Cholesky)
 *     and SDV_ECUDA for CUDA faults; sdv_last_error() returns a thread-local
 *     message; nothing throws across the ABI;
 *   - dense blocks are fp64 column-major with the vector index slowest
 *     (an n x s block is [s][n]); observation vectors are time-major
 *     [n_t][n_obs] (proj/src/fourdvar.cpp:156, :170);
 *   - plain pointers are HOST buffers unless the name ends in _dev (device
 *     pointers, e.g. from sdv_dev_alloc);
 *   - a problem owns one CUDA stream; calls on one problem are serialised by
 *     the caller (not re-entrant); distinct problems may run concurrently.
 */
#ifndef SDV_H_
#define SDV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDV_OK 0
#define SDV_EINVAL (-22)
#define SDV_ENUMERIC (-34)
#define SDV_ECUDA (-5)

/* SDV_MODEL_BURGERS_DIRICHLET: the reference's own Burgers (proj/src/burgers.cpp,
 * n interior points, zero walls, RK3-TVD); requires SDV_PRIOR_LAPLACIAN. */
enum { SDV_MODEL_BURGERS = 1, SDV_MODEL_BVE = 2, SDV_MODEL_BURGERS_DIRICHLET = 3, SDV_MODEL_BVE_DIRICHLET = 4 };
/* SDV_MODEL_BVE_DIRICHLET: the reference's own barotropic-vorticity model
 * (proj/src/bve.cpp: n = nx columns x ny rows, zero walls, beta-term 1/Ro,
 * forcing sin(pi y), RK3-TVD, DST Poisson); requires SDV_PRIOR_LAPLACIAN (2-D,
 * unscaled stencil) and the ny / reynolds / rossby fields. */
/* SDV_PRIOR_FOURIER: B = sigma^2 C, Fourier-diagonal (control-variable form).
 * SDV_PRIOR_LAPLACIAN: Gamma = (alpha I - beta Lap*)^{-2} on the Dirichlet grid,
 * stencil scale 1 (proj/src/prior.cpp:9-62), x-space background term. */
enum { SDV_PRIOR_FOURIER = 0, SDV_PRIOR_LAPLACIAN = 1 };
enum { SDV_SKETCH_RANDSVD = 0, SDV_SKETCH_NYSTROM = 1, SDV_SKETCH_SINGLEVIEW = 2, SDV_SKETCH_LANCZOS = 3 };
/* proj/include/sketchdav/fourdvar.hpp:91-98 */
enum {
  SDV_MODE_SKETCHSOLV = 0,
  SDV_MODE_SKETCHPREC = 1,
  SDV_MODE_SKETCHPRECA = 2,
  SDV_MODE_PRECGAMMA = 3,
  SDV_MODE_PRECLANCZOS = 4,
  SDV_MODE_PRECALANCZOS = 5
};

typedef struct sdv_problem sdv_problem;
typedef struct sdv_traj sdv_traj;

/* Model + prior description (replaces constructing BurgersModel/BVEModel and
 * PriorCovariance, proj/include/sketchdav/{burgers,bve,prior}.hpp; periodic
 * RK4 / Arakawa / Fourier-Gaussian variants of SURVEY.md Appendix A). */
typedef struct {
  int model;            /* SDV_MODEL_* */
  int n;                /* grid points per dimension (power of two) */
  double nu;            /* viscosity */
  double dt;            /* inner time step */
  int n_t;              /* observation intervals */
  int steps_per_interval;
  double prior_sigma;   /* B = sigma^2 C */
  double prior_length;  /* Gaussian correlation length */
  int block_group;      /* BVE: vectors per L2-resident sweep group (0 = auto) */
  int prior_kind;       /* SDV_PRIOR_* */
  double prior_alpha;   /* Laplacian prior: alpha */
  double prior_beta;    /* Laplacian prior: beta */
  int ny;               /* SDV_MODEL_BVE_DIRICHLET: rows */
  double reynolds;      /* SDV_MODEL_BVE_DIRICHLET: Re */
  double rossby;        /* SDV_MODEL_BVE_DIRICHLET: Ro */
} sdv_problem_desc;

const char* sdv_last_error(void);
const char* sdv_version(void);
int sdv_device_init(int device);
/* Number of kernels this library has launched so far (process-wide). */
unsigned long long sdv_launch_count(void);
/* Per-variant launch counters of the sweep kernels (process-wide, atomic):
 * out[i] for i < min(n, count), returns count; sdv_path_name(i) names
 * variant i ("bve_stage_fused", "bve_carry", "bve_stage_lite", ...). A CUDA
 * graph replay is counted once, when it is captured. Lets callers and tests
 * assert which kernel path a call took. */
int sdv_path_counts(uint64_t* out, int n);
const char* sdv_path_name(int i);

/* AssimilationProblem (proj/include/sketchdav/fourdvar.hpp:25-40) + validate
 * (proj/src/fourdvar.cpp:25-58). obs_values/obs_variances: n_obs x n_t
 * column-major (= time-major [n_t][n_obs]). */
int sdv_problem_create(const sdv_problem_desc* desc, int64_t n_obs, const int64_t* obs_indices,
                       const double* obs_values, const double* obs_variances, const double* background,
                       sdv_problem** out);
void sdv_problem_destroy(sdv_problem* p);
/* dims = {state_dim, misfit_dim, n_obs, n_t, steps_per_interval, total_steps} */
int sdv_problem_dims(const sdv_problem* p, int64_t dims[6]);

/* DynamicalModel::forward (proj/include/sketchdav/model.hpp:33) */
int sdv_forward(sdv_problem* p, const double* x0, int steps, double* out);
/* DynamicalModel::linearize (proj/include/sketchdav/model.hpp:36-40): one FWD
 * sweep storing every RK4 stage input on the device. */
int sdv_linearize(sdv_problem* p, const double* x0, sdv_traj** out);
int sdv_linearize_dev(sdv_problem* p, const double* x0_dev, sdv_traj** out);
/* DynamicalModel::linearize(x0, steps, checkpoint_stride) with its stride
 * (proj/include/sketchdav/model.hpp:36-40; the reference's checkpointed
 * trajectory is proj/src/burgers.cpp:114-191). policy:
 *   SDV_STORE_AUTO       every RK stage in HBM when it fits (the contract's
 *                        "implementations may store more"), else checkpoints
 *                        every min(checkpoint_stride, what fits) steps;
 *   SDV_STORE_FULL       every RK stage (sdv_linearize);
 *   SDV_STORE_CHECKPOINT states every checkpoint_stride (>= 1) steps; the
 *                        sweeps recompute one segment of stage inputs at a
 *                        time from its checkpoint (results bitwise equal to
 *                        the full store).
 * The Dirichlet BVE (SDV_MODEL_BVE_DIRICHLET) stores every stage whatever the
 * policy, as the reference BVE (proj/src/bve.cpp:221-225). sdv_linearize is
 * SDV_STORE_AUTO with the problem's steps per interval as the stride. */
#define SDV_STORE_AUTO 0
#define SDV_STORE_FULL 1
#define SDV_STORE_CHECKPOINT 2
int sdv_linearize_ex(sdv_problem* p, const double* x0, int checkpoint_stride, int policy, sdv_traj** out);
int sdv_linearize_ex_dev(sdv_problem* p, const double* x0_dev, int checkpoint_stride, int policy, sdv_traj** out);
/* info = {total_steps, checkpoint stride (0 = every stage stored), segments,
 * bytes of HBM the trajectory holds} */
int sdv_traj_info(const sdv_traj* t, int64_t info[4]);
/* A problem destroyed while trajectories of it are alive is released with its
 * last trajectory (handles are reference-counted; the problem handle itself
 * is invalid after sdv_problem_destroy). */
void sdv_traj_destroy(sdv_traj* t);
/* How a block of s vectors is swept (the batching seam, proj/src/sketch.cpp:116-140):
 * n_sub = 0: as one block; n_sub > 0: as n_sub consecutive L2-resident
 * sub-blocks of near-equal width (wide blocks on grids whose per-vector RK
 * workspace would stream from HBM, e.g. 512^2: 8 vectors each), each one
 * CUDA-graph replay through the whole window. Results are identical. */
int sdv_sub_blocks(const sdv_problem* p, int s, int* n_sub);
/* LinearizedTrajectory::state_at / tlm_range / adj_range
 * (proj/include/sketchdav/model.hpp:17-21), batched over s vectors. */
int sdv_traj_state_at(const sdv_traj* t, int step, double* out);
int sdv_tlm_range(sdv_traj* t, int begin, int end, const double* dx, int s, double* out);
int sdv_adj_range(sdv_traj* t, int begin, int end, const double* lambda, int s, double* out);

/* PriorCovariance::apply_sqrt (proj/include/sketchdav/prior.hpp:34-35), s vectors. */
int sdv_prior_sqrt_block(sdv_problem* p, const double* v, int s, double* out);

/* MisfitOperator::apply / adjoint_apply (proj/src/fourdvar.cpp:145-176) and
 * GramMap::apply (proj/include/sketchdav/linalg.hpp:72-74) over a block of s
 * columns — the batched apply_columns seam (proj/src/sketch.cpp:116-140).
 * V: n x s, Y/W: m x s, Z/HV: n x s. */
int sdv_misfit_apply_block(sdv_traj* t, const double* V, int s, double* Y);
int sdv_misfit_adjoint_block(sdv_traj* t, const double* W, int s, double* Z);
int sdv_gram_apply_block(sdv_traj* t, const double* V, int s, double* HV);
int sdv_misfit_apply_block_dev(sdv_traj* t, const double* V_dev, int s, double* Y_dev);
int sdv_misfit_adjoint_block_dev(sdv_traj* t, const double* W_dev, int s, double* Z_dev);
int sdv_gram_apply_block_dev(sdv_traj* t, const double* V_dev, int s, double* HV_dev);

/* evaluate (proj/src/fourdvar.cpp:92-132), control-variable background term:
 * x0 = xb + B^{1/2} z; cost = 0.5|z|^2 + 0.5 sum innov^2/var;
 * ctrl_grad = z + B^{1/2} lambda0 (= Gamma^{1/2} g). z may be NULL (z = 0).
 * ctrl_grad / lambda0 may be NULL. */
int sdv_evaluate(sdv_problem* p, const double* x0, const double* z, double* cost, double* ctrl_grad,
                 double* lambda0);

/* woodbury_apply (proj/src/linalg.cpp:32-50) on s vectors: basis n x l. */
int sdv_woodbury_apply(sdv_problem* p, int64_t l, const double* basis, const double* eigenvalues, const double* v,
                       int s, double* out);
/* Device Householder thin QR (proj/src/linalg.cpp:108-134): y (n x l) ->
 * q (n x l), r (l x l); returns the deficient-column count in *ndef. */
int sdv_thin_qr(sdv_problem* p, int64_t n, int64_t l, const double* y, double* q, double* r, int* ndef);

/* Device-buffer forms for the sharded sketch: thin QR of a
 * device block in place (y_dev n x l -> Q, r host l x l; the sketches' QR:
 * CholQR2 on the fp64 tensor cores when the block is well conditioned, else
 * Householder, R(i,i) >= 0 either way), and the RandSVD /
 * Nystrom tail evd_from_gram_factor (proj/src/sketch.cpp:27-33, :191-197):
 * from the tall factor Wt (n x l, device, unchanged) the basis Q_W U (device
 * n x l, may be NULL) and eigenvalues S^2 - shift (floored at 0 if floor0). */
int sdv_thin_qr_dev(sdv_problem* p, int64_t n, int64_t l, double* y_dev, double* r, int* ndef);
int sdv_evd_from_tall_dev(sdv_problem* p, int64_t n, int64_t l, double* wt_dev, double shift, int floor0,
                          double* basis_dev, double* eig);
/* Nystrom tail (nystrom_assemble, proj/src/sketch.cpp:162-200) from device
 * Omega and Y = H Omega (n x l each): basis (device n x l, may be NULL) and
 * eigenvalues max(0, sigma^2 - nu). */
int sdv_nystrom_assemble_dev(sdv_problem* p, int64_t n, int64_t l, const double* omega_dev, const double* y_dev,
                             double* basis_dev, double* eig);

/* Sketch of the misfit Hessian at trajectory t (randsvd_sketch,
 * nystrom_sketch, singleview_sketch, lanczos_sketch; proj/src/sketch.cpp).
 * eig: rank values; basis: n x rank (may be NULL);
 * counts = {tlm_applies, adj_applies, final_rank}. Lanczos starts from a
 * gaussian_vector(n, seed). */
int sdv_sketch(sdv_traj* t, int method, int rank, int rank2, uint64_t seed, double* eig, double* basis,
               int64_t counts[3]);

/* lanczos_sketch(h, rank, start) (proj/src/sketch.cpp:292-389) from a caller
 * vector start (host, n; nonzero), as first_iterate_study calls it with the
 * GN right-hand side (proj/src/harness.cpp:590-592). Same outputs as
 * sdv_sketch. */
int sdv_lanczos_sketch(sdv_traj* t, int rank, const double* start, double* eig, double* basis, int64_t counts[3]);

/* adaptive_randsvd / adaptive_nystrom / adaptive_singleview
 * (proj/src/sketch.cpp:402-564): start at rank, grow by growth while the
 * cond_estimate probe kappa_sk > eps_sketch, capped at max_rank (rank2: the
 * SingleView adjoint width cap, <= 0 for 2 max_rank + 1). eig/basis sized
 * for max_rank; counts = {tlm, adj, final_rank, probes, tolerance_met};
 * kappa (may be NULL) receives the kappa_sk history, up to max_kappa values. */
int sdv_sketch_adaptive(sdv_traj* t, int method, int rank, int growth, int max_rank, int rank2, double eps_sketch,
                        uint64_t seed, double* eig, double* basis, int64_t counts[5], double* kappa, int max_kappa);

/* cond_estimate (proj/src/sketch.cpp:391-400): kappa of (I + H)(I + H_hat)^{-1}
 * from one seeded probe, H_hat = (basis, eig) of rank l. */
int sdv_cond_estimate(sdv_traj* t, int64_t l, const double* basis, const double* eig, uint64_t seed, double* kappa);

/* pcg_solve (proj/src/linalg.cpp:52-106) on (I + H) x = rhs at trajectory t,
 * preconditioned by woodbury_apply with (basis, eig) when l > 0.
 * info = {iterations, converged}. */
int sdv_pcg_solve(sdv_traj* t, const double* rhs, int64_t l, const double* basis, const double* eig, double tol,
                  int max_iter, double* x, int info[2]);

/* gn_solve (proj/src/fourdvar.cpp:213-422). */
typedef struct {
  int mode;           /* SDV_MODE_* */
  int method;         /* SDV_SKETCH_* */
  int rank, rank2, growth, max_rank;
  double eps_sketch, eps_reuse;
  uint64_t seed;
  double grad_tol, pcg_tol;
  int max_gn_iters, pcg_max_iter;
} sdv_gn_config;
/* log: max_log records of 16 doubles {k, cost, grad_inf_norm, step, pcg_iters,
 * ls_trials, pcg_converged, sketch_recomputed, final_rank, kappa_sk, kappa_re,
 * fwd, tlm, adj, offline_tlm, offline_adj}; summary = {final_cost,
 * final_grad_inf_norm, total_pcg, converged, line_search_failed};
 * eig0: first sketch's eigenvalues (max_eig entries, NaN padded). */
int sdv_gn_solve(sdv_problem* p, const sdv_gn_config* cfg, double* analysis, double* log, int max_log, int* n_iters,
                 double summary[5], double* eig0, int max_eig);

/* mix_seed / gaussian_matrix (proj/src/rng.cpp:9-44), bit-exact host RNG
 * used for every test block (n x l column-major). */
uint64_t sdv_mix_seed(uint64_t seed, uint64_t stream);
int sdv_gaussian_matrix(int64_t n, int64_t l, uint64_t seed, double* out);

/* Memory helpers (device-resident inputs for benchmarking, pinned host). */
int sdv_dev_alloc(size_t bytes, void** ptr);
int sdv_dev_free(void* ptr);
int sdv_host_alloc(size_t bytes, void** ptr);
int sdv_host_free(void* ptr);
int sdv_memcpy_htod(void* dst_dev, const void* src, size_t bytes);
int sdv_memcpy_dtoh(void* dst, const void* src_dev, size_t bytes);
int sdv_synchronize(sdv_problem* p);
/* CUDA events on the problem's stream (device timing for benchmarks). */
int sdv_event_create(void** ev);
int sdv_event_destroy(void* ev);
int sdv_event_record(sdv_problem* p, void* ev);
int sdv_event_elapsed_ms(void* start, void* stop, float* ms);
/* Per-kernel timing probe: runs `stages` TLM stages of a BVE block sweep
 * (group of s vectors) with events around every launch; returns the mean
 * duration of the fused stage kernel and of the column-FFT kernel (ms). */
int sdv_probe_stage_kernels(sdv_traj* t, int s, int stages, float* ms_stage, float* ms_col);
/* The same for `stages` adjoint RK stages (periodic BVE): mean duration of the
 * fused ADJ stage kernel and of the carry / column pass before it (ms). */
int sdv_probe_adj_stage_kernels(sdv_traj* t, int s, int stages, float* ms_stage, float* ms_col);

#ifdef __cplusplus
}
#endif

#endif /* SDV_H_ */

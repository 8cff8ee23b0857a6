// Device linear-algebra primitives for the sketch / PCG / Woodbury layer.
// All reductions are deterministic (fixed grid, fixed-order tree).
#pragma once

#include <atomic>

#include "common.cuh"

namespace sdv {

// Number of kernel launches issued by this library (for bench gpu_launches),
// process-wide (atomic) and per calling thread (graph capture subtracts the
// launches it only recorded, without racing other threads' counts).
extern std::atomic<unsigned long long> g_launches;
extern thread_local unsigned long long t_launches;
inline void count_launch(unsigned long long k = 1) {
  g_launches.fetch_add(k, std::memory_order_relaxed);
  t_launches += k;
}

// Which kernel variant the sweeps took (sdv_path_counts): one count per
// host-side launch decision (a CUDA-graph replay is counted once, at capture).
enum KernelPath {
  kPathBveStageFused = 0,  // stage_kernel<N, TLM/ADJ, 8, stage, fused> (the hot path)
  kPathBveCarry,           // carry_kernel<N> (tile carries of the fused Poisson path)
  kPathBveStageLite,       // fused kernel as a plain stage on 2-row tiles (small blocks)
  kPathBveStagePlain,      // unfused stage_kernel (8- or 2-row tiles, NL forward)
  kPathBveColSolve,        // col_solve_kernel (recurrence column pass)
  kPathBveColFft,          // col_kernel (y-FFT column pass)
  kPathBurgers,            // whole-sweep Burgers kernels
  kPathCount
};
extern std::atomic<unsigned long long> g_path[kPathCount];
inline void count_path(int p, unsigned long long k = 1) { g_path[p].fetch_add(k, std::memory_order_relaxed); }
const char* path_name(int p);

// Device workspaces owned by one CUDA stream (reduction partials, QR
// scratch, a host-readable dot result). Thread-safe lookup; released when the
// owning Problem destroys the stream.
struct StreamWork {
  DevBuf<double> partial, qr_house, qr_w, qr_scal, qr_q, qr_sgn, dot;
};
StreamWork& stream_work(cudaStream_t st);
void release_stream_work(cudaStream_t st);

// out[0] = sum_i a[i] * b[i] (device scalar), deterministic.
void dev_dot(const double* a, const double* b, long long n, double* out, cudaStream_t st);
// Column dots: out[j] = sum_i a[i + j*lda] * b[i + j*ldb], j < ncols.
void dev_coldots(const double* a, long long lda, const double* b, long long ldb, long long n, int ncols, double* out,
                 cudaStream_t st);
// Fused PCG steps (dots bitwise equal to dev_dot): q <- p + q and *pq = <p, q>;
// alpha = rz / *pq (device), x <- x + alpha p, r <- r - alpha q, *rr = <r, r>.
void dev_pcg_q(long long n, const double* p, double* q, double* pq, cudaStream_t st);
void dev_pcg_xr(long long n, double rz, const double* pq, const double* p, const double* q, double* x, double* r,
                double* rr, cudaStream_t st);
// y = alpha x + beta y   (alpha/beta host scalars)
void dev_axpby(long long n, double alpha, const double* x, double beta, double* y, cudaStream_t st);
// y = alpha x + beta y with alpha = (*num / *den) * sa (device scalars), used by PCG without host sync.
void dev_scale_copy(long long n, double a, const double* x, double* y, cudaStream_t st);
void dev_fill(long long n, double v, double* y, cudaStream_t st);
// C (k x l) = A^T B with A (n x k), B (n x l) column-major, leading dims n. Deterministic.
void dev_gemm_tn(long long n, int k, int l, const double* a, const double* b, double* c, cudaStream_t st);
// G (l x l) = A^T A on the fp64 tensor cores (mma.sync.m8n8k4.f64), l <= 128.
bool dev_gram_dmma_ok(int l);
void dev_gram_dmma(long long n, int l, const double* a, double* c, cudaStream_t st);
// C (n x l) = alpha * A (n x k) * B (k x l) + beta * C; B small, device, column-major (ldb = k).
void dev_gemm_nn_small(long long n, int k, int l, double alpha, const double* a, const double* b, double beta,
                       double* c, cudaStream_t st);
// Row-wise lower-triangular solve: for every row r of Y (n x l), x = L^{-1} y_r,
// stored as row r of X (n x l). L is l x l lower (device, column-major).
void dev_trsm_rows_lower(long long n, int l, const double* lmat, const double* y, double* x, cudaStream_t st);

// Householder thin QR on the device (same arithmetic as the reference's
// Eigen HouseholderQR + sign fix, proj/src/linalg.cpp:108-134).
// y (n x l) is overwritten by Q; r_host receives R (l x l, column-major).
// Returns the number of deficient columns.
int dev_householder_qr(long long n, int l, double* y, double* r_host, cudaStream_t st);
// CholQR2 on the DMMA Gram (l <= 128); returns -1 without touching y when the
// block is too ill-conditioned or deficient for it.
int dev_cholqr2(long long n, int l, double* y, double* r_host, cudaStream_t st);
// Thin QR used by the sketches: CholQR2 when it applies (default; SDV_QR=
// householder forces the Householder path), else Householder.
int dev_thin_qr(long long n, int l, double* y, double* r_host, cudaStream_t st);

}  // namespace sdv

// Device linear algebra for the sketch / PCG / Woodbury layer (sm_100a, fp64).
// Deterministic reductions: a fixed grid writes per-block partials that one
// block folds in a fixed order (warp-shuffle trees inside each block).
#include <string>

#include "linalg_kernels.cuh"
#include "hostla.hpp"

#include <cfloat>
#include <map>
#include <memory>
#include <mutex>
#include <cmath>

namespace sdv {

std::atomic<unsigned long long> g_launches{0};

// Per-stream device workspaces (a Problem owns its streams, so two problems
// driven from two threads never share a buffer; work on one stream is
// ordered, so reuse within a stream is safe).
namespace {
std::mutex g_work_mu;
std::map<cudaStream_t, std::unique_ptr<StreamWork>>& work_registry() {
  static auto* reg = new std::map<cudaStream_t, std::unique_ptr<StreamWork>>();  // outlives static dtors
  return *reg;
}
}  // namespace
StreamWork& stream_work(cudaStream_t st) {
  std::lock_guard<std::mutex> l(g_work_mu);
  auto& w = work_registry()[st];
  if (!w) w = std::make_unique<StreamWork>();
  return *w;
}
void release_stream_work(cudaStream_t st) {
  std::unique_ptr<StreamWork> dead;
  {
    std::lock_guard<std::mutex> l(g_work_mu);
    auto it = work_registry().find(st);
    if (it == work_registry().end()) return;
    dead = std::move(it->second);
    work_registry().erase(it);
  }
}
thread_local unsigned long long t_launches = 0;
std::atomic<unsigned long long> g_path[kPathCount];
const char* path_name(int p) {
  static const char* const names[kPathCount] = {"bve_stage_fused", "bve_carry",     "bve_stage_lite", "bve_stage_plain",
                                                "bve_col_solve",   "bve_col_fft",   "burgers_sweep"};
  return p >= 0 && p < kPathCount ? names[p] : nullptr;
}

namespace {
constexpr int kRedBlocks = 296;  // 2 CTAs per SM on 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
template <int TH>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < TH / 32 ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

__global__ void __launch_bounds__(kRedThreads) dot_partial_kernel(const double* __restrict__ a,
                                                                  const double* __restrict__ b, long long n,
                                                                  double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(kRedThreads) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kRedThreads)
    s = fma(a[i], b[i], s);
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void __launch_bounds__(kRedThreads) sum_partials_kernel(const double* __restrict__ part, int np, int ncols,
                                                                   double* __restrict__ out) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += kRedThreads) s += part[static_cast<long long>(c) * np + i];
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) out[c] = s;
  (void)ncols;
}

// out[e] = sum_c part[c * ne + e], c in order (one thread per output element)
__global__ void sum_partials_t_kernel(const double* __restrict__ part, int np, int ne, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  double s = 0.0;
  for (int c = 0; c < np; ++c) s += part[static_cast<long long>(c) * ne + e];
  out[e] = s;
}

DevBuf<double>& partial_buf(size_t n, cudaStream_t st) {
  DevBuf<double>& buf = stream_work(st).partial;
  buf.ensure(n);
  return buf;
}

// ---- column dots over a column range: out[j] = sum_i a[i+j*lda] b[i+j*ldb]
__global__ void __launch_bounds__(kRedThreads) coldot_partial_kernel(const double* __restrict__ a, long long lda,
                                                                     const double* __restrict__ b, long long ldb,
                                                                     long long n, int nchunks,
                                                                     double* __restrict__ part) {
  __shared__ double sh[32];
  const int col = blockIdx.y;
  const long long chunk = (n + nchunks - 1) / nchunks;
  const long long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  const double* ac = a + col * lda;
  const double* bc = b + col * ldb;
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += kRedThreads) s = fma(ac[i], bc[i], s);
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[static_cast<long long>(col) * nchunks + blockIdx.x] = s;
}

// ---- fused PCG updates (proj/src/linalg.cpp:52-106). Same grid, grid-stride
// partition and fma order as dot_partial_kernel, so every dot equals dev_dot's
// bit for bit; the axpy arithmetic equals axpby_kernel's.
// q <- p + q; part <- partial sums of <p, q>
__global__ void __launch_bounds__(kRedThreads) pcg_q_kernel(long long n, const double* __restrict__ p,
                                                            double* __restrict__ q, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(kRedThreads) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kRedThreads) {
    const double pi = p[i];
    const double qi = fma(1.0, pi, 1.0 * q[i]);
    q[i] = qi;
    s = fma(pi, qi, s);
  }
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// alpha = rz / *pq; x <- x + alpha p; r <- r - alpha q; part <- partial sums of <r, r>
__global__ void __launch_bounds__(kRedThreads) pcg_xr_kernel(long long n, double rz, const double* __restrict__ pq,
                                                             const double* __restrict__ p, const double* __restrict__ q,
                                                             double* __restrict__ x, double* __restrict__ r,
                                                             double* __restrict__ part) {
  __shared__ double sh[32];
  const double alpha = rz / *pq;
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(kRedThreads) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kRedThreads) {
    x[i] = fma(alpha, p[i], 1.0 * x[i]);
    const double ri = fma(-alpha, q[i], 1.0 * r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void axpby_kernel(long long n, double alpha, const double* __restrict__ x, double beta,
                             double* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = beta == 0.0 ? alpha * x[i] : fma(alpha, x[i], beta * y[i]);
}
__global__ void fill_kernel(long long n, double v, double* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = v;
}

// ---- C = A^T B, tiles of 32x32 outputs per block over a row chunk.
constexpr int kGT = 32;
constexpr int kGRows = 64;
__global__ void __launch_bounds__(256) gemm_tn_partial_kernel(long long n, int k, int l, const double* __restrict__ a,
                                                              const double* __restrict__ b, int nchunks,
                                                              double* __restrict__ part) {
  __shared__ double as[kGRows][kGT + 1];
  __shared__ double bs[kGRows][kGT + 1];
  const int ti = blockIdx.y * kGT, tj = blockIdx.z * kGT;
  const long long chunk = ((n + nchunks - 1) / nchunks + kGRows - 1) / kGRows * kGRows;
  const long long r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int tx = threadIdx.x % kGT, ty = threadIdx.x / kGT;  // ty in [0,8)
  double acc[4] = {0, 0, 0, 0};
  for (long long rb = r0; rb < r1; rb += kGRows) {
    for (int e = threadIdx.x; e < kGRows * kGT; e += 256) {
      const int rr = e % kGRows, cc = e / kGRows;
      const long long row = rb + rr;
      as[rr][cc] = (row < r1 && ti + cc < k) ? a[row + static_cast<long long>(ti + cc) * n] : 0.0;
      bs[rr][cc] = (row < r1 && tj + cc < l) ? b[row + static_cast<long long>(tj + cc) * n] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < kGRows; ++rr) {
      const double bv = bs[rr][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(as[rr][ty + 8 * q], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = ti + ty + 8 * q, j = tj + tx;
    if (i < k && j < l) part[(static_cast<long long>(j) * k + i) * nchunks + blockIdx.x] = acc[q];
  }
}

// ---- C = alpha A B + beta C, A tall (n x k), B small (k x l).
constexpr int kNNCols = 16;
__global__ void __launch_bounds__(256) gemm_nn_small_kernel(long long n, int k, int l, double alpha,
                                                            const double* __restrict__ a, const double* __restrict__ b,
                                                            double beta, double* __restrict__ c) {
  extern __shared__ double bsh[];  // k x kNNCols
  const int c0 = blockIdx.y * kNNCols;
  const int nc = min(kNNCols, l - c0);
  for (int e = threadIdx.x; e < k * kNNCols; e += blockDim.x) {
    const int kk = e % k, cc = e / k;
    bsh[e] = cc < nc ? b[kk + static_cast<long long>(c0 + cc) * k] : 0.0;
  }
  __syncthreads();
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  double acc[kNNCols];
#pragma unroll
  for (int q = 0; q < kNNCols; ++q) acc[q] = 0.0;
  for (int kk = 0; kk < k; ++kk) {
    const double av = a[r + static_cast<long long>(kk) * n];
#pragma unroll
    for (int q = 0; q < kNNCols; ++q) acc[q] = fma(av, bsh[kk + q * k], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < kNNCols; ++q)
    if (q < nc) {
      double* cp = c + r + static_cast<long long>(c0 + q) * n;
      *cp = beta == 0.0 ? alpha * acc[q] : fma(alpha, acc[q], beta * *cp);
    }
}

// ---- row-wise lower triangular solve
__global__ void __launch_bounds__(64) trsm_rows_lower_kernel(long long n, int l, const double* __restrict__ lm,
                                                             const double* __restrict__ y, double* __restrict__ x) {
  extern __shared__ double xs[];  // 64 x (l+1)
  const long long r = blockIdx.x * 64LL + threadIdx.x;
  if (r >= n) return;
  double* xr = xs + threadIdx.x * (l + 1);
  for (int i = 0; i < l; ++i) {
    double s = y[r + static_cast<long long>(i) * n];
    for (int kk = 0; kk < i; ++kk) s -= __ldg(lm + i + static_cast<long long>(kk) * l) * xr[kk];
    const double v = s / __ldg(lm + i + static_cast<long long>(i) * l);
    xr[i] = v;
    x[r + static_cast<long long>(i) * n] = v;
  }
}

// ---- fp64 tensor-core (DMMA, mma.sync.m8n8k4.f64) Gram of a tall block -----
// G = A^T A for A n x l column-major (l <= 8 LT). Each CTA accumulates a row
// chunk: 32-row slabs of A are staged in shared memory as [col][row] with a
// stride of 36 doubles (the 8-byte fragment loads of a half-warp hit 16
// distinct bank pairs), and warp w owns the upper-triangle 8 x 8 output tiles
// of tile rows w, w + 8, ...: per 4-row k-step it loads one A fragment per
// tile row and one B fragment per tile column and issues one DMMA per tile.
// Partials [chunk][l][l] are reduced in a fixed order (deterministic).
constexpr int kDmmaRows = 32, kDmmaStride = 36;
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
template <int LT>
__global__ void __launch_bounds__(256) gram_dmma_kernel(long long n, int l, const double* __restrict__ a,
                                                        long long rows_per_cta, double* __restrict__ part) {
  constexpr int LP = 8 * LT;
  constexpr int TPW = (LT + 7) / 8;  // tile rows per warp
  __shared__ __align__(16) double sa[LP * kDmmaStride];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r0 = blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
  double acc[TPW][LT][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u)
#pragma unroll
    for (int tj = 0; tj < LT; ++tj) acc[u][tj][0] = acc[u][tj][1] = 0.0;
  const int fr = lane % 4, fc = lane / 4;  // fragment row (k) and column (tile-local)
  for (long long rb = r0; rb < r1; rb += kDmmaRows) {
    __syncthreads();
    for (int e = threadIdx.x; e < LP * kDmmaRows; e += 256) {
      const int c = e / kDmmaRows, r = e % kDmmaRows;
      const long long row = rb + r;
      sa[c * kDmmaStride + r] = (c < l && row < r1) ? a[row + static_cast<long long>(c) * n] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < kDmmaRows; k0 += 4) {
      double bf[LT];
#pragma unroll
      for (int tj = 0; tj < LT; ++tj) bf[tj] = sa[(8 * tj + fc) * kDmmaStride + k0 + fr];
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        const int ti = warp + 8 * u;
        if (ti < LT) {
          const double af = sa[(8 * ti + fc) * kDmmaStride + k0 + fr];  // A fragment of tile row ti
#pragma unroll
          for (int tj = 0; tj < LT; ++tj)
            if (tj >= ti) dmma_884(acc[u][tj][0], acc[u][tj][1], af, bf[tj]);
        }
      }
    }
  }
  double* out = part + static_cast<long long>(blockIdx.x) * l * l;
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int ti = warp + 8 * u;
    if (ti >= LT) continue;
#pragma unroll
    for (int tj = 0; tj < LT; ++tj) {
      if (tj < ti) continue;
      const int i = 8 * ti + fc;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 8 * tj + 2 * fr + h;
        if (i < l && j < l) {
          out[i + static_cast<long long>(j) * l] = acc[u][tj][h];
          out[j + static_cast<long long>(i) * l] = acc[u][tj][h];
        }
      }
    }
  }
}

// ---- Householder QR pieces ---------------------------------------------------
struct House {
  double beta, tau, inv;
};
__global__ void house_scalar_kernel(const double* __restrict__ c0p, const double* __restrict__ tailp,
                                    House* __restrict__ h) {
  const double c0 = *c0p, tail = *tailp;
  House o;
  if (tail <= DBL_MIN) {
    o.tau = 0.0;
    o.beta = c0;
    o.inv = 0.0;
  } else {
    double beta = sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    o.beta = beta;
    o.inv = 1.0 / (c0 - beta);
    o.tau = (beta - c0) / beta;
  }
  *h = o;
}
// Column j: y[j] = beta, y[i>j] *= inv (or 0 when tau == 0).
__global__ void house_scale_kernel(long long n, int j, double* __restrict__ y, const House* __restrict__ h) {
  const House hh = *h;
  double* col = y + static_cast<long long>(j) * n;
  for (long long i = j + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i == j) col[i] = hh.beta;
    else col[i] = hh.tau == 0.0 ? 0.0 : col[i] * hh.inv;
  }
}
// partials of sum_{i>j} v_i t[i, c] for columns c in [c0, c1) of t (ld n).
__global__ void __launch_bounds__(kRedThreads) house_dot_partial_kernel(long long n, int j, const double* __restrict__ v,
                                                                        const double* __restrict__ t, int c0,
                                                                        int nchunks, double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = c0 + blockIdx.y;
  const long long len = n - j - 1;
  const long long chunk = (len + nchunks - 1) / nchunks;
  const long long i0 = j + 1 + blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  const double* tc = t + static_cast<long long>(c) * n;
  double s = 0.0;
  for (long long i = i0 + threadIdx.x; i < i1; i += kRedThreads) s = fma(v[i], tc[i], s);
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[static_cast<long long>(blockIdx.y) * nchunks + blockIdx.x] = s;
}
// w_c = t[j,c] + sum partials; stored scaled by tau.
__global__ void __launch_bounds__(kRedThreads) house_dot_final_kernel(int j, long long n, const double* __restrict__ t,
                                                                      int c0, int nchunks, const double* __restrict__ part,
                                                                      const House* __restrict__ h,
                                                                      double* __restrict__ w) {
  __shared__ double sh[32];
  const int c = c0 + blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nchunks; i += kRedThreads) s += part[static_cast<long long>(blockIdx.x) * nchunks + i];
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) w[blockIdx.x] = (t[j + static_cast<long long>(c) * n] + s) * h->tau;
}
// t[i, c] -= w_c v_i for i >= j (v_j = 1), c in [c0, c0+nc).
__global__ void house_update_kernel(long long n, int j, const double* __restrict__ v, double* __restrict__ t, int c0,
                                    int nc, const double* __restrict__ w) {
  const int c = c0 + blockIdx.y;
  const double wc = w[blockIdx.y];
  double* tc = t + static_cast<long long>(c) * n;
  for (long long i = j + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    tc[i] -= wc * (i == j ? 1.0 : v[i]);
  (void)nc;
}
__global__ void eye_kernel(long long n, int l, double* __restrict__ q) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n * l;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % n, c = e / n;
    q[e] = (i == c) ? 1.0 : 0.0;
  }
}
__global__ void col_sign_kernel(long long n, int l, const double* __restrict__ sgn, double* __restrict__ q) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n * l;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    q[e] *= sgn[e / n];
}
__global__ void sumsq_tail_partial_kernel(long long n, int j, const double* __restrict__ y, double* __restrict__ part) {
  __shared__ double sh[32];
  const double* col = y + static_cast<long long>(j) * n;
  double s = 0.0;
  for (long long i = j + 1 + blockIdx.x * static_cast<long long>(kRedThreads) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * kRedThreads)
    s = fma(col[i], col[i], s);
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int grid_for(long long n, int th = 256) {
  long long g = (n + th - 1) / th;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}
}  // namespace

void dev_dot(const double* a, const double* b, long long n, double* out, cudaStream_t st) {
  DevBuf<double>& part = partial_buf(kRedBlocks, st);
  dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, n, part.get());
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(part.get(), kRedBlocks, 1, out);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}

void dev_coldots(const double* a, long long lda, const double* b, long long ldb, long long n, int ncols, double* out,
                 cudaStream_t st) {
  if (ncols <= 0) return;
  const int nchunks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, n / 4096)));
  DevBuf<double>& part = partial_buf(static_cast<size_t>(nchunks) * ncols, st);
  coldot_partial_kernel<<<dim3(nchunks, ncols), kRedThreads, 0, st>>>(a, lda, b, ldb, n, nchunks, part.get());
  sum_partials_kernel<<<ncols, kRedThreads, 0, st>>>(part.get(), nchunks, ncols, out);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}

void dev_pcg_q(long long n, const double* p, double* q, double* pq, cudaStream_t st) {
  DevBuf<double>& part = partial_buf(kRedBlocks, st);
  pcg_q_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, p, q, part.get());
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(part.get(), kRedBlocks, 1, pq);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}
void dev_pcg_xr(long long n, double rz, const double* pq, const double* p, const double* q, double* x, double* r,
                double* rr, cudaStream_t st) {
  DevBuf<double>& part = partial_buf(kRedBlocks, st);
  pcg_xr_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, rz, pq, p, q, x, r, part.get());
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(part.get(), kRedBlocks, 1, rr);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}
void dev_axpby(long long n, double alpha, const double* x, double beta, double* y, cudaStream_t st) {
  axpby_kernel<<<grid_for(n), 256, 0, st>>>(n, alpha, x, beta, y);
  count_launch();
  SDV_LAUNCH_CHECK();
}
void dev_scale_copy(long long n, double a, const double* x, double* y, cudaStream_t st) {
  dev_axpby(n, a, x, 0.0, y, st);
}
void dev_fill(long long n, double v, double* y, cudaStream_t st) {
  fill_kernel<<<grid_for(n), 256, 0, st>>>(n, v, y);
  count_launch();
  SDV_LAUNCH_CHECK();
}

void dev_gemm_tn(long long n, int k, int l, const double* a, const double* b, double* c, cudaStream_t st) {
  if (k <= 0 || l <= 0) return;
  const int tk = (k + kGT - 1) / kGT, tl = (l + kGT - 1) / kGT;
  int nchunks = static_cast<int>(std::max<long long>(1, std::min<long long>((n + 4095) / 4096, 592 / (tk * tl) + 1)));
  DevBuf<double>& part = partial_buf(static_cast<size_t>(nchunks) * k * l, st);
  gemm_tn_partial_kernel<<<dim3(nchunks, tk, tl), 256, 0, st>>>(n, k, l, a, b, nchunks, part.get());
  sum_partials_kernel<<<k * l, kRedThreads, 0, st>>>(part.get(), nchunks, k * l, c);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}

void dev_gemm_nn_small(long long n, int k, int l, double alpha, const double* a, const double* b, double beta,
                       double* c, cudaStream_t st) {
  if (l <= 0 || n <= 0) return;
  if (k <= 0) {
    for (int j = 0; j < l; ++j) dev_axpby(n, 0.0, c + static_cast<long long>(j) * n, beta, c + static_cast<long long>(j) * n, st);
    return;
  }
  const size_t smem = sizeof(double) * k * kNNCols;
  if (smem > 48 * 1024)
    SDV_CUDA(cudaFuncSetAttribute(gemm_nn_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  gemm_nn_small_kernel<<<dim3(ceil_div(n, 256), ceil_div(l, kNNCols)), 256, smem, st>>>(n, k, l, alpha, a, b, beta,
                                                                                        c);
  count_launch();
  SDV_LAUNCH_CHECK();
}

void dev_trsm_rows_lower(long long n, int l, const double* lmat, const double* y, double* x, cudaStream_t st) {
  const size_t smem = sizeof(double) * 64 * (l + 1);
  if (smem > 48 * 1024)
    SDV_CUDA(cudaFuncSetAttribute(trsm_rows_lower_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  trsm_rows_lower_kernel<<<ceil_div(n, 64), 64, smem, st>>>(n, l, lmat, y, x);
  count_launch();
  SDV_LAUNCH_CHECK();
}

namespace {
template <int LT>
void gram_dmma_launch(long long n, int l, const double* a, double* c, cudaStream_t st) {
  // ~2 CTAs per SM, each over a contiguous chunk of 32-row slabs
  const long long slabs = (n + kDmmaRows - 1) / kDmmaRows;
  const int nchunks = static_cast<int>(std::max<long long>(1, std::min<long long>(296, slabs)));
  const long long rows = ((slabs + nchunks - 1) / nchunks) * kDmmaRows;
  const int used = static_cast<int>((n + rows - 1) / rows);
  DevBuf<double>& part = partial_buf(static_cast<size_t>(used) * l * l, st);
  gram_dmma_kernel<LT><<<used, 256, 0, st>>>(n, l, a, rows, part.get());
  sum_partials_t_kernel<<<ceil_div(static_cast<long long>(l) * l, 256), 256, 0, st>>>(part.get(), used, l * l, c);
  count_launch(2);
  SDV_LAUNCH_CHECK();
}
}  // namespace

bool dev_gram_dmma_ok(int l) { return l >= 1 && l <= 128; }

void dev_gram_dmma(long long n, int l, const double* a, double* c, cudaStream_t st) {
  if (!dev_gram_dmma_ok(l)) throw std::invalid_argument("dev_gram_dmma: need 1 <= l <= 128");
  const int lt = (l + 7) / 8;
  if (lt <= 4) gram_dmma_launch<4>(n, l, a, c, st);
  else if (lt <= 8) gram_dmma_launch<8>(n, l, a, c, st);
  else if (lt <= 12) gram_dmma_launch<12>(n, l, a, c, st);
  else gram_dmma_launch<16>(n, l, a, c, st);
}

int dev_householder_qr(long long n, int l, double* y, double* r_host, cudaStream_t st) {
  if (n < l) throw std::invalid_argument("thin_qr: need rows >= cols");
  StreamWork& ws = stream_work(st);
  DevBuf<double>& hs = ws.qr_house;  // House records (3 doubles each)
  DevBuf<double>& w = ws.qr_w;
  DevBuf<double>& scal = ws.qr_scal;
  DevBuf<double>& qbuf = ws.qr_q;
  DevBuf<double>& sgn = ws.qr_sgn;
  hs.ensure(static_cast<size_t>(3) * l);
  w.ensure(static_cast<size_t>(l));
  scal.ensure(2);
  qbuf.ensure(static_cast<size_t>(n) * l);
  sgn.ensure(static_cast<size_t>(l));
  const int nchunks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, n / 8192)));
  DevBuf<double> part(static_cast<size_t>(std::max(kRedBlocks, nchunks * l)));
  for (int j = 0; j < l; ++j) {
    // tail norm^2 and c0
    sumsq_tail_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, j, y, part.get());
    sum_partials_kernel<<<1, kRedThreads, 0, st>>>(part.get(), kRedBlocks, 1, scal.get() + 1);
    house_scalar_kernel<<<1, 1, 0, st>>>(y + j + static_cast<long long>(j) * n, scal.get() + 1, reinterpret_cast<House*>(hs.get()) + j);
    house_scale_kernel<<<grid_for(n - j), 256, 0, st>>>(n, j, y, reinterpret_cast<House*>(hs.get()) + j);
    count_launch(4);
    const int nc = l - j - 1;
    if (nc > 0) {
      const double* v = y + static_cast<long long>(j) * n;
      house_dot_partial_kernel<<<dim3(nchunks, nc), kRedThreads, 0, st>>>(n, j, v, y, j + 1, nchunks, part.get());
      house_dot_final_kernel<<<nc, kRedThreads, 0, st>>>(j, n, y, j + 1, nchunks, part.get(), reinterpret_cast<House*>(hs.get()) + j, w.get());
      house_update_kernel<<<dim3(grid_for(n - j) / 4 + 1, nc), 256, 0, st>>>(n, j, v, y, j + 1, nc, w.get());
      count_launch(3);
    }
    SDV_LAUNCH_CHECK();
  }
  // R (upper triangle of the factored block) to the host.
  std::vector<double> rr(static_cast<size_t>(l) * l);
  SDV_CUDA(cudaMemcpy2DAsync(rr.data(), sizeof(double) * l, y, sizeof(double) * n, sizeof(double) * l, l,
                             cudaMemcpyDeviceToHost, st));
  // Q = H_0 ... H_{l-1} [I; 0]
  double* q = qbuf.get();
  eye_kernel<<<grid_for(n * l), 256, 0, st>>>(n, l, q);
  count_launch();
  for (int j = l - 1; j >= 0; --j) {
    const double* v = y + static_cast<long long>(j) * n;
    const int nc = l - j;
    house_dot_partial_kernel<<<dim3(nchunks, nc), kRedThreads, 0, st>>>(n, j, v, q, j, nchunks, part.get());
    house_dot_final_kernel<<<nc, kRedThreads, 0, st>>>(j, n, q, j, nchunks, part.get(), reinterpret_cast<House*>(hs.get()) + j, w.get());
    house_update_kernel<<<dim3(grid_for(n - j) / 4 + 1, nc), 256, 0, st>>>(n, j, v, q, j, nc, w.get());
    count_launch(3);
  }
  SDV_LAUNCH_CHECK();
  SDV_CUDA(cudaStreamSynchronize(st));
  std::vector<double> sg(static_cast<size_t>(l), 1.0);
  for (int j = 0; j < l; ++j) {
    for (int i = 0; i < l; ++i) r_host[i + static_cast<size_t>(j) * l] = i <= j ? rr[i + static_cast<size_t>(j) * l] : 0.0;
  }
  for (int i = 0; i < l; ++i)
    if (r_host[i + static_cast<size_t>(i) * l] < 0.0) {
      sg[i] = -1.0;
      for (int j = 0; j < l; ++j) r_host[i + static_cast<size_t>(j) * l] = -r_host[i + static_cast<size_t>(j) * l];
    }
  SDV_CUDA(cudaMemcpyAsync(sgn.get(), sg.data(), sizeof(double) * l, cudaMemcpyHostToDevice, st));
  col_sign_kernel<<<grid_for(n * l), 256, 0, st>>>(n, l, sgn.get(), q);
  count_launch();
  SDV_CUDA(cudaMemcpyAsync(y, q, sizeof(double) * n * l, cudaMemcpyDeviceToDevice, st));
  SDV_CUDA(cudaStreamSynchronize(st));
  double dmax = 0.0;
  for (int i = 0; i < l; ++i) dmax = std::max(dmax, std::abs(r_host[i + static_cast<size_t>(i) * l]));
  const double tol = static_cast<double>(std::max<long long>(n, l)) * DBL_EPSILON * dmax;
  int ndef = 0;
  for (int i = 0; i < l; ++i)
    if (std::abs(r_host[i + static_cast<size_t>(i) * l]) <= tol) ++ndef;
  return ndef;
}

// ---- CholQR2 on the fp64 tensor cores ------------------------------------------
// Y = Q R by two Cholesky-QR passes (G = Y^T Y on DMMA, R = chol(G)^T on the
// host, Q = Y R^{-1} as a tall x small product), R = R2 R1 with R(i,i) > 0 (the
// reference's sign convention, proj/src/linalg.cpp:108-134). Declines (returns
// -1, Y untouched) when a Cholesky factor breaks down or its diagonal spans
// more than 1e5 (kappa(Y) beyond what two passes restore to orthogonality):
// the caller then runs the Householder path, which also handles deficiency.
namespace {
bool chol_upper(const std::vector<double>& g, int l, std::vector<double>& r) {
  HMat a(l, l);
  for (int j = 0; j < l; ++j)
    for (int i = 0; i < l; ++i) a(i, j) = 0.5 * (g[i + static_cast<size_t>(j) * l] + g[j + static_cast<size_t>(i) * l]);
  HMat lo;
  try {
    lo = hcholesky(a);
  } catch (const std::exception&) {
    return false;
  }
  double dmin = lo(0, 0), dmax = lo(0, 0);
  for (int i = 0; i < l; ++i) {
    dmin = std::min(dmin, lo(i, i));
    dmax = std::max(dmax, lo(i, i));
  }
  if (!(dmin > 1e-5 * dmax)) return false;
  r.assign(static_cast<size_t>(l) * l, 0.0);
  for (int j = 0; j < l; ++j)
    for (int i = 0; i <= j; ++i) r[i + static_cast<size_t>(j) * l] = lo(j, i);
  return true;
}
// inverse of an upper-triangular l x l (column-major) by back substitution
std::vector<double> upper_inv(const std::vector<double>& r, int l) {
  std::vector<double> x(static_cast<size_t>(l) * l, 0.0);
  for (int j = 0; j < l; ++j) {
    x[j + static_cast<size_t>(j) * l] = 1.0 / r[j + static_cast<size_t>(j) * l];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += r[i + static_cast<size_t>(k) * l] * x[k + static_cast<size_t>(j) * l];
      x[i + static_cast<size_t>(j) * l] = -s / r[i + static_cast<size_t>(i) * l];
    }
  }
  return x;
}
}  // namespace

int dev_cholqr2(long long n, int l, double* y, double* r_host, cudaStream_t st) {
  if (n < l) throw std::invalid_argument("thin_qr: need rows >= cols");
  if (!dev_gram_dmma_ok(l)) return -1;
  StreamWork& ws = stream_work(st);
  DevBuf<double>& qbuf = ws.qr_q;
  DevBuf<double>& small = ws.qr_w;
  qbuf.ensure(static_cast<size_t>(n) * l);
  small.ensure(static_cast<size_t>(l) * l);
  std::vector<double> g(static_cast<size_t>(l) * l), r1, r2;
  auto gram_host = [&](const double* a) {
    dev_gram_dmma(n, l, a, small.get(), st);
    SDV_CUDA(cudaMemcpyAsync(g.data(), small.get(), sizeof(double) * l * l, cudaMemcpyDeviceToHost, st));
    SDV_CUDA(cudaStreamSynchronize(st));
  };
  gram_host(y);
  if (!chol_upper(g, l, r1)) return -1;
  std::vector<double> inv = upper_inv(r1, l);
  SDV_CUDA(cudaMemcpyAsync(small.get(), inv.data(), sizeof(double) * l * l, cudaMemcpyHostToDevice, st));
  dev_gemm_nn_small(n, l, l, 1.0, y, small.get(), 0.0, qbuf.get(), st);  // Q1 = Y R1^{-1}
  gram_host(qbuf.get());
  if (!chol_upper(g, l, r2)) return -1;
  inv = upper_inv(r2, l);
  SDV_CUDA(cudaMemcpyAsync(small.get(), inv.data(), sizeof(double) * l * l, cudaMemcpyHostToDevice, st));
  dev_gemm_nn_small(n, l, l, 1.0, qbuf.get(), small.get(), 0.0, y, st);  // Q = Q1 R2^{-1}
  // R = R2 R1 (upper)
  for (int j = 0; j < l; ++j)
    for (int i = 0; i < l; ++i) {
      double acc = 0.0;
      for (int k = i; k <= j; ++k) acc += r2[i + static_cast<size_t>(k) * l] * r1[k + static_cast<size_t>(j) * l];
      r_host[i + static_cast<size_t>(j) * l] = i <= j ? acc : 0.0;
    }
  SDV_CUDA(cudaStreamSynchronize(st));
  return 0;  // full rank (a deficient Y would have declined)
}

int dev_thin_qr(long long n, int l, double* y, double* r_host, cudaStream_t st) {
  static const bool householder = [] {
    const char* e = std::getenv("SDV_QR");
    return e && std::string(e) == "householder";
  }();
  if (!householder) {
    const int nd = dev_cholqr2(n, l, y, r_host, st);
    if (nd >= 0) return nd;
  }
  return dev_householder_qr(n, l, y, r_host, st);
}

}  // namespace sdv

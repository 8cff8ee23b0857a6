// Batched fp64 barotropic-vorticity stage kernels (periodic n x n, Arakawa
// Jacobian, 5-point viscosity, spectral Poisson), sm_100a.
//
// Replaces the reference's per-vector CPU loops BVETrajectory::tlm_range/
// adj_range + jac/jac_adj + DirichletSolver2D::solve
// (/root/reference/proj/src/bve.cpp:138-211, proj/src/dirichlet.cpp:134-155)
// for the BASELINE.json periodic/RK4/Arakawa configs.
//
// Layout in HBM: a block of s fields is [s][n][n] (x fastest, index i + n*j,
// as the reference, proj/include/sketchdav/bve.hpp:20). "Row spectra" are
// [s][n][n/2] double2: the x-FFT of each row with the (real) k=0 and k=n/2
// coefficients packed into element 0 (re = X(0), im = X(n/2)).
//
// Every RK4 stage is two launches:
//   col kernel  : y-FFT of the row spectra, spectral multiply, inverse y-FFT;
//   stage kernel: inverse x-FFT of the T owned rows + 2 halo rows, the
//                 Arakawa/Laplacian stencils with the stored base stage fields,
//                 the RK4 (TLM/NL) or adjoint-RK4 (ADJ) update, and the forward
//                 x-FFT of the next stage's Poisson input for the owned rows.
#include "bve_kernels.cuh"
#include "fft.cuh"

#include <type_traits>

namespace sdv {

namespace {

template <int N>
struct RowCfg {
  static constexpr int kThreads = 256;
  static constexpr int kTeam = N / 4 < kThreads ? N / 4 : kThreads;
  static constexpr int kTeams = kThreads / kTeam;
};

// Packed half spectra of rows a, b -> full spectrum of z = a + i b.
template <int N>
__device__ __forceinline__ void unpack_pair(const double2* __restrict__ ra, const double2* __restrict__ rb, double2* z,
                                            int t, int nt) {
  for (int k = t; k < N / 2; k += nt) {
    const double2 a = ra[k], b = rb[k];
    if (k == 0) {
      z[0] = make_double2(a.x, b.x);
      z[N / 2] = make_double2(a.y, b.y);
    } else {
      z[k] = make_double2(a.x - b.y, a.y + b.x);
      z[N - k] = make_double2(a.x + b.y, b.x - a.y);
    }
  }
}
// Full spectrum Z of z = a + i b -> packed half spectra of a and b.
template <int N>
__device__ __forceinline__ void pack_pair(const double2* z, double2* __restrict__ ra, double2* __restrict__ rb, int t,
                                          int nt) {
  for (int k = t; k < N / 2; k += nt) {
    if (k == 0) {
      const double2 z0 = z[0], zn = z[N / 2];
      ra[0] = make_double2(z0.x, zn.x);
      rb[0] = make_double2(z0.y, zn.y);
    } else {
      const double2 zk = z[k], zm = z[N - k];
      ra[k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      rb[k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
  }
}

// Arakawa Jacobian J(a,b) at (x, row r) given 3x3 neighbourhoods
// a[dy][dx], b[dy][dx] with dy,dx in {0,1,2} <-> offsets {-1,0,+1}.
// Returns 12 h^2 J (the caller scales).
__device__ __forceinline__ double arakawa12(const double a[3][3], const double b[3][3]) {
  // J++
  const double jpp = (a[1][2] - a[1][0]) * (b[2][1] - b[0][1]) - (a[2][1] - a[0][1]) * (b[1][2] - b[1][0]);
  // J+x
  const double jpx = a[1][2] * (b[2][2] - b[0][2]) - a[1][0] * (b[2][0] - b[0][0]) -
                     a[2][1] * (b[2][2] - b[2][0]) + a[0][1] * (b[0][2] - b[0][0]);
  // Jx+
  const double jxp = b[2][1] * (a[2][2] - a[2][0]) - b[0][1] * (a[0][2] - a[0][0]) -
                     b[1][2] * (a[2][2] - a[0][2]) + b[1][0] * (a[2][0] - a[0][0]);
  return jpp + jpx + jxp;
}

template <int N>
__device__ __forceinline__ void load3x3_smem(const double* f, int r, int x, double o[3][3]) {
#pragma unroll
  for (int dy = 0; dy < 3; ++dy)
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) o[dy][dx] = f[(r + dy - 1) * N + ((x + dx - 1) & (N - 1))];
}
template <int N>
__device__ __forceinline__ void load3x3_glob(const double* __restrict__ f, int gy, int x, double o[3][3]) {
#pragma unroll
  for (int dy = 0; dy < 3; ++dy) {
    const double* row = f + static_cast<long long>((gy + dy - 1) & (N - 1)) * N;
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) o[dy][dx] = __ldg(row + ((x + dx - 1) & (N - 1)));
  }
}
__device__ __forceinline__ double lap5(const double o[3][3]) { return o[1][0] + o[1][2] + o[0][1] + o[2][1] - 4.0 * o[1][1]; }

}  // namespace

// ---------------------------------------------------------------- row FFTs --
template <int N>
__global__ void __launch_bounds__(256) row_fwd_kernel(const double* __restrict__ f, double2* __restrict__ s, const double2* __restrict__ tw) {
  using C = RowCfg<N>;
  extern __shared__ double2 sm[];
  const int team = threadIdx.x / C::kTeam, t = threadIdx.x % C::kTeam;
  const int pair = blockIdx.x * C::kTeams + team;
  const bool active = pair < N / 2;
  const long long v = blockIdx.y;
  double2* a = sm + team * 2 * N;
  double2* b = a + N;
  if (active) {
    const double* r0 = f + v * N * N + static_cast<long long>(2 * pair) * N;
    for (int x = t; x < N; x += C::kTeam) a[x] = make_double2(r0[x], r0[x + N]);
  }
  __syncthreads();
  double2* z = fft_team<N, false>(a, b, tw, t, C::kTeam, active);
  if (active) {
    double2* ra = s + v * N * (N / 2) + static_cast<long long>(2 * pair) * (N / 2);
    pack_pair<N>(z, ra, ra + N / 2, t, C::kTeam);
  }
}

template <int N>
__global__ void __launch_bounds__(256) row_inv_kernel(const double2* __restrict__ s, double* __restrict__ f, const double2* __restrict__ tw) {
  using C = RowCfg<N>;
  extern __shared__ double2 sm[];
  const int team = threadIdx.x / C::kTeam, t = threadIdx.x % C::kTeam;
  const int pair = blockIdx.x * C::kTeams + team;
  const bool active = pair < N / 2;
  const long long v = blockIdx.y;
  double2* a = sm + team * 2 * N;
  double2* b = a + N;
  if (active) {
    const double2* ra = s + v * N * (N / 2) + static_cast<long long>(2 * pair) * (N / 2);
    unpack_pair<N>(ra, ra + N / 2, a, t, C::kTeam);
  }
  __syncthreads();
  double2* z = fft_team<N, true>(a, b, tw, t, C::kTeam, active);
  if (active) {
    double* r0 = f + v * N * N + static_cast<long long>(2 * pair) * N;
    for (int x = t; x < N; x += C::kTeam) {
      const double2 q = z[x];
      r0[x] = q.x;
      r0[x + N] = q.y;
    }
  }
}

// ------------------------------------------------------------- column pass --
// y-FFT of CW adjacent kx columns, multiply by sym[kx*N + ky], inverse y-FFT.
// Column kx = 0 holds X(0) + i X(n/2) per row; both are real-input columns, so
// the multiplier is applied through the Hermitian split
//   Z'(ky) = (s0+sN)/2 Z(ky) + (s0-sN)/2 conj(Z(-ky)).
template <int N, int CW>
__global__ void __launch_bounds__(CW*(N / 4)) col_kernel(double2* __restrict__ s, const double* __restrict__ sym, const double2* __restrict__ tw) {
  constexpr int kTeam = N / 4;
  constexpr int kThreads = CW * kTeam;
  extern __shared__ double2 sm[];
  const int team = threadIdx.x / kTeam, t = threadIdx.x % kTeam;
  const int kx0 = blockIdx.x * CW;
  const long long v = blockIdx.y;
  double2* base = s + v * N * (N / 2) + kx0;
  for (int e = threadIdx.x; e < CW * N; e += kThreads) {
    const int y = e / CW, c = e % CW;
    sm[c * 2 * N + y] = base[static_cast<long long>(y) * (N / 2) + c];
  }
  __syncthreads();
  double2* a = sm + team * 2 * N;
  double2* b = a + N;
  double2* z = fft_team<N, false>(a, b, tw, t, kTeam, true);
  double2* o = (z == a) ? b : a;
  const int kx = kx0 + team;
  if (kx == 0) {
    const double* s0 = sym;
    const double* sn = sym + static_cast<long long>(N / 2) * N;
    for (int ky = t; ky < N; ky += kTeam) {
      const double p = 0.5 * (__ldg(s0 + ky) + __ldg(sn + ky)), m = 0.5 * (__ldg(s0 + ky) - __ldg(sn + ky));
      const double2 zk = z[ky], zm = z[(N - ky) & (N - 1)];
      o[ky] = make_double2(p * zk.x + m * zm.x, p * zk.y - m * zm.y);
    }
  } else {
    const double* sk = sym + static_cast<long long>(kx) * N;
    for (int ky = t; ky < N; ky += kTeam) {
      const double w = __ldg(sk + ky);
      o[ky] = make_double2(w * z[ky].x, w * z[ky].y);
    }
  }
  __syncthreads();
  double2* r = fft_team<N, true>(o, z, tw, t, kTeam, true);
  const int roff = static_cast<int>(r - a);  // 0 or N (same for every team)
  for (int e = threadIdx.x; e < CW * N; e += kThreads) {
    const int y = e / CW, c = e % CW;
    base[static_cast<long long>(y) * (N / 2) + c] = sm[c * 2 * N + roff + y];
  }
}

// --------------------------------------------------------- fused RK stage --
template <int N, int T, int MODE>
__global__ void __launch_bounds__(256) stage_kernel(StageArgs p) {
  using C = RowCfg<N>;
  constexpr int R = T + 2;        // rows incl. halo
  constexpr int PTS = T * N / 256;  // owned points per thread
  extern __shared__ double smd[];
  double* P = smd;                // R x N  inverse-FFT field
  double* X = P + R * N;          // R x N  stencil input
  double2* F = reinterpret_cast<double2*>(X + R * N);  // kTeams x 2N
  const int tid = threadIdx.x;
  const int team = tid / C::kTeam, t = tid % C::kTeam;
  const int y0 = blockIdx.x * T;
  const long long v = blockIdx.y;
  const long long off = v * N * N;
  const long long soff = v * N * (N / 2);
  const double2* tw = p.tw;
  double2* fa = F + team * 2 * N;
  double2* fb = fa + N;
  const bool has_prev = MODE != kModeAdj || (p.flags & kFlagHasPrev);
  const bool finish = MODE == kModeAdj && (p.flags & kFlagFinish);

  // Phase 1: inverse x-FFT of rows y0-1 .. y0+T (P field).
  if (has_prev) {
    constexpr int kPairs = R / 2;
    for (int base = 0; base < kPairs; base += C::kTeams) {
      const int pr = base + team;
      const bool act = pr < kPairs;
      if (act) {
        const int ga = (y0 - 1 + 2 * pr) & (N - 1), gb = (y0 + 2 * pr) & (N - 1);
        unpack_pair<N>(p.s_in + soff + static_cast<long long>(ga) * (N / 2),
                       p.s_in + soff + static_cast<long long>(gb) * (N / 2), fa, t, C::kTeam);
      }
      __syncthreads();
      const double2* z = fft_team<N, true>(fa, fb, tw, t, C::kTeam, act);
      if (act) {
        for (int x = t; x < N; x += C::kTeam) {
          const double2 q = z[x];
          P[(2 * pr) * N + x] = q.x;
          P[(2 * pr + 1) * N + x] = q.y;
        }
      }
      __syncthreads();
    }
  }

  // Phase 2: stencil input rows.
  if (MODE != kModeAdj) {
    const double* xin = p.x_in + off;
    for (int e = tid; e < R * N; e += 256) {
      const int r = e / N, x = e % N;
      X[e] = xin[static_cast<long long>((y0 - 1 + r) & (N - 1)) * N + x];
    }
  } else {
    const double dt = p.dt;
    for (int e = tid; e < R * N; e += 256) {
      const int r = e / N, x = e % N;
      const int gy = (y0 - 1 + r) & (N - 1);
      const long long g = off + static_cast<long long>(gy) * N + x;
      const bool owned = r >= 1 && r <= T;
      const double mu = has_prev ? p.q_in[g] + P[e] : 0.0;
      double a;
      if (finish) {
        if (owned) p.d[g] = p.acc[g] + mu;
        continue;
      }
      switch (p.stage) {
        case 3: {
          const double lam = has_prev ? p.acc[g] + mu : p.d[g];
          if (owned && has_prev) p.d[g] = lam;
          a = dt / 6.0 * lam;
          break;
        }
        case 2: {
          const double lam = p.d[g];
          if (owned) p.acc[g] = lam + mu;
          a = dt / 3.0 * lam + dt * mu;
          break;
        }
        case 1: {
          const double lam = p.d[g];
          if (owned) p.acc[g] += mu;
          a = dt / 3.0 * lam + 0.5 * dt * mu;
          break;
        }
        default: {
          const double lam = p.d[g];
          if (owned) p.acc[g] += mu;
          a = dt / 6.0 * lam + 0.5 * dt * mu;
          break;
        }
      }
      X[e] = a;
    }
    if (finish) return;
  }
  __syncthreads();

  // Phase 3: stencils + RK update on owned rows.
  const double js = p.inv12h2, ls = p.invh2, nu = p.nu, dt = p.dt;
  double res[PTS];
#pragma unroll
  for (int q = 0; q < PTS; ++q) {
    const int e = tid + q * 256;
    const int r = 1 + e / N, x = e % N;
    const int gy = (y0 + r - 1) & (N - 1);
    const long long g = off + static_cast<long long>(gy) * N + x;
    double xs[3][3];
    load3x3_smem<N>(X, r, x, xs);
    if (MODE == kModeNl) {
      double ps[3][3];
      load3x3_smem<N>(P, r, x, ps);
      const double kk = arakawa12(ps, xs) * js + nu * lap5(xs) * ls;
      if (p.store_w) {
        p.store_w[static_cast<long long>(gy) * N + x] = xs[1][1];
        p.store_p[static_cast<long long>(gy) * N + x] = ps[1][1];
      }
      res[q] = kk;
    } else if (MODE == kModeTlm) {
      double ps[3][3], bp[3][3], bw[3][3];
      load3x3_smem<N>(P, r, x, ps);
      load3x3_glob<N>(p.base_p, gy, x, bp);
      load3x3_glob<N>(p.base_w, gy, x, bw);
      res[q] = (arakawa12(bp, xs) + arakawa12(ps, bw)) * js + nu * lap5(xs) * ls;
    } else {
      double bp[3][3], bw[3][3];
      load3x3_glob<N>(p.base_p, gy, x, bp);
      load3x3_glob<N>(p.base_w, gy, x, bw);
      p.q_out[g] = -arakawa12(bp, xs) * js + nu * lap5(xs) * ls;
      res[q] = -arakawa12(xs, bw) * js;
    }
    if (MODE != kModeAdj) {
      const double kk = res[q];
      double xn;
      switch (p.stage) {
        case 0: {
          const double d = p.d[g];
          p.acc[g] = d + dt / 6.0 * kk;
          xn = d + 0.5 * dt * kk;
          p.x_out[g] = xn;
          break;
        }
        case 1: {
          const double d = p.d[g];
          p.acc[g] += dt / 3.0 * kk;
          xn = d + 0.5 * dt * kk;
          p.x_out[g] = xn;
          break;
        }
        case 2: {
          const double d = p.d[g];
          p.acc[g] += dt / 3.0 * kk;
          xn = d + dt * kk;
          p.x_out[g] = xn;
          break;
        }
        default: {
          xn = p.acc[g] + dt / 6.0 * kk;
          p.d[g] = xn;
          break;
        }
      }
      res[q] = xn;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PTS; ++q) P[N + tid + q * 256] = res[q];
  __syncthreads();

  // Phase 4: forward x-FFT of the owned rows -> next row spectra.
  constexpr int kOwnPairs = T / 2;
  for (int base = 0; base < kOwnPairs; base += C::kTeams) {
    const int pr = base + team;
    const bool act = pr < kOwnPairs;
    if (act)
      for (int x = t; x < N; x += C::kTeam) fa[x] = make_double2(P[(1 + 2 * pr) * N + x], P[(2 + 2 * pr) * N + x]);
    __syncthreads();
    const double2* z = fft_team<N, false>(fa, fb, tw, t, C::kTeam, act);
    if (act) {
      double2* ra = p.s_out + soff + static_cast<long long>(y0 + 2 * pr) * (N / 2);
      pack_pair<N>(z, ra, ra + N / 2, t, C::kTeam);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ obs kernels --
__global__ void gather_obs_kernel(const double* __restrict__ f, long long dim, const long long* __restrict__ idx,
                                  int n_obs, const double* __restrict__ w, double* __restrict__ y, long long m,
                                  int nvec) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<long long>(n_obs) * nvec) return;
  const int v = static_cast<int>(e / n_obs), k = static_cast<int>(e % n_obs);
  y[v * m + k] = f[v * dim + idx[k]] * w[k];
}
__global__ void scatter_obs_kernel(double* __restrict__ f, long long dim, const long long* __restrict__ idx,
                                   int n_obs, const double* __restrict__ w, const double* __restrict__ y, long long m,
                                   int nvec) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<long long>(n_obs) * nvec) return;
  const int v = static_cast<int>(e / n_obs), k = static_cast<int>(e % n_obs);
  f[v * dim + idx[k]] += y[v * m + k] * w[k];
}

// ---------------------------------------------------------------- launchers --
namespace {
template <int N>
struct Launch {
  static constexpr int kT = 8;
  static constexpr int kCW = N >= 256 ? 4 : (N >= 128 ? 8 : 16);
  static size_t row_smem() { return sizeof(double2) * 2 * N * RowCfg<N>::kTeams; }
  static size_t stage_smem() { return sizeof(double) * 2 * (kT + 2) * N + row_smem(); }
  static size_t col_smem() { return sizeof(double2) * 2 * N * kCW; }
  static void setup() {
    static bool done = false;
    if (done) return;
    SDV_CUDA(cudaFuncSetAttribute(stage_kernel<N, kT, kModeTlm>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(stage_smem())));
    SDV_CUDA(cudaFuncSetAttribute(stage_kernel<N, kT, kModeAdj>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(stage_smem())));
    SDV_CUDA(cudaFuncSetAttribute(stage_kernel<N, kT, kModeNl>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(stage_smem())));
    SDV_CUDA(cudaFuncSetAttribute(col_kernel<N, kCW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(col_smem())));
    SDV_CUDA(cudaFuncSetAttribute(row_fwd_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(row_smem())));
    SDV_CUDA(cudaFuncSetAttribute(row_inv_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(row_smem())));
    done = true;
  }
  static void row_fwd(const double* f, double2* s, int nvec, cudaStream_t st) {
    setup();
    dim3 g(ceil_div(N / 2, RowCfg<N>::kTeams), nvec);
    row_fwd_kernel<N><<<g, 256, row_smem(), st>>>(f, s, twiddle_table(N));
    SDV_LAUNCH_CHECK();
  }
  static void row_inv(const double2* s, double* f, int nvec, cudaStream_t st) {
    setup();
    dim3 g(ceil_div(N / 2, RowCfg<N>::kTeams), nvec);
    row_inv_kernel<N><<<g, 256, row_smem(), st>>>(s, f, twiddle_table(N));
    SDV_LAUNCH_CHECK();
  }
  static void col(double2* s, const double* sym, int nvec, cudaStream_t st) {
    setup();
    dim3 g((N / 2) / kCW, nvec);
    col_kernel<N, kCW><<<g, kCW * (N / 4), col_smem(), st>>>(s, sym, twiddle_table(N));
    SDV_LAUNCH_CHECK();
  }
  static void stage(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    setup();
    dim3 g(N / kT, nvec);
    switch (mode) {
      case kModeTlm: stage_kernel<N, kT, kModeTlm><<<g, 256, stage_smem(), st>>>(a); break;
      case kModeAdj: stage_kernel<N, kT, kModeAdj><<<g, 256, stage_smem(), st>>>(a); break;
      default: stage_kernel<N, kT, kModeNl><<<g, 256, stage_smem(), st>>>(a); break;
    }
    SDV_LAUNCH_CHECK();
  }
};

template <class F>
void dispatch_n(int n, F&& f) {
  switch (n) {
    case 32: f(std::integral_constant<int, 32>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 256: f(std::integral_constant<int, 256>{}); break;
    case 512: f(std::integral_constant<int, 512>{}); break;
    default: throw std::invalid_argument("BVE grid size must be one of 32, 64, 128, 256, 512");
  }
}
}  // namespace

void bve_row_fwd(int n, const double* f, double2* s, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::row_fwd(f, s, nvec, st); });
}
void bve_row_inv(int n, const double2* s, double* f, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::row_inv(s, f, nvec, st); });
}
void bve_col(int n, double2* s, const double* sym, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::col(s, sym, nvec, st); });
}
void bve_stage(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::stage(mode, a, nvec, st); });
}
void gather_obs(const double* f, long long dim, const long long* idx, int n_obs, const double* w, double* y,
                long long m, int nvec, cudaStream_t st) {
  const long long tot = static_cast<long long>(n_obs) * nvec;
  if (tot == 0) return;
  gather_obs_kernel<<<ceil_div(tot, 256), 256, 0, st>>>(f, dim, idx, n_obs, w, y, m, nvec);
  SDV_LAUNCH_CHECK();
}
void scatter_obs(double* f, long long dim, const long long* idx, int n_obs, const double* w, const double* y,
                 long long m, int nvec, cudaStream_t st) {
  const long long tot = static_cast<long long>(n_obs) * nvec;
  if (tot == 0) return;
  scatter_obs_kernel<<<ceil_div(tot, 256), 256, 0, st>>>(f, dim, idx, n_obs, w, y, m, nvec);
  SDV_LAUNCH_CHECK();
}

}  // namespace sdv

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
// coefficients packed into element 0 (re = X(0), im = X(n/2)); two real rows
// are transformed by one complex FFT (z = a + i b).
//
// Every RK4 stage is two launches:
//   col kernel  : y-FFT of the row spectra, spectral multiply, inverse y-FFT;
//   stage kernel: inverse x-FFT of the T owned rows + 2 halo rows, the
//                 Arakawa/Laplacian stencils with the stored base stage fields,
//                 the RK4 (TLM/NL) or adjoint-RK4 (ADJ) update, and the forward
//                 x-FFT of the next stage's Poisson input for the owned rows.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "bve_kernels.cuh"
#include "fft.cuh"
#include "linalg_kernels.cuh"
#include "stencil.cuh"

namespace sdv {

namespace {

constexpr int kThreads = 256;

// TT: owned rows per stage CTA (8; 2 for small blocks, where 8-row tiles
// would leave most SMs idle). CWW: columns per col-kernel CTA (0 = default).
template <int N, int TT = 8, int CWW = 0>
struct Cfg {
  static constexpr int kTeam = N / 8;                        // threads per FFT
  static constexpr int kTeams = kThreads / kTeam;            // FFTs in flight per CTA
  static constexpr int kPad = FftSize<N>::kPadded;           // double2 per FFT buffer
  static constexpr int kT = TT;                              // owned rows per stage CTA
  static constexpr int kNCT = N < kThreads ? N : kThreads;   // column threads
  static constexpr int kRG = kThreads / kNCT;                // row groups
  static constexpr int kRPG = kT / kRG;                      // rows per group
  static constexpr int kCPT = N / kNCT;                      // columns per thread
  static constexpr int kCWDefault = (N / 2) < (kThreads / kTeam) ? (N / 2) : (kThreads / kTeam);
  static constexpr int kCW = CWW > 0 ? CWW : kCWDefault;     // col-kernel columns
  static constexpr size_t kFftBytes = sizeof(double2) * kPad * kTeams;
  static constexpr size_t kTileBytes = sizeof(double) * (kT + 2) * N;
  static constexpr size_t kXBytes = kTileBytes > kFftBytes ? kTileBytes : kFftBytes;
  static constexpr size_t kStageSmem = kTileBytes + kXBytes;
  static constexpr size_t kRowSmem = kFftBytes;
  static constexpr int kColStride = kPad + 2;  // team buffers 8 banks apart (conflict-free staging)
  static constexpr size_t kColSmem = sizeof(double2) * kColStride * kCW;
};

// Packed half spectra (ra, rb) of two real rows -> element i of the full
// spectrum of z = a + i b.
template <int N>
__device__ __forceinline__ double2 unpack_elem(const double2* __restrict__ ra, const double2* __restrict__ rb, int i) {
  if (i == 0) return make_double2(ra[0].x, rb[0].x);
  if (i == N / 2) return make_double2(ra[0].y, rb[0].y);
  if (i < N / 2) {
    const double2 a = ra[i], b = rb[i];
    return make_double2(a.x - b.y, a.y + b.x);
  }
  const double2 a = ra[N - i], b = rb[N - i];
  return make_double2(a.x + b.y, b.x - a.y);
}
// Full spectrum z (padded smem) -> packed half spectra of the two real rows.
template <int N>
__device__ __forceinline__ void pack_pair(const double2* z, double2* __restrict__ ra, double2* __restrict__ rb, int t,
                                          int nt) {
  for (int k = t; k < N / 2; k += nt) {
    if (k == 0) {
      const double2 z0 = z[0], zn = z[fpad(N / 2)];
      ra[0] = make_double2(z0.x, zn.x);
      rb[0] = make_double2(z0.y, zn.y);
    } else {
      const double2 zk = z[fpad(k)], zm = z[fpad(N - k)];
      ra[k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      rb[k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
  }
}

// Asynchronous global -> shared 16-byte copy (LDGSTS): every copy of a tile is
// in flight at once instead of one load-use round trip per element.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Cache-line prefetch of `rows` periodic rows starting at row y of a field
// (one 128-byte line per thread-iteration): L1 for the shared base tiles the
// stencil walks, L2 for the per-vector RK state it streams.
template <int N, bool L1>
__device__ __forceinline__ void prefetch_rows(const double* f, int y, int rows, int tid, int nt) {
  constexpr int kLines = N / 16;  // 128-byte lines per row
  for (int i = tid; i < rows * kLines; i += nt) {
    const double* a = f + static_cast<long long>((y + i / kLines) & (N - 1)) * N + (i % kLines) * 16;
    if (L1) asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
    else asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  }
}

__device__ __forceinline__ void shift3(double w[3][3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    w[0][c] = w[1][c];
    w[1][c] = w[2][c];
  }
}

}  // namespace

// ---------------------------------------------------------------- row FFTs --
template <int N>
__global__ void __launch_bounds__(kThreads) row_fwd_kernel(const double* __restrict__ f, double2* __restrict__ s,
                                                           const double2* __restrict__ tw) {
  using C = Cfg<N>;
  pdl_wait();
  pdl_trigger();
  extern __shared__ double2 sm[];
  const int team = threadIdx.x / C::kTeam, t = threadIdx.x % C::kTeam;
  const int pair = blockIdx.x * C::kTeams + team;
  const bool active = pair < N / 2;
  const long long v = blockIdx.y;
  double2* buf = sm + team * C::kPad;
  const double* r0 = f + v * N * N + static_cast<long long>(2 * pair) * N;
  auto load = [&](int i) { return make_double2(r0[i], r0[i + N]); };
  auto store = [&](int i, double2 z) { buf[fpad(i)] = z; };
  fft_team<N, false>(buf, tw, t, active, load, store);
  __syncthreads();
  if (active) {
    double2* ra = s + v * N * (N / 2) + static_cast<long long>(2 * pair) * (N / 2);
    pack_pair<N>(buf, ra, ra + N / 2, t, C::kTeam);
  }
}

template <int N>
__global__ void __launch_bounds__(kThreads) row_inv_kernel(const double2* __restrict__ s, double* __restrict__ f,
                                                           const double2* __restrict__ tw) {
  using C = Cfg<N>;
  pdl_wait();
  pdl_trigger();
  extern __shared__ double2 sm[];
  const int team = threadIdx.x / C::kTeam, t = threadIdx.x % C::kTeam;
  const int pair = blockIdx.x * C::kTeams + team;
  const bool active = pair < N / 2;
  const long long v = blockIdx.y;
  double2* buf = sm + team * C::kPad;
  const double2* ra = s + v * N * (N / 2) + static_cast<long long>(2 * pair) * (N / 2);
  double* r0 = f + v * N * N + static_cast<long long>(2 * pair) * N;
  auto load = [&](int i) { return unpack_elem<N>(ra, ra + N / 2, i); };
  auto store = [&](int i, double2 z) {
    r0[i] = z.x;
    r0[i + N] = z.y;
  };
  fft_team<N, true>(buf, tw, t, active, load, store);
}

// ------------------------------------------------------------- column pass --
// y-FFT of kCW adjacent kx columns, multiply by sym[kx*N + ky], inverse y-FFT.
// Column kx = 0 holds X(0) + i X(n/2) per row; both are real-input columns, so
// the multiplier is applied through the Hermitian split
//   Z'(ky) = (s0+sN)/2 Z(ky) + (s0-sN)/2 conj(Z(-ky)).
// Body shared by col_kernel and the column-0 CTA of col_solve_kernel. All
// threads of the CTA call it (barriers); inactive ones only synchronise.
template <int N, int CW>
__device__ __forceinline__ void col_fft_body(double2* __restrict__ s, const double* __restrict__ sym,
                                             const double2* __restrict__ tw, double2* sm, int kx0, int team, int t,
                                             bool active, long long v) {
  using C = Cfg<N, 8, CW>;
  double2* col = s + v * N * (N / 2) + kx0 + team;
  double2* buf = sm + team * C::kColStride;
  auto ld_glob = [&](int i) { return col[static_cast<long long>(i) * (N / 2)]; };
  auto st_own = [&](int i, double2 z) { buf[fpad(i)] = z; };
  fft_team<N, false>(buf, tw, t, active, ld_glob, st_own);
  __syncthreads();
  const int kx = kx0 + team;
  const double* sk = sym + static_cast<long long>(kx) * N;
  const double* sn = sym + static_cast<long long>(N / 2) * N;
  auto ld_mul = [&](int ky) {
    const double2 z = buf[fpad(ky)];
    if (kx != 0) {
      const double w = __ldg(sk + ky);
      return make_double2(w * z.x, w * z.y);
    }
    const double a = __ldg(sk + ky), b = __ldg(sn + ky);
    const double pp = 0.5 * (a + b), mm = 0.5 * (a - b);
    const double2 zm = buf[fpad((N - ky) & (N - 1))];
    return make_double2(pp * z.x + mm * zm.x, pp * z.y - mm * zm.y);
  };
  auto st_glob = [&](int i, double2 z) { col[static_cast<long long>(i) * (N / 2)] = z; };
  fft_team<N, true>(buf, tw, t, active, ld_mul, st_glob);
}
template <int N, int CW>
__global__ void __launch_bounds__(CW*(N / 8)) col_kernel(double2* __restrict__ s, const double* __restrict__ sym,
                                                         const double2* __restrict__ tw) {
  extern __shared__ double2 sm[];
  pdl_wait();
  pdl_trigger();
  // Lanes interleave the kCW columns (team = column), so every warp-wide
  // global access covers kCW adjacent double2 of a few rows (coalesced); the
  // first forward pass reads global memory directly and the last inverse
  // pass writes it back (no staging pass).
  col_fft_body<N, CW>(s, sym, tw, sm, blockIdx.x * CW, threadIdx.x % CW, threadIdx.x / CW, true, blockIdx.y);
}

// ------------------------------------------------ column Poisson solve --
// Cyclic carries of one column across its 32 segments (lane = segment q).
// FWD: slot holds L_q, the zero-carry forward recurrence value at the last row
// of segment q; it becomes the closed carry into q,
//   C_q = sum_{p<q} rho^{RPS (q-1-p)} L_p + rho^{RPS q} F_{-1},
//   F_{-1} = F_{N-1} = C_32 / (1 - rho^N)   (clos = 1/(1 - rho^N)).
// BWD: the mirror image for the backward recurrence (carries from above).
template <bool FWD>
__device__ __forceinline__ void carry_scan(double2& slot, double rhoR, double clos, int lane) {
  constexpr unsigned kAll = 0xffffffffu;
  double A = rhoR, bx = slot.x, by = slot.y;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double Ap = FWD ? __shfl_up_sync(kAll, A, d) : __shfl_down_sync(kAll, A, d);
    const double px = FWD ? __shfl_up_sync(kAll, bx, d) : __shfl_down_sync(kAll, bx, d);
    const double py = FWD ? __shfl_up_sync(kAll, by, d) : __shfl_down_sync(kAll, by, d);
    if (FWD ? lane >= d : lane + d < 32) {
      bx = fma(A, px, bx);
      by = fma(A, py, by);
      A *= Ap;
    }
  }
  const int end = FWD ? 31 : 0, first = FWD ? 0 : 31;
  const double tx = __shfl_sync(kAll, bx, end) * clos, ty = __shfl_sync(kAll, by, end) * clos;
  double cx = FWD ? __shfl_up_sync(kAll, bx, 1) : __shfl_down_sync(kAll, bx, 1);
  double cy = FWD ? __shfl_up_sync(kAll, by, 1) : __shfl_down_sync(kAll, by, 1);
  double ae = FWD ? __shfl_up_sync(kAll, A, 1) : __shfl_down_sync(kAll, A, 1);
  if (lane == first) {
    cx = cy = 0.0;
    ae = 1.0;
  }
  slot = make_double2(fma(ae, tx, cx), fma(ae, ty, cy));
}
// For each kx >= 1 the 5-point Poisson operator restricted to one x-Fourier
// mode is the circulant (1/h^2)(d - S - S^-1) in y, d = 2 + 4 sin^2(pi kx/N),
// S the cyclic row shift. With rho + 1/rho = d (rho < 1),
//   (d - S - S^-1)^-1 = rho (1 - rho S^-1)^-1 (1 - rho S)^-1,
// i.e. a forward first-order recurrence F_j = w_j + rho F_{j-1} followed by a
// backward one G_j = F_j + rho G_{j+1}, both cyclic. This is the exact
// inverse the y-FFT/multiply/inverse-y-FFT of col_kernel applies (same
// operator, same eigenvalues mu(kx, ky)), at ~10 flops per point instead of
// two 512-point FFTs, with coalesced row-segment access and no twiddles.
// Each thread owns RPS = N/32 consecutive rows of one column in registers;
// the 32 segment carries of a column are chained through shared memory, and
// the cyclic closure uses 1/(1 - rho^N). tab[kx] = {rho, rho^RPS,
// 1/(1 - rho^N), h^2 rho / N} (the 1/N is the unnormalised inverse x-FFT).
// Column kx = 0 (packed X(0) + i X(N/2), singular at kx = 0) stays on the
// FFT path: the grid's last CTA column runs col_kernel's body on it.
template <int N>
__global__ void __launch_bounds__(256, N >= 512 ? 2 : 3)
    col_solve_kernel(double2* __restrict__ s, const double4* __restrict__ tab, const double* __restrict__ sym,
                     const double2* __restrict__ tw) {
  constexpr int CS = 8, SEG = 32, RPS = N / SEG;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == gridDim.x - 1) {
    extern __shared__ double2 sm[];
    col_fft_body<N, 1>(s, sym, tw, sm, 0, 0, threadIdx.x, threadIdx.x < N / 8, blockIdx.y);
    return;
  }
  __shared__ double2 car[2][CS][SEG];
  const int c = threadIdx.x % CS, sg = threadIdx.x / CS;
  const int kx = blockIdx.x * CS + c;
  const bool live = kx != 0;
  const long long v = blockIdx.y;
  double2* col = s + v * N * (N / 2) + kx + static_cast<long long>(sg) * RPS * (N / 2);
  const double4 tb = tab[kx];
  const double rho = tb.x, rhoR = tb.y, clos = tb.z, scale = tb.w;
  double2 x[RPS];
#pragma unroll
  for (int k = 0; k < RPS; ++k) x[k] = live ? col[static_cast<long long>(k) * (N / 2)] : make_double2(0.0, 0.0);
  // forward local recurrence (zero carry-in)
  double2 f = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < RPS; ++k) {
    f = make_double2(fma(rho, f.x, x[k].x), fma(rho, f.y, x[k].y));
    x[k] = f;
  }
  car[0][c][sg] = f;
  __syncthreads();
  // Segment carries: warp w chains column w's 32 segments (lane = segment)
  // with a Kogge-Stone scan of the affine maps C -> rho^RPS C + L.
  const int wc = threadIdx.x / 32, lane = threadIdx.x % 32;
  const double4 tw4 = tab[blockIdx.x * CS + wc];
  const bool wlive = blockIdx.x * CS + wc != 0;
  if (wlive) carry_scan<true>(car[0][wc][lane], tw4.y, tw4.z, lane);
  __syncthreads();
  {
    const double2 cin = car[0][c][sg];
    double pw = rho;
#pragma unroll
    for (int k = 0; k < RPS; ++k) {
      x[k] = make_double2(fma(pw, cin.x, x[k].x), fma(pw, cin.y, x[k].y));
      pw *= rho;
    }
  }
  // backward local recurrence (zero carry-in from above)
  double2 g = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = RPS - 1; k >= 0; --k) {
    g = make_double2(fma(rho, g.x, x[k].x), fma(rho, g.y, x[k].y));
    x[k] = g;
  }
  car[1][c][sg] = g;
  __syncthreads();
  if (wlive) carry_scan<false>(car[1][wc][lane], tw4.y, tw4.z, lane);
  __syncthreads();
  if (!live) return;
  const double2 cin = car[1][c][sg];
  double pw = rho;
#pragma unroll
  for (int k = RPS - 1; k >= 0; --k) {
    const double2 z = make_double2(fma(pw, cin.x, x[k].x), fma(pw, cin.y, x[k].y));
    col[static_cast<long long>(k) * (N / 2)] = make_double2(scale * z.x, scale * z.y);
    pw *= rho;
  }
}

// ----------------------------------------------- tile carries (fused path) --
// Packed kx = 0 column of one vector, one warp, exact O(N) solves (lane l owns
// rows l*RPS .. l*RPS + RPS - 1):
//  * real part, x-mode 0: the zero-mean pseudo-inverse of the periodic second
//    difference L = 2 - S - S^-1 (the (0,0) mode of psi is 0): with
//    w' = w - mean(w), P_j = sum_{m<j} w'_m, S_j = sum_{i=1}^{j} P_i,
//    D_0 = S_N / N, psi_j = j D_0 - S_j minus its mean;
//  * imaginary part, x-mode N/2: (6 - S - S^-1)^-1 by the cyclic forward and
//    backward recurrences with rho = 3 - 2 sqrt 2, as col_solve_kernel.
// Both times h^2 / N (the 1/N is the unnormalised inverse x-FFT): the same
// operator as the spectral column pass (mu = 4 sin^2(pi ky / N) / h^2).
// t0 = tab[0] = {rho_{N/2}, h^2 / N, 1 / (1 - rho_{N/2}^N), h^2 rho_{N/2} / N}.
template <int N>
__device__ __forceinline__ void col0_warp_solve(double2* __restrict__ col, double4 t0, int lane) {
  constexpr unsigned kAll = 0xffffffffu;
  constexpr int RPS = N / 32;
  double2 x[RPS];
#pragma unroll
  for (int k = 0; k < RPS; ++k) x[k] = col[static_cast<long long>(lane * RPS + k) * (N / 2)];
  auto warp_sum = [&](double a) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) a += __shfl_xor_sync(kAll, a, d);
    return a;
  };
  auto warp_excl = [&](double a) {  // exclusive prefix sum over lanes
    double incl = a;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(kAll, incl, d);
      if (lane >= d) incl += o;
    }
    return incl - a;
  };
  // ---- real part (singular) ----
  double ls = 0.0;
#pragma unroll
  for (int k = 0; k < RPS; ++k) ls += x[k].x;
  const double mean = warp_sum(ls) / N;
  double pre[RPS];  // P_j at row j = lane*RPS + k (exclusive prefix of w')
  {
    double run = warp_excl(ls - RPS * mean);
#pragma unroll
    for (int k = 0; k < RPS; ++k) {
      pre[k] = run;
      run += x[k].x - mean;
    }
  }
  // S_j = sum_{i=1}^{j} P_i (P_0 = 0, so S_j = inclusive prefix of P)
  double lp = 0.0;
#pragma unroll
  for (int k = 0; k < RPS; ++k) lp += pre[k];
  const double d0 = warp_sum(lp) / N;  // S_N / N (P_N = 0)
  double ps = 0.0;
  {
    double run = warp_excl(lp);
#pragma unroll
    for (int k = 0; k < RPS; ++k) {
      run += pre[k];
      pre[k] = static_cast<double>(lane * RPS + k) * d0 - run;  // psi_j before centring
      ps += pre[k];
    }
  }
  const double pm = warp_sum(ps) / N;
  // ---- imaginary part (x-mode N/2) ----
  const double rho = t0.x;
  double2 slot;
  double f = 0.0;
#pragma unroll
  for (int k = 0; k < RPS; ++k) {
    f = fma(rho, f, x[k].y);
    x[k].y = f;
  }
  double rR = 1.0;
#pragma unroll
  for (int k = 0; k < RPS; ++k) rR *= rho;
  slot = make_double2(f, 0.0);
  carry_scan<true>(slot, rR, t0.z, lane);
  {
    double pw = rho;
#pragma unroll
    for (int k = 0; k < RPS; ++k) {
      x[k].y = fma(pw, slot.x, x[k].y);
      pw *= rho;
    }
  }
  double g = 0.0;
#pragma unroll
  for (int k = RPS - 1; k >= 0; --k) {
    g = fma(rho, g, x[k].y);
    x[k].y = g;
  }
  slot = make_double2(g, 0.0);
  carry_scan<false>(slot, rR, t0.z, lane);
  double pw = rho;
#pragma unroll
  for (int k = RPS - 1; k >= 0; --k) {
    x[k].y = t0.w * fma(pw, slot.x, x[k].y);
    pw *= rho;
  }
#pragma unroll
  for (int k = 0; k < RPS; ++k)
    col[static_cast<long long>(lane * RPS + k) * (N / 2)] = make_double2(t0.y * (pre[k] - pm), x[k].y);
}

// Tile carries per x-mode kx >= 1 (32 adjacent modes per CTA, lane = mode;
// warp = part of QP = Q/8 consecutive 8-row tiles): the forward carries C_q
// (F at the last row of tile q-1) from the tile end values L_q,
// C_{q+1} = L_q + rho^8 C_q, and the backward carries E_q (G at the first row
// of tile q+1) from V_q = M_q + alpha_0 C_q + rho^8 V_{q+1}, M_q = H at the
// first row of tile q, both cyclic (closure 1/(1 - rho^N)). The 8 part maps
// are composed through shared memory. The grid's last CTA column solves the
// packed kx = 0 column in place (col0_warp_solve).
template <int N>
__global__ void __launch_bounds__(256, 2) carry_kernel(double2* __restrict__ s, const double2* __restrict__ lsum,
                                                    double2* __restrict__ car_c, double2* __restrict__ car_e,
                                                    const double4* __restrict__ tab) {
  constexpr int T = 8, Q = N / T, NPT = 8, QP = Q / NPT;
  static_assert(Q % NPT == 0, "carry_kernel: N / 8 tiles must split into 8 parts");
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x % 32, pt = threadIdx.x / 32;
  const long long v = blockIdx.y;
  if (blockIdx.x == gridDim.x - 1) {
    if (pt == 0) col0_warp_solve<N>(s + v * N * (N / 2), tab[0], lane);
    return;
  }
  __shared__ double2 part[NPT][32];
  const int kx = blockIdx.x * 32 + lane;
  const bool live = kx != 0 && kx < N / 2;
  const int kxs = live ? kx : 1;
  const double4 tb = tab[kxs];
  const long long cb = v * Q * (N / 2) + kxs;
  double2 Lv[QP], Mv[QP];
#pragma unroll
  for (int i = 0; i < QP; ++i) {
    const int q = pt * QP + i;
    Lv[i] = lsum[cb + static_cast<long long>(q) * (N / 2)];
    Mv[i] = s[v * N * (N / 2) + static_cast<long long>(q) * T * (N / 2) + kxs];
  }
  const double rho = tb.x, clos = tb.z;
  double rT = rho * rho;
  rT *= rT;
  rT *= rT;  // rho^8
  double A = 1.0;  // part map multiplier rho^(8 QP)
#pragma unroll
  for (int i = 0; i < QP; ++i) A *= rT;
  double a0 = 0.0;  // alpha_0 = sum_{m<8} rho^(2m+1)
  {
    double pw = rho;
#pragma unroll
    for (int m = 0; m < T; ++m) {
      a0 += pw;
      pw *= rho * rho;
    }
  }
  // forward: part composition with zero carry-in, then the closed carry
  double2 f = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < QP; ++i) f = make_double2(fma(rT, f.x, Lv[i].x), fma(rT, f.y, Lv[i].y));
  part[pt][lane] = f;
  __syncthreads();
  double2 tot = make_double2(0.0, 0.0);
#pragma unroll
  for (int p = 0; p < NPT; ++p) {
    const double2 fp = part[p][lane];
    tot = make_double2(fma(A, tot.x, fp.x), fma(A, tot.y, fp.y));
  }
  double2 cin = make_double2(clos * tot.x, clos * tot.y);  // C_0
  for (int p = 0; p < pt; ++p) {
    const double2 fp = part[p][lane];
    cin = make_double2(fma(A, cin.x, fp.x), fma(A, cin.y, fp.y));
  }
#pragma unroll
  for (int i = 0; i < QP; ++i) {
    if (live) car_c[cb + static_cast<long long>(pt * QP + i) * (N / 2)] = cin;
    Mv[i] = make_double2(fma(a0, cin.x, Mv[i].x), fma(a0, cin.y, Mv[i].y));  // u_q
    cin = make_double2(fma(rT, cin.x, Lv[i].x), fma(rT, cin.y, Lv[i].y));
  }
  // backward: V at the first tile of each part with zero carry from above
  double2 g = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = QP - 1; i >= 0; --i) g = make_double2(fma(rT, g.x, Mv[i].x), fma(rT, g.y, Mv[i].y));
  __syncthreads();
  part[pt][lane] = g;
  __syncthreads();
  double2 vt = make_double2(0.0, 0.0);
#pragma unroll
  for (int p = NPT - 1; p >= 0; --p) {
    const double2 gp = part[p][lane];
    vt = make_double2(fma(A, vt.x, gp.x), fma(A, vt.y, gp.y));
  }
  double2 e = make_double2(clos * vt.x, clos * vt.y);  // V at tile 0 (= part NPT, cyclic)
  for (int p = NPT - 1; p > pt; --p) {
    const double2 gp = part[p][lane];
    e = make_double2(fma(A, e.x, gp.x), fma(A, e.y, gp.y));
  }
  if (!live) return;
#pragma unroll
  for (int i = QP - 1; i >= 0; --i) {
    const long long o = cb + static_cast<long long>(pt * QP + i) * (N / 2);
    car_e[o] = e;
    e = make_double2(fma(rT, e.x, Mv[i].x), fma(rT, e.y, Mv[i].y));
  }
}

// --------------------------------------------------------- fused RK stage --
// ST: RK stage as a compile-time constant (TLM/ADJ; -1 = runtime p.stage).
// FUS: fused Poisson path (TLM/ADJ, T = 8). The launch stages its spectrum
// rows and stencil-input rows into shared memory with cp.async up front,
// reconstructs the y-solved spectra from the tile-local recurrence values
// and the tile carries of bve_carry, runs both x-FFTs in place in P (swizzled
// layout, no scratch buffer), and ends with the tile-local forward/backward
// recurrences of the next Poisson solve on its own rows, so the full-field
// column pass (read + write of every spectrum) drops out of each stage.
template <int N, int MODE, int T, int ST = -1, bool FUS = false>
__global__ void __launch_bounds__(kThreads, 2) stage_kernel(StageArgs p) {
  using C = Cfg<N, T>;
  constexpr int R = T + 2;
  const int stage = ST >= 0 ? ST : p.stage;
  extern __shared__ double smd[];
  double* P = smd;                             // R x N inverse-FFT field
  double* X = P + R * N;                       // R x N stencil input
  double2* F = reinterpret_cast<double2*>(X);  // FFT buffers alias X
  const int tid = threadIdx.x;
  const int team = tid / C::kTeam, t = tid % C::kTeam;
  const int y0 = blockIdx.x * T;
  const long long v = blockIdx.y;
  const long long off = v * N * N;
  const long long soff = v * N * (N / 2);
  const double2* tw = p.tw;
  double2* fbuf = F + team * C::kPad;
  const bool has_prev = MODE != kModeAdj || (p.flags & kFlagHasPrev);
  const bool finish = MODE == kModeAdj && (p.flags & kFlagFinish);
  const bool pf = !(p.flags & kFlagNoPrefetch);

  // Prefetch what the later phases read, so it streams in under the inverse
  // FFT: the stencil's first base tile into L1 (shared by the whole tile,
  // walked row by row), the per-vector RK state and stencil input into L2.
  if (pf) {
    if (MODE == kModeTlm) {
      prefetch_rows<N, true>(p.base_p, y0 - 1, R, tid, kThreads);
      if (!FUS) prefetch_rows<N, false>(p.x_in + off, y0 - 1, R, tid, kThreads);
      if (stage >= 1 && stage <= 2) prefetch_rows<N, false>(p.d + off, y0, T, tid, kThreads);
      if (stage >= (FUS ? 2 : 1)) prefetch_rows<N, false>(p.acc + off, y0, T, tid, kThreads);
    } else if (MODE == kModeAdj && !finish) {
      prefetch_rows<N, true>(p.base_p, y0 - 1, R, tid, kThreads);
      if (has_prev && !FUS) prefetch_rows<N, false>(p.q_in + off, y0 - 1, R, tid, kThreads);
      prefetch_rows<N, false>(p.acc + off, y0 - 1, R, tid, kThreads);
      prefetch_rows<N, false>(p.d + off, y0 - 1, R, tid, kThreads);
    }
  }

  pdl_wait();  // everything below reads what the previous launch wrote

  constexpr int kPairs = R / 2;
  constexpr bool kTail = FUS && kPairs > C::kTeams;
  // fused path: inverse x-FFT of row pair pr in place in its P region
  auto pair_fft = [&](int pr, bool act, auto bar_c) {
    double* pa = P + (2 * pr) * N;
    double2* buf = reinterpret_cast<double2*>(pa);
    auto load = [&](int i) { return buf[i]; };
    auto store = [&](int i, double2 z) {
      pa[i] = z.x;
      pa[i + N] = z.y;
    };
    fft_team<N, true, 0, true, decltype(bar_c)::value, true>(buf, tw, t, act, load, store);
  };
  if constexpr (FUS) {
    // Phase 0: every global tile read of the launch in flight at once. The
    // stencil input (TLM x_in, ADJ q_in) streams into X by cp.async; the
    // spectrum rows y0-1 .. y0+T go through registers into P (a packed
    // spectrum row is N doubles, the size of a field row): thread kx loads its
    // column of the R rows plus the carries of the three tiles involved and
    // stores the y-solved values psi = scale (H + alpha_o C_q + rho^(T-o) E_q)
    // (row offset o of tile q, alpha_o = sum_{m=o}^{T-1} rho^(2m-o+1), see
    // bve_carry). kx = 0 and first-stage (kFlagRawIn) spectra are final.
    const bool inv = has_prev && !(p.flags & kFlagSkipInvFft);
    const double* xsrc = MODE == kModeTlm ? p.x_in : (has_prev ? p.q_in : nullptr);
    if (xsrc) {
      xsrc += off;
      for (int e = 2 * tid; e < R * N; e += 2 * kThreads) {
        const int r = e / N, x = e % N;
        cp_async16(X + e, xsrc + static_cast<long long>((y0 - 1 + r) & (N - 1)) * N + x);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (inv) {
      constexpr int Q = N / T;
      const bool raw = p.flags & kFlagRawIn;
      const int q0 = blockIdx.x, qm = (q0 + Q - 1) % Q, qp = (q0 + 1) % Q;
      for (int kx = tid; kx < N / 2; kx += kThreads) {
        const double2* hs = p.s_in + soff + kx;
        double2 h[R];
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = hs[static_cast<long long>((y0 - 1 + r) & (N - 1)) * (N / 2)];
        if (kx != 0 && !raw) {
          const long long cb = static_cast<long long>(v) * Q * (N / 2) + kx;
          const double2 cm = p.car_c[cb + qm * (N / 2)], c0 = p.car_c[cb + q0 * (N / 2)],
                        cq = p.car_c[cb + qp * (N / 2)];
          const double2 em = p.car_e[cb + qm * (N / 2)], e0 = p.car_e[cb + q0 * (N / 2)],
                        eq = p.car_e[cb + qp * (N / 2)];
          const double4 tb = p.stab[kx];
          const double rho = tb.x, scale = tb.w;
          double pw[T + 1], al[T];
          pw[0] = 1.0;
#pragma unroll
          for (int i = 1; i <= T; ++i) pw[i] = pw[i - 1] * rho;
          al[T - 1] = pw[T];
#pragma unroll
          for (int o = T - 2; o >= 0; --o) al[o] = fma(rho, al[o + 1], pw[o + 1]);
          auto fix = [&](double2& z, double a, double b, double2 c, double2 e) {
            z = make_double2(scale * fma(b, e.x, fma(a, c.x, z.x)), scale * fma(b, e.y, fma(a, c.y, z.y)));
          };
          fix(h[0], al[T - 1], pw[1], cm, em);
#pragma unroll
          for (int o = 0; o < T; ++o) fix(h[1 + o], al[o], pw[T - o], c0, e0);
          fix(h[R - 1], al[0], pw[T], cq, eq);
        }
        // unpack each row pair (a, b) into the full spectrum of z = a + i b
        // (pass-0 input of the inverse FFT, natural order, in the pair region)
#pragma unroll
        for (int pr = 0; pr < R / 2; ++pr) {
          double2* z = reinterpret_cast<double2*>(P + (2 * pr) * N);
          const double2 a = h[2 * pr], b = h[2 * pr + 1];
          if (kx == 0) {
            z[0] = make_double2(a.x, b.x);
            z[N / 2] = make_double2(a.y, b.y);
          } else {
            z[kx] = make_double2(a.x - b.y, a.y + b.x);
            z[N - kx] = make_double2(a.x + b.y, b.x - a.y);
          }
        }
      }
    }
    if (xsrc) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (inv) {
      // Phase 1: inverse x-FFT of the R rows, in place (pair region of P).
      // With N = 512 (4 teams) the fifth (halo) pair is a tail round: in the
      // TLM team 0 runs it under a named barrier while the other warps start
      // stencil sweep A (which reads X and psi_b, not P); the ADJ runs it here.
      static_assert(kPairs <= 2 * C::kTeams, "fused path: at most two inverse FFT rounds");
      pair_fft(team, team < kPairs, std::integral_constant<int, -1>{});
      // TLM: sweep A reads X and psi_b only; the barrier before sweep B
      // orders these P rows (and the tail pair's)
      if (MODE != kModeTlm || !kTail) __syncthreads();
      // (ADJ: the tail pair runs under a named barrier at the start of
      // phase 2, overlapped with the combination of rows 0 .. 2 kTeams - 1)
    }
  }
  // Phase 1: inverse x-FFT of rows y0-1 .. y0+T -> P.
  if (!FUS && has_prev && !(p.flags & kFlagSkipInvFft)) {
#pragma unroll 1
    for (int b0 = 0; b0 < kPairs; b0 += C::kTeams) {
      const int pr = b0 + team;
      const bool act = pr < kPairs;
      const int ga = (y0 - 1 + 2 * pr) & (N - 1), gb = (y0 + 2 * pr) & (N - 1);
      const double2* ra = p.s_in + soff + static_cast<long long>(ga) * (N / 2);
      const double2* rb = p.s_in + soff + static_cast<long long>(gb) * (N / 2);
      double* pa = P + (2 * pr) * N;
      auto load = [&](int i) { return unpack_elem<N>(ra, rb, i); };
      auto store = [&](int i, double2 z) {
        pa[i] = z.x;
        pa[i + N] = z.y;
      };
      fft_team<N, true>(fbuf, tw, t, act, load, store);
      __syncthreads();
    }
  }

  // Phase 2: stencil-input rows (overwrite the FFT buffers).
  if (FUS && MODE == kModeTlm) {
    // staged in phase 0
  } else if (MODE != kModeAdj) {
    const double* xin = p.x_in + off;
    for (int e = 2 * tid; e < R * N; e += 2 * kThreads) {
      const int r = e / N, x = e % N;
      cp_async16(X + e, xin + static_cast<long long>((y0 - 1 + r) & (N - 1)) * N + x);
    }
    cp_async_wait_all();
  } else {
    if (pf && !finish) prefetch_rows<N, true>(p.base_w, y0 - 1, R, tid, kThreads);
    // lambda/mu combination of SURVEY.md B.1, batched kB elements per thread
    // (all loads issued before any dependent arithmetic).
    // Row-wise: each thread owns column pairs (16-byte loads/stores), row
    // offsets are computed once per row (only the two halo rows wrap), and
    // kRB rows of loads are issued before the dependent arithmetic.
    const double dt = p.dt;
    const double2* __restrict__ qin = reinterpret_cast<const double2*>(p.q_in);
    double2* __restrict__ lamp = reinterpret_cast<double2*>(p.d);
    double2* __restrict__ accp = reinterpret_cast<double2*>(p.acc);
    const bool need_a = finish || stage <= 1 || (stage == 3 && has_prev);
    const bool need_l = !(finish || (stage == 3 && has_prev));
    const double2 z2 = make_double2(0.0, 0.0);
    // one batch of RB rows from rb: all loads first, then the arithmetic
    auto batch = [&](int x2, int rb, auto rb_c) {
      constexpr int kRB = decltype(rb_c)::value;
      {
        double2 qv[kRB], av[kRB], lv[kRB];
        long long go[kRB];
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          const int r = rb + u;
          go[u] = (off + static_cast<long long>((y0 - 1 + r) & (N - 1)) * N) / 2 + x2;
          if (FUS) qv[u] = has_prev ? reinterpret_cast<const double2*>(X + r * N)[x2] : z2;  // staged
          else qv[u] = has_prev ? qin[go[u]] : z2;
          // the accumulator enters a (halo rows) only at stage 3; stages 1, 0
          // and the finish update it on the owned rows alone
          const bool own_r = r >= 1 && r <= T;
          av[u] = (need_a && (stage == 3 || own_r)) ? accp[go[u]] : z2;
          lv[u] = need_l ? lamp[go[u]] : z2;
        }
#pragma unroll
        for (int u = 0; u < kRB; ++u) {
          const int r = rb + u;
          const bool owned = r >= 1 && r <= T;
          const double2 pp = reinterpret_cast<const double2*>(P + r * N)[x2];
          const double2 mu = has_prev ? make_double2(qv[u].x + pp.x, qv[u].y + pp.y) : z2;
          if (finish) {
            if (owned) lamp[go[u]] = make_double2(av[u].x + mu.x, av[u].y + mu.y);
            continue;
          }
          double2 a;
          if (stage == 3) {
            const double2 lam = has_prev ? make_double2(av[u].x + mu.x, av[u].y + mu.y) : lv[u];
            if (owned && has_prev) lamp[go[u]] = lam;
            a = make_double2(dt / 6.0 * lam.x, dt / 6.0 * lam.y);
          } else if (stage == 2) {
            if (owned) accp[go[u]] = make_double2(lv[u].x + mu.x, lv[u].y + mu.y);
            a = make_double2(dt / 3.0 * lv[u].x + dt * mu.x, dt / 3.0 * lv[u].y + dt * mu.y);
          } else if (stage == 1) {
            if (owned) accp[go[u]] = make_double2(av[u].x + mu.x, av[u].y + mu.y);
            a = make_double2(dt / 3.0 * lv[u].x + 0.5 * dt * mu.x, dt / 3.0 * lv[u].y + 0.5 * dt * mu.y);
          } else {
            if (owned) accp[go[u]] = make_double2(av[u].x + mu.x, av[u].y + mu.y);
            a = make_double2(dt / 6.0 * lv[u].x + 0.5 * dt * mu.x, dt / 6.0 * lv[u].y + 0.5 * dt * mu.y);
          }
          reinterpret_cast<double2*>(X + r * N)[x2] = a;
        }
      }
    };
    constexpr bool kAdjTail = FUS && kTail && MODE == kModeAdj;
    if constexpr (kAdjTail) {
      // tail inverse-FFT pair (rows 2 kTeams, 2 kTeams + 1) on team 0 while
      // the other warps combine the rows of the first round
      constexpr int kR1 = 2 * C::kTeams;  // rows done by round 1
      static_assert(kR1 % 4 == 0 && R - kR1 == 2, "ADJ tail layout");
      const bool inv = has_prev && !(p.flags & kFlagSkipInvFft);
      if (inv && team == 0) pair_fft(C::kTeams, true, std::integral_constant<int, 1>{});
      for (int x2 = tid; x2 < N / 2; x2 += kThreads)
#pragma unroll 1
        for (int rb = 0; rb < kR1; rb += 4) batch(x2, rb, std::integral_constant<int, 4>{});
      __syncthreads();  // tail rows of P complete
      for (int x2 = tid; x2 < N / 2; x2 += kThreads) batch(x2, kR1, std::integral_constant<int, 2>{});
    } else {
      constexpr int kRB = R % 5 == 0 ? 5 : (R % 2 == 0 ? 2 : 1);
#pragma unroll 1
      for (int x2 = tid; x2 < N / 2; x2 += kThreads)
#pragma unroll 1
        for (int rb = 0; rb < R; rb += kRB) batch(x2, rb, std::integral_constant<int, kRB>{});
    }
    if (finish) return;
  }
  __syncthreads();

  if constexpr (FUS && MODE != kModeNl) {
    // Phase 3 (fused TLM/ADJ): each thread owns two adjacent columns x0, x0+1 of
    // RPG rows; per window row and field one 16-byte load (x0, x0+1) plus the
    // two outer neighbours (4 values for 2 points instead of 3 per point).
    //   A: J(psi_b, X) + nu Lap X (smem X, global psi_b)
    //   B: + J(P, omega_b), RK4 update (smem P, global omega_b)
    constexpr int NCP = N / 2, RG = kThreads / NCP, RPG = T / RG;
    static_assert(RG * NCP == kThreads && RPG * RG == T, "fused TLM stencil mapping");
    const double js = p.inv12h2, nls = p.nu * p.invh2, dt = p.dt;
    const int x0 = 2 * (tid % NCP), rg = tid / NCP;
    const int xm = (x0 - 1) & (N - 1), xq = (x0 + 2) & (N - 1);
    const int r0 = 1 + rg * RPG;
    const long long gb0 = static_cast<long long>(y0 + r0 - 1) * N;
    const long long gbm = static_cast<long long>((y0 + r0 - 2) & (N - 1)) * N;
    const long long gbp = static_cast<long long>((y0 + r0 - 1 + RPG) & (N - 1)) * N;
    auto goff = [&](int j) { return j < 0 ? gbm : (j >= RPG ? gbp : gb0 + static_cast<long long>(j) * N); };
    auto lds = [&](const double* S, int j, double* w) {
      const double* row = S + (r0 + j) * N;
      const double2 c = *reinterpret_cast<const double2*>(row + x0);
      w[0] = row[xm];
      w[1] = c.x;
      w[2] = c.y;
      w[3] = row[xq];
    };
    auto ldg = [&](const double* G, int j, double* w) {
      const double* row = G + goff(j);
      const double2 c = __ldg(reinterpret_cast<const double2*>(row + x0));
      w[0] = __ldg(row + xm);
      w[1] = c.x;
      w[2] = c.y;
      w[3] = __ldg(row + xq);
    };
    double2 rc[RPG];
    const long long g0 = off + gb0 + x0;
    auto sweep = [&](const double* S, const double* G, auto pass_c) {
      constexpr int pass = decltype(pass_c)::value;
      double ws[3][4], wg[3][4];  // 3-slot rings (base rows are L1-prefetched)
      lds(S, -1, ws[0]);
      lds(S, 0, ws[1]);
      ldg(G, -1, wg[0]);
      ldg(G, 0, wg[1]);
      double2 dn[2] = {}, an[2] = {};
      auto rkload = [&](int j) {  // RK state of owned row j, one row ahead
        const long long g = g0 + static_cast<long long>(j) * N;
        if (stage >= 1 && stage <= 2) dn[j & 1] = *reinterpret_cast<const double2*>(p.d + g);
        // (fused TLM: stage 1 rebuilds the accumulator from d and its input)
        if (stage >= 2) an[j & 1] = *reinterpret_cast<const double2*>(p.acc + g);
      };
      if (MODE == kModeTlm && pass == 1) rkload(0);
#pragma unroll
      for (int q = 0; q < RPG; ++q) {
        const int s0 = q % 3, s1 = (q + 1) % 3, s2 = (q + 2) % 3;
        lds(S, q + 1, ws[s2]);
        ldg(G, q + 1, wg[s2]);
        if (MODE == kModeTlm && pass == 1 && q + 1 < RPG) rkload(q + 1);
        double kk[2];
        {
          // rows -1, 0, +1 of the field and base windows (ring slots renamed)
          const double Wr[3][4] = {{ws[s0][0], ws[s0][1], ws[s0][2], ws[s0][3]},
                                   {ws[s1][0], ws[s1][1], ws[s1][2], ws[s1][3]},
                                   {ws[s2][0], ws[s2][1], ws[s2][2], ws[s2][3]}};
          const double Br[3][4] = {{wg[s0][0], wg[s0][1], wg[s0][2], wg[s0][3]},
                                   {wg[s1][0], wg[s1][1], wg[s1][2], wg[s1][3]},
                                   {wg[s2][0], wg[s2][1], wg[s2][2], wg[s2][3]}};
          double jj[2];  // 12 h^2 J(base, field) at the two columns
          arakawa12_pair(Br, Wr, jj);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double lap = Wr[1][c] + Wr[1][c + 2] + Wr[0][c + 1] + Wr[2][c + 1] - 4.0 * Wr[1][c + 1];
            // TLM A: J(psi_b, X) + nu Lap X;  B: + J(P, omega_b) = - J(omega_b, P)
            // ADJ A: -J(psi_b, a) + nu Lap a;  B: -J(a, omega_b) = + J(omega_b, a)
            if (MODE == kModeAdj) kk[c] = pass == 0 ? fma(-jj[c], js, nls * lap) : jj[c] * js;
            else if (pass == 0) kk[c] = fma(jj[c], js, nls * lap);
            else kk[c] = fma(-jj[c], js, c ? rc[q].y : rc[q].x);
          }
        }
        if (MODE == kModeAdj) {
          // A: q_out = -J(psi_b, a) + nu Lap a (non-Poisson part of mu);
          // B: -J(a, omega_b), the next Poisson input
          if (pass == 0) *reinterpret_cast<double2*>(p.q_out + g0 + static_cast<long long>(q) * N) = make_double2(kk[0], kk[1]);
          else rc[q] = make_double2(kk[0], kk[1]);
        } else if (pass == 0) {
          rc[q] = make_double2(kk[0], kk[1]);
        } else {
          const long long g = g0 + static_cast<long long>(q) * N;
          // stage 0: x_in is d itself, already in the X tile
          const double2 dcur = stage == 0 ? *reinterpret_cast<const double2*>(X + (r0 + q) * N + x0) : dn[q & 1];
          const double2 acur = an[q & 1];
          double2 out;
          if (stage == 0) {
            // no accumulator write: with x1 = d + dt/2 k1 (this stage's
            // output), d + dt/6 k1 = (2 d + x1) / 3, rebuilt in stage 1
            out = make_double2(dcur.x + 0.5 * dt * kk[0], dcur.y + 0.5 * dt * kk[1]);
            *reinterpret_cast<double2*>(p.x_out + g) = out;
          } else if (stage == 1) {
            const double2 x1 = *reinterpret_cast<const double2*>(X + (r0 + q) * N + x0);  // this stage's input
            // (times 1/3, not a division: an fp64 divide is ~12 instructions per point)
            constexpr double kThird = 1.0 / 3.0;
            const double2 a1 = make_double2((2.0 * dcur.x + x1.x) * kThird, (2.0 * dcur.y + x1.y) * kThird);
            *reinterpret_cast<double2*>(p.acc + g) = make_double2(a1.x + dt / 3.0 * kk[0], a1.y + dt / 3.0 * kk[1]);
            out = make_double2(dcur.x + 0.5 * dt * kk[0], dcur.y + 0.5 * dt * kk[1]);
            *reinterpret_cast<double2*>(p.x_out + g) = out;
          } else if (stage == 2) {
            *reinterpret_cast<double2*>(p.acc + g) = make_double2(acur.x + dt / 3.0 * kk[0], acur.y + dt / 3.0 * kk[1]);
            out = make_double2(dcur.x + dt * kk[0], dcur.y + dt * kk[1]);
            *reinterpret_cast<double2*>(p.x_out + g) = out;
          } else {
            out = make_double2(acur.x + dt / 6.0 * kk[0], acur.y + dt / 6.0 * kk[1]);
            *reinterpret_cast<double2*>(p.d + g) = out;
          }
          rc[q] = out;
        }
      }
    };
    constexpr bool kTlmTail = kTail && MODE == kModeTlm;
    if constexpr (kTlmTail) {
      if (has_prev && !(p.flags & kFlagSkipInvFft) && team == 0)
        pair_fft(C::kTeams, true, std::integral_constant<int, 1>{});
    }
    if (!(p.flags & kFlagSkipStencil)) {
      if (pf) prefetch_rows<N, true>(p.base_w, y0 - 1, R, tid, kThreads);
      sweep(X, p.base_p, std::integral_constant<int, 0>{});
      if constexpr (kTlmTail) __syncthreads();  // tail pair rows of P complete
      // ADJ: both sweeps walk X; a barrier keeps the compiler from merging
      // them into one schedule with both windows live (register spills)
      if constexpr (MODE == kModeAdj) __syncthreads();
      sweep(MODE == kModeTlm ? P : X, p.base_w, std::integral_constant<int, 1>{});
    } else {
      if constexpr (kTlmTail) __syncthreads();
#pragma unroll
      for (int q = 0; q < RPG; ++q) rc[q] = make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RPG; ++q) *reinterpret_cast<double2*>(P + (r0 + q) * N + x0) = rc[q];
    __syncthreads();
  } else {
  // Phase 3: stencils + RK update on owned rows. Each thread walks kCPT
  // columns of kRPG rows with a 3x3 sliding window per field (3 new loads per
  // field per row).
  const double js = p.inv12h2, ls = p.invh2, nu = p.nu, dt = p.dt;
  const int xt = tid % C::kNCT, rg = tid / C::kNCT;
  const int r0 = 1 + rg * C::kRPG;  // first owned smem row of this group
  double res[C::kCPT][C::kRPG] = {};
  // TLM: two sweeps per column strip, each with one shared-memory window
  // (X or P) and one global base-field window (L1-prefetched):
  //   A: J(psi_b, X) + nu Lap X          B: + J(P, omega_b), RK4 update
  // Windows are 4-slot rings indexed by the (unrolled, compile-time) row, so
  // advancing a row renames registers instead of moving them; owned-row
  // global addresses are one base pointer plus compile-time row offsets.
  // NL: one smem-only sweep J(P, X) + nu Lap X with the RK4 update.
  // Global row j (relative to the first owned row of this thread) of a field;
  // only j = -1 and j = kRPG can wrap periodically.
  const long long grow0 = static_cast<long long>(y0 + r0 - 1) * N;
  const long long grow_m = static_cast<long long>((y0 + r0 - 2) & (N - 1)) * N;
  const long long grow_p = static_cast<long long>((y0 + r0 - 1 + C::kRPG) & (N - 1)) * N;
  auto grow_off = [&](int j) { return j < 0 ? grow_m : (j >= C::kRPG ? grow_p : grow0 + static_cast<long long>(j) * N); };
  auto sweep = [&](int cc, const double* S, const double* G, auto pass_c, double(&rc)[C::kRPG]) {
    constexpr int pass = decltype(pass_c)::value;
    const int x = xt + cc * C::kNCT;
    const int xm = (x - 1) & (N - 1), xp = (x + 1) & (N - 1);
    const double* S0 = S + r0 * N;
    double ws[4][3], wg[4][3];
    auto srow = [&](int j, double* w) {
      const double* row = S0 + j * N;
      w[0] = row[xm];
      w[1] = row[x];
      w[2] = row[xp];
    };
    auto grow = [&](int j, double* w) {
      const double* row = G + grow_off(j);
      w[0] = __ldg(row + xm);
      w[1] = __ldg(row + x);
      w[2] = __ldg(row + xp);
    };
    // RK state of owned row j (pass B), prefetched one row ahead
    const long long g0 = off + grow0 + x;
    double dn[2] = {0.0, 0.0}, an[2] = {0.0, 0.0};
    auto rkload = [&](int j) {  // (stage 0 reads d from the X tile instead)
      if (stage >= 1 && stage <= 2) dn[j & 1] = p.d[g0 + static_cast<long long>(j) * N];
      if (stage >= 1) an[j & 1] = p.acc[g0 + static_cast<long long>(j) * N];
    };
    srow(-1, ws[0]);
    srow(0, ws[1]);
    grow(-1, wg[0]);
    grow(0, wg[1]);
    grow(1, wg[2]);
    if (pass == 1) rkload(0);
#pragma unroll
    for (int q = 0; q < C::kRPG; ++q) {
      const int sa = q & 3, sb = (q + 1) & 3, sc = (q + 2) & 3, sd = (q + 3) & 3;
      srow(q + 1, ws[sc]);
      if (q + 2 <= C::kRPG) grow(q + 2, wg[sd]);
      if (pass == 1 && q + 1 < C::kRPG) rkload(q + 1);
      const double W[3][3] = {{ws[sa][0], ws[sa][1], ws[sa][2]},
                              {ws[sb][0], ws[sb][1], ws[sb][2]},
                              {ws[sc][0], ws[sc][1], ws[sc][2]}};
      const double B[3][3] = {{wg[sa][0], wg[sa][1], wg[sa][2]},
                              {wg[sb][0], wg[sb][1], wg[sb][2]},
                              {wg[sc][0], wg[sc][1], wg[sc][2]}};
      if (pass == 0) {
        rc[q] = arakawa12(B, W) * js + nu * lap5(W) * ls;
      } else {
        const long long g = g0 + static_cast<long long>(q) * N;
        const double kk = rc[q] + arakawa12(W, B) * js;
        // stage 0: x_in is d itself, already in the X tile
        const double dcur = stage == 0 ? X[(r0 + q) * N + x] : dn[q & 1];
        const double acur = an[q & 1];
        double out;
        if (stage == 0) {
          p.acc[g] = dcur + dt / 6.0 * kk;
          out = dcur + 0.5 * dt * kk;
          p.x_out[g] = out;
        } else if (stage == 1) {
          p.acc[g] = acur + dt / 3.0 * kk;
          out = dcur + 0.5 * dt * kk;
          p.x_out[g] = out;
        } else if (stage == 2) {
          p.acc[g] = acur + dt / 3.0 * kk;
          out = dcur + dt * kk;
          p.x_out[g] = out;
        } else {
          out = acur + dt / 6.0 * kk;
          p.d[g] = out;
        }
        rc[q] = out;
      }
    }
  };
  if (!(p.flags & kFlagSkipStencil)) {
    if (MODE == kModeTlm) {
      // all A sweeps (base psi_b), then all B sweeps (base omega_b): one base
      // tile is walked at a time, the other streams into L1 meanwhile
      if (pf) prefetch_rows<N, true>(p.base_w, y0 - 1, R, tid, kThreads);
#pragma unroll
      for (int cc = 0; cc < C::kCPT; ++cc) sweep(cc, X, p.base_p, std::integral_constant<int, 0>{}, res[cc]);
#pragma unroll
      for (int cc = 0; cc < C::kCPT; ++cc) sweep(cc, P, p.base_w, std::integral_constant<int, 1>{}, res[cc]);
    } else if (MODE == kModeAdj) {
      // one sweep, one smem window (a) and two prefetched base windows
#pragma unroll 1
      for (int cc = 0; cc < C::kCPT; ++cc) {
        const int x = xt + cc * C::kNCT;
        const int xm = (x - 1) & (N - 1), xp = (x + 1) & (N - 1);
        const double* S0 = X + r0 * N;
        auto srow = [&](int j, double* w) {
          const double* row = S0 + j * N;
          w[0] = row[xm];
          w[1] = row[x];
          w[2] = row[xp];
        };
        auto grow = [&](const double* G, int j, double* w) {
          const double* row = G + grow_off(j);
          w[0] = __ldg(row + xm);
          w[1] = __ldg(row + x);
          w[2] = __ldg(row + xp);
        };
        // 4-slot ring windows (row j in slot (j+1) & 3), see the TLM sweep
        double wa[4][3], bp[4][3], bw[4][3];
        srow(-1, wa[0]);
        srow(0, wa[1]);
        grow(p.base_p, -1, bp[0]);
        grow(p.base_p, 0, bp[1]);
        grow(p.base_p, 1, bp[2]);
        grow(p.base_w, -1, bw[0]);
        grow(p.base_w, 0, bw[1]);
        grow(p.base_w, 1, bw[2]);
        const long long g0 = off + grow0 + x;
#pragma unroll
        for (int q = 0; q < C::kRPG; ++q) {
          const int sa = q & 3, sb = (q + 1) & 3, sc = (q + 2) & 3, sd = (q + 3) & 3;
          srow(q + 1, wa[sc]);
          if (q + 2 <= C::kRPG) {
            grow(p.base_p, q + 2, bp[sd]);
            grow(p.base_w, q + 2, bw[sd]);
          }
          const double A[3][3] = {{wa[sa][0], wa[sa][1], wa[sa][2]},
                                  {wa[sb][0], wa[sb][1], wa[sb][2]},
                                  {wa[sc][0], wa[sc][1], wa[sc][2]}};
          const double BP[3][3] = {{bp[sa][0], bp[sa][1], bp[sa][2]},
                                   {bp[sb][0], bp[sb][1], bp[sb][2]},
                                   {bp[sc][0], bp[sc][1], bp[sc][2]}};
          const double BW[3][3] = {{bw[sa][0], bw[sa][1], bw[sa][2]},
                                   {bw[sb][0], bw[sb][1], bw[sb][2]},
                                   {bw[sc][0], bw[sc][1], bw[sc][2]}};
          p.q_out[g0 + static_cast<long long>(q) * N] = -arakawa12(BP, A) * js + nu * lap5(A) * ls;
          const double out = -arakawa12(A, BW) * js;
          if (cc == 0) res[0][q] = out;
          else res[C::kCPT - 1][q] = out;
        }
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < C::kCPT; ++cc) {
        const int x = xt + cc * C::kNCT;
        const int xs[3] = {(x - 1) & (N - 1), x, (x + 1) & (N - 1)};
        double wx[3][3], wp[3][3];
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            wx[dy][c] = X[(r0 - 1 + dy) * N + xs[c]];
            wp[dy][c] = P[(r0 - 1 + dy) * N + xs[c]];
          }
#pragma unroll
        for (int q = 0; q < C::kRPG; ++q) {
          const int r = r0 + q;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            wx[2][c] = X[(r + 1) * N + xs[c]];
            wp[2][c] = P[(r + 1) * N + xs[c]];
          }
          const int gy = (y0 + r - 1) & (N - 1);
          const long long g = off + static_cast<long long>(gy) * N + x;
          if (p.store_w) {
            p.store_w[static_cast<long long>(gy) * N + x] = wx[1][1];
            p.store_p[static_cast<long long>(gy) * N + x] = wp[1][1];
          }
          const double kk = arakawa12(wp, wx) * js + nu * lap5(wx) * ls;
          double out;
          switch (p.stage) {
            case 0: {
              const double d = p.d[g];
              p.acc[g] = d + dt / 6.0 * kk;
              out = d + 0.5 * dt * kk;
              p.x_out[g] = out;
              break;
            }
            case 1: {
              const double d = p.d[g];
              p.acc[g] += dt / 3.0 * kk;
              out = d + 0.5 * dt * kk;
              p.x_out[g] = out;
              break;
            }
            case 2: {
              const double d = p.d[g];
              p.acc[g] += dt / 3.0 * kk;
              out = d + dt * kk;
              p.x_out[g] = out;
              break;
            }
            default: {
              out = p.acc[g] + dt / 6.0 * kk;
              p.d[g] = out;
              break;
            }
          }
          res[cc][q] = out;
          shift3(wx);
          shift3(wp);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int cc = 0; cc < C::kCPT; ++cc)
#pragma unroll
    for (int q = 0; q < C::kRPG; ++q) P[(r0 + q) * N + xt + cc * C::kNCT] = res[cc][q];
  __syncthreads();

  }

  // The successor (PDL launches only) may be scheduled from here: it starts
  // while this launch runs its last phase and waits for its completion.
  // Small-block variants (T < 8) leave it to the implicit trigger at exit: their
  // column-pass successor, scheduled early, lands on the few SMs with room
  // left and runs there unbalanced (512^2, one vector: 16.2 vs 11.1 us).
  if (T == 8) pdl_trigger();
  // Phase 4: forward x-FFT of the owned rows -> next row spectra.
  constexpr int kOwnPairs = T / 2;
  if constexpr (FUS) {
    if (p.flags & kFlagSkipFwdFft) return;
    // in place per pair region (rows 1+2pr, 2+2pr of P); T = 8 rows are one
    // round (kTeams >= 4 for every N <= 512)
    static_assert(kOwnPairs <= C::kTeams, "fused path: one forward FFT round");
    {
      const int pr = team;
      const bool act = pr < kOwnPairs;
      const double* pa = P + (1 + 2 * pr) * N;
      double2* buf = reinterpret_cast<double2*>(P + (1 + 2 * pr) * N);
      auto load = [&](int i) { return make_double2(pa[i], pa[i + N]); };
      auto store = [&](int i, double2 z) { buf[fswz(i)] = z; };
      fft_team<N, false, 0, true, -1, true>(buf, tw, t, act, load, store);
      __syncthreads();
    }
    // Tile-local y-recurrences of the next Poisson solve, per x-mode kx
    // (thread kx unpacks the two real rows of each pair from Z(kx), Z(N-kx)):
    // F_o = w_o + rho F_{o-1} (F_{-1} = 0), L = F_{T-1};
    // H_o = F_o + rho H_{o+1} (H_T = 0). Column kx = 0 is stored raw
    // (packed X(0) + i X(N/2)).
    constexpr int Q = N / T;
    for (int kx = tid; kx < N / 2; kx += kThreads) {
      double2 w[T];
#pragma unroll
      for (int pr = 0; pr < kOwnPairs; ++pr) {
        const double2* z = reinterpret_cast<const double2*>(P + (1 + 2 * pr) * N);
        if (kx == 0) {
          const double2 z0 = z[0], zn = z[fswz(N / 2)];
          w[2 * pr] = make_double2(z0.x, zn.x);
          w[2 * pr + 1] = make_double2(z0.y, zn.y);
        } else {
          const double2 zk = z[fswz(kx)], zm = z[fswz(N - kx)];
          w[2 * pr] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
          w[2 * pr + 1] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        }
      }
      double2* out = p.s_out + soff + static_cast<long long>(y0) * (N / 2) + kx;
      if (kx != 0 && !(p.flags & kFlagNoRecur)) {
        const double rho = p.stab[kx].x;
        double2 f = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < T; ++o) {
          f = make_double2(fma(rho, f.x, w[o].x), fma(rho, f.y, w[o].y));
          w[o] = f;
        }
        p.lsum[(v * Q + blockIdx.x) * (N / 2) + kx] = f;
        double2 g = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = T - 1; o >= 0; --o) {
          g = make_double2(fma(rho, g.x, w[o].x), fma(rho, g.y, w[o].y));
          w[o] = g;
        }
      }
#pragma unroll
      for (int o = 0; o < T; ++o) out[static_cast<long long>(o) * (N / 2)] = w[o];
    }
    if constexpr (MODE == kModeTlm) {
      // fused observation gather (stage 3 at an interval end): this CTA wrote
      // the new state of its own rows in sweep B
      if (stage == 3 && p.obs_y) {
        __syncthreads();
        const int o0 = p.obs_tile[blockIdx.x], o1 = p.obs_tile[blockIdx.x + 1];
        for (int o = o0 + tid; o < o1; o += kThreads) p.obs_y[v * p.obs_m + o] = p.d[off + p.obs_idx[o]] * p.obs_w[o];
      }
    }
    return;
  }
#pragma unroll 1
  for (int b0 = 0; b0 < ((p.flags & kFlagSkipFwdFft) ? 0 : kOwnPairs); b0 += C::kTeams) {
    const int pr = b0 + team;
    const bool act = pr < kOwnPairs;
    const double* pa = P + (1 + 2 * pr) * N;
    auto load = [&](int i) { return make_double2(pa[i], pa[i + N]); };
    auto store = [&](int i, double2 z) { fbuf[fpad(i)] = z; };
    fft_team<N, false>(fbuf, tw, t, act, load, store);
    __syncthreads();
    if (act) {
      double2* ra = p.s_out + soff + static_cast<long long>(y0 + 2 * pr) * (N / 2);
      pack_pair<N>(fbuf, ra, ra + N / 2, t, C::kTeam);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ obs kernels --
__global__ void gather_obs_kernel(const double* __restrict__ f, long long dim, const long long* __restrict__ idx,
                                  int n_obs, const double* __restrict__ w, double* __restrict__ y, long long m,
                                  int nvec) {
  pdl_wait();
  pdl_trigger();
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<long long>(n_obs) * nvec) return;
  const int v = static_cast<int>(e / n_obs), k = static_cast<int>(e % n_obs);
  y[v * m + k] = f[v * dim + idx[k]] * w[k];
}
__global__ void scatter_obs_kernel(double* __restrict__ f, long long dim, const long long* __restrict__ idx,
                                   int n_obs, const double* __restrict__ w, const double* __restrict__ y, long long m,
                                   int nvec) {
  pdl_wait();
  pdl_trigger();
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<long long>(n_obs) * nvec) return;
  const int v = static_cast<int>(e / n_obs), k = static_cast<int>(e % n_obs);
  f[v * dim + idx[k]] += y[v * m + k] * w[k];
}

// ---------------------------------------------------------------- launchers --
// 8-row stage CTAs below which a sweep lane counts as a small block. Measured
// on B200 (tools/small_block.py, profiles/r2_small_blocks.md): the fused path
// (8-row tiles + carry pass) beats the 2-row small-block path from 128 CTAs
// per lane on every grid (512^2: 2 vectors, 256^2: 4, 128^2: 8), well below
// the 296 CTA slots of one wave. SDV_FILL overrides (experiments).
int bve_stage_fill() {
  static const int f = [] {
    const char* e = std::getenv("SDV_FILL");
    return e ? std::max(1, std::atoi(e)) : 128;
  }();
  return f;
}

namespace {
template <int N>
struct Launch {
  using C = Cfg<N>;
  // Small-block variants: when the 8-row / kCW-column grids would not fill
  // the 148 SMs (PCG and line-search sweeps run one vector), use 2-row stage
  // tiles and 1-column col CTAs (more, shorter CTAs: lower per-stage latency).
  static constexpr int kSmallT = N >= 128 ? 2 : 8;
  using CS = Cfg<N, kSmallT>;
  static constexpr int kFill = 2 * 148;
  static bool small_stage(int nvec) { return (N / C::kT) * nvec < bve_stage_fill(); }
  static bool small_col(int nvec) { return ((N / 2) / C::kCW) * nvec < kFill; }
  template <class K>
  static void smem_attr(K k, size_t bytes) {
    SDV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  }
  static void setup() {
    static const bool once = [] {  // thread-safe one-time kernel attributes (magic static)
      setup_once();
      return true;
    }();
    (void)once;
  }
  static void setup_once() {
    stage_attrs<8>(std::make_integer_sequence<int, 4>{});
    stage_attrs<kSmallT>(std::make_integer_sequence<int, 4>{});
    if constexpr (N >= 64) fused_attrs(std::make_integer_sequence<int, 4>{});
    smem_attr(col_kernel<N, C::kCW>, C::kColSmem);
    smem_attr(col_kernel<N, 1>, Cfg<N, 8, 1>::kColSmem);
    smem_attr(row_fwd_kernel<N>, C::kRowSmem);
    smem_attr(row_inv_kernel<N>, C::kRowSmem);
  }
  static void row_fwd(const double* f, double2* s, int nvec, cudaStream_t st) {
    setup();
    dim3 g(ceil_div(N / 2, C::kTeams), nvec);
    launch_pdl(row_fwd_kernel<N>, g, kThreads, C::kRowSmem, st, f, s, twiddle_table(N));
  }
  static void row_inv(const double2* s, double* f, int nvec, cudaStream_t st) {
    setup();
    dim3 g(ceil_div(N / 2, C::kTeams), nvec);
    launch_pdl(row_inv_kernel<N>, g, kThreads, C::kRowSmem, st, s, f, twiddle_table(N));
  }
  static void col(double2* s, const double* sym, int nvec, cudaStream_t st) {
    setup();
    count_path(kPathBveColFft);
    if (small_col(nvec)) {
      launch_pdl(col_kernel<N, 1>, dim3(N / 2, nvec), C::kTeam, Cfg<N, 8, 1>::kColSmem, st, s, sym,
                 twiddle_table(N));
    } else {
      launch_pdl(col_kernel<N, C::kCW>, dim3((N / 2) / C::kCW, nvec), C::kCW * C::kTeam, C::kColSmem, st, s, sym,
                 twiddle_table(N));
    }
  }
  // Poisson column pass: kx >= 1 by the recurrence solver, kx = 0 (packed,
  // singular) by the FFT column kernel on that one column.
  static void col_solve(double2* s, const double4* tab, const double* sym, int nvec, cudaStream_t st) {
    setup();
    // Small blocks (PCG / line-search sweeps, one vector): the solver's N/16+1
    // CTAs per vector would leave most SMs idle; the 1-column FFT kernel has
    // N/2 CTAs per vector.
    if (small_col(nvec)) return col(s, sym, nvec, st);
    count_path(kPathBveColSolve);
    launch_pdl(col_solve_kernel<N>, dim3((N / 2) / 8 + 1, nvec), 256, Cfg<N, 8, 1>::kColSmem, st, s, tab, sym,
               twiddle_table(N));
  }
  // fused Poisson path: 8-row tiles, P + X only (the x-FFTs run in place)
  static constexpr size_t kFusSmem = 2 * Cfg<N, 8>::kTileBytes;
  template <int... S>
  static void fused_attrs(std::integer_sequence<int, S...>) {
    (smem_attr(stage_kernel<N, kModeTlm, 8, S, true>, kFusSmem), ...);
    (smem_attr(stage_kernel<N, kModeAdj, 8, S, true>, kFusSmem), ...);
    if constexpr (kLite) {
      (smem_attr(stage_kernel<N, kModeTlm, kSmallT, S, true>, kLiteSmem), ...);
      (smem_attr(stage_kernel<N, kModeAdj, kSmallT, S, true>, kLiteSmem), ...);
    }
  }
  // lite path: the two-column stencil mapping needs N/2 >= 256/T column pairs
  static constexpr bool kLite = N >= 256;
  static constexpr size_t kLiteSmem = 2 * Cfg<N, kSmallT>::kTileBytes;
  static void stage_lite(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    if constexpr (kLite) {
      setup();
      count_path(kPathBveStageLite);
      const dim3 g(N / kSmallT, nvec), b(kThreads);
      const bool tlm = mode == kModeTlm;
      switch (a.stage) {
        case 0: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, kSmallT, 0, true> : stage_kernel<N, kModeAdj, kSmallT, 0, true>, g, b, kLiteSmem, st, a);
        case 1: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, kSmallT, 1, true> : stage_kernel<N, kModeAdj, kSmallT, 1, true>, g, b, kLiteSmem, st, a);
        case 2: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, kSmallT, 2, true> : stage_kernel<N, kModeAdj, kSmallT, 2, true>, g, b, kLiteSmem, st, a);
        default: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, kSmallT, 3, true> : stage_kernel<N, kModeAdj, kSmallT, 3, true>, g, b, kLiteSmem, st, a);
      }
    } else {
      throw std::invalid_argument("bve_stage_lite: needs n >= 256");
    }
  }
  static void stage_fused(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    if constexpr (N < 64) {
      throw std::invalid_argument("bve_stage: the fused path needs n >= 64");
    } else {
      stage_fused_impl(mode, a, nvec, st);
    }
  }
  static void stage_fused_impl(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    setup();
    count_path(kPathBveStageFused);
    const dim3 g(N / 8, nvec), b(kThreads);
    const bool tlm = mode == kModeTlm;
    if (mode == kModeNl) throw std::invalid_argument("bve_stage: the fused path covers TLM/ADJ");
    switch (a.stage) {
      case 0: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, 8, 0, true> : stage_kernel<N, kModeAdj, 8, 0, true>, g, b, kFusSmem, st, a);
      case 1: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, 8, 1, true> : stage_kernel<N, kModeAdj, 8, 1, true>, g, b, kFusSmem, st, a);
      case 2: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, 8, 2, true> : stage_kernel<N, kModeAdj, 8, 2, true>, g, b, kFusSmem, st, a);
      default: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, 8, 3, true> : stage_kernel<N, kModeAdj, 8, 3, true>, g, b, kFusSmem, st, a);
    }
  }
  static void carry(double2* s, const double2* lsum, double2* cc, double2* ce, const double4* tab, const double* sym,
                    int nvec, cudaStream_t st) {
    setup();
    if constexpr (N >= 64) {
      count_path(kPathBveCarry);
      launch_pdl(carry_kernel<N>, dim3(ceil_div(N / 2, 32) + 1, nvec), 256, 0, st, s, lsum, cc, ce, tab);
    } else {
      throw std::invalid_argument("bve_carry: the fused path needs n >= 64");
    }
  }
  template <int T>
  static void stage_t(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    using CT = Cfg<N, T>;
    const dim3 g(N / T, nvec), b(kThreads);
    const size_t sm = CT::kStageSmem;
    if (mode == kModeNl) return launch_pdl(stage_kernel<N, kModeNl, T>, g, b, sm, st, a);
    // TLM / ADJ: the RK stage is a template constant (no per-point branches)
    const bool tlm = mode == kModeTlm;
    switch (a.stage) {
      case 0: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, T, 0> : stage_kernel<N, kModeAdj, T, 0>, g, b, sm, st, a);
      case 1: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, T, 1> : stage_kernel<N, kModeAdj, T, 1>, g, b, sm, st, a);
      case 2: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, T, 2> : stage_kernel<N, kModeAdj, T, 2>, g, b, sm, st, a);
      default: return launch_pdl(tlm ? stage_kernel<N, kModeTlm, T, 3> : stage_kernel<N, kModeAdj, T, 3>, g, b, sm, st, a);
    }
  }
  template <int T, int... S>
  static void stage_attrs(std::integer_sequence<int, S...>) {
    const size_t sm = Cfg<N, T>::kStageSmem;
    (smem_attr(stage_kernel<N, kModeTlm, T, S>, sm), ...);
    (smem_attr(stage_kernel<N, kModeAdj, T, S>, sm), ...);
    smem_attr(stage_kernel<N, kModeNl, T>, sm);
  }
  static void stage(int mode, const StageArgs& a, int nvec, cudaStream_t st) {
    setup();
    count_path(kPathBveStagePlain);
    if (small_stage(nvec)) stage_t<kSmallT>(mode, a, nvec, st);
    else stage_t<8>(mode, a, nvec, st);
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
void bve_col_solve(int n, double2* s, const double4* tab, const double* sym, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::col_solve(s, tab, sym, nvec, st); });
}
void bve_stage(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st, bool fused) {
  dispatch_n(n, [&](auto c) {
    constexpr int NN = decltype(c)::value;
    if (fused && (NN < 64 || Launch<NN>::small_stage(nvec)))
      throw std::invalid_argument("bve_stage: block too small for the fused path");
    if (fused) Launch<decltype(c)::value>::stage_fused(mode, a, nvec, st);
    else Launch<decltype(c)::value>::stage(mode, a, nvec, st);
  });
}
bool bve_fused_ok(int n, int nvec) {
  if (n < 64 || std::getenv("SDV_NO_FUSE")) return false;
  bool ok = false;
  dispatch_n(n, [&](auto c) { ok = !Launch<decltype(c)::value>::small_stage(nvec); });
  return ok;
}
bool bve_lite_ok(int n, int nvec) {
  if (n < 256 || nvec < 1 || std::getenv("SDV_NO_LITE")) return false;
  bool small = false;
  dispatch_n(n, [&](auto c) { small = Launch<decltype(c)::value>::small_stage(nvec); });
  return small;
}
void bve_stage_lite(int n, int mode, const StageArgs& a, int nvec, cudaStream_t st) {
  if (!(a.flags & kFlagRawIn) || !(a.flags & kFlagNoRecur))
    throw std::invalid_argument("bve_stage_lite: needs kFlagRawIn | kFlagNoRecur");
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::stage_lite(mode, a, nvec, st); });
}
void bve_carry(int n, double2* s, const double2* lsum, double2* car_c, double2* car_e, const double4* tab,
               const double* sym, int nvec, cudaStream_t st) {
  dispatch_n(n, [&](auto c) { Launch<decltype(c)::value>::carry(s, lsum, car_c, car_e, tab, sym, nvec, st); });
}
void gather_obs(const double* f, long long dim, const long long* idx, int n_obs, const double* w, double* y,
                long long m, int nvec, cudaStream_t st) {
  const long long tot = static_cast<long long>(n_obs) * nvec;
  if (tot == 0) return;
  launch_pdl(gather_obs_kernel, ceil_div(tot, 256), 256, 0, st, f, dim, idx, n_obs, w, y, m, nvec);
}
void scatter_obs(double* f, long long dim, const long long* idx, int n_obs, const double* w, const double* y,
                 long long m, int nvec, cudaStream_t st) {
  const long long tot = static_cast<long long>(n_obs) * nvec;
  if (tot == 0) return;
  launch_pdl(scatter_obs_kernel, ceil_div(tot, 256), 256, 0, st, f, dim, idx, n_obs, w, y, m, nvec);
}

}  // namespace sdv

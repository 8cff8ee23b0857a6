// Cluster-resident TLM / ADJ sweeps of the periodic barotropic-vorticity model
// for small blocks (the PCG, line-search and probe regime: one or a few
// vectors per sweep), sm_100a.
//
// Replaces, for s <= a few vectors on grids up to 256^2, the per-stage launch
// pairs of the block path (bve_kernels.cu), whose cost at one vector is pure
// launch and grid-drain latency (~8 us per RK stage at 128^2). One thread-block
// cluster owns one vector for the whole sweep (reference: the per-vector
// BVETrajectory::tlm_range / adj_range loops, /root/reference/proj/src/bve.cpp:138-161,
// run by pcg_solve through GramMap, proj/src/linalg.cpp:52-106):
//   * CTA rank q of the CL-CTA cluster holds rows [q TR, (q+1) TR) of the
//     RK state (d, accumulator, stage input, streamfunction) in shared memory
//     for all 4 * steps stages; only the base trajectory (global, L2) and the
//     observation gathers/scatters touch HBM;
//   * the Poisson solve per stage is the x-FFT (in place, swizzled, one round
//     of row pairs) + the y-recurrence solver of bve_col_solve split into
//     per-CTA segments: the CL segment end values are exchanged through
//     distributed shared memory and every CTA forms its own cyclic carries
//     (O(CL) per mode), so one cluster barrier per recurrence direction
//     replaces the column pass; the singular x-mode 0 (zero-mean periodic
//     second difference) is solved in closed form from per-segment moments
//     exchanged with the forward carries;
//   * stencil halo rows come from the neighbouring CTAs' shared memory.
// Three cluster barriers per RK stage.
#include <cooperative_groups.h>

#include "bve_kernels.cuh"
#include "fft.cuh"
#include "stencil.cuh"

namespace cg = cooperative_groups;

namespace sdv {

namespace {

constexpr int kCThreads = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

template <int N>
struct ClusterCfg {
  static constexpr int CL = N <= 64 ? 4 : (N == 128 ? 8 : 16);
  static constexpr int TR = N / CL;  // rows per CTA (16)
  static constexpr int NCT = N < kCThreads ? N : kCThreads;
  static constexpr int RG = kCThreads / NCT;
  static constexpr int RPG = TR / RG;
  static constexpr int KX = N / 2;
  static constexpr size_t kOwn = static_cast<size_t>(TR) * N;       // doubles
  static constexpr size_t kHalo = static_cast<size_t>(TR + 2) * N;  // doubles
  // D, A (own rows) + X, P and the two base-field tiles BP, BW (halo rows)
  static constexpr size_t kFields = 2 * kOwn + 4 * kHalo;
  static constexpr int kTw = N == 64 ? 56 : (N == 128 ? 120 : 248);  // fft_twiddle_count(N)
  static constexpr size_t kSmem =
      sizeof(double) * kFields + sizeof(double2) * 2 * KX + sizeof(double) * 4 + sizeof(double2) * kTw;
  static_assert(TR % 2 == 0 && TR * CL == N, "cluster tiling");
  static_assert((TR / 2) <= kCThreads / (N / 8), "one forward FFT round of row pairs");
  static_assert(KX <= kCThreads, "one x-mode per thread");
};

struct ClusterArgs {
  double* state = nullptr;       // [nvec][N][N]
  const double* base_w = nullptr;  // [steps][4][N^2] stored stage inputs
  const double* base_p = nullptr;  // [steps][4][N^2] their streamfunctions
  int k0 = 0, k1 = 0;
  const long long* idx = nullptr;
  int n_obs = 0;
  int spi = 1;
  const double* w = nullptr;  // R^{-1/2}, [n_t][n_obs]
  double* y = nullptr;        // [nvec][m] (TLM out / ADJ in), or null
  long long m = 0;
  const double4* tab = nullptr;
  const double2* tw = nullptr;
  double dt = 0, nu = 0, js = 0, ls = 0;
};

template <int N, int MODE>
__global__ void __launch_bounds__(kCThreads, 1) cluster_sweep_kernel(ClusterArgs a) {
  using C = ClusterCfg<N>;
  constexpr int CL = C::CL, TR = C::TR, KX = C::KX, NCT = C::NCT, RPG = C::RPG;
  constexpr int kTeam = N / 8;
  cg::cluster_group cl = cg::this_cluster();
  const int q = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x;
  const int team = tid / kTeam, t = tid % kTeam;
  const long long v = blockIdx.y;
  const long long dim = static_cast<long long>(N) * N;
  const int y0 = q * TR;  // first global row of this CTA

  extern __shared__ double smd[];
  double* D = smd;
  double* A = D + C::kOwn;
  double* X = A + C::kOwn;    // TLM stage input / ADJ a, then q (non-Poisson part of mu); rows y0-1 .. y0+TR
  double* P0 = X + C::kHalo;  // streamfunction / Poisson input, FFT buffers
  double* BP = P0 + C::kHalo; // base psi_b tile of the stage (cp.async)
  double* BW = BP + C::kHalo; // base omega_b tile of the stage
  double2* Lx = reinterpret_cast<double2*>(smd + C::kFields);  // segment forward end values
  double2* Vx = Lx + KX;                                          // segment backward start values
  double* Mo = reinterpret_cast<double*>(Vx + KX);                // x-mode 0 real-part moments s0, s1, s2
  // twiddles in shared memory: every cluster barrier (acquire) invalidates L1
  double2* TW = reinterpret_cast<double2*>(Mo + 4);
  for (int e = tid; e < C::kTw; e += kCThreads) TW[e] = a.tw[e];

  // load this CTA's rows of the vector
  double* gst = a.state + v * dim + static_cast<long long>(y0) * N;
  for (int e = tid; e < TR * N; e += kCThreads) D[e] = gst[e];
  if (MODE == kModeAdj)
    for (int e = tid; e < TR * N; e += kCThreads) A[e] = 0.0;
  __syncthreads();

  // x-mode constants of this thread (kx = tid)
  const int kx = tid;
  const bool kl = kx < KX;
  double rho = 0.0, scale = 0.0, clos = 0.0, rT = 0.0;
  if (kl) {
    const double4 tb = a.tab[kx];  // kx = 0: x-mode N/2 constants (imaginary part)
    rho = tb.x;
    clos = tb.z;
    scale = tb.w;
    rT = 1.0;
#pragma unroll
    for (int i = 0; i < TR; ++i) rT *= rho;
  }
  const double h2n = a.tab[0].y;  // h^2 / N (x-mode 0)

  // ---- Poisson solve of the TR own rows held as a physical field in the
  // pair regions of Pb rows 1..TR (in place): x-FFT, y-recurrences with
  // cluster-exchanged carries, inverse x-FFT. Two cluster barriers.
  auto poisson = [&](double* Pb) {
    // forward x-FFT per row pair (swizzled in place)
    {
      const int pr = team;
      const bool act = pr < TR / 2;
      double* pa = Pb + (1 + 2 * pr) * N;
      double2* buf = reinterpret_cast<double2*>(pa);
      auto load = [&](int i) { return make_double2(pa[i], pa[i + N]); };
      auto store = [&](int i, double2 z) { buf[fswz(i)] = z; };
      fft_team<N, false, 0, true, 0, true, true>(buf, TW, t, act, load, store);
    }
    __syncthreads();
    double2 f[TR];
    if (kl) {
#pragma unroll
      for (int pr = 0; pr < TR / 2; ++pr) {
        const double2* z = reinterpret_cast<const double2*>(Pb + (1 + 2 * pr) * N);
        if (kx == 0) {
          const double2 z0 = z[0], zn = z[fswz(N / 2)];
          f[2 * pr] = make_double2(z0.x, zn.x);
          f[2 * pr + 1] = make_double2(z0.y, zn.y);
        } else {
          const double2 zk = z[fswz(kx)], zm = z[fswz(N - kx)];
          f[2 * pr] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
          f[2 * pr + 1] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        }
      }
      if (kx == 0) {  // moments of the x-mode-0 (real) part of this segment
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int o = 0; o < TR; ++o) {
          s0 += f[o].x;
          s1 += o * f[o].x;
          s2 += static_cast<double>(o * o) * f[o].x;
        }
        Mo[0] = s0;
        Mo[1] = s1;
        Mo[2] = s2;
      }
      double2 g = make_double2(0.0, 0.0);  // zero-carry forward recurrence
#pragma unroll
      for (int o = 0; o < TR; ++o) {
        g = make_double2(fma(rho, g.x, f[o].x), fma(rho, g.y, f[o].y));
        if (kx != 0) f[o] = g;
        else f[o].y = g.y;
      }
      Lx[kx] = g;
    }
    cl.sync();  // (1) segment end values and moments visible
    double psi0[TR];
    if (kl) {
      // forward carry into this segment: C_q = clos sum_m rT^m L_{q-1-m}
      double2 c = make_double2(0.0, 0.0);
      double pw = 1.0;
#pragma unroll 4
      for (int m = 0; m < CL; ++m) {
        const double2 L = cl.map_shared_rank(Lx, (q - 1 - m + 2 * CL) % CL)[kx];
        c = make_double2(fma(pw, L.x, c.x), fma(pw, L.y, c.y));
        pw *= rT;
      }
      c = make_double2(clos * c.x, clos * c.y);
      pw = rho;
#pragma unroll
      for (int o = 0; o < TR; ++o) {
        if (kx != 0) f[o] = make_double2(fma(pw, c.x, f[o].x), fma(pw, c.y, f[o].y));
        else f[o].y = fma(pw, c.y, f[o].y);
        pw *= rho;
      }
      double2 g = make_double2(0.0, 0.0);  // zero-carry backward recurrence
#pragma unroll
      for (int o = TR - 1; o >= 0; --o) {
        g = make_double2(fma(rho, g.x, f[o].x), fma(rho, g.y, f[o].y));
        if (kx != 0) f[o] = g;
        else f[o].y = g.y;
      }
      Vx[kx] = g;
      if (kx == 0) {
        // x-mode 0: zero-mean pseudo-inverse of the periodic second
        // difference from the segment moments (see col0_warp_solve):
        // P_j = sum_{m<j} w'_m, S_j = sum_{i<=j} P_i, D0 = S_{N-1}/N,
        // psi_j = j D0 - S_j - mean(psi).
        double s0[CL], s1[CL], s2[CL], tot = 0.0;
#pragma unroll
        for (int p = 0; p < CL; ++p) {
          const double* mo = cl.map_shared_rank(Mo, p);
          s0[p] = mo[0];
          s1[p] = mo[1];
          s2[p] = mo[2];
          tot += s0[p];
        }
        const double mean = tot / N;
        double wq = 0.0, wmine = 0.0, sp_sum = 0.0, send_mine = 0.0, ni = 0.0;
#pragma unroll
        for (int p = 0; p < CL; ++p) {
          const double a0 = s0[p] - TR * mean;
          const double a1 = s1[p] - mean * (TR * (TR - 1) / 2);
          const double a2 = s2[p] - mean * ((TR - 1) * TR * (2 * TR - 1) / 6);
          const double sp = TR * wq + (TR - 1) * a0 - a1;
          if (p == q) {
            wmine = wq;
            send_mine = sp_sum;
          }
          const double nb = static_cast<double>(N - p * TR);
          ni += wq * (TR * nb - TR * (TR - 1) / 2) + nb * ((TR - 1) * a0 - a1) - (TR - 1) * TR / 2 * a0 + 0.5 * (a2 + a1);
          sp_sum += sp;
          wq += a0;
        }
        const double d0 = sp_sum / N;
        const double mpsi = (d0 * (0.5 * N * (N - 1)) - ni) / N;
        double pp = wmine, ss = send_mine;
#pragma unroll
        for (int o = 0; o < TR; ++o) {
          ss += pp;
          psi0[o] = h2n * (static_cast<double>(y0 + o) * d0 - ss - mpsi);
          pp += f[o].x - mean;
        }
      }
    }
    cl.sync();  // (2) segment backward start values visible
    if (kl) {
      // backward carry from above: E_q = clos sum_m rT^m V_{q+1+m}
      double2 e = make_double2(0.0, 0.0);
      double pw = 1.0;
#pragma unroll 4
      for (int m = 0; m < CL; ++m) {
        const double2 V = cl.map_shared_rank(Vx, (q + 1 + m) % CL)[kx];
        e = make_double2(fma(pw, V.x, e.x), fma(pw, V.y, e.y));
        pw *= rT;
      }
      e = make_double2(clos * e.x, clos * e.y);
      double pb = rho;
#pragma unroll
      for (int o = TR - 1; o >= 0; --o) {  // psi_o = scale (H_o + rho^(TR-o) E)
        f[o] = make_double2(scale * fma(pb, e.x, f[o].x), scale * fma(pb, e.y, f[o].y));
        if (kx == 0) f[o].x = psi0[o];
        pb *= rho;
      }
      // unpacked spectra z = a + i b of each row pair (inverse-FFT input)
#pragma unroll
      for (int pr = 0; pr < TR / 2; ++pr) {
        double2* z = reinterpret_cast<double2*>(Pb + (1 + 2 * pr) * N);
        const double2 ra = f[2 * pr], rb = f[2 * pr + 1];
        if (kx == 0) {
          z[0] = make_double2(ra.x, rb.x);
          z[N / 2] = make_double2(ra.y, rb.y);
        } else {
          z[kx] = make_double2(ra.x - rb.y, ra.y + rb.x);
          z[N - kx] = make_double2(ra.x + rb.y, rb.x - ra.y);
        }
      }
    }
    __syncthreads();
    {
      const int pr = team;
      const bool act = pr < TR / 2;
      double* pa = Pb + (1 + 2 * pr) * N;
      double2* buf = reinterpret_cast<double2*>(pa);
      auto load = [&](int i) { return buf[i]; };
      auto store = [&](int i, double2 z) {
        pa[i] = z.x;
        pa[i + N] = z.y;
      };
      fft_team<N, true, 0, true, 0, true, true>(buf, TW, t, act, load, store);
    }
    __syncthreads();
  };

  // halo rows (0 and TR+1) of a TR+2-row field: pull from the neighbouring
  // CTAs' own boundary rows, or push this CTA's boundary rows into theirs
  auto pull_halo = [&](double* F) {
    const double* up = cl.map_shared_rank(F, (q + CL - 1) % CL) + TR * N;  // its last own row
    const double* dn = cl.map_shared_rank(F, (q + 1) % CL) + N;           // its first own row
    for (int e = tid; e < N; e += kCThreads) {
      F[e] = up[e];
      F[(TR + 1) * N + e] = dn[e];
    }
  };
  auto push_halo = [&](double* F) {
    double* up = cl.map_shared_rank(F, (q + CL - 1) % CL) + (TR + 1) * N;  // its bottom halo row
    double* dn = cl.map_shared_rank(F, (q + 1) % CL);                       // its top halo row
    for (int e = tid; e < N; e += kCThreads) {
      up[e] = F[N + e];
      dn[e] = F[TR * N + e];
    }
  };
  // base-field tiles of stage (k, s): rows y0-1 .. y0+TR, async into BP/BW
  auto load_base = [&](int k, int s) {
    const double* bw = a.base_w + (static_cast<long long>(k) * 4 + s) * dim;
    const double* bp = a.base_p + (static_cast<long long>(k) * 4 + s) * dim;
    for (int e = 2 * tid; e < (TR + 2) * N; e += 2 * kCThreads) {
      const int r = e / N, xx = e % N;
      const long long go = static_cast<long long>((y0 - 1 + r) & (N - 1)) * N + xx;
      cp_async16(BP + e, bp + go);
      cp_async16(BW + e, bw + go);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  // stencil thread mapping: column x, rows r0 .. r0+RPG-1 (1-based in the
  // halo layout)
  const int x = tid % NCT, rg = tid / NCT;
  const int r0 = 1 + rg * RPG;
  const int xm = (x - 1) & (N - 1), xp = (x + 1) & (N - 1);
  auto srow = [&](const double* S, int r, double* w3) {
    const double* row = S + r * N;
    w3[0] = row[xm];
    w3[1] = row[x];
    w3[2] = row[xp];
  };
  auto win = [](const double (*ring)[3], int i0, int i1, int i2, double out[3][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[0][c] = ring[i0][c];
      out[1][c] = ring[i1][c];
      out[2][c] = ring[i2][c];
    }
  };

  const double dt = a.dt, nu = a.nu, js = a.js, ls = a.ls;
  const long long lo = static_cast<long long>(y0) * N, hi = lo + TR * N;  // own flat index range

  if constexpr (MODE == kModeTlm) {
    // stage-0 input of the first step: the state itself
    for (int e = tid; e < TR * N; e += kCThreads) X[N + e] = D[e];
    __syncthreads();
    for (int k = a.k0; k < a.k1; ++k) {
      for (int s = 0; s < 4; ++s) {
        load_base(k, s);  // lands under the Poisson solve
        for (int e = tid; e < TR * N; e += kCThreads) P0[N + e] = X[N + e];
        __syncthreads();
        poisson(P0);
        pull_halo(X);    // the neighbours' stage inputs are final until barrier (3)
        push_halo(P0);   // psi boundary rows into the neighbours' halo rows
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        cl.sync();  // (3) psi halos in place; X halo pulls of all CTAs done before any X write
        double xo[RPG];
        {
          double wx[3][3], wp[3][3], gp[3][3], gw[3][3];
          srow(X, r0 - 1, wx[0]);
          srow(X, r0, wx[1]);
          srow(P0, r0 - 1, wp[0]);
          srow(P0, r0, wp[1]);
          srow(BP, r0 - 1, gp[0]);
          srow(BP, r0, gp[1]);
          srow(BW, r0 - 1, gw[0]);
          srow(BW, r0, gw[1]);
#pragma unroll
          for (int j = 0; j < RPG; ++j) {
            const int i0 = j % 3, i1 = (j + 1) % 3, i2 = (j + 2) % 3;
            srow(X, r0 + j + 1, wx[i2]);
            srow(P0, r0 + j + 1, wp[i2]);
            srow(BP, r0 + j + 1, gp[i2]);
            srow(BW, r0 + j + 1, gw[i2]);
            double W[3][3], Pw[3][3], Bp[3][3], Bw[3][3];
            win(wx, i0, i1, i2, W);
            win(wp, i0, i1, i2, Pw);
            win(gp, i0, i1, i2, Bp);
            win(gw, i0, i1, i2, Bw);
            const double kk = arakawa12(Bp, W) * js + nu * lap5(W) * ls + arakawa12(Pw, Bw) * js;
            const int e = (r0 - 1 + j) * N + x;  // own-row index
            const double d = D[e];
            if (s == 0) {
              A[e] = d + dt / 6.0 * kk;
              xo[j] = d + 0.5 * dt * kk;
            } else if (s == 1) {
              A[e] += dt / 3.0 * kk;
              xo[j] = d + 0.5 * dt * kk;
            } else if (s == 2) {
              A[e] += dt / 3.0 * kk;
              xo[j] = d + dt * kk;
            } else {
              const double dn = A[e] + dt / 6.0 * kk;
              D[e] = dn;
              xo[j] = dn;
            }
          }
        }
        __syncthreads();  // all stencil reads of X done
#pragma unroll
        for (int j = 0; j < RPG; ++j) X[(r0 + j) * N + x] = xo[j];
        __syncthreads();
      }
      if (a.y && (k + 1) % a.spi == 0) {
        const int iv = (k + 1) / a.spi - 1;
        const double* w = a.w + static_cast<long long>(iv) * a.n_obs;
        double* yv = a.y + v * a.m + static_cast<long long>(iv) * a.n_obs;
        for (int o = tid; o < a.n_obs; o += kCThreads) {
          const long long g = a.idx[o];
          if (g >= lo && g < hi) yv[o] = D[g - lo] * w[o];
        }
      }
    }
  } else {
    // ---- adjoint sweep, steps k1-1 .. k0, stages 3..0
    bool first = true;
    for (int k = a.k1 - 1; k >= a.k0; --k) {
      if (a.y && (k + 1) % a.spi == 0) {
        const int iv = (k + 1) / a.spi - 1;
        const double* w = a.w + static_cast<long long>(iv) * a.n_obs;
        const double* yv = a.y + v * a.m + static_cast<long long>(iv) * a.n_obs;
        double* tgt = first ? D : A;
        for (int o = tid; o < a.n_obs; o += kCThreads) {
          const long long g = a.idx[o];
          if (g >= lo && g < hi) tgt[g - lo] += yv[o] * w[o];
        }
        __syncthreads();
      }
      for (int s = 3; s >= 0; --s) {
        const bool has_prev = !first;
        load_base(k, s);  // lands under the combination and the halo exchange
        // lambda / mu combination (pointwise on own rows; X holds q of the
        // previous stage, P0 the Poisson part) -> a in X
        for (int e = tid; e < TR * N; e += kCThreads) {
          const double mu = has_prev ? X[N + e] + P0[N + e] : 0.0;
          const double lam = D[e];
          double av;
          if (s == 3) {
            if (has_prev) {
              const double l2 = A[e] + mu;
              D[e] = l2;
              av = dt / 6.0 * l2;
            } else {
              av = dt / 6.0 * lam;
            }
          } else if (s == 2) {
            A[e] = lam + mu;
            av = dt / 3.0 * lam + dt * mu;
          } else if (s == 1) {
            A[e] += mu;
            av = dt / 3.0 * lam + 0.5 * dt * mu;
          } else {
            A[e] += mu;
            av = dt / 6.0 * lam + 0.5 * dt * mu;
          }
          X[N + e] = av;
        }
        __syncthreads();
        push_halo(X);  // a boundary rows into the neighbours' halo rows
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        cl.sync();  // (a) halos of a in place
        double qo[RPG];
        {
          double wa[3][3], gp[3][3], gw[3][3];
          srow(X, r0 - 1, wa[0]);
          srow(X, r0, wa[1]);
          srow(BP, r0 - 1, gp[0]);
          srow(BP, r0, gp[1]);
          srow(BW, r0 - 1, gw[0]);
          srow(BW, r0, gw[1]);
#pragma unroll
          for (int j = 0; j < RPG; ++j) {
            const int i0 = j % 3, i1 = (j + 1) % 3, i2 = (j + 2) % 3;
            srow(X, r0 + j + 1, wa[i2]);
            srow(BP, r0 + j + 1, gp[i2]);
            srow(BW, r0 + j + 1, gw[i2]);
            double W[3][3], Bp[3][3], Bw[3][3];
            win(wa, i0, i1, i2, W);
            win(gp, i0, i1, i2, Bp);
            win(gw, i0, i1, i2, Bw);
            qo[j] = -arakawa12(Bp, W) * js + nu * lap5(W) * ls;
            P0[r0 * N + j * N + x] = -arakawa12(W, Bw) * js;  // next Poisson input
          }
        }
        __syncthreads();  // all stencil reads of a done
#pragma unroll
        for (int j = 0; j < RPG; ++j) X[(r0 + j) * N + x] = qo[j];
        poisson(P0);
        first = false;
      }
    }
    // finish: lambda = acc + mu_1
    for (int e = tid; e < TR * N; e += kCThreads) D[e] = first ? D[e] : A[e] + X[N + e] + P0[N + e];
    __syncthreads();
  }
  for (int e = tid; e < TR * N; e += kCThreads) gst[e] = D[e];
  cl.sync();  // no CTA leaves while a neighbour may still read its shared memory
}

template <int N>
struct ClusterLaunch {
  using C = ClusterCfg<N>;
  template <int MODE>
  static void run(const ClusterArgs& a, int nvec, cudaStream_t st) {
    auto k = cluster_sweep_kernel<N, MODE>;
    static bool attr = false;
    if (!attr) {
      SDV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem)));
      if (C::CL > 8) SDV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C::CL, nvec);
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C::CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SDV_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  }
};

}  // namespace

// Opt-in (SDV_CLUSTER=<max vectors>). Measured on B200 (tools/small_block.py,
// CUDA-graph replay): one vector per RK stage-step takes 10.5 us at 128^2 and
// 12.6 us at 256^2 here against 7.9 / 8.4 us for the two-launch block path; the
// sweep is barrier- and latency-bound at one CTA (8 warps) per SM, three
// cluster barriers (each with an L1-invalidating acquire) per stage. It wins
// only at 256^2 with 3-7 vectors (4: 12.5 vs 14.9 us), a block width the GN
// solver does not use, so the default stays with the block path.
bool bve_cluster_ok(int n, int nvec) {
  const char* e = std::getenv("SDV_CLUSTER");
  const int maxv = e ? std::atoi(e) : 0;
  return (n == 64 || n == 128 || n == 256) && nvec >= 1 && nvec <= maxv;
}

void bve_cluster_sweep(int n, int mode, double* state, int nvec, const double* base_w, const double* base_p, int k0,
                       int k1, const long long* idx, int n_obs, int spi, const double* w, double* y, long long m,
                       const double4* tab, double dt, double nu, double js, double ls, cudaStream_t st) {
  ClusterArgs a;
  a.state = state;
  a.base_w = base_w;
  a.base_p = base_p;
  a.k0 = k0;
  a.k1 = k1;
  a.idx = idx;
  a.n_obs = n_obs;
  a.spi = spi;
  a.w = w;
  a.y = y;
  a.m = m;
  a.tab = tab;
  a.tw = twiddle_table(n);
  a.dt = dt;
  a.nu = nu;
  a.js = js;
  a.ls = ls;
  auto go = [&](auto launcher) {
    if (mode == kModeTlm) launcher.template run<kModeTlm>(a, nvec, st);
    else launcher.template run<kModeAdj>(a, nvec, st);
  };
  switch (n) {
    case 64: go(ClusterLaunch<64>{}); break;
    case 128: go(ClusterLaunch<128>{}); break;
    case 256: go(ClusterLaunch<256>{}); break;
    default: throw std::invalid_argument("bve_cluster_sweep: n must be 64, 128 or 256");
  }
}

}  // namespace sdv

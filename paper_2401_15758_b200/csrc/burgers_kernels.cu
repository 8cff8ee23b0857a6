// Batched fp64 1-D viscous Burgers RK4 TLM / ADJ / FWD sweeps, sm_100a.
//
// Replaces BurgersTrajectory::tlm_range / adj_range + step_tlm / step_adj +
// rhs_jacobian(_adjoint) (/root/reference/proj/src/burgers.cpp:152-236) for
// the periodic RK4 configs. One CTA owns one
// vector of the block for the whole sweep: the tangent/adjoint field lives in
// registers + shared memory across all stages (no HBM round trip per stage);
// the stored base stage inputs u_s, [steps][4][n], are streamed from L2/HBM
// and are shared by every CTA of the block at the same step.
// Observation gathers (TLM) and scatters (ADJ) are fused at interval ends.
#include "burgers_kernels.cuh"
#include "fft.cuh"

#include <type_traits>

namespace sdv {

namespace {
__device__ __forceinline__ int wrapm(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
}  // namespace

// Forward nonlinear sweep (one vector). Stores the 4 RK4 stage inputs of
// every step in base (if non-null) and the final state in out.
template <int NPT>
__global__ void __launch_bounds__(1024) burgers_fwd_kernel(BurgersArgs p, const double* __restrict__ x0,
                                                           double* __restrict__ base, double* __restrict__ out,
                                                           int steps) {
  extern __shared__ double sh[];
  double* X = sh;
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  double U[NPT], A[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) U[q] = x0[tid + q * nt];
  for (int k = 0; k < steps; ++k) {
    for (int s = 0; s < 4; ++s) {
      double xs[NPT];
      if (s == 0) {
#pragma unroll
        for (int q = 0; q < NPT; ++q) X[tid + q * nt] = U[q];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const int i = tid + q * nt, im = wrapm(i - 1, n), ip = wrapm(i + 1, n);
        const double xi = X[i], xm = X[im], xp = X[ip];
        if (base) base[(static_cast<long long>(k) * 4 + s) * n + i] = xi;
        const double kk = -xi * (xp - xm) * p.c1 + p.nu * (xm - 2.0 * xi + xp) * p.c2;
        switch (s) {
          case 0: A[q] = U[q] + p.dt / 6.0 * kk; xs[q] = U[q] + 0.5 * p.dt * kk; break;
          case 1: A[q] += p.dt / 3.0 * kk; xs[q] = U[q] + 0.5 * p.dt * kk; break;
          case 2: A[q] += p.dt / 3.0 * kk; xs[q] = U[q] + p.dt * kk; break;
          default: U[q] = A[q] + p.dt / 6.0 * kk; break;
        }
      }
      __syncthreads();
      if (s < 3) {
#pragma unroll
        for (int q = 0; q < NPT; ++q) X[tid + q * nt] = xs[q];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q) out[tid + q * nt] = U[q];
}

// Double-buffered base stage inputs in shared memory: the row of stage t+1
// (n doubles, contiguous in [steps][4][n]) arrives by one TMA bulk copy issued
// at the start of stage t, so the stored trajectory's L2/HBM latency overlaps
// the current stage. Thread 0 issues; every thread waits on the row's mbarrier.
struct BaseRows {
  double* row[2];
  unsigned long long* bar;  // [2]
  unsigned ph[2];
  __device__ __forceinline__ void issue(const double* src, int n, int slot) {
    fence_proxy_async();
    mbar_arm(&bar[slot], sizeof(double) * n);
    bulk_g2s(row[slot], src, sizeof(double) * n, &bar[slot]);
  }
  __device__ __forceinline__ const double* wait(int slot) {
    mbar_wait(&bar[slot], ph[slot]);
    ph[slot] ^= 1u;
    return row[slot];
  }
};

// Block TLM over steps [k0, k1). state: [nvec][n] in/out. Shared memory:
// two stage-input buffers (alternating, one barrier per RK stage) and two
// base rows (TMA-fed one stage ahead).
template <int NPT>
__global__ void __launch_bounds__(1024) burgers_tlm_kernel(BurgersArgs p, double* __restrict__ state) {
  extern __shared__ __align__(128) double sh[];
  __shared__ __align__(8) unsigned long long bars[2];
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  const long long v = blockIdx.x;
  BaseRows br{{sh + 2 * n, sh + 3 * n}, bars, {0u, 0u}};
  const long long t0 = static_cast<long long>(p.k0) * 4, t1 = static_cast<long long>(p.k1) * 4;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init_fence();
  }
  double D[NPT], A[NPT];
  int cur = 0;
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    D[q] = state[v * n + tid + q * nt];
    sh[tid + q * nt] = D[q];
  }
  __syncthreads();
  if (tid == 0 && t0 < t1) br.issue(p.base + (t0 - 4LL * p.base_k0) * n, n, 0);
  for (int k = p.k0; k < p.k1; ++k) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const long long t = static_cast<long long>(k) * 4 + s;
      const int slot = static_cast<int>((t - t0) & 1);
      if (tid == 0 && t + 1 < t1) br.issue(p.base + (t + 1 - 4LL * p.base_k0) * n, n, slot ^ 1);
      const double* u = br.wait(slot);
      const double* X = sh + cur * n;
      double* Xn = sh + (cur ^ 1) * n;
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const int i = tid + q * nt, im = wrapm(i - 1, n), ip = wrapm(i + 1, n);
        const double xi = X[i], xm = X[im], xp = X[ip];
        const double ui = u[i], um = u[im], up = u[ip];
        const double kk = -xi * (up - um) * p.c1 - ui * (xp - xm) * p.c1 + p.nu * (xm - 2.0 * xi + xp) * p.c2;
        double xs;
        switch (s) {
          case 0: A[q] = D[q] + p.dt / 6.0 * kk; xs = D[q] + 0.5 * p.dt * kk; break;
          case 1: A[q] += p.dt / 3.0 * kk; xs = D[q] + 0.5 * p.dt * kk; break;
          case 2: A[q] += p.dt / 3.0 * kk; xs = D[q] + p.dt * kk; break;
          default: D[q] = A[q] + p.dt / 6.0 * kk; xs = D[q]; break;
        }
        Xn[i] = xs;  // next stage input (after stage 3: the next step's state)
      }
      cur ^= 1;
      __syncthreads();
    }
    if (p.y && (k + 1) % p.spi == 0) {
      const int iv = (k + 1) / p.spi - 1;
      const double* X = sh + cur * n;
      for (int o = tid; o < p.n_obs; o += nt)
        p.y[v * p.m + static_cast<long long>(iv) * p.n_obs + o] = X[p.idx[o]] * p.w[static_cast<long long>(iv) * p.n_obs + o];
    }
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q) state[v * n + tid + q * nt] = D[q];
}

// Block ADJ over steps [k0, k1) backwards:
//   a4 = dt/6 L, m4 = J4^T a4; a3 = dt/3 L + dt m4, ...; L <- L + sum m.
// Observation scatter L[idx] += y*w before each interval's last step. L stays
// in registers (own points); a alternates between two shared buffers (one
// barrier per stage); base rows TMA-fed one stage ahead as in the TLM.
template <int NPT>
__global__ void __launch_bounds__(1024) burgers_adj_kernel(BurgersArgs p, double* __restrict__ state) {
  extern __shared__ __align__(128) double sh[];
  __shared__ __align__(8) unsigned long long bars[2];
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  const long long v = blockIdx.x;
  BaseRows br{{sh + 2 * n, sh + 3 * n}, bars, {0u, 0u}};
  double* Ls = sh + 4 * n;  // observation scatter
  const long long tlast = static_cast<long long>(p.k1) * 4 - 1, tfirst = static_cast<long long>(p.k0) * 4;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init_fence();
  }
  double L[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) L[q] = state[v * n + tid + q * nt];
  __syncthreads();
  if (tid == 0 && tfirst <= tlast) br.issue(p.base + (tlast - 4LL * p.base_k0) * n, n, 0);
  int cur = 0;
  for (int k = p.k1 - 1; k >= p.k0; --k) {
    if (p.y && (k + 1) % p.spi == 0) {
#pragma unroll
      for (int q = 0; q < NPT; ++q) Ls[tid + q * nt] = L[q];
      __syncthreads();
      const int iv = (k + 1) / p.spi - 1;
      for (int o = tid; o < p.n_obs; o += nt)
        Ls[p.idx[o]] += p.y[v * p.m + static_cast<long long>(iv) * p.n_obs + o] * p.w[static_cast<long long>(iv) * p.n_obs + o];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NPT; ++q) L[q] = Ls[tid + q * nt];
    }
    double acc[NPT], mu[NPT];
#pragma unroll
    for (int s = 3; s >= 0; --s) {
      const long long t = static_cast<long long>(k) * 4 + s;
      const int slot = static_cast<int>((tlast - t) & 1);
      double* Ab = sh + cur * n;
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const double l = L[q];
        double a;
        switch (s) {
          case 3: a = p.dt / 6.0 * l; break;
          case 2: a = p.dt / 3.0 * l + p.dt * mu[q]; break;
          case 1: a = p.dt / 3.0 * l + 0.5 * p.dt * mu[q]; break;
          default: a = p.dt / 6.0 * l + 0.5 * p.dt * mu[q]; break;
        }
        Ab[tid + q * nt] = a;
      }
      const double* u = br.wait(slot);
      __syncthreads();  // also: every thread is past the previous stage's reads of the other base row
      if (tid == 0 && t - 1 >= tfirst) br.issue(p.base + (t - 1 - 4LL * p.base_k0) * n, n, slot ^ 1);
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const int i = tid + q * nt, im = wrapm(i - 1, n), ip = wrapm(i + 1, n);
        const double ai = Ab[i], am = Ab[im], ap = Ab[ip];
        const double ui = u[i], um = u[im], up = u[ip];
        const double m = -ai * (up - um) * p.c1 + (up * ap - um * am) * p.c1 + p.nu * (am - 2.0 * ai + ap) * p.c2;
        mu[q] = m;
        acc[q] = (s == 3) ? m : acc[q] + m;
      }
      cur ^= 1;  // the next stage writes the other buffer
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) L[q] += acc[q];
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q) state[v * n + tid + q * nt] = L[q];
}

// 1-D periodic circulant apply out = Re IFFT(sym .* FFT(in)), one CTA per vector.
template <int N>
__global__ void __launch_bounds__(N / 8) spectral1d_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                          const double* __restrict__ sym, const double2* __restrict__ tw) {
  extern __shared__ double2 sm2[];
  const long long v = blockIdx.x;
  const int t = threadIdx.x;
  const double* src = in + v * N;
  double* dst = out + v * N;
  auto ld_real = [&](int i) { return make_double2(src[i], 0.0); };
  auto st_buf = [&](int i, double2 z) { sm2[fpad(i)] = z; };
  fft_team<N, false>(sm2, tw, t, true, ld_real, st_buf);
  __syncthreads();
  auto ld_mul = [&](int k) {
    const double w = __ldg(sym + k);
    const double2 z = sm2[fpad(k)];
    return make_double2(w * z.x, w * z.y);
  };
  auto st_out = [&](int i, double2 z) { dst[i] = z.x; };
  fft_team<N, true>(sm2, tw, t, true, ld_mul, st_out);
}

namespace {
template <class F>
void dispatch_npt(int npt, F&& f) {
  switch (npt) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: throw std::invalid_argument("Burgers: n must be a power of two in [32, 4096]");
  }
}
void geometry(int n, int& threads, int& npt) {
  if (n < 32 || (n & (n - 1)) || n > 4096) throw std::invalid_argument("Burgers: n must be a power of two in [32, 4096]");
  threads = n < 1024 ? n : 1024;
  npt = n / threads;
}
}  // namespace

void burgers_fwd(const BurgersArgs& p, const double* x0, double* base, double* out, int steps, cudaStream_t st) {
  int th, npt;
  geometry(p.n, th, npt);
  dispatch_npt(npt, [&](auto c) {
    burgers_fwd_kernel<decltype(c)::value><<<1, th, sizeof(double) * p.n, st>>>(p, x0, base, out, steps);
  });
  SDV_LAUNCH_CHECK();
}
void burgers_tlm(const BurgersArgs& p, double* state, int nvec, cudaStream_t st) {
  int th, npt;
  geometry(p.n, th, npt);
  dispatch_npt(npt, [&](auto c) {
    const size_t smem = sizeof(double) * 4 * p.n;
    if (smem > 48 * 1024)
      SDV_CUDA(cudaFuncSetAttribute(burgers_tlm_kernel<decltype(c)::value>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    burgers_tlm_kernel<decltype(c)::value><<<nvec, th, smem, st>>>(p, state);
  });
  SDV_LAUNCH_CHECK();
}
void burgers_adj(const BurgersArgs& p, double* state, int nvec, cudaStream_t st) {
  int th, npt;
  geometry(p.n, th, npt);
  dispatch_npt(npt, [&](auto c) {
    const size_t smem = sizeof(double) * 5 * p.n;
    if (smem > 48 * 1024)
      SDV_CUDA(cudaFuncSetAttribute(burgers_adj_kernel<decltype(c)::value>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    burgers_adj_kernel<decltype(c)::value><<<nvec, th, smem, st>>>(p, state);
  });
  SDV_LAUNCH_CHECK();
}

namespace {
template <int N>
void spectral1d_launch(const double* in, double* out, const double* sym, int nvec, cudaStream_t st) {
  constexpr int kTeam = FftSize<N>::kTeam;
  const size_t smem = sizeof(double2) * FftSize<N>::kPadded;
  static const bool init = [&] {  // thread-safe one-time attribute (magic static)
    SDV_CUDA(cudaFuncSetAttribute(spectral1d_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    return true;
  }();
  (void)init;
  spectral1d_kernel<N><<<nvec, kTeam, smem, st>>>(in, out, sym, twiddle_table(N));
  SDV_LAUNCH_CHECK();
}
}  // namespace

void spectral1d(int n, const double* in, double* out, const double* sym, int nvec, cudaStream_t st) {
  switch (n) {
    case 32: spectral1d_launch<32>(in, out, sym, nvec, st); break;
    case 64: spectral1d_launch<64>(in, out, sym, nvec, st); break;
    case 128: spectral1d_launch<128>(in, out, sym, nvec, st); break;
    case 256: spectral1d_launch<256>(in, out, sym, nvec, st); break;
    case 512: spectral1d_launch<512>(in, out, sym, nvec, st); break;
    case 1024: spectral1d_launch<1024>(in, out, sym, nvec, st); break;
    case 2048: spectral1d_launch<2048>(in, out, sym, nvec, st); break;
    case 4096: spectral1d_launch<4096>(in, out, sym, nvec, st); break;
    default: throw std::invalid_argument("spectral1d: n must be a power of two in [32, 4096]");
  }
}

}  // namespace sdv

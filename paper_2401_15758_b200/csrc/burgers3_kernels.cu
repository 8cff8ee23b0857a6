// The reference's own 1-D Burgers model on the GPU:
// n interior points of (0,1), homogeneous Dirichlet walls, dx = 1/(n+1),
// advective centred differences, Shu-Osher RK3-TVD, with the exact
// stage-differentiated TLM / ADJ of proj/src/burgers.cpp:56-92, :218-236 and
// the (alpha I - beta Lap*)^{-2} prior of proj/src/prior.cpp / the Thomas
// solver of proj/src/dirichlet.cpp:157-187. One CTA owns one vector for the
// whole sweep (field in registers + shared memory); the stored stage inputs
// [steps][3][n] stream from L2.
#include <type_traits>

#include "burgers_kernels.cuh"

namespace sdv {

namespace {

// centred first/second differences with zero walls (proj/src/burgers.cpp:13-31)
__device__ __forceinline__ double val(const double* f, int i, int n) { return (i >= 0 && i < n) ? f[i] : 0.0; }
__device__ __forceinline__ double gval(const double* __restrict__ f, int i, int n) {
  return (i >= 0 && i < n) ? __ldg(f + i) : 0.0;
}

// rhs(u)_i = -u_i D1u_i + nu D2u_i, u in shared memory
__device__ __forceinline__ double rhs3(const double* u, int i, int n, const BurgersArgs& p) {
  const double l = val(u, i - 1, n), c = u[i], r = val(u, i + 1, n);
  const double a = (r - l) * p.c1, b = (l - 2.0 * c + r) * p.c2;
  return -c * a + p.nu * b;
}
// J(u) d, d in shared memory, u global
__device__ __forceinline__ double jac3(const double* __restrict__ u, const double* d, int i, int n,
                                      const BurgersArgs& p) {
  const double du = (gval(u, i + 1, n) - gval(u, i - 1, n)) * p.c1;
  const double dl = val(d, i - 1, n), dc = d[i], dr = val(d, i + 1, n);
  double out = -dc * du;
  out -= __ldg(u + i) * ((dr - dl) * p.c1);
  out += p.nu * ((dl - 2.0 * dc + dr) * p.c2);
  return out;
}
// J(u)^T l = -l D1u + D1(u l) + nu D2 l, l in shared memory, u global
__device__ __forceinline__ double jac3t(const double* __restrict__ u, const double* l, int i, int n,
                                       const BurgersArgs& p) {
  const double um = gval(u, i - 1, n), uc = __ldg(u + i), up = gval(u, i + 1, n);
  const double lm = val(l, i - 1, n), lc = l[i], lp = val(l, i + 1, n);
  double out = -lc * ((up - um) * p.c1);
  out += (up * lp - um * lm) * p.c1;
  out += p.nu * ((lm - 2.0 * lc + lp) * p.c2);
  return out;
}

}  // namespace

template <int NPT>
__global__ void __launch_bounds__(1024) burgers3_fwd_kernel(BurgersArgs p, const double* __restrict__ x0,
                                                            double* __restrict__ base, double* __restrict__ out,
                                                            int steps) {
  extern __shared__ double X[];
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  double U[NPT], U1[NPT], R[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) U[q] = (tid + q * nt < n) ? x0[tid + q * nt] : 0.0;
  for (int k = 0; k < steps; ++k) {
    double* bk = base ? base + static_cast<long long>(k) * 3 * n : nullptr;
    // u1 = u + dt rhs(u)
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = U[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) {
        R[q] = rhs3(X, i, n, p);
        U1[q] = U[q] + p.dt * R[q];
        if (bk) bk[i] = U[q];
      }
    }
    __syncthreads();
    // u2 = 0.75 u + 0.25 (u1 + dt rhs(u1))
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = U1[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) {
        R[q] = 0.75 * U[q] + 0.25 * (U1[q] + p.dt * rhs3(X, i, n, p));
        if (bk) {
          bk[n + i] = U1[q];
          bk[2 * n + i] = R[q];
        }
      }
    }
    __syncthreads();
    // u' = u/3 + 2/3 (u2 + dt rhs(u2))
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = R[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) U[q] = U[q] / 3.0 + (2.0 / 3.0) * (R[q] + p.dt * rhs3(X, i, n, p));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q)
    if (tid + q * nt < n) out[tid + q * nt] = U[q];
}

// Block TLM (proj/src/burgers.cpp:218-225) over steps [k0, k1).
template <int NPT>
__global__ void __launch_bounds__(1024) burgers3_tlm_kernel(BurgersArgs p, double* __restrict__ state) {
  extern __shared__ double X[];
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  const long long v = blockIdx.x;
  double D[NPT], D1[NPT], D2[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) D[q] = (tid + q * nt < n) ? state[v * n + tid + q * nt] : 0.0;
  for (int k = p.k0; k < p.k1; ++k) {
    const double* u0 = p.base + static_cast<long long>(k - p.base_k0) * 3 * n;
    const double* u1 = u0 + n;
    const double* u2 = u0 + 2 * n;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = D[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) D1[q] = D[q] + p.dt * jac3(u0, X, i, n, p);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = D1[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) D2[q] = 0.75 * D[q] + 0.25 * (D1[q] + p.dt * jac3(u1, X, i, n, p));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) X[tid + q * nt] = D2[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) D[q] = D[q] / 3.0 + (2.0 / 3.0) * (D2[q] + p.dt * jac3(u2, X, i, n, p));
    }
    __syncthreads();
    if (p.y && (k + 1) % p.spi == 0) {
      const int iv = (k + 1) / p.spi - 1;
#pragma unroll
      for (int q = 0; q < NPT; ++q)
        if (tid + q * nt < n) X[tid + q * nt] = D[q];
      __syncthreads();
      for (int o = tid; o < p.n_obs; o += nt)
        p.y[v * p.m + static_cast<long long>(iv) * p.n_obs + o] =
            X[p.idx[o]] * p.w[static_cast<long long>(iv) * p.n_obs + o];
      __syncthreads();
    }
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q)
    if (tid + q * nt < n) state[v * n + tid + q * nt] = D[q];
}

// Block ADJ (proj/src/burgers.cpp:227-236) over steps [k0, k1) backwards, with
// the observation scatter of MisfitOperator::adjoint_apply at interval ends.
template <int NPT>
__global__ void __launch_bounds__(1024) burgers3_adj_kernel(BurgersArgs p, double* __restrict__ state) {
  extern __shared__ double sm3[];
  double* L = sm3;
  double* T = sm3 + p.n;
  const int n = p.n, tid = threadIdx.x, nt = blockDim.x;
  const long long v = blockIdx.x;
#pragma unroll
  for (int q = 0; q < NPT; ++q)
    if (tid + q * nt < n) L[tid + q * nt] = state[v * n + tid + q * nt];
  __syncthreads();
  for (int k = p.k1 - 1; k >= p.k0; --k) {
    if (p.y && (k + 1) % p.spi == 0) {
      const int iv = (k + 1) / p.spi - 1;
      for (int o = tid; o < p.n_obs; o += nt)
        L[p.idx[o]] += p.y[v * p.m + static_cast<long long>(iv) * p.n_obs + o] *
                       p.w[static_cast<long long>(iv) * p.n_obs + o];
      __syncthreads();
    }
    const double* u0 = p.base + static_cast<long long>(k - p.base_k0) * 3 * n;
    const double* u1 = u0 + n;
    const double* u2 = u0 + 2 * n;
    double T2[NPT], T1[NPT];
    // t2 = 2/3 (lam + dt J2^T lam)
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) T2[q] = (2.0 / 3.0) * (L[i] + p.dt * jac3t(u2, L, i, n, p));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) T[tid + q * nt] = T2[q];
    __syncthreads();
    // t1 = 0.25 (t2 + dt J1^T t2)
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) T1[q] = 0.25 * (T2[q] + p.dt * jac3t(u1, T, i, n, p));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) T[tid + q * nt] = T1[q];
    __syncthreads();
    // lam' = lam/3 + 0.75 t2 + t1 + dt J0^T t1
    double Ln[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int i = tid + q * nt;
      if (i < n) Ln[q] = L[i] / 3.0 + 0.75 * T2[q] + T1[q] + p.dt * jac3t(u0, T, i, n, p);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (tid + q * nt < n) L[tid + q * nt] = Ln[q];
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q)
    if (tid + q * nt < n) state[v * n + tid + q * nt] = L[tid + q * nt];
}

// Thomas algorithm with cached pivots (proj/src/dirichlet.cpp:172-187); one
// CTA per vector, the recurrences run on thread 0 over shared memory.
__global__ void thomas_kernel(int n, double off, const double* __restrict__ pivot, const double* __restrict__ in,
                              double* __restrict__ out) {
  extern __shared__ double ys[];
  const long long v = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ys[i] = in[v * n + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < n; ++i) ys[i] = ys[i] - off / pivot[i - 1] * ys[i - 1];
    ys[n - 1] = ys[n - 1] / pivot[n - 1];
    for (int i = n - 2; i >= 0; --i) ys[i] = (ys[i] - off * ys[i + 1]) / pivot[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[v * n + i] = ys[i];
}

__global__ void lap_inv_sqrt_kernel(int n, double alpha, double b, const double* __restrict__ in,
                                    double* __restrict__ out, long long total) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= total) return;
  const int i = static_cast<int>(e % n);
  const double* r = in + (e - i);
  const double c = r[i], l = i > 0 ? r[i - 1] : 0.0, rr = i + 1 < n ? r[i + 1] : 0.0;
  out[e] = alpha * c + b * (2.0 * c - l - rr);
}

namespace {
template <class F>
void dispatch3(int n, int& th, F&& f) {
  if (n < 3 || n > 4096) throw std::invalid_argument("Burgers (Dirichlet): need 3 <= n <= 4096");
  th = n < 1024 ? ((n + 31) / 32) * 32 : 1024;
  const int npt = (n + th - 1) / th;
  switch (npt) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    default: f(std::integral_constant<int, 4>{}); break;
  }
}
}  // namespace

void burgers3_fwd(const BurgersArgs& p, const double* x0, double* base, double* out, int steps, cudaStream_t st) {
  int th = 0;
  dispatch3(p.n, th, [&](auto c) {
    burgers3_fwd_kernel<decltype(c)::value><<<1, th, sizeof(double) * p.n, st>>>(p, x0, base, out, steps);
  });
  SDV_LAUNCH_CHECK();
}
void burgers3_tlm(const BurgersArgs& p, double* state, int nvec, cudaStream_t st) {
  int th = 0;
  dispatch3(p.n, th, [&](auto c) {
    burgers3_tlm_kernel<decltype(c)::value><<<nvec, th, sizeof(double) * p.n, st>>>(p, state);
  });
  SDV_LAUNCH_CHECK();
}
void burgers3_adj(const BurgersArgs& p, double* state, int nvec, cudaStream_t st) {
  int th = 0;
  dispatch3(p.n, th, [&](auto c) {
    const size_t smem = sizeof(double) * 2 * p.n;
    if (smem > 48 * 1024)
      SDV_CUDA(cudaFuncSetAttribute(burgers3_adj_kernel<decltype(c)::value>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    burgers3_adj_kernel<decltype(c)::value><<<nvec, th, smem, st>>>(p, state);
  });
  SDV_LAUNCH_CHECK();
}
void thomas_solve(int n, double off, const double* pivot, const double* in, double* out, int nvec, cudaStream_t st) {
  thomas_kernel<<<nvec, 128, sizeof(double) * n, st>>>(n, off, pivot, in, out);
  SDV_LAUNCH_CHECK();
}
void lap_inv_sqrt(int n, double alpha, double b, const double* in, double* out, int nvec, cudaStream_t st) {
  const long long total = static_cast<long long>(n) * nvec;
  lap_inv_sqrt_kernel<<<ceil_div(total, 256), 256, 0, st>>>(n, alpha, b, in, out, total);
  SDV_LAUNCH_CHECK();
}

}  // namespace sdv

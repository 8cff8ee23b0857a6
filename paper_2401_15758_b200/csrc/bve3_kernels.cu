// The reference's own barotropic-vorticity model (proj/src/bve.cpp,
// proj/src/dirichlet.cpp), batched over s vectors:
// nx x ny interior points of [0,1] x [-1,1] with homogeneous Dirichlet walls,
// central differences, 5-point Laplacian, beta-term (1/Ro) psi_x, forcing
// sin(pi y), Shu-Osher RK3-TVD. The Poisson inverse psi = (-Lap_h)^-1 omega is
// the reference's dense sine-transform form S_x [Lambda^-1 o (S_x W S_y)] S_y
// (proj/src/dirichlet.cpp:82-155), done here as batched fp64 GEMMs (cuBLAS,
// which uses the DMMA tensor pipe on sm_100) with a fused spectral scale.
//
// Layout: a block is [s][ny][nx] (x fastest, i + nx j), as the reference.
// Stencil/RK kernels are one thread per point; every formula keeps the
// reference's operation order (proj/src/bve.cpp:28-82, :171-211), so the
// tangent/adjoint match the reference's arithmetic to rounding.

#include "bve3_kernels.cuh"
#include "linalg_kernels.cuh"

namespace sdv {

namespace {

struct Pt {
  int i, j;
  long long base;  // vector offset
};

__device__ __forceinline__ double at(const double* f, const Bve3Args& a, long long base, int i, int j) {
  return (i < 0 || i >= a.nx || j < 0 || j >= a.ny) ? 0.0 : f[base + i + static_cast<long long>(a.nx) * j];
}
// d_x, d_y (proj/src/bve.cpp:28-47): (e - w) * 0.5 (nx+1), (n - s) * 0.25 (ny+1)
__device__ __forceinline__ double ddx(const double* f, const Bve3Args& a, long long b, int i, int j) {
  return (at(f, a, b, i + 1, j) - at(f, a, b, i - 1, j)) * a.cx;
}
__device__ __forceinline__ double ddy(const double* f, const Bve3Args& a, long long b, int i, int j) {
  return (at(f, a, b, i, j + 1) - at(f, a, b, i, j - 1)) * a.cy;
}
// laplacian = -neg_laplacian_2d(f, 1/dx^2, 1/dy^2) (proj/src/dirichlet.cpp:30-47)
__device__ __forceinline__ double lap(const double* f, const Bve3Args& a, long long b, int i, int j) {
  const double c = at(f, a, b, i, j);
  return -(a.lx * (2.0 * c - at(f, a, b, i - 1, j) - at(f, a, b, i + 1, j)) +
           a.ly * (2.0 * c - at(f, a, b, i, j - 1) - at(f, a, b, i, j + 1)));
}
__device__ __forceinline__ bool point(const Bve3Args& a, int nvec, Pt& p, long long& g) {
  const long long dim = static_cast<long long>(a.nx) * a.ny;
  g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (g >= dim * nvec) return false;
  const long long v = g / dim, e = g % dim;
  p.base = v * dim;
  p.i = static_cast<int>(e % a.nx);
  p.j = static_cast<int>(e / a.nx);
  return true;
}

// Nonlinear RK3 stage: r = rhs(w_s, psi_s) (proj/src/bve.cpp:64-82), then the
// Shu-Osher combination with the step-start state u.
__global__ void nl_stage_kernel(Bve3Args a, int stage, const double* __restrict__ u, const double* __restrict__ ws,
                                const double* __restrict__ ps, double* __restrict__ out, int nvec) {
  Pt p;
  long long g;
  if (!point(a, nvec, p, g)) return;
  const double ox = ddx(ws, a, p.base, p.i, p.j), oy = ddy(ws, a, p.base, p.i, p.j);
  const double px = ddx(ps, a, p.base, p.i, p.j), py = ddy(ps, a, p.base, p.i, p.j);
  double r = -(py * ox - px * oy);
  r += a.inv_ro * (px + a.forcing[p.j]);
  r += a.inv_re * lap(ws, a, p.base, p.i, p.j);
  const double w = ws[g];
  if (stage == 0) out[g] = u[g] + a.dt * r;
  else if (stage == 1) out[g] = 0.75 * u[g] + 0.25 * (w + a.dt * r);
  else out[g] = u[g] / 3.0 + (2.0 / 3.0) * (w + a.dt * r);
}

// Tangent-linear stage (proj/src/bve.cpp:184-197) + the RK3 combination
// (tlm_range, :138-148): d1 = d + dt j0, d2 = 0.75 d + 0.25 (d1 + dt j1),
// d' = d/3 + 2/3 (d2 + dt j2). wb/pb: the stored base stage omega/psi (one
// field shared by the block).
__global__ void tlm_stage_kernel(Bve3Args a, int stage, const double* __restrict__ d, const double* __restrict__ ds,
                                 const double* __restrict__ dp, const double* __restrict__ wb,
                                 const double* __restrict__ pb, double* __restrict__ out, int nvec) {
  Pt p;
  long long g;
  if (!point(a, nvec, p, g)) return;
  const double ox = ddx(wb, a, 0, p.i, p.j), oy = ddy(wb, a, 0, p.i, p.j);
  const double px = ddx(pb, a, 0, p.i, p.j), py = ddy(pb, a, 0, p.i, p.j);
  const double dx = ddx(ds, a, p.base, p.i, p.j), dy = ddy(ds, a, p.base, p.i, p.j);
  const double dpx = ddx(dp, a, p.base, p.i, p.j), dpy = ddy(dp, a, p.base, p.i, p.j);
  double jv = -(dpy * ox + py * dx - dpx * oy - px * dy);
  jv += a.inv_ro * dpx;
  jv += a.inv_re * lap(ds, a, p.base, p.i, p.j);
  const double s = ds[g];
  if (stage == 0) out[g] = d[g] + a.dt * jv;
  else if (stage == 1) out[g] = 0.75 * d[g] + 0.25 * (s + a.dt * jv);
  else out[g] = d[g] / 3.0 + (2.0 / 3.0) * (s + a.dt * jv);
}

// Adjoint stage, part 1 (proj/src/bve.cpp:199-211): the Poisson right-hand
// side vp = d_y(ox L) - d_x(oy L) - (1/Ro) d_x(L).
__global__ void adj_vp_kernel(Bve3Args a, const double* __restrict__ L, const double* __restrict__ wb,
                              double* __restrict__ vp, int nvec) {
  Pt p;
  long long g;
  if (!point(a, nvec, p, g)) return;
  auto oxl = [&](int i, int j) {
    return (i < 0 || i >= a.nx || j < 0 || j >= a.ny) ? 0.0 : ddx(wb, a, 0, i, j) * at(L, a, p.base, i, j);
  };
  auto oyl = [&](int i, int j) {
    return (i < 0 || i >= a.nx || j < 0 || j >= a.ny) ? 0.0 : ddy(wb, a, 0, i, j) * at(L, a, p.base, i, j);
  };
  const double dyox = (oxl(p.i, p.j + 1) - oxl(p.i, p.j - 1)) * a.cy;
  const double dxoy = (oyl(p.i + 1, p.j) - oyl(p.i - 1, p.j)) * a.cx;
  const double dxl = ddx(L, a, p.base, p.i, p.j);
  vp[g] = dyox - dxoy - a.inv_ro * dxl;
}

// Adjoint stage, part 2: a = d_x(py L) - d_y(px L) + P[vp] + (1/Re) Lap L and
// the reverse RK3 combination (adj_range, :150-161):
//   stage 2: t2 = 2/3 (lam + dt a2); stage 1: t1 = 0.25 (t2 + dt a1);
//   stage 0: lam' = lam/3 + 0.75 t2 + t1 + dt a0.
__global__ void adj_stage_kernel(Bve3Args a, int stage, const double* __restrict__ L, const double* __restrict__ ps,
                                 const double* __restrict__ pb, const double* __restrict__ lam,
                                 const double* __restrict__ t2, double* __restrict__ out, int nvec) {
  Pt p;
  long long g;
  if (!point(a, nvec, p, g)) return;
  auto pyl = [&](int i, int j) {
    return (i < 0 || i >= a.nx || j < 0 || j >= a.ny) ? 0.0 : ddy(pb, a, 0, i, j) * at(L, a, p.base, i, j);
  };
  auto pxl = [&](int i, int j) {
    return (i < 0 || i >= a.nx || j < 0 || j >= a.ny) ? 0.0 : ddx(pb, a, 0, i, j) * at(L, a, p.base, i, j);
  };
  double o = (pyl(p.i + 1, p.j) - pyl(p.i - 1, p.j)) * a.cx;
  o -= (pxl(p.i, p.j + 1) - pxl(p.i, p.j - 1)) * a.cy;
  o += ps[g] + a.inv_re * lap(L, a, p.base, p.i, p.j);
  if (stage == 2) out[g] = (2.0 / 3.0) * (lam[g] + a.dt * o);
  else if (stage == 1) out[g] = 0.25 * (L[g] + a.dt * o);
  else out[g] = lam[g] / 3.0 + 0.75 * t2[g] + L[g] + a.dt * o;
}

// Orthonormal sine transform along x of every row (proj/src/dirichlet.cpp:
// 110-122 restricted to one dimension): out(i, j) = sum_k S(i, k) in(k, j),
// S(i, k) = sqrt(2 / (nx + 1)) sin((i + 1)(k + 1) pi / (nx + 1)). One CTA per
// row chunk; the row and the nx x nx table are staged in shared memory. S is
// symmetric and orthogonal (S^2 = I), so the same kernel is its own inverse.
__global__ void sine_x_kernel(int nx, int ny, const double* __restrict__ sx, const double* __restrict__ in,
                              double* __restrict__ out, int rows_per_cta) {
  extern __shared__ double sm3[];
  double* tab = sm3;               // nx x nx
  double* row = sm3 + nx * nx;     // rows_per_cta x nx
  const long long dim = static_cast<long long>(nx) * ny;
  const long long v = blockIdx.y;
  const int j0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, ny - j0);
  for (int e = threadIdx.x; e < nx * nx; e += blockDim.x) tab[e] = sx[e];
  for (int e = threadIdx.x; e < nr * nx; e += blockDim.x)
    row[e] = in[v * dim + static_cast<long long>(j0) * nx + e];
  __syncthreads();
  for (int e = threadIdx.x; e < nr * nx; e += blockDim.x) {
    const int r = e / nx, i = e % nx;
    const double* rr = row + r * nx;
    double acc = 0.0;
    for (int k = 0; k < nx; ++k) acc = fma(tab[i + k * nx], rr[k], acc);
    out[v * dim + static_cast<long long>(j0) * nx + e] = acc;
  }
}

// Per x-mode i, the exact solve of the Dirichlet tridiagonal system in y,
// ((a + bx mu_i) I + by tridiag(-1, 2, -1)) x = d (Thomas; the elimination
// multipliers m[j][i] = 1 / pivot_j and c[j][i] = -by / pivot_j depend only on
// the mode and are tabulated once). Same operator the reference diagonalises
// by the sine transform in y (proj/src/dirichlet.cpp:82-99, :149-153).
// Thread = mode, walking the ny rows (coalesced across the modes of a warp).
__global__ void thomas_y_kernel(int nx, int ny, double off, const double* __restrict__ m, const double* __restrict__ c,
                                double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  double* f = x + static_cast<long long>(blockIdx.y) * nx * ny + i;
  double prev = 0.0;
  for (int j = 0; j < ny; ++j) {
    const long long o = static_cast<long long>(j) * nx;
    prev = (f[o] - off * prev) * m[o + i];
    f[o] = prev;
  }
  double nxt = f[static_cast<long long>(ny - 1) * nx];
  for (int j = ny - 2; j >= 0; --j) {
    const long long o = static_cast<long long>(j) * nx;
    nxt = f[o] - c[o + i] * nxt;
    f[o] = nxt;
  }
}

// alpha v + neg_laplacian_2d(v, b, b) (proj/src/prior.cpp:53-62)
__global__ void lap2_inv_sqrt_kernel(int nx, int ny, double alpha, double b, const double* __restrict__ in,
                                     double* __restrict__ out, int nvec) {
  const long long dim = static_cast<long long>(nx) * ny;
  const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (g >= dim * nvec) return;
  const long long base = (g / dim) * dim, e = g % dim;
  const int i = static_cast<int>(e % nx), j = static_cast<int>(e / nx);
  auto f = [&](int ii, int jj) {
    return (ii < 0 || ii >= nx || jj < 0 || jj >= ny) ? 0.0 : in[base + ii + static_cast<long long>(nx) * jj];
  };
  const double c = f(i, j);
  out[g] = alpha * c + (b * (2.0 * c - f(i - 1, j) - f(i + 1, j)) + b * (2.0 * c - f(i, j - 1) - f(i, j + 1)));
}

constexpr int kTpb = 256;
int blocks(long long n) { return ceil_div(n, kTpb); }

}  // namespace

// ---------------------------------------------------------- DST solver --
DstSolver::DstSolver(int nx, int ny, double a, double bx, double by, cudaStream_t st)
    : nx_(nx), ny_(ny), off_(-by), st_(st) {
  // proj/src/dirichlet.cpp:82-99: the operator must be positive definite
  // (a + bx mu_x + by mu_y > 0 for every mode, mu = 2 - 2 cos(k pi / (n + 1))).
  auto mu = [](int k, int n) { return 2.0 - 2.0 * std::cos(static_cast<double>(k) * M_PI / (n + 1.0)); };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      if (!(a + bx * mu(i + 1, nx) + by * mu(j + 1, ny) > 0.0))
        throw std::invalid_argument("DirichletSolver2D: operator is not positive definite");
  // orthonormal sine matrix in x (proj/src/dirichlet.cpp:110-120)
  std::vector<double> sx(static_cast<size_t>(nx) * nx);
  const double nr = std::sqrt(2.0 / (nx + 1));
  for (int i = 0; i < nx; ++i)
    for (int k = 0; k < nx; ++k) sx[i + static_cast<size_t>(nx) * k] = nr * std::sin((i + 1.0) * (k + 1.0) * M_PI / (nx + 1));
  // Thomas multipliers per x-mode for (a + bx mu_i + 2 by) on the diagonal, -by off it
  std::vector<double> m(static_cast<size_t>(nx) * ny), c(static_cast<size_t>(nx) * ny);
  for (int i = 0; i < nx; ++i) {
    const double diag = a + bx * mu(i + 1, nx) + 2.0 * by;
    double cp = 0.0;
    for (int j = 0; j < ny; ++j) {
      const double piv = diag - off_ * cp;
      if (!(piv > 0.0)) throw std::invalid_argument("DirichletSolver2D: operator is not positive definite");
      m[i + static_cast<size_t>(nx) * j] = 1.0 / piv;
      cp = off_ / piv;
      c[i + static_cast<size_t>(nx) * j] = cp;
    }
  }
  sx_.upload(sx.data(), sx.size(), st);
  m_.upload(m.data(), m.size(), st);
  c_.upload(c.data(), c.size(), st);
}
DstSolver::~DstSolver() = default;

size_t DstSolver::sine_smem(int rows) const { return sizeof(double) * (static_cast<size_t>(nx_) * nx_ + static_cast<size_t>(rows) * nx_); }

// out = S_x T^{-1} S_x in, T^{-1} the per-mode tridiagonal solves in y
// (= S_x [inv o (S_x in S_y)] S_y, the reference's dense-sine solve, up to
// roundoff). Three launches, no library call; in may alias out.
void DstSolver::solve(const double* in, double* out, int nvec) const {
  const long long dim = static_cast<long long>(nx_) * ny_;
  tmp_.ensure(static_cast<size_t>(dim) * nvec);
  constexpr int kRows = 8;
  const size_t sm = sine_smem(kRows);
  static const bool once = [] {
    SDV_CUDA(cudaFuncSetAttribute(sine_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return true;
  }();
  (void)once;
  if (sm > 200 * 1024) throw std::invalid_argument("DirichletSolver2D: nx too large for the shared-memory sine table");
  const dim3 gx(ceil_div(ny_, kRows), nvec);
  sine_x_kernel<<<gx, kTpb, sm, st_>>>(nx_, ny_, sx_.get(), in, tmp_.get(), kRows);
  SDV_LAUNCH_CHECK();
  thomas_y_kernel<<<dim3(ceil_div(nx_, 64), nvec), 64, 0, st_>>>(nx_, ny_, off_, m_.get(), c_.get(), tmp_.get());
  SDV_LAUNCH_CHECK();
  sine_x_kernel<<<gx, kTpb, sm, st_>>>(nx_, ny_, sx_.get(), tmp_.get(), out, kRows);
  SDV_LAUNCH_CHECK();
}

// ------------------------------------------------------------- launchers --
void bve3_nl_stage(const Bve3Args& a, int stage, const double* u, const double* ws, const double* ps, double* out,
                   int nvec, cudaStream_t st) {
  nl_stage_kernel<<<blocks(static_cast<long long>(a.nx) * a.ny * nvec), kTpb, 0, st>>>(a, stage, u, ws, ps, out, nvec);
  SDV_LAUNCH_CHECK();
}
void bve3_tlm_stage(const Bve3Args& a, int stage, const double* d, const double* ds, const double* dp,
                    const double* wb, const double* pb, double* out, int nvec, cudaStream_t st) {
  tlm_stage_kernel<<<blocks(static_cast<long long>(a.nx) * a.ny * nvec), kTpb, 0, st>>>(a, stage, d, ds, dp, wb, pb,
                                                                                         out, nvec);
  SDV_LAUNCH_CHECK();
}
void bve3_adj_vp(const Bve3Args& a, const double* L, const double* wb, double* vp, int nvec, cudaStream_t st) {
  adj_vp_kernel<<<blocks(static_cast<long long>(a.nx) * a.ny * nvec), kTpb, 0, st>>>(a, L, wb, vp, nvec);
  SDV_LAUNCH_CHECK();
}
void bve3_adj_stage(const Bve3Args& a, int stage, const double* L, const double* ps, const double* pb,
                    const double* lam, const double* t2, double* out, int nvec, cudaStream_t st) {
  adj_stage_kernel<<<blocks(static_cast<long long>(a.nx) * a.ny * nvec), kTpb, 0, st>>>(a, stage, L, ps, pb, lam, t2,
                                                                                         out, nvec);
  SDV_LAUNCH_CHECK();
}
void lap2_inv_sqrt(int nx, int ny, double alpha, double b, const double* in, double* out, int nvec, cudaStream_t st) {
  lap2_inv_sqrt_kernel<<<blocks(static_cast<long long>(nx) * ny * nvec), kTpb, 0, st>>>(nx, ny, alpha, b, in, out,
                                                                                         nvec);
  SDV_LAUNCH_CHECK();
}

}  // namespace sdv

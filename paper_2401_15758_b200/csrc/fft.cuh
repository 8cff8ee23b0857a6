// Hand-written shared-memory FFT building blocks (no cuFFT on the hot path).
//
// fft_team<N, INV>: one length-N complex transform per "team" of threads,
// Stockham autosort formulation (radix-4 passes, one radix-2 pass when log2 N
// is odd), ping-ponging between two shared-memory buffers. Twiddles come from
// a per-length table tw[m] = exp(-2 pi i m / N) in global memory (L1 resident).
// Unnormalised in both directions; the 1/N^d factors are folded into the
// spectral multipliers (Poisson symbol, B^{1/2} symbol).
#pragma once

#include "common.cuh"

namespace sdv {

__host__ __device__ constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <bool CONJ>
__device__ __forceinline__ double2 cmul_tw(double2 a, double2 w) {
  if (CONJ) return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.y, w.x, a.x * w.y));
}

// Radix-4 butterfly; forward uses -i, inverse +i.
template <bool INV>
__device__ __forceinline__ void bfly4(double2& v0, double2& v1, double2& v2, double2& v3) {
  const double2 y0 = cadd(v0, v2), y1 = csub(v0, v2), y2 = cadd(v1, v3);
  const double2 d = csub(v1, v3);
  const double2 y3 = INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
  v0 = cadd(y0, y2);
  v2 = csub(y0, y2);
  v1 = cadd(y1, y3);
  v3 = csub(y1, y3);
}

// All threads of the CTA must call this (it synchronises with __syncthreads
// after every pass). Team thread t in [0, nt) works on the transform held in
// a[0..N); b is scratch of the same size. Returns the buffer holding the
// result (a or b).
template <int N, bool INV>
__device__ __forceinline__ double2* fft_team(double2* a, double2* b, const double2* __restrict__ tw, int t, int nt,
                                             bool active) {
  constexpr int LOG = ilog2_c(N);
  int ns = 1;
#pragma unroll
  for (int pass = 0; pass < LOG / 2; ++pass) {
    if (active) {
      for (int j = t; j < N / 4; j += nt) {
        const int k = j & (ns - 1);
        double2 v0 = a[j], v1 = a[j + N / 4], v2 = a[j + N / 2], v3 = a[j + 3 * N / 4];
        if (ns > 1) {
          const int st = N / (ns * 4);
          v1 = cmul_tw<INV>(v1, __ldg(tw + k * st));
          v2 = cmul_tw<INV>(v2, __ldg(tw + 2 * k * st));
          v3 = cmul_tw<INV>(v3, __ldg(tw + 3 * k * st));
        }
        bfly4<INV>(v0, v1, v2, v3);
        const int base = (j - k) * 4 + k;
        b[base] = v0;
        b[base + ns] = v1;
        b[base + 2 * ns] = v2;
        b[base + 3 * ns] = v3;
      }
    }
    __syncthreads();
    double2* tmp = a;
    a = b;
    b = tmp;
    ns *= 4;
  }
  if (LOG & 1) {
    if (active) {
      for (int j = t; j < N / 2; j += nt) {
        const int k = j & (ns - 1);
        double2 v0 = a[j], v1 = a[j + N / 2];
        if (ns > 1) v1 = cmul_tw<INV>(v1, __ldg(tw + k * (N / (2 * ns))));
        const int base = (j - k) * 2 + k;
        b[base] = cadd(v0, v1);
        b[base + ns] = csub(v0, v1);
      }
    }
    __syncthreads();
    double2* tmp = a;
    a = b;
    b = tmp;
  }
  return a;
}

// Device twiddle table exp(-2 pi i m / N), m in [0, N); cached per length.
const double2* twiddle_table(int n);

}  // namespace sdv

// Hand-written shared-memory FFT building blocks (no cuFFT on the hot path).
//
// fft_team<N, INV>: one length-N complex transform per "team" of N/8 threads.
// Register-blocked Stockham autosort: every thread holds 8 complex values per
// pass and performs 8/R radix-R butterflies in registers (radix-8 passes,
// one trailing radix-4 or radix-2 pass when log2 N is not a multiple of 3:
// 512 = 8*8*8, 256 = 8*8*4, 128 = 8*8*2, 4096 = 8^4). Passes exchange data
// in place through one padded shared buffer (index i -> i + i/8, which makes
// the stride-8 Stockham stores bank-conflict free). The first pass reads
// through a caller functor (e.g. straight from global memory, unpacking
// packed real spectra) and the last pass writes through one, so a transform
// costs P-1 shared-memory round trips. Twiddles come from a per-length table
// tw[m] = exp(-2 pi i m / N) (L1 resident). Unnormalised in both directions;
// the 1/N^d factors are folded into the spectral multipliers.
#pragma once

#include "common.cuh"

namespace sdv {

__host__ __device__ constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }
__host__ __device__ __forceinline__ int fpad(int i) { return i + (i >> 3); }
// Unpadded in-place layout: XOR-swizzle within aligned groups of 8 elements
// (16 B each). The stride-8 Stockham stores of 8 consecutive lanes then hit 8
// distinct 16-byte bank groups, like the padded layout, but a length-N buffer
// occupies exactly N elements, so a transform can run in place over the rows
// it reads (no separate scratch buffer).
__host__ __device__ __forceinline__ int fswz(int i) { return i ^ ((i >> 3) & 7); }
template <bool SWZ>
__host__ __device__ __forceinline__ int fidx(int i) {
  return SWZ ? fswz(i) : fpad(i);
}
template <int N>
struct FftSize {
  static constexpr int kPadded = N + N / 8;  // double2 elements per team buffer
  static constexpr int kTeam = N / 8;        // threads per transform
};

__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
template <bool CONJ>
__host__ __device__ __forceinline__ double2 cmul_tw(double2 a, double2 w) {
  if (CONJ) return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.y, w.x, a.x * w.y));
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__host__ __device__ __forceinline__ double2 mul_mi(double2 d) {
  return INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
}

// In-register natural-order DFTs.
template <bool INV>
__host__ __device__ __forceinline__ void dft2(double2* v) {
  const double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <bool INV>
__host__ __device__ __forceinline__ void dft4(double2* v) {
  const double2 y0 = cadd(v[0], v[2]), y1 = csub(v[0], v[2]), y2 = cadd(v[1], v[3]);
  const double2 y3 = mul_mi<INV>(csub(v[1], v[3]));
  v[0] = cadd(y0, y2);
  v[2] = csub(y0, y2);
  v[1] = cadd(y1, y3);
  v[3] = csub(y1, y3);
}
template <bool INV>
__host__ __device__ __forceinline__ void dft8(double2* v) {
  constexpr double c = 0.70710678118654752440;
  double2 e[4] = {v[0], v[2], v[4], v[6]};
  double2 o[4] = {v[1], v[3], v[5], v[7]};
  dft4<INV>(e);
  dft4<INV>(o);
  // o[k] *= w8^k (forward w8 = e^{-i pi/4}; inverse conjugate)
  const double2 o1 = INV ? make_double2(c * (o[1].x - o[1].y), c * (o[1].x + o[1].y))
                         : make_double2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
  const double2 o2 = mul_mi<INV>(o[2]);
  const double2 o3 = INV ? make_double2(-c * (o[3].x + o[3].y), c * (o[3].x - o[3].y))
                         : make_double2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}
template <int R, bool INV>
__host__ __device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 8) dft8<INV>(v);
  else if constexpr (R == 4) dft4<INV>(v);
  else dft2<INV>(v);
}

template <int N, int PASS>
struct FftPass {
  static constexpr int L = ilog2_c(N);
  static constexpr int n8 = L / 3;
  static constexpr int rem = L % 3;
  static constexpr int NP = n8 + (rem ? 1 : 0);
  static constexpr int R = PASS < n8 ? 8 : (rem == 2 ? 4 : 2);
  static constexpr int NS = 1 << (3 * PASS);
  static constexpr bool LAST = PASS == NP - 1;
  // Offset of this pass's twiddle block in the per-pass table (pass 0 has
  // none; every pass before the last is radix 8).
  static constexpr int tw_off() {
    int off = 0, ns = 8;
    for (int p = 1; p < PASS; ++p) {
      off += 7 * ns;
      ns *= 8;
    }
    return off;
  }
  static constexpr int kTwOff = tw_off();
};

// Per-pass twiddle table of a length-n transform: pass p >= 1 owns a block of
// (R_p - 1) NS_p entries, entry (r-1) NS_p + k = exp(-2 pi i r k S_p / n),
// S_p = n / (NS_p R_p). Lanes of a warp hold consecutive k, so each twiddle
// load is one contiguous 16-byte-per-lane access (a table indexed by r k S
// gathers from up to 32 cache lines per load and dominated the L1 traffic).
// Values are bit-identical to exp(-2 pi i m / n) at m = r k S.
inline int fft_twiddle_count(int n) {
  int tot = 0, ns = 8, rest = n / 8;
  while (rest > 1) {
    const int r = rest >= 8 ? 8 : rest;
    tot += (r - 1) * ns;
    ns *= r;
    rest /= r;
  }
  return tot;
}
template <class Cplx, class Make>
void fft_build_twiddles(int n, Cplx* out, Make make) {
  int off = 0, ns = 8, rest = n / 8;
  while (rest > 1) {
    const int r = rest >= 8 ? 8 : rest, s = n / (ns * r);
    for (int rr = 1; rr < r; ++rr)
      for (int k = 0; k < ns; ++k) {
        const long m = static_cast<long>(rr) * k * s;
        const double ang = -2.0 * 3.14159265358979323846 * static_cast<double>(m) / static_cast<double>(n);
        out[off + (rr - 1) * ns + k] = make(ang);
      }
    off += (r - 1) * ns;
    ns *= r;
    rest /= r;
  }
}

// One Stockham pass for team thread t: 8/R butterflies b = t + (N/8) q.
// Input index of (q, r): b + r N/R; output index: (b - k) R + k + r NS.
// TWP: radix-8 passes load w^k and w^2k and form w^3k .. w^7k by products
// (5 complex multiplies instead of 5 more L1 loads; within a few ulp of the
// exact-rounded table). Used by the L1-bound fused stage kernels.
// TSM: the twiddle table is in shared memory (plain loads instead of __ldg).
template <bool TSM>
__host__ __device__ __forceinline__ double2 tw_load(const double2* p) {
#ifdef __CUDA_ARCH__
  if constexpr (TSM) return *p;
  else return __ldg(p);
#else
  return *p;
#endif
}
template <int N, int PASS, bool INV, bool TWP = false, bool TSM = false>
__host__ __device__ __forceinline__ void fft_pass_compute(double2* v, int t, const double2* __restrict__ tw) {
  using P = FftPass<N, PASS>;
  constexpr int R = P::R, G = 8 / R, T = N / 8;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int b = t + T * q;
    const int k = b & (P::NS - 1);
    if (P::NS > 1) {
      const double2* twp = tw + P::kTwOff + k;
      if constexpr (R == 8 && TWP) {
        const double2 w1 = tw_load<TSM>(twp), w2 = tw_load<TSM>(twp + P::NS);
        double2 w[8];
        w[1] = w1;
        w[2] = w2;
        w[3] = cmul_tw<false>(w2, w1);
        w[4] = cmul_tw<false>(w2, w2);
        w[5] = cmul_tw<false>(w[4], w1);
        w[6] = cmul_tw<false>(w[3], w[3]);
        w[7] = cmul_tw<false>(w[4], w[3]);
#pragma unroll
        for (int r = 1; r < R; ++r) v[q * R + r] = cmul_tw<INV>(v[q * R + r], w[r]);
      } else {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[q * R + r] = cmul_tw<INV>(v[q * R + r], tw_load<TSM>(twp + (r - 1) * P::NS));
        }
      }
    }
    dftR<R, INV>(v + q * R);
  }
}
template <int N, int PASS>
__host__ __device__ __forceinline__ int fft_in_index(int t, int q, int r) {
  using P = FftPass<N, PASS>;
  return t + (N / 8) * q + r * (N / P::R);
}
template <int N, int PASS>
__host__ __device__ __forceinline__ int fft_out_index(int t, int q, int r) {
  using P = FftPass<N, PASS>;
  const int b = t + (N / 8) * q;
  const int k = b & (P::NS - 1);
  return (b - k) * P::R + k + r * P::NS;
}

#ifdef __CUDACC__
// All threads of the CTA must call this (it synchronises with __syncthreads).
// buf: this team's padded buffer (FftSize<N>::kPadded double2). load(i) gives
// input element i; store(i, v) receives output element i (natural order).
// Threads with active == false only take part in the barriers. The caller
// must __syncthreads() before reusing buf or reading what store() wrote to
// shared memory.
// Barrier of fft_team: BAR = 0 synchronises the CTA; BAR > 0 is named
// barrier BAR over the calling team's N/8 threads only (warp-aligned teams),
// so one team can run a transform while the rest of the CTA does other work.
// BAR = -1: every team syncs on its own named barrier 1 + threadIdx.x / COUNT
// (teams are contiguous thread ranges; sub-warp teams use __syncwarp), so the
// teams of a CTA run their transforms without waiting for each other.
template <int BAR, int COUNT>
__device__ __forceinline__ void team_sync() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else if constexpr (BAR < 0) {
    if constexpr (COUNT < 32) {
      __syncwarp();
    } else {
      const int id = 1 + static_cast<int>(threadIdx.x) / COUNT;
      asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(COUNT) : "memory");
    }
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(COUNT) : "memory");
  }
}

// SWZ selects the buffer layout: padded (fpad, FftSize<N>::kPadded elements)
// or swizzled in place (fswz, exactly N elements).
template <int N, bool INV, int PASS = 0, bool SWZ = false, int BAR = 0, bool TWP = false, bool TSM = false, class Load,
          class Store>
__device__ __forceinline__ void fft_team(double2* buf, const double2* __restrict__ tw, int t, bool active, Load& load,
                                         Store& store) {
  using P = FftPass<N, PASS>;
  constexpr int R = P::R, G = 8 / R;
  double2 v[8];
  if (active) {
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = fft_in_index<N, PASS>(t, q, r);
        if constexpr (PASS == 0) v[q * R + r] = load(i);
        else v[q * R + r] = buf[fidx<SWZ>(i)];
      }
    fft_pass_compute<N, PASS, INV, TWP, TSM>(v, t, tw);
  }
  if constexpr (P::LAST) {
    team_sync<BAR, N / 8>();  // store() may target buf: all reads of this pass come first
    if (active) {
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) store(fft_out_index<N, PASS>(t, q, r), v[q * R + r]);
    }
  } else {
    team_sync<BAR, N / 8>();  // every read of buf in this pass precedes the in-place writes
    if (active) {
#pragma unroll
      for (int q = 0; q < G; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) buf[fidx<SWZ>(fft_out_index<N, PASS>(t, q, r))] = v[q * R + r];
    }
    team_sync<BAR, N / 8>();
    fft_team<N, INV, PASS + 1, SWZ, BAR, TWP, TSM>(buf, tw, t, active, load, store);
  }
}

#endif

// Device twiddle table exp(-2 pi i m / N), m in [0, N); cached per length.
const double2* twiddle_table(int n);

}  // namespace sdv

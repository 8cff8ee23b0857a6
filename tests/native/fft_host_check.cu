// Host-side check of the register-blocked Stockham FFT pass math in
// paper_2401_15758_b200/csrc/fft.cuh (all team threads emulated serially)
// against a naive DFT. Built and run by tests/test_native.py (no GPU needed).
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../paper_2401_15758_b200/csrc/fft.cuh"

using namespace sdv;

template <int N, bool INV, int PASS>
void run_pass(std::vector<double2>& a, const std::vector<double2>& tw) {
  using P = FftPass<N, PASS>;
  constexpr int R = P::R, G = 8 / R;
  std::vector<double2> b(N);
  for (int t = 0; t < N / 8; ++t) {
    double2 v[8];
    for (int q = 0; q < G; ++q)
      for (int r = 0; r < R; ++r) v[q * R + r] = a[fft_in_index<N, PASS>(t, q, r)];
    fft_pass_compute<N, PASS, INV>(v, t, tw.data());
    for (int q = 0; q < G; ++q)
      for (int r = 0; r < R; ++r) b[fft_out_index<N, PASS>(t, q, r)] = v[q * R + r];
  }
  a = b;
  if constexpr (!P::LAST) run_pass<N, INV, PASS + 1>(a, tw);
}

template <int N>
double check(bool inv) {
  std::vector<double2> tw(std::max(1, fft_twiddle_count(N))), x(N), y;
  fft_build_twiddles(N, tw.data(), [](double a) { return make_double2(std::cos(a), std::sin(a)); });
  for (int i = 0; i < N; ++i) x[i] = make_double2(std::sin(1.3 * i + 0.2), std::cos(0.7 * i * i + 1.0));
  y = x;
  if (inv) run_pass<N, true, 0>(y, tw);
  else run_pass<N, false, 0>(y, tw);
  double err = 0, nrm = 0;
  for (int k = 0; k < N; ++k) {
    double re = 0, im = 0;
    for (int n = 0; n < N; ++n) {
      const double ang = (inv ? 2 : -2) * M_PI * (double)((long long)n * k % N) / N;
      re += x[n].x * std::cos(ang) - x[n].y * std::sin(ang);
      im += x[n].x * std::sin(ang) + x[n].y * std::cos(ang);
    }
    err = std::fmax(err, std::hypot(y[k].x - re, y[k].y - im));
    nrm = std::fmax(nrm, std::hypot(re, im));
  }
  return err / nrm;
}

int main() {
  double worst = 0;
  auto rep = [&](int n, double e) {
    std::printf("N=%d rel err %.3e\n", n, e);
    worst = std::fmax(worst, e);
  };
  for (int inv = 0; inv < 2; ++inv) {
    rep(32, check<32>(inv));
    rep(64, check<64>(inv));
    rep(128, check<128>(inv));
    rep(256, check<256>(inv));
    rep(512, check<512>(inv));
    rep(1024, check<1024>(inv));
    rep(4096, check<4096>(inv));
  }
  std::printf("worst %.3e\n", worst);
  return worst < 1e-13 ? 0 : 1;
}

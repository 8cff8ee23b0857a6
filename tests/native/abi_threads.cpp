// Concurrency contract of the C-ABI (include/sdv.h): a plain C++ program that
// links libsdv_cuda.so and drives it the way the reference's callers do.
//
//  1. two threads, two problems (a Burgers and a BVE problem, each with its
//     own stream and workspaces) running Gram blocks concurrently;
//  2. eight threads on ONE trajectory, each pushing single columns through
//     sdv_misfit_apply_block / sdv_misfit_adjoint_block, as the reference's
//     apply_columns fans a GramMap out over std::threads
//     (proj/src/sketch.cpp:116-140, :212; "safe to call concurrently",
//     proj/include/sketchdav/model.hpp:9-13, linalg.hpp:14-16).
//
// Every concurrent result must be BITWISE equal to the serial one. Built and
// run by tests/test_native_abi.py (build on CPU, run with -m gpu).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/sdv.h"

namespace {
int fails = 0;
#define CHECK(x)                                                                   \
  do {                                                                             \
    if (!(x)) {                                                                    \
      std::fprintf(stderr, "FAIL %s:%d %s (%s)\n", __FILE__, __LINE__, #x, sdv_last_error()); \
      ++fails;                                                                     \
    }                                                                              \
  } while (0)

struct Setup {
  sdv_problem* p = nullptr;
  sdv_traj* t = nullptr;
  int64_t n = 0, m = 0;
};

// A periodic problem with deterministic observations (values from a smooth
// field), observing every 4th point (Burgers) / every 4th row and column (BVE).
Setup make(int model, int n, int steps_per_interval, double dt) {
  Setup s;
  sdv_problem_desc d{};
  d.model = model;
  d.n = n;
  d.nu = model == SDV_MODEL_BURGERS ? 0.005 : 1e-4;
  d.dt = dt;
  d.n_t = 2;
  d.steps_per_interval = steps_per_interval;
  d.prior_sigma = 0.1;
  d.prior_length = model == SDV_MODEL_BURGERS ? 0.05 : 0.3;
  d.prior_kind = SDV_PRIOR_FOURIER;
  const int64_t dim = model == SDV_MODEL_BURGERS ? n : static_cast<int64_t>(n) * n;
  std::vector<int64_t> idx;
  if (model == SDV_MODEL_BURGERS)
    for (int i = 0; i < n; i += 4) idx.push_back(i);
  else
    for (int j = 0; j < n; j += 4)
      for (int i = 0; i < n; i += 4) idx.push_back(i + static_cast<int64_t>(n) * j);
  const int64_t no = static_cast<int64_t>(idx.size());
  std::vector<double> bg(dim), val(no * d.n_t), var(no * d.n_t, 1e-4);
  for (int64_t i = 0; i < dim; ++i) bg[i] = std::sin(2.0 * M_PI * (i % n) / n) + 0.3 * std::cos(2.0 * M_PI * (i / n) / n);
  for (int64_t k = 0; k < no * d.n_t; ++k) val[k] = 0.9 * bg[idx[k % no]];
  CHECK(sdv_problem_create(&d, no, idx.data(), val.data(), var.data(), bg.data(), &s.p) == SDV_OK);
  CHECK(sdv_linearize(s.p, bg.data(), &s.t) == SDV_OK);
  int64_t dims[6];
  CHECK(sdv_problem_dims(s.p, dims) == SDV_OK);
  s.n = dims[0];
  s.m = dims[1];
  return s;
}

std::vector<double> randn(int64_t n, int64_t l, uint64_t seed) {
  std::vector<double> g(static_cast<size_t>(n * l));
  CHECK(sdv_gaussian_matrix(n, l, seed, g.data()) == SDV_OK);
  return g;
}
}  // namespace

int main() {
  CHECK(sdv_device_init(0) == SDV_OK);
  Setup a = make(SDV_MODEL_BURGERS, 256, 10, 1e-3);
  Setup b = make(SDV_MODEL_BVE, 64, 4, 0.02);
  const int s = 6;
  const auto va = randn(a.n, s, 11), vb = randn(b.n, s, 12);

  // serial references
  std::vector<double> ha(va.size()), hb(vb.size());
  CHECK(sdv_gram_apply_block(a.t, va.data(), s, ha.data()) == SDV_OK);
  CHECK(sdv_gram_apply_block(b.t, vb.data(), s, hb.data()) == SDV_OK);

  // 1. two threads, two problems, 10 Gram blocks each
  {
    int bad = 0;
    auto worker = [&](const Setup& x, const std::vector<double>& v, const std::vector<double>& ref) {
      std::vector<double> out(v.size());
      for (int r = 0; r < 10; ++r) {
        if (sdv_gram_apply_block(x.t, v.data(), s, out.data()) != SDV_OK || std::memcmp(out.data(), ref.data(), sizeof(double) * ref.size()))
          ++bad;
      }
    };
    std::thread t1(worker, std::cref(a), std::cref(va), std::cref(ha));
    std::thread t2(worker, std::cref(b), std::cref(vb), std::cref(hb));
    t1.join();
    t2.join();
    CHECK(bad == 0);
    std::printf("two problems x two threads: %d mismatching blocks of 20\n", bad);
  }

  // 2. eight threads on one trajectory, one column per call (apply_columns)
  for (const Setup* x : {&a, &b}) {
    const int cols = 16;
    const auto v = randn(x->n, cols, 21);
    const auto w = randn(x->m, cols, 22);
    std::vector<double> y_ser(static_cast<size_t>(x->m * cols)), z_ser(static_cast<size_t>(x->n * cols));
    for (int j = 0; j < cols; ++j) {
      CHECK(sdv_misfit_apply_block(x->t, v.data() + j * x->n, 1, y_ser.data() + j * x->m) == SDV_OK);
      CHECK(sdv_misfit_adjoint_block(x->t, w.data() + j * x->m, 1, z_ser.data() + j * x->n) == SDV_OK);
    }
    std::vector<double> y(y_ser.size()), z(z_ser.size());
    std::vector<std::thread> pool;
    for (int t = 0; t < 8; ++t)
      pool.emplace_back([&, t] {
        for (int j = t; j < cols; j += 8) {  // strided, as apply_columns
          CHECK(sdv_misfit_apply_block(x->t, v.data() + j * x->n, 1, y.data() + j * x->m) == SDV_OK);
          CHECK(sdv_misfit_adjoint_block(x->t, w.data() + j * x->m, 1, z.data() + j * x->n) == SDV_OK);
        }
      });
    for (auto& th : pool) th.join();
    const bool same = !std::memcmp(y.data(), y_ser.data(), sizeof(double) * y.size()) &&
                      !std::memcmp(z.data(), z_ser.data(), sizeof(double) * z.size());
    CHECK(same);
    std::printf("eight threads on one trajectory (n = %lld): %s\n", static_cast<long long>(x->n),
                same ? "bitwise equal to serial" : "MISMATCH");
  }

  sdv_traj_destroy(a.t);
  sdv_traj_destroy(b.t);
  sdv_problem_destroy(a.p);
  sdv_problem_destroy(b.p);
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}

// extern "C" boundary (include/sdv.h). Converts C++ exceptions into status
// codes + a thread-local message, never throwing across the ABI.
#include <atomic>
#include <cstring>
#include <mutex>
#include <limits>
#include <string>

#include "../../include/sdv.h"
#include "engine.hpp"
#include "solver.hpp"

// Scratch device buffers for the host-pointer entry points.
struct Scratch {
  sdv::DevBuf<double> a, b;
};
// One problem = one CUDA stream + its workspaces. Calls on one problem (and on
// its trajectories) are serialised by `mu`, so the reference's concurrent
// callers (apply_columns worker threads on one trajectory,
// proj/src/sketch.cpp:129-139; "safe to call concurrently",
// proj/include/sketchdav/model.hpp:9-13) are safe; distinct problems share no
// mutable state and run concurrently on their own streams.
// The handle is reference-counted: one reference for the caller's handle and
// one per live trajectory, so destroying a problem before its trajectories
// (finalisers of garbage-collected host languages run in no particular
// order) defers its release to the last sdv_traj_destroy instead of leaving
// their owner pointers dangling.
struct sdv_problem {
  std::unique_ptr<sdv::Problem> p;
  mutable std::mutex mu;
  Scratch sc;
  std::atomic<int> refs{1};
};
struct sdv_traj {
  sdv_problem* owner = nullptr;
  std::unique_ptr<sdv::Trajectory> t;
  explicit sdv_traj(sdv_problem* o) : owner(o) { o->refs.fetch_add(1, std::memory_order_relaxed); }
  // never the last reference: the creating call or sdv_traj_destroy holds one
  ~sdv_traj() { owner->refs.fetch_sub(1, std::memory_order_acq_rel); }
};
namespace {
void release(sdv_problem* p) {
  if (p->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete p;
}
}  // namespace

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SDV_OK;
  } catch (const sdv::CudaError& e) {
    g_err = e.what();
    return SDV_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SDV_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SDV_ENUMERIC;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

using Lock = std::lock_guard<std::mutex>;
}  // namespace

namespace {
template <class F>
int block_host(sdv_traj* t, const double* in, long long in_rows, int s, double* out, long long out_rows, F&& f) {
  return guard([&] {
    need(t, "trajectory");
    if (s < 1) throw std::invalid_argument("block: need s >= 1");
    Lock lk(t->owner->mu);
    auto& q = *t->owner->p;
    auto& sc = t->owner->sc;
    sc.a.upload(in, static_cast<size_t>(in_rows) * s, q.stream());
    sc.b.ensure(static_cast<size_t>(out_rows) * s);
    f(q, sc.a.get(), sc.b.get());
    sc.b.download(out, static_cast<size_t>(out_rows) * s, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}
}  // namespace

extern "C" {

const char* sdv_last_error(void) { return g_err.c_str(); }
const char* sdv_version(void) { return "sdv-b200 0.1 (sm_100a)"; }
unsigned long long sdv_launch_count(void) { return sdv::g_launches.load(); }
int sdv_path_counts(uint64_t* out, int n) {
  for (int i = 0; i < n && i < sdv::kPathCount; ++i) out[i] = sdv::g_path[i].load();
  return sdv::kPathCount;
}
const char* sdv_path_name(int i) { return sdv::path_name(i); }

int sdv_device_init(int device) {
  return guard([&] {
    SDV_CUDA(cudaSetDevice(device));
    SDV_CUDA(cudaFree(nullptr));
  });
}

int sdv_problem_create(const sdv_problem_desc* desc, int64_t n_obs, const int64_t* idx, const double* values,
                       const double* variances, const double* background, sdv_problem** out) {
  return guard([&] {
    need(desc, "desc");
    need(out, "out");
    need(background, "background");
    if (n_obs > 0) {
      need(idx, "obs_indices");
      need(values, "obs_values");
      need(variances, "obs_variances");
    }
    sdv::ProblemDesc d;
    d.model = desc->model;
    d.n = desc->n;
    d.nu = desc->nu;
    d.dt = desc->dt;
    d.n_t = desc->n_t;
    d.spi = desc->steps_per_interval;
    d.prior_sigma = desc->prior_sigma;
    d.prior_length = desc->prior_length;
    d.block_group = desc->block_group;
    d.prior_kind = desc->prior_kind;
    d.prior_alpha = desc->prior_alpha;
    d.prior_beta = desc->prior_beta;
    d.ny = desc->ny;
    d.reynolds = desc->reynolds;
    d.rossby = desc->rossby;
    auto p = std::make_unique<sdv_problem>();
    static_assert(sizeof(long long) == sizeof(int64_t), "int64");
    p->p = std::make_unique<sdv::Problem>(d, n_obs, reinterpret_cast<const long long*>(idx), values, variances,
                                          background);
    *out = p.release();
  });
}
void sdv_problem_destroy(sdv_problem* p) {
  if (p) release(p);
}

int sdv_problem_dims(const sdv_problem* p, int64_t dims[6]) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    const auto& q = *p->p;
    dims[0] = q.dim();
    dims[1] = q.m();
    dims[2] = q.n_obs();
    dims[3] = q.desc().n_t;
    dims[4] = q.desc().spi;
    dims[5] = q.total_steps();
  });
}

int sdv_forward(sdv_problem* p, const double* x0, int steps, double* out) {
  return guard([&] {
    need(p, "problem");
    if (steps < 0) throw std::invalid_argument("forward: steps must be >= 0");
    Lock lk(p->mu);
    auto& q = *p->p;
    auto& s = p->sc;
    s.a.upload(x0, static_cast<size_t>(q.dim()), q.stream());
    s.b.ensure(static_cast<size_t>(q.dim()));
    q.forward(s.a.get(), steps, s.b.get());
    s.b.download(out, static_cast<size_t>(q.dim()), q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}

int sdv_linearize_ex_dev(sdv_problem* p, const double* x0_dev, int checkpoint_stride, int policy, sdv_traj** out) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(x0_dev, "x0");
    need(out, "out");
    auto t = std::make_unique<sdv_traj>(p);
    t->t = p->p->linearize(x0_dev, checkpoint_stride, policy);
    *out = t.release();
  });
}
int sdv_linearize_ex(sdv_problem* p, const double* x0, int checkpoint_stride, int policy, sdv_traj** out) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(x0, "x0");
    need(out, "out");
    auto& q = *p->p;
    sdv::DevBuf<double> d;
    d.upload(x0, static_cast<size_t>(q.dim()), q.stream());
    auto t = std::make_unique<sdv_traj>(p);
    t->t = q.linearize(d.get(), checkpoint_stride, policy);
    *out = t.release();
  });
}
int sdv_traj_info(const sdv_traj* t, int64_t info[4]) {
  return guard([&] {
    need(t, "trajectory");
    need(info, "info");
    Lock lk(t->owner->mu);
    info[0] = t->t->steps;
    info[1] = t->t->stride;
    info[2] = t->t->segments();
    info[3] = static_cast<int64_t>(t->t->stored_bytes());
  });
}
int sdv_sub_blocks(const sdv_problem* p, int s, int* n_sub) {
  return guard([&] {
    need(p, "problem");
    need(n_sub, "n_sub");
    *n_sub = p->p->sub_blocks(s);
  });
}
int sdv_linearize_dev(sdv_problem* p, const double* x0_dev, sdv_traj** out) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(out, "out");
    auto t = std::make_unique<sdv_traj>(p);
    t->t = p->p->linearize(x0_dev, p->p->desc().spi, sdv::kStoreAuto);
    *out = t.release();
  });
}
int sdv_linearize(sdv_problem* p, const double* x0, sdv_traj** out) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(x0, "x0");
    auto& q = *p->p;
    sdv::DevBuf<double> d;
    d.upload(x0, static_cast<size_t>(q.dim()), q.stream());
    auto t = std::make_unique<sdv_traj>(p);
    t->t = q.linearize(d.get(), q.desc().spi, sdv::kStoreAuto);
    *out = t.release();
  });
}
void sdv_traj_destroy(sdv_traj* t) {
  if (!t) return;
  sdv_problem* owner = t->owner;
  owner->refs.fetch_add(1, std::memory_order_relaxed);
  {
    Lock lk(owner->mu);
    delete t;
  }
  release(owner);
}

int sdv_traj_state_at(const sdv_traj* t, int step, double* out) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    auto& q = *t->owner->p;
    SDV_CUDA(cudaMemcpyAsync(out, t->t->state_at(step), sizeof(double) * q.dim(), cudaMemcpyDeviceToHost,
                             q.stream()));
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}


int sdv_tlm_range(sdv_traj* t, int begin, int end, const double* dx, int s, double* out) {
  const long long n = t ? t->owner->p->dim() : 0;
  return block_host(t, dx, n, s, out, n, [&](sdv::Problem& q, double* a, double* b) {
    SDV_CUDA(cudaMemcpyAsync(b, a, sizeof(double) * n * s, cudaMemcpyDeviceToDevice, q.stream()));
    q.tlm(*t->t, b, s, begin, end, nullptr, nullptr);
  });
}
int sdv_adj_range(sdv_traj* t, int begin, int end, const double* lam, int s, double* out) {
  const long long n = t ? t->owner->p->dim() : 0;
  return block_host(t, lam, n, s, out, n, [&](sdv::Problem& q, double* a, double* b) {
    SDV_CUDA(cudaMemcpyAsync(b, a, sizeof(double) * n * s, cudaMemcpyDeviceToDevice, q.stream()));
    q.adj(*t->t, b, s, begin, end, nullptr, nullptr);
  });
}

int sdv_prior_sqrt_block(sdv_problem* p, const double* v, int s, double* out) {
  return guard([&] {
    need(p, "problem");
    if (s < 1) throw std::invalid_argument("block: need s >= 1");
    Lock lk(p->mu);
    auto& q = *p->p;
    auto& sc = p->sc;
    sc.a.upload(v, static_cast<size_t>(q.dim()) * s, q.stream());
    sc.b.ensure(static_cast<size_t>(q.dim()) * s);
    q.prior_sqrt(sc.a.get(), sc.b.get(), s);
    sc.b.download(out, static_cast<size_t>(q.dim()) * s, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}

int sdv_misfit_apply_block(sdv_traj* t, const double* V, int s, double* Y) {
  if (!t) return guard([] { throw std::invalid_argument("null argument: trajectory"); });
  auto& q0 = *t->owner->p;
  return block_host(t, V, q0.dim(), s, Y, q0.m(),
                    [&](sdv::Problem& q, double* a, double* b) { q.misfit_apply(*t->t, a, s, b); });
}
int sdv_misfit_adjoint_block(sdv_traj* t, const double* W, int s, double* Z) {
  if (!t) return guard([] { throw std::invalid_argument("null argument: trajectory"); });
  auto& q0 = *t->owner->p;
  return block_host(t, W, q0.m(), s, Z, q0.dim(),
                    [&](sdv::Problem& q, double* a, double* b) { q.misfit_adjoint(*t->t, a, s, b); });
}
int sdv_gram_apply_block(sdv_traj* t, const double* V, int s, double* HV) {
  if (!t) return guard([] { throw std::invalid_argument("null argument: trajectory"); });
  auto& q0 = *t->owner->p;
  return block_host(t, V, q0.dim(), s, HV, q0.dim(),
                    [&](sdv::Problem& q, double* a, double* b) { q.gram_apply(*t->t, a, s, b); });
}
int sdv_misfit_apply_block_dev(sdv_traj* t, const double* V, int s, double* Y) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    t->owner->p->misfit_apply(*t->t, V, s, Y);
  });
}
int sdv_misfit_adjoint_block_dev(sdv_traj* t, const double* W, int s, double* Z) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    t->owner->p->misfit_adjoint(*t->t, W, s, Z);
  });
}
int sdv_gram_apply_block_dev(sdv_traj* t, const double* V, int s, double* HV) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    t->owner->p->gram_apply(*t->t, V, s, HV);
  });
}

int sdv_evaluate(sdv_problem* p, const double* x0, const double* z, double* cost, double* ctrl_grad,
                 double* lambda0) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(x0, "x0");
    need(cost, "cost");
    auto& q = *p->p;
    const size_t n = static_cast<size_t>(q.dim());
    sdv::DevBuf<double> dx, dz, dg(n), dl(n);
    dx.upload(x0, n, q.stream());
    if (z) dz.upload(z, n, q.stream());
    auto tr = q.linearize(dx.get());
    *cost = q.evaluate(*tr, z ? dz.get() : nullptr, dg.get(), dl.get());
    if (ctrl_grad) dg.download(ctrl_grad, n, q.stream());
    if (lambda0) dl.download(lambda0, n, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}

int sdv_woodbury_apply(sdv_problem* p, int64_t l, const double* basis, const double* eig, const double* v, int s,
                       double* out) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    auto& q = *p->p;
    sdv::DeviceEVD e;
    e.upload(q.dim(), static_cast<int>(l), basis, eig, q.stream());
    const size_t n = static_cast<size_t>(q.dim());
    sdv::DevBuf<double> dv, dout(n * s);
    dv.upload(v, n * s, q.stream());
    for (int j = 0; j < s; ++j) sdv::woodbury_apply(e, dv.get() + j * n, dout.get() + j * n, q.dim(), q.stream());
    dout.download(out, n * s, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
  });
}

int sdv_thin_qr(sdv_problem* p, int64_t n, int64_t l, const double* y, double* q, double* r, int* ndef) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    cudaStream_t st = p->p->stream();
    sdv::DevBuf<double> d;
    d.upload(y, static_cast<size_t>(n * l), st);
    const int nd = sdv::dev_householder_qr(n, static_cast<int>(l), d.get(), r, st);
    d.download(q, static_cast<size_t>(n * l), st);
    SDV_CUDA(cudaStreamSynchronize(st));
    if (ndef) *ndef = nd;
  });
}

int sdv_thin_qr_dev(sdv_problem* p, int64_t n, int64_t l, double* y_dev, double* r, int* ndef) {
  return guard([&] {
    need(p, "problem");
    need(y_dev, "y");
    need(r, "r");
    Lock lk(p->mu);
    cudaStream_t st = p->p->stream();
    const int nd = sdv::dev_thin_qr(n, static_cast<int>(l), y_dev, r, st);  // the sketches' QR (CholQR2 / Householder)
    SDV_CUDA(cudaStreamSynchronize(st));
    if (ndef) *ndef = nd;
  });
}

int sdv_evd_from_tall_dev(sdv_problem* p, int64_t n, int64_t l, double* wt_dev, double shift, int floor0,
                          double* basis_dev, double* eig) {
  return guard([&] {
    need(p, "problem");
    need(wt_dev, "wt");
    need(eig, "eig");
    if (n < 1 || l < 1 || l > n) throw std::invalid_argument("evd_from_tall: need 1 <= l <= n");
    Lock lk(p->mu);
    cudaStream_t st = p->p->stream();
    const size_t nl = static_cast<size_t>(n) * static_cast<size_t>(l);
    sdv::DevBuf<double> wt(nl);
    SDV_CUDA(cudaMemcpyAsync(wt.get(), wt_dev, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    sdv::DeviceEVD e = sdv::evd_from_tall(wt, n, static_cast<int>(l), shift, floor0 != 0, st);
    if (basis_dev)
      SDV_CUDA(cudaMemcpyAsync(basis_dev, e.basis.get(), sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    SDV_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < l; ++i) eig[i] = e.eig[static_cast<size_t>(i)];
  });
}

int sdv_nystrom_assemble_dev(sdv_problem* p, int64_t n, int64_t l, const double* omega_dev, const double* y_dev,
                             double* basis_dev, double* eig) {
  return guard([&] {
    need(p, "problem");
    need(omega_dev, "omega");
    need(y_dev, "y");
    need(eig, "eig");
    if (n < 1 || l < 1 || l > n) throw std::invalid_argument("nystrom_assemble: need 1 <= l <= n");
    Lock lk(p->mu);
    cudaStream_t st = p->p->stream();
    sdv::DeviceEVD e = sdv::nystrom_assemble(omega_dev, y_dev, n, static_cast<int>(l), st);
    const size_t nl = static_cast<size_t>(n) * static_cast<size_t>(l);
    if (basis_dev)
      SDV_CUDA(cudaMemcpyAsync(basis_dev, e.basis.get(), sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    SDV_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < l; ++i) eig[i] = e.eig[static_cast<size_t>(i)];
  });
}

int sdv_sketch(sdv_traj* t, int method, int rank, int rank2, uint64_t seed, double* eig, double* basis,
               int64_t counts[3]) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    need(eig, "eig");
    auto& q = *t->owner->p;
    sdv::MisfitOp op(q, *t->t);
    sdv::SketchResult r = sdv::sketch(op, method, rank, rank2, seed);
    std::memcpy(eig, r.evd.eig.data(), sizeof(double) * r.evd.l);
    if (basis) r.evd.basis.download(basis, static_cast<size_t>(q.dim()) * r.evd.l, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
    if (counts) {
      counts[0] = r.tlm;
      counts[1] = r.adj;
      counts[2] = r.final_rank;
    }
  });
}

int sdv_lanczos_sketch(sdv_traj* t, int rank, const double* start, double* eig, double* basis, int64_t counts[3]) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    need(start, "start");
    need(eig, "eig");
    auto& q = *t->owner->p;
    sdv::MisfitOp op(q, *t->t);
    sdv::DevBuf<double> st;
    st.upload(start, static_cast<size_t>(q.dim()), q.stream());
    sdv::SketchResult r = sdv::lanczos_sketch(op, rank, st.get());
    std::memcpy(eig, r.evd.eig.data(), sizeof(double) * r.evd.l);
    if (basis) r.evd.basis.download(basis, static_cast<size_t>(q.dim()) * r.evd.l, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
    if (counts) {
      counts[0] = r.tlm;
      counts[1] = r.adj;
      counts[2] = r.final_rank;
    }
  });
}

int sdv_sketch_adaptive(sdv_traj* t, int method, int rank, int growth, int max_rank, int rank2, double eps_sketch,
                        uint64_t seed, double* eig, double* basis, int64_t counts[5], double* kappa, int max_kappa) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    need(eig, "eig");
    need(counts, "counts");
    if (method < 0 || method > 2) throw std::invalid_argument("sdv_sketch_adaptive: method must be 0, 1 or 2");
    auto& q = *t->owner->p;
    sdv::SketchCfg c;
    c.method = method;
    c.rank = rank;
    c.growth = growth;
    c.max_rank = max_rank;
    c.rank2 = rank2;
    c.eps_sketch = eps_sketch;
    c.seed = seed;
    // offline (sketch) and online (probe) applications are charged separately,
    // as gn_solve does (proj/src/fourdvar.cpp:257-324)
    sdv::MisfitOp off(q, *t->t), on(q, *t->t);
    sdv::SketchResult r = method == 0   ? sdv::adaptive_randsvd(off, c, on)
                          : method == 1 ? sdv::adaptive_nystrom(off, c, on)
                                        : sdv::adaptive_singleview(off, c, on);
    std::memcpy(eig, r.evd.eig.data(), sizeof(double) * r.evd.l);
    if (basis) r.evd.basis.download(basis, static_cast<size_t>(q.dim()) * r.evd.l, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
    counts[0] = r.tlm;
    counts[1] = r.adj;
    counts[2] = r.final_rank;
    counts[3] = r.probes;
    counts[4] = r.tolerance_met;
    if (kappa)
      for (int i = 0; i < max_kappa && i < static_cast<int>(r.kappa.size()); ++i) kappa[i] = r.kappa[i];
  });
}

int sdv_cond_estimate(sdv_traj* t, int64_t l, const double* basis, const double* eig, uint64_t seed, double* kappa) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    need(kappa, "kappa");
    auto& q = *t->owner->p;
    sdv::DeviceEVD e;
    if (l > 0) e.upload(q.dim(), static_cast<int>(l), basis, eig, q.stream());
    sdv::MisfitOp op(q, *t->t);
    *kappa = sdv::cond_estimate(op, e, seed);
  });
}

int sdv_pcg_solve(sdv_traj* t, const double* rhs, int64_t l, const double* basis, const double* eig, double tol,
                  int max_iter, double* x, int info[2]) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    auto& q = *t->owner->p;
    const size_t n = static_cast<size_t>(q.dim());
    sdv::DeviceEVD e;
    if (l > 0) e.upload(q.dim(), static_cast<int>(l), basis, eig, q.stream());
    sdv::MisfitOp op(q, *t->t);
    sdv::DevBuf<double> db, dx(n);
    db.upload(rhs, n, q.stream());
    const sdv::PCGResult r = sdv::pcg_solve(op, db.get(), l > 0 ? &e : nullptr, tol, max_iter, dx.get());
    dx.download(x, n, q.stream());
    SDV_CUDA(cudaStreamSynchronize(q.stream()));
    info[0] = r.iterations;
    info[1] = r.converged;
  });
}

int sdv_gn_solve(sdv_problem* p, const sdv_gn_config* cfg, double* analysis, double* log, int max_log, int* n_iters,
                 double summary[5], double* eig0, int max_eig) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    need(cfg, "config");
    sdv::GNConfig g;
    g.mode = cfg->mode;
    g.method = cfg->method;
    g.rank = cfg->rank;
    g.rank2 = cfg->rank2;
    g.growth = cfg->growth;
    g.max_rank = cfg->max_rank;
    g.eps_sketch = cfg->eps_sketch;
    g.eps_reuse = cfg->eps_reuse;
    g.seed = cfg->seed;
    g.grad_tol = cfg->grad_tol;
    g.pcg_tol = cfg->pcg_tol;
    g.max_gn_iters = cfg->max_gn_iters;
    g.pcg_max_iter = cfg->pcg_max_iter;
    const sdv::GNResult r = sdv::gn_solve(*p->p, g);
    std::memcpy(analysis, r.analysis.data(), sizeof(double) * r.analysis.size());
    if (n_iters) *n_iters = static_cast<int>(r.iterations.size());
    for (size_t i = 0; log && i < r.iterations.size() && static_cast<int>(i) < max_log; ++i)
      std::memcpy(log + 16 * i, r.iterations[i].rec, sizeof(double) * 16);
    if (summary) {
      summary[0] = r.final_cost;
      summary[1] = r.final_grad_inf_norm;
      summary[2] = static_cast<double>(r.total_pcg);
      summary[3] = r.converged;
      summary[4] = r.line_search_failed;
    }
    if (eig0) {
      for (int i = 0; i < max_eig; ++i)
        eig0[i] = i < static_cast<int>(r.eig0.size()) ? r.eig0[i] : std::numeric_limits<double>::quiet_NaN();
    }
  });
}

uint64_t sdv_mix_seed(uint64_t seed, uint64_t stream) { return sdv::mix_seed(seed, stream); }
int sdv_gaussian_matrix(int64_t n, int64_t l, uint64_t seed, double* out) {
  return guard([&] {
    need(out, "out");
    const std::vector<double> g = sdv::gaussian_matrix(n, l, seed);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

int sdv_dev_alloc(size_t bytes, void** ptr) { return guard([&] { SDV_CUDA(cudaMalloc(ptr, bytes)); }); }
int sdv_dev_free(void* ptr) { return guard([&] { SDV_CUDA(cudaFree(ptr)); }); }
int sdv_host_alloc(size_t bytes, void** ptr) { return guard([&] { SDV_CUDA(cudaMallocHost(ptr, bytes)); }); }
int sdv_host_free(void* ptr) { return guard([&] { SDV_CUDA(cudaFreeHost(ptr)); }); }
int sdv_memcpy_htod(void* dst, const void* src, size_t bytes) {
  return guard([&] { SDV_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); });
}
int sdv_memcpy_dtoh(void* dst, const void* src, size_t bytes) {
  return guard([&] { SDV_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}
int sdv_synchronize(sdv_problem* p) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    SDV_CUDA(cudaStreamSynchronize(p->p->stream()));
  });
}
int sdv_event_create(void** ev) {
  return guard([&] {
    cudaEvent_t e;
    SDV_CUDA(cudaEventCreate(&e));
    *ev = e;
  });
}
int sdv_event_destroy(void* ev) { return guard([&] { SDV_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev))); }); }
int sdv_event_record(sdv_problem* p, void* ev) {
  return guard([&] {
    need(p, "problem");
    Lock lk(p->mu);
    SDV_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), p->p->stream()));
  });
}
int sdv_event_elapsed_ms(void* a, void* b, float* ms) {
  return guard([&] {
    SDV_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(b)));
    SDV_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  });
}
int sdv_probe_stage_kernels(sdv_traj* t, int s, int stages, float* ms_stage, float* ms_col) {
  return guard([&] {
    need(t, "trajectory");
    Lock lk(t->owner->mu);
    t->owner->p->probe_stage_kernels(*t->t, s, stages, ms_stage, ms_col);
  });
}
int sdv_probe_adj_stage_kernels(sdv_traj* t, int s, int stages, float* ms_stage, float* ms_col) {
  return guard([&] {
    need(t, "trajectory");
    need(ms_stage, "ms_stage");
    need(ms_col, "ms_col");
    Lock lk(t->owner->mu);
    t->owner->p->probe_adj_stage_kernels(*t->t, s, stages, ms_stage, ms_col);
  });
}

}  // extern "C"

// Common device/host helpers for the sm_100a SC-4DVAR Hessian-product engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sdv {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SDV_CUDA(call)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::sdv::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

#define SDV_LAUNCH_CHECK() SDV_CUDA(cudaGetLastError())

// RAII device buffer.
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t n) {
    if (n == n_ && p_) return;
    release();
    if (n) SDV_CUDA(cudaMalloc(&p_, n * sizeof(T)));
    n_ = n;
  }
  void ensure(size_t n) {
    if (n > n_) alloc(n);
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* h, size_t n, cudaStream_t s) {
    ensure(n);
    SDV_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* h, size_t n, cudaStream_t s) const {
    SDV_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Programmatic dependent launch (PDL): a kernel launched through launch_pdl
// may start while its stream predecessor is still running; it must call
// pdl_wait() before touching anything the predecessor writes, and calls
// pdl_trigger() once all its CTAs are resident so its own successor can be
// scheduled into the tail. Measured on B200 (tools/small_block.py, C3): the
// one-vector Gram sweep took 100.6 ms with PDL vs 81.0 ms without, and the
// s = 110 block was unchanged, so PDL is opt-in (SDV_PDL=1); without it
// the griddepcontrol instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
inline bool pdl_enabled() {
  static const bool on = std::getenv("SDV_PDL") != nullptr;
  return on;
}
template <class... KArgs, class... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SDV_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

}  // namespace sdv

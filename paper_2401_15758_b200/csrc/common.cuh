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

// ---- TMA bulk copies + mbarriers (sm_90+ PTX; sm_100a here) ----
// 1-D bulk copy global -> shared (the TMA engine; UBLKCP in SASS), completion
// counted in bytes on an mbarrier; one elected thread arms and issues.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arm(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// Orders earlier generic-proxy accesses to shared memory (made CTA-visible by
// a preceding barrier) before async-proxy (bulk copy) writes to it.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Programmatic dependent launch (PDL): a kernel launched through launch_pdl
// may be scheduled while its stream predecessor is still running. It calls
// pdl_wait() before touching anything the predecessor writes (the wait returns
// when the predecessor has completed and flushed) and pdl_trigger() AFTER the
// wait, so at most one successor is resident behind a running kernel and only
// its launch latency and prologue overlap. (Round 1 triggered before the
// wait: chains of waiting grids piled up on the SMs and the one-vector sweep
// got slower.) Where the trigger sits matters, because an early successor's
// CTAs land on whatever SMs have room at that moment: the 8-row stage kernels
// trigger before their last phase, the small-block (2-row) stage kernels only
// at exit, the column / carry / row kernels right after their wait. Measured
// on B200 (tools/small_block.py, us per stage-step, PDL vs not;
// profiles/r2_small_blocks.md): 512^2 s = 1 / 2 / 4: 11.1 / 15.2 / 20.5 vs
// 12.4 / 16.8 / 22.9; 256^2 s = 1 / 4 / 8: 7.3 / 10.1 / 13.1 vs 8.4 / 11.4 /
// 14.5; 128^2 s = 1 / 2: 6.8 / 7.1 vs 8.0 / 8.9. SDV_NO_PDL turns PDL off
// (without the launch attribute the griddepcontrol instructions are no-ops).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
inline bool pdl_enabled() {
  static const bool on = std::getenv("SDV_NO_PDL") == nullptr;
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

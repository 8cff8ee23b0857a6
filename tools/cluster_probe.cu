// Feasibility probe: max co-resident thread-block clusters of size 8/16 at a
// given dynamic smem, and the latency of cluster.sync() / DSMEM reads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_loop(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  sm[threadIdx.x] = threadIdx.x + cl.block_rank();
  cl.sync();
  double acc = 0;
  const unsigned r = (cl.block_rank() + 1) % cl.num_blocks();
  double* rem = cl.map_shared_rank(sm, r);
  for (int i = 0; i < iters; ++i) {
    acc += rem[(threadIdx.x + i) & 255];
    cl.sync();
  }
  if (threadIdx.x == 0) out[blockIdx.x + gridDim.x * blockIdx.y] = acc;
}

int main() {
  cudaFuncSetAttribute(sync_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {4, 8, 16}) {
    for (int kb : {64, 140, 200, 220}) {
      size_t smem = kb * 1024;
      cudaFuncSetAttribute(sync_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, sync_loop, &cfg);
      printf("cluster %2d smem %3d KB: max active clusters %d (%s)\n", cs, kb, n, cudaGetErrorString(e));
      if (kb == 200 && n > 0) {
        double* out;
        cudaMalloc(&out, 8 * 1024);
        cfg.gridDim = dim3(cs, 1);
        const int iters = 20000;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaLaunchKernelEx(&cfg, sync_loop, 100, out);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, sync_loop, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("   cluster.sync + 1 DSMEM load per iteration: %.3f us (err %s)\n", ms * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(out);
      }
    }
  }
  return 0;
}

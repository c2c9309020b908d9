// probe: cooperative launch combined with thread-block clusters; max active clusters for a
// persistent-kernel-like configuration (512 threads, ~60 KB dynamic smem, 64 regs).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(512, 2) k(int* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  sm[threadIdx.x] = blockIdx.x;
  cl.sync();
  double* peer = cl.map_shared_rank(sm, (cl.block_rank() + 1) % cl.num_blocks());
  double v = peer[threadIdx.x];
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (int)v;
}
int main() {
  int* out; cudaMalloc(&out, 4096 * 4);
  const size_t smem = 60 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs * 4);
    int ncl = -1;
    cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(ncl > 0 ? ncl * cs : cs);
    cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[4] = {0};
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("cluster %2d: max active clusters %4d (%s) -> CTAs %4d; coop launch %s / %s; out[0..1] = %d %d\n", cs, ncl,
           cudaGetErrorString(e0), ncl * cs, cudaGetErrorString(e1), cudaGetErrorString(e2), h[0], h[1]);
    cudaGetLastError();
  }
  return 0;
}

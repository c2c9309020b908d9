// 2-D tensor-map TMA streaming microbenchmark
#include <cuda.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { uint32_t ok = 0; while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory"); }
template <int NS, int BR>
__global__ void __launch_bounds__(512, 1) k_tma2d(const __grid_constant__ CUtensorMap tm, int64_t n, int nc, int stage_bytes, double* out) {
  extern __shared__ __align__(1024) double ring[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int CB = (nc + 7) / 8;
  int RB = (stage_bytes / (BR * 64)) / CB; if (RB < 1) RB = 1; if (RB > 16) RB = 16;
  const int TR = RB * BR;
  const int64_t nb = n / BR;   // n multiple of BR
  const int64_t b0 = (int64_t)blockIdx.x * nb / gridDim.x, b1 = (int64_t)(blockIdx.x + 1) * nb / gridDim.x;
  const int64_t r0 = b0 * BR, r1 = b1 * BR;
  const int ntile = (int)((r1 - r0 + TR - 1) / TR);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[i])), "r"(15));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  if (wid == 15) {
    for (int t = 0; t < ntile; ++t) {
      int s = t % NS;
      if (t >= NS) wait(&empty[s], (uint32_t)((t / NS - 1) & 1));
      double* stg = ring + (size_t)s * (stage_bytes / 8);
      const int64_t rb = r0 + (int64_t)t * TR;
      const int nrb = (int)min((int64_t)RB, (r1 - rb) / BR);
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"((uint32_t)(nrb * CB * BR * 64)) : "memory");
      __syncwarp();
      for (int op = lane; op < nrb * CB; op += 32) {
        const int rbx = op % nrb, cbx = op / nrb;
        double* dst = stg + (size_t)(cbx * 8) * TR + rbx * BR;   // column-major tile, column stride TR
        // box lands as 8 columns of BR rows contiguous: we need column stride TR -> only valid when RB == 1;
        // for RB > 1 store boxes side by side: [cbx][rbx][8][BR]
        dst = stg + ((size_t)cbx * nrb + rbx) * (8 * BR);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(dst)), "l"(&tm), "r"((int)(rb + rbx * BR)), "r"(cbx * 8), "r"(su(&full[s])) : "memory");
      }
    }
  } else {
    for (int t = 0; t < ntile; ++t) {
      int s = t % NS;
      wait(&full[s], (uint32_t)((t / NS) & 1));
      double* stg = ring + (size_t)s * (stage_bytes / 8);
      const int64_t rb = r0 + (int64_t)t * TR;
      const int nrb = (int)min((int64_t)RB, (r1 - rb) / BR);
      const int tot = nrb * CB * 8 * BR;
      for (int e = threadIdx.x; e < tot; e += 480) acc += stg[e];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
  }
  if (acc == 12345.678) out[0] = acc;
}
int main() {
  const int64_t NMAX = 2097152; const int NC = 64;
  double *Z, *out; cudaMalloc(&Z, 8ull * NMAX * NC); cudaMalloc(&out, 8); cudaMemset(Z, 0, 8ull * NMAX * NC);
  double* flush; cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int64_t n : {262144ll, 2097152ll}) for (int nc : {2, 8, 32, 64}) {
    CUtensorMap tm128, tm256;
    cuuint64_t gd[2] = {(cuuint64_t)n, (cuuint64_t)nc}; cuuint64_t gs[1] = {(cuuint64_t)n * 8};
    cuuint32_t es[2] = {1, 1};
    cuuint32_t bd[2] = {128, 8};
    CUresult r1 = cuTensorMapEncodeTiled(&tm128, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Z, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t bd2[2] = {256, 8};
    CUresult r2 = cuTensorMapEncodeTiled(&tm256, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Z, gd, gs, bd2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) { printf("encode failed %d %d\n", r1, r2); return 1; }
    auto run = [&](auto launch, const char* name) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) { cudaMemset(flush, it, 512ull << 20); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best; }
      printf("n=%7lld nc=%2d %-24s %8.2f us %7.0f GB/s\n", (long long)n, nc, name, best * 1e3, 8.0 * n * nc / (best * 1e-3) / 1e9);
    };
    for (int sb : {32768, 65536}) {
      int ns = (200 * 1024) / sb; char nm[64];
      if (ns >= 6) { cudaFuncSetAttribute(k_tma2d<6, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * sb); snprintf(nm, 64, "2d128 6x%dK", sb / 1024); run([&] { k_tma2d<6, 128><<<148, 512, 6 * sb>>>(tm128, n, nc, sb, out); }, nm); }
      else { cudaFuncSetAttribute(k_tma2d<3, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * sb); snprintf(nm, 64, "2d128 3x%dK", sb / 1024); run([&] { k_tma2d<3, 128><<<148, 512, 3 * sb>>>(tm128, n, nc, sb, out); }, nm);
             cudaFuncSetAttribute(k_tma2d<3, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * sb); snprintf(nm, 64, "2d256 3x%dK", sb / 1024); run([&] { k_tma2d<3, 256><<<148, 512, 3 * sb>>>(tm256, n, nc, sb, out); }, nm); }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

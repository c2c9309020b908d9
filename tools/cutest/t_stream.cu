// microbenchmark: stream `nc` columns of n doubles (column-major, ld) and dot each with column 0.
// variants: (a) LDG thread-per-row, (b) TMA 1-D bulk copies into a multi-stage smem ring.
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(512) k_ldg(const double* Z, int64_t ld, int64_t n, int nc, double* out) {
  double acc = 0;
  for (int64_t r = blockIdx.x * 512ll + threadIdx.x; r < n; r += (int64_t)gridDim.x * 512) {
    double z[8]; int c = 0;
    for (; c + 8 <= nc; c += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) z[u] = __ldcs(Z + (c + u) * ld + r);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += z[u];
    }
    for (; c < nc; ++c) acc += __ldcs(Z + c * ld + r);
  }
  if (acc == 12345.678) out[0] = acc;
}
template <int NS>
__global__ void __launch_bounds__(512, 1) k_tma(const double* Z, int64_t ld, int64_t n, int nc, int stage_bytes, double* out) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  int TR = (stage_bytes / 8) / nc; TR = TR >= 4096 ? 4096 : (TR & ~31);
  const int64_t ng = n >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5, r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
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
      if (t >= NS) { uint32_t ok = 0; while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(&empty[s])), "r"((uint32_t)((t / NS - 1) & 1)) : "memory"); }
      double* stg = ring + (size_t)s * (stage_bytes / 8);
      int64_t rb = r0 + (int64_t)t * TR; uint32_t bytes = (uint32_t)min((int64_t)TR, r1 - rb) * 8u;
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(bytes * nc) : "memory");
      __syncwarp();
      for (int c = lane; c < nc; c += 32)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(stg + (size_t)c * TR)), "l"(Z + c * ld + rb), "r"(bytes), "r"(su(&full[s])) : "memory");
    }
  } else {
    for (int t = 0; t < ntile; ++t) {
      int s = t % NS;
      uint32_t ok = 0; while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(&full[s])), "r"((uint32_t)((t / NS) & 1)) : "memory");
      double* stg = ring + (size_t)s * (stage_bytes / 8);
      int64_t rb = r0 + (int64_t)t * TR; int rows = (int)min((int64_t)TR, r1 - rb);
      for (int c = wid; c < nc; c += 15) for (int r = lane; r < rows; r += 32) acc += stg[(size_t)c * TR + r];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
  }
  if (acc == 12345.678) out[0] = acc;
}
int main() {
  const int64_t n = 2097152; const int NCMAX = 64;
  double *Z, *out; cudaMalloc(&Z, 8ull * n * NCMAX); cudaMalloc(&out, 8); cudaMemset(Z, 0, 8ull * n * NCMAX);
  double* flush; cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int64_t nn : {262144ll, 2097152ll}) for (int nc : {2, 8, 32, 61}) {
    auto run = [&](auto launch, const char* name) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) { cudaMemset(flush, it, 512ull << 20); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best; }
      double gb = 8.0 * nn * nc / (best * 1e-3) / 1e9;
      printf("n=%lld nc=%2d %-22s %8.2f us %7.0f GB/s\n", (long long)nn, nc, name, best * 1e3, gb);
    };
    run([&] { k_ldg<<<296, 512>>>(Z, n, nn, nc, out); }, "ldg 296x512");
    for (int sb : {16384, 32768, 49152}) {
      cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * sb);
      char nm[64]; snprintf(nm, 64, "tma4 stage %dK", sb / 1024);
      run([&] { k_tma<4><<<148, 512, 4 * sb>>>(Z, n, nn, nc, sb, out); }, nm);
    }
    cudaFuncSetAttribute(k_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 24576);
    run([&] { k_tma<8><<<148, 512, 8 * 24576>>>(Z, n, nn, nc, 24576, out); }, "tma8 stage 24K");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

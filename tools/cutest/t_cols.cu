// probe: cold-L2 streaming of nc basis columns (n = 2M rows, column-major, ld = n) by 1-D TMA bulk
// copies into a shared-memory ring, the DK1 / DK2 access pattern.  Parameters: rows per copy TR,
// columns per stage CPS (stage = CPS copies of TR rows), ring depth NS, order (tile-outer: for each
// row tile all columns; chunk-outer: for each chunk of CPS columns all row tiles), L2 policy.
// Consumers (16 warps) only sum what lands.  L2 flushed (512 MB memset) before every launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cutest/t_cols tools/cutest/t_cols.cu
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
}
constexpr int NSMAX = 16;
__global__ void __launch_bounds__(544, 1) k_tma(const double* Z, int64_t ld, int64_t n, int nc, int TR, int CPS, int NS,
                                              int tile_outer, int evict_first, double* out, int desc = 0) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[NSMAX], empty[NSMAX];
  const int64_t ng = n >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5, r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const int ntile = (int)((r1 - r0 + TR - 1) / TR), nch = (nc + CPS - 1) / CPS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int SD = TR * CPS;  // doubles per stage
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[i])), "r"(16));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nst = ntile * nch;
  double acc = 0;
  if (wid == 16) {
    if (lane == 0) {
      uint64_t pol;
      if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      for (int t = 0; t < nst; ++t) {
        const int s = t % NS;
        if (t >= NS) wait(&empty[s], (uint32_t)((t / NS - 1) & 1));
        int ti = tile_outer ? t / nch : t % ntile;
        const int q = tile_outer ? t % nch : t / ntile;
        if (desc) ti = ntile - 1 - ti;
        const int64_t rb = r0 + (int64_t)ti * TR;
        const uint32_t rows = (uint32_t)min((int64_t)TR, r1 - rb);
        const int ncs = min(CPS, nc - q * CPS);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(rows * 8u * ncs) : "memory");
        for (int c = 0; c < ncs; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(su(ring + (size_t)s * SD + (size_t)c * TR)), "l"(Z + (int64_t)(q * CPS + c) * ld + rb),
                       "r"(rows * 8u), "r"(su(&full[s])), "l"(pol) : "memory");
      }
    }
  } else {
    for (int t = 0; t < nst; ++t) {
      const int s = t % NS;
      wait(&full[s], (uint32_t)((t / NS) & 1));
      const double* stg = ring + (size_t)s * SD;
      for (int i = threadIdx.x; i < SD; i += 512) acc += stg[i];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
  }
  if (acc == 12345.678) out[0] = acc;
}
// plain loads: thread per row, 8 columns in flight per thread, rows grid-strided
__global__ void __launch_bounds__(512, 2) k_ldg(const double* Z, int64_t ld, int64_t n, int nc, double* out) {
  double acc = 0;
  for (int64_t r = blockIdx.x * 512ll + threadIdx.x; r < n; r += (int64_t)gridDim.x * 512) {
    int c = 0;
    for (; c + 8 <= nc; c += 8) {
      double z[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) z[u] = __ldcs(Z + (c + u) * ld + r);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += z[u];
    }
    for (; c < nc; ++c) acc += __ldcs(Z + c * ld + r);
  }
  if (acc == 12345.678) out[0] = acc;
}
// ideal: the nc columns as one flat array, 16-byte loads, 4 in flight per thread
__global__ void __launch_bounds__(512, 2) k_flat(const double2* Z, int64_t n2, double* out) {
  double acc = 0;
  const int64_t st = (int64_t)gridDim.x * 512;
  int64_t i = blockIdx.x * 512ll + threadIdx.x;
  for (; i + 3 * st < n2; i += 4 * st) {
    double2 a = __ldcs(Z + i), b = __ldcs(Z + i + st), c = __ldcs(Z + i + 2 * st), d = __ldcs(Z + i + 3 * st);
    acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  for (; i < n2; i += st) acc += Z[i].x + Z[i].y;
  if (acc == 12345.678) out[0] = acc;
}
int main(int argc, char**) {
  const int64_t n = 2097152;
  const int NCMAX = 56;
  double *Z, *out, *flush;
  cudaMalloc(&Z, 8ull * n * NCMAX);
  cudaMalloc(&out, 8);
  cudaMemset(Z, 0, 8ull * n * NCMAX);
  cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nc : {11, 21, 35, 51}) {
    if (argc > 1) break;  // "pair": only the L2-reuse experiment
    auto run = [&](auto launch, const char* name) {
      float best = 1e9, warm = 1e9;
      for (int it = 0; it < 7; ++it) {
        cudaMemset(flush, it, 512ull << 20);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      for (int it = 0; it < 5; ++it) {  // back to back (what the solver sees: no flush)
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        warm = ms < warm ? ms : warm;
      }
      const double gb = 8.0 * n * nc / 1e9;
      printf("nc=%2d %-40s cold %8.2f us %6.0f GB/s   b2b %8.2f us %6.0f GB/s\n", nc, name, best * 1e3, gb / (best * 1e-3),
             warm * 1e3, gb / (warm * 1e-3));
    };
    run([&] { k_flat<<<296, 512>>>((const double2*)Z, n * nc / 2, out); }, "flat 16B loads");
    run([&] { k_ldg<<<296, 512>>>(Z, n, n, nc, out); }, "ldg thread/row 8 cols");
    struct V { int TR, CPS, NS, to; };
    for (V v : {V{512, 8, 4, 0}, V{512, 8, 4, 1}, V{512, 8, 6, 1}, V{512, 8, 6, 0}, V{1024, 4, 6, 1}, V{2048, 2, 6, 1},
                V{4096, 1, 6, 1}, V{4096, 1, 6, 0}, V{2048, 1, 12, 1}, V{1024, 2, 12, 1}, V{8192, 1, 3, 1}}) {
      for (int ef : {1, 0}) {
        char nm[96];
        snprintf(nm, 96, "tma TR=%d CPS=%d NS=%d %s %s", v.TR, v.CPS, v.NS, v.to ? "tile-outer" : "chunk-outer", ef ? "EF" : "EN");
        const int smem = v.TR * v.CPS * v.NS * 8;
        run([&] { k_tma<<<148, 544, smem>>>(Z, n, n, nc, v.TR, v.CPS, v.NS, v.to, ef, out); }, nm);
      }
    }
  }
  // L2 reuse between consecutive passes: pass 1 (tile-outer ascending, evict-normal), optionally a
  // 217 MB evict-first stream in between (the Arnoldi SpMV's matrix), then pass 2 timed alone
  double* A2;
  cudaMalloc(&A2, 220ull << 20);
  cudaMemset(A2, 0, 220ull << 20);
  for (int nc : {21, 35, 51}) {
    for (int mid : {0, 1})
      for (int v = 0; v < 4; ++v) {
        const int desc = v & 1, ef1 = v >> 1;  // pass-2 direction; pass-1 policy
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
          cudaMemset(flush, it, 512ull << 20);
          k_tma<<<148, 544, 512 * 8 * 6 * 8>>>(Z, n, n, nc, 512, 8, 6, 1, ef1, out, 0);
          if (mid) k_flat<<<296, 512>>>((const double2*)A2, (220ll << 20) / 16, out);
          cudaEventRecord(a);
          k_tma<<<148, 544, 512 * 8 * 6 * 8>>>(Z, n, n, nc, 512, 8, 6, 1, 0, out, desc);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        printf("pair nc=%2d pass1 %s, %s, pass2 %s EN: %8.2f us %6.0f GB/s\n", nc, ef1 ? "EF" : "EN",
               mid ? "220 MB stream between" : "back to back", desc ? "DESC" : "asc ", best * 1e3, 8.0 * n * nc / 1e9 / (best * 1e-3));
      }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

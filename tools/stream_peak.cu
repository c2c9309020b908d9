// Read-only and copy HBM stream peaks on this box ("also measure a read-only stream
// peak").  fp64 arrays of 2 GiB (16x the L2), LDG with 8 independent loads in flight per thread,
// grid = 148 SMs x 8 CTAs x 512 threads, best of 10 launches timed with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_peak tools/stream_peak.cu
// Prints one JSON line.
#include <cstdio>
#include <cstdint>

template <bool STREAM>
__global__ void __launch_bounds__(512) k_read_t(const double* __restrict__ a, int64_t n, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = STREAM ? __ldcs(a + i + u * stride) : a[i + u * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; i < n; i += stride) acc += STREAM ? __ldcs(a + i) : a[i];
  if (acc == 1.2345e300) out[0] = acc;  // keeps the loads alive
}
#define k_read k_read_t<true>

// L2-resident read: the same `n` doubles read `reps` times inside one launch (no launch gaps)
__global__ void __launch_bounds__(512) k_read_rep(const double* __restrict__ a, int64_t n, int reps, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int rep = 0; rep < reps; ++rep) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a[i + u * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; i < n; i += stride) acc += a[i];
  }
  if (acc == 1.2345e300) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(b + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(b + i, __ldcs(a + i));
}

__global__ void k_init(double* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = 1.0 + (double)(i & 1023);
}

int main() {
  const int64_t n = (int64_t)1 << 28;  // 2 GiB of fp64
  double *a, *b, *out;
  if (cudaMalloc(&a, n * 8) || cudaMalloc(&b, n * 8) || cudaMalloc(&out, 8)) { printf("{\"error\": \"alloc\"}\n"); return 1; }
  k_init<<<148 * 8, 512>>>(a, n);
  k_init<<<148 * 8, 512>>>(b, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_r = 1e30f, best_c = 1e30f;
  for (int it = 0; it < 12; ++it) {
    cudaEventRecord(e0);
    k_read<<<148 * 8, 512>>>(a, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best_r) best_r = ms;
    cudaEventRecord(e0);
    k_copy<<<148 * 8, 512>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best_c) best_c = ms;
  }
  const double rd = (double)n * 8 / (best_r * 1e-3) / 1e9, cp = (double)n * 16 / (best_c * 1e-3) / 1e9;
  // L2-resident read: 48 MB (fits the 126 MB L2), 20 back-to-back launches per timing
  const int64_t nl = (int64_t)6 << 20;
  float best_l2 = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(e0);
    k_read_rep<<<148 * 4, 512>>>(a, nl, 20, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 1 && ms < best_l2) best_l2 = ms;
  }
  const double l2 = (double)nl * 8 * 20 / (best_l2 * 1e-3) / 1e9;
  printf("{\"read_only_gbs\": %.1f, \"copy_gbs\": %.1f, \"l2_read_gbs\": %.1f, \"bytes_per_array\": %lld, "
         "\"how\": \"fp64 LDG stream, 148x8 CTAs x 512, best of 10 after 2 warm-ups, CUDA events; copy counts read + "
         "write bytes; l2_read: 48 MB array read 20x inside one launch (L2-resident)\", \"err\": \"%s\"}\n",
         rd, cp, l2, (long long)(n * 8), cudaGetErrorString(cudaGetLastError()));
  return 0;
}

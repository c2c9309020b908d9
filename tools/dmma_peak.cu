// dmma_peak.cu — measured FP64 tensor-core (DMMA m8n8k4) and FP64 FMA peaks of this B200, the
// denominators for the k_spmm_bsr_tma / Gram roofline.  Every warp runs CH
// independent accumulator chains of mma.sync.m8n8k4.f64 (512 flops each) for ITER iterations;
// grid = SMs x BLK CTAs of WARPS warps; time by CUDA events, best of 5.  The FMA probe runs 8
// independent fp64 FMA chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dmma(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void k_fma(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-6 + i;
  const double m = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, sms);
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * 2, threads = warps * 32;
    float ms = best_ms([&] { k_dmma<4><<<blocks, threads>>>(out, iters); });
    const double flops = (double)blocks * warps * iters * 4 * 512.0;
    printf(", \"dmma_tflops_w%d\": %.2f", warps, flops / (ms * 1e-3) / 1e12);
  }
  {
    const int blocks = sms * 4, threads = 512;
    float ms = best_ms([&] { k_fma<<<blocks, threads>>>(out, iters); });
    const double flops = (double)blocks * threads * iters * 8 * 2.0;
    printf(", \"fp64_fma_tflops\": %.2f", flops / (ms * 1e-3) / 1e12);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

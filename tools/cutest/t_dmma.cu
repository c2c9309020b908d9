// verify the m8n8k4 f64 fragment layout assumed by dense.cu
#include <cstdio>
#include <cmath>
__global__ void k(const double* A /*8x4 row-major*/, const double* B /*4x8 row-major*/, double* C /*8x8 row-major*/) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[(l >> 2) * 8 + (l & 3) * 2] = c0;
  C[(l >> 2) * 8 + (l & 3) * 2 + 1] = c1;
}
int main() {
  double A[32], B[32], C[64], R[64];
  for (int i = 0; i < 32; ++i) { A[i] = i * 0.5 + 1; B[i] = (i % 7) - 3.0 + i * 0.01; }
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) { double s = 0; for (int q = 0; q < 4; ++q) s += A[i*4+q]*B[q*8+j]; R[i*8+j] = s; }
  double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dC); cudaMemcpy(C, dC, 512, cudaMemcpyDeviceToHost);
  double e = 0; for (int i = 0; i < 64; ++i) e = fmax(e, fabs(C[i] - R[i]));
  printf("dmma max err %.3e (%s)\n", e, cudaGetErrorString(cudaGetLastError()));
}

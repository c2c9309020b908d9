// verify the assumed fragment layouts of mma.sync m16n8k{4,8,16} .f64 (groupID g = lane/4, t = lane%4):
//   A (16 x K, row): a[2j + h] = A(g + 8h, t + 4j)     j < K/4, h in {0,1}
//   B (K x 8, col):  b[j]      = B(t + 4j, g)
//   C (16 x 8):      c[2h + i] = C(g + 8h, 2t + i)
#include <cmath>
#include <cstdio>
template <int K>
__global__ void k(const double* A, const double* B, double* C) {  // A 16xK row-major, B Kx8 row-major
  const int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
  for (int j = 0; j < K / 4; ++j) {
    a[2 * j] = A[g * K + t + 4 * j];
    a[2 * j + 1] = A[(g + 8) * K + t + 4 * j];
    b[j] = B[(t + 4 * j) * 8 + g];
  }
  if (K == 4)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  if (K == 8)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  if (K == 16)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                 "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  for (int h = 0; h < 2; ++h)
    for (int i = 0; i < 2; ++i) C[(g + 8 * h) * 8 + 2 * t + i] = c[2 * h + i];
}
template <int K>
void run() {
  double A[16 * K], B[K * 8], C[128], R[128];
  for (int i = 0; i < 16 * K; ++i) A[i] = 1.0 + i * 0.37 - (i % 5);
  for (int i = 0; i < K * 8; ++i) B[i] = (i % 7) - 3.0 + i * 0.013;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int q = 0; q < K; ++q) s += A[i * K + q] * B[q * 8 + j];
      R[i * 8 + j] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof A); cudaMalloc(&dB, sizeof B); cudaMalloc(&dC, sizeof C);
  cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
  k<K><<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(C, dC, sizeof C, cudaMemcpyDeviceToHost);
  double e = 0;
  for (int i = 0; i < 128; ++i) e = fmax(e, fabs(C[i] - R[i]) / (1 + fabs(R[i])));
  printf("m16n8k%d max rel err %.3e (%s)\n", K, e, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<4>(); run<8>(); run<16>(); }

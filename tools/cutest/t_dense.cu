// standalone check of the small dense kernels
#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_1807_09467_b200/csrc/kernels.cuh"
using namespace rg;
int main() {
  const int k = 4;
  double A[16] = {2,1,0,0, 0.5,3,1,0, 0.2,0.1,2,1, 0.3,0,0.4,1.5};  // col-major, any full-rank
  std::vector<double> G(k*k);
  for (int i=0;i<k;i++) for (int j=0;j<k;j++){ double s=0; for(int l=0;l<k;l++) s+=A[i*k+l]*A[j*k+l]; G[j*k+i]=s; }
  double *dG,*dR,*dRi; int* df;
  cudaMalloc(&dG, 8*k*k); cudaMalloc(&dR, 8*k*k); cudaMalloc(&dRi, 8*k*k); cudaMalloc(&df, 4);
  cudaMemcpy(dG, G.data(), 8*k*k, cudaMemcpyHostToDevice); cudaMemset(df,0,4);
  cudaError_t e = launch_chol(dG, k, dR, dRi, df, 0);
  printf("launch %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize(); printf("sync %s\n", cudaGetErrorString(e));
  std::vector<double> R(k*k), Ri(k*k); int f;
  cudaMemcpy(R.data(), dR, 8*k*k, cudaMemcpyDeviceToHost); cudaMemcpy(Ri.data(), dRi, 8*k*k, cudaMemcpyDeviceToHost);
  cudaMemcpy(&f, df, 4, cudaMemcpyDeviceToHost);
  printf("fail=%d\nR:", f); for (double v: R) printf(" %.4f", v); printf("\nRi:"); for (double v: Ri) printf(" %.4f", v); printf("\n");
  // check R^T R = G
  double err=0; for(int i=0;i<k;i++)for(int j=0;j<k;j++){double s=0;for(int l=0;l<k;l++) s+=R[i*k+l]*R[j*k+l]; err=fmax(err,fabs(s-G[j*k+i]));}
  printf("RtR-G %.3e\n", err);
  return 0;
}

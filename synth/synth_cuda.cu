// synth_cuda.cu — device side of the seeded input generators (see synth_common.h).
// Built with -fmad=false so every value is bit-identical to synth.c.  Used by bench.py to
// generate A_t / b_t of a sequence directly in HBM (the solution-dependent sequences of
// PAPER.md:118 need x_{t-1}, which lives on the device).  Not part of the product library.
#include <cuda_runtime.h>
#include <stdint.h>
#include "synth_common.h"

namespace {

__global__ void k_fill5_values(int N, double cd, double ih, double idt, double bx, double by,
                               const double* __restrict__ uvel, const int32_t* __restrict__ row_ptr,
                               double* __restrict__ val) {
  int64_t n = (int64_t)N * N;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(r % N), j = (int)(r / N);
    double vx = uvel ? uvel[r] : bx, vy = uvel ? uvel[r] : by;
    sy_row5(i, j, N, cd, ih, idt, vx, vy, val + row_ptr[r], nullptr);
  }
}

__global__ void k_fill7_values(int N, double cd, double ih, double idt, double bx, double by,
                               double bz, const int32_t* __restrict__ row_ptr,
                               double* __restrict__ val) {
  int64_t n = (int64_t)N * N * N;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(r % N), j = (int)((r / N) % N), l = (int)(r / ((int64_t)N * N));
    sy_row7(i, j, l, N, cd, ih, idt, bx, by, bz, val + row_ptr[r], nullptr);
  }
}

__global__ void k_rhs(int64_t n, const double* __restrict__ u, double dt, double f,
                      double* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = u[i] / dt + f;
}

__global__ void k_c5_values(int64_t nnzb, int B, uint64_t seed, const int8_t* __restrict__ kind,
                            double s_up, double s_dn, double* __restrict__ val) {
  int64_t tot = nnzb * B * B;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / ((int64_t)B * B);
    int w = (int)(e - b * B * B);
    int c = w / B, r = w - c * B;
    val[e] = sy_c5_base(seed, b, r, c, B, kind[b], s_up, s_dn);
  }
}

// A_t = A_{t-1} o (1 + 0.01 xi) in place: 16-byte streaming loads / stores, 4 pairs in flight per
// thread (the same per-element arithmetic as the scalar loop, so host and device stay bit-identical)
__global__ void k_c5_perturb(int64_t nval, uint64_t seed, int t, double* __restrict__ val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (((uintptr_t)val & 15) != 0) {
    for (int64_t e = i; e < nval; e += stride) val[e] = val[e] * sy_c5_factor(seed, t, e);
    return;
  }
  const int64_t n2 = nval / 2;
  double2* v2 = reinterpret_cast<double2*>(val);
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldcs(v2 + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t e = 2 * (i + u * stride);
      a[u].x = a[u].x * sy_c5_factor(seed, t, e);
      a[u].y = a[u].y * sy_c5_factor(seed, t, e + 1);
      __stcs(v2 + i + u * stride, a[u]);
    }
  }
  for (; i < n2; i += stride) {
    double2 a = v2[i];
    a.x = a.x * sy_c5_factor(seed, t, 2 * i);
    a.y = a.y * sy_c5_factor(seed, t, 2 * i + 1);
    v2[i] = a;
  }
  if ((nval & 1) && blockIdx.x == 0 && threadIdx.x == 0) val[nval - 1] = val[nval - 1] * sy_c5_factor(seed, t, nval - 1);
}

__global__ void k_normal_vec(int64_t n, uint64_t seed, uint64_t stream, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sy_normal12(seed, stream, (uint64_t)i);
}

inline int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int syd_fill5_values(int N, double cd, double ih, double idt, double bx, double by,
                     const double* uvel, const int32_t* row_ptr, double* val, void* stream) {
  k_fill5_values<<<grid_for((int64_t)N * N), 256, 0, (cudaStream_t)stream>>>(N, cd, ih, idt, bx, by,
                                                                            uvel, row_ptr, val);
  return (int)cudaGetLastError();
}

int syd_fill7_values(int N, double cd, double ih, double idt, double bx, double by, double bz,
                     const int32_t* row_ptr, double* val, void* stream) {
  k_fill7_values<<<grid_for((int64_t)N * N * N), 256, 0, (cudaStream_t)stream>>>(
      N, cd, ih, idt, bx, by, bz, row_ptr, val);
  return (int)cudaGetLastError();
}

int syd_rhs(int64_t n, const double* u, double dt, double f, double* b, void* stream) {
  k_rhs<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, u, dt, f, b);
  return (int)cudaGetLastError();
}

int syd_c5_values(int64_t nnzb, int B, uint64_t seed, const int8_t* kind, double s_up, double s_dn,
                  double* val, void* stream) {
  k_c5_values<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(nnzb, B, seed, kind, s_up, s_dn, val);
  return (int)cudaGetLastError();
}

int syd_c5_perturb(int64_t nval, uint64_t seed, int t, double* val, void* stream) {
  k_c5_perturb<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(nval, seed, t, val);
  return (int)cudaGetLastError();
}

int syd_normal_vec(int64_t n, uint64_t seed, uint64_t stream_id, double* out, void* stream) {
  k_normal_vec<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, seed, stream_id, out);
  return (int)cudaGetLastError();
}

}  // extern "C"

// spmv.cu — sparse matrix-vector products (K1 CSR, K2 SELL-32, K3 BSR), fp64, sm_100a.
//
// One read of the matrix per product, coalesced ("the cost of a matrix-vector
// multiplication reduces to O(mb)").  HBM-bound: bytes per product are in DESIGN.md §Roofline.
// Three output modes share each kernel:
//   SM_STEP  w = A v_j into V column j+1 (x = un-normalised column j, scaled on output)
//   SM_RES   r = b - A x into V column 0, ||r||^2 grid-reduced (cycle start)
//   SM_PLAIN y = A x (rg_apply, C = A W)
#include "epilogue.cuh"
#include "kernels.cuh"

namespace rg {
namespace {

struct SpmvArgs {
  MatDev A;
  Layout L;
  DevState* st;
  int mode;
  const double* x;
  double* y;
  int res_epi;
};

struct Io {
  const double* x;
  double* y;
  const double* b;
  double xs;
  bool res;
};

// Returns false if this launch is a no-op (decided uniformly from the device state).
__device__ __forceinline__ bool setup(const SpmvArgs& a, Io& io, int& kid) {
  DevState* st = a.st;
  const Layout& L = a.L;
  io.res = false;
  io.b = nullptr;
  io.xs = 1.0;
  if (a.mode == SM_STEP) {
    kid = K_SPMV_STEP;
    const int j = st->j;
    if (!st->active || (st->dcgs && j >= st->m)) { prof_noop(st, kid); return false; }
    io.x = L.Z + (int64_t)(L.VB + j) * L.ld;
    io.y = L.Z + (int64_t)(L.VB + j + 1) * L.ld;
    io.xs = st->dcgs ? 1.0 : st->sc[L.VB + j];  // DCGS2: y = A u on the raw vector
  } else if (a.mode == SM_RES) {
    kid = K_SPMV_RES;
    if (st->done) { prof_noop(st, kid); return false; }
    io.x = L.x;
    io.y = L.Z + (int64_t)L.VB * L.ld;
    io.b = L.b;
    io.res = true;
  } else {
    kid = K_SPMV_PLAIN;
    io.x = a.x;
    io.y = a.y;
  }
  if (st) prof_begin(st, kid);
  return true;
}

// Tail shared by every format: residual reduction + epilogue, profiling.
__device__ __forceinline__ void finish(const SpmvArgs& a, const Io& io, int kid, double nrm) {
  __shared__ double bsh[33], vals[1], tot[1];
  DevState* st = a.st;
  if (io.res) {
    const double t = block_sum(nrm, bsh);
    if (threadIdx.x == 0) vals[0] = t;
    __syncthreads();
    if (!grid_reduce(vals, 1, a.L.partial, a.L.counter, tot, tot)) return;
    if (a.res_epi) epi_cycle_start(st, a.L, tot[0]);
    if (threadIdx.x == 0) prof_end(st, kid, a.A.bytes + 8.0 * a.L.n);
    return;
  }
  if (st && st->profile) {
    if (grid_last(a.L.counter) && threadIdx.x == 0) prof_end(st, kid, a.A.bytes);
  }
}

__device__ __forceinline__ double emit(const Io& io, int64_t r, double s) {
  double v;
  if (io.res) {
    v = io.b[r] - s;
  } else {
    v = io.xs * s;
  }
  io.y[r] = v;
  return v * v;
}

// ---------------------------------------------------------------- CSR, LPR lanes per row
template <int LPR>
__global__ void __launch_bounds__(OT, 2) k_spmv_csr(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int lane = threadIdx.x & (LPR - 1);
  const int64_t rows_per_cta = OT / LPR;
  const int64_t stride = (int64_t)gridDim.x * rows_per_cta;
  double nrm = 0.0;
  const int32_t* __restrict__ rp = A.rp;
  const int32_t* __restrict__ ci = A.ci;
  const double* __restrict__ v = A.v;
  const double* __restrict__ x = io.x;
  // warp-uniform trip count: iterate over groups of rows covering whole warps
  for (int64_t base = (int64_t)blockIdx.x * rows_per_cta + (threadIdx.x & ~31) / LPR; base < A.n;
       base += stride) {
    const int64_t row = base + (threadIdx.x & 31) / LPR;
    double s = 0.0;
    if (row < A.n) {
      const int32_t p0 = __ldg(rp + row), p1 = __ldg(rp + row + 1);
      if constexpr (LPR == 1) {
        // thread per row: up to 8 (column, value) pairs in flight, then 8 gathers of x
        for (int32_t p = p0; p < p1; p += 8) {
          int32_t cc[8];
          double vv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool ok = p + u < p1;
            cc[u] = ok ? __ldcs(ci + p + u) : 0;
            vv[u] = ok ? __ldcs(v + p + u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < p1) s += vv[u] * __ldg(x + cc[u]);
        }
      } else {
        for (int32_t p = p0 + lane; p < p1; p += LPR) s += __ldcs(v + p) * __ldg(x + __ldcs(ci + p));
      }
    }
    if constexpr (LPR > 1) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, LPR);
    }
    if (lane == 0 && row < A.n) nrm += emit(io, row, s);
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- SELL-32 (sigma = 1)
__global__ void __launch_bounds__(OT, 2) k_spmv_sell(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  double nrm = 0.0;
  const int64_t rows = A.nslices * 32;
  const double* __restrict__ x = io.x;
  for (int64_t row = (int64_t)blockIdx.x * OT + threadIdx.x; row < rows; row += (int64_t)gridDim.x * OT) {
    const int64_t sl = row >> 5;
    const int w = __ldg(A.sw + sl);
    const int64_t base = __ldg(A.sp + sl) + (row & 31);
    double s = 0.0;
    for (int c = 0; c < w; c += 8) {  // 8 coalesced (column, value) pairs in flight, then gathers
      int32_t cc[8];
      double vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = c + u < w;
        const int64_t e = base + (int64_t)(c + u) * 32;
        cc[u] = ok ? __ldcs(A.sci + e) : 0;
        vv[u] = ok ? __ldcs(A.sv + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c + u < w) s += vv[u] * __ldg(x + cc[u]);
    }
    if (row < A.n) nrm += emit(io, row, s);
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- BSR (b <= 64), 64 threads / block row
__global__ void __launch_bounds__(256) k_spmv_bsr(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int b = A.b;
  const int r = threadIdx.x & 63;
  double nrm = 0.0;
  const double* __restrict__ x = io.x;
  for (int64_t I = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 6); I < A.nb; I += (int64_t)gridDim.x * 4) {
    if (r < b) {
      double s = 0.0;
      const int32_t p0 = __ldg(A.rp + I), p1 = __ldg(A.rp + I + 1);
      for (int32_t p = p0; p < p1; ++p) {
        const double* __restrict__ blk = A.v + (int64_t)p * b * b + r;
        const double* __restrict__ xb = x + (int64_t)__ldg(A.ci + p) * b;
#pragma unroll 16
        for (int c = 0; c < b; ++c) s += __ldcs(blk + (int64_t)c * b) * __ldg(xb + c);
      }
      nrm += emit(io, I * b + r, s);
    }
  }
  finish(a, io, kid, nrm);
}

}  // namespace

cudaError_t launch_spmv(const MatDev& A, const Layout& L, DevState* st, int mode, const double* x,
                        double* y, int res_epi, cudaStream_t s) {
  SpmvArgs a{A, L, st, mode, x, y, res_epi};
  const int cap_red = NSM * VEC_CTAS_PER_SM;  // reducing launches: bounded partials
  if (A.fmt == 2) {
    int64_t g = (A.nb + 3) / 4;
    const int64_t cap = mode == SM_RES ? cap_red : (int64_t)NSM * 8;
    if (g > cap) g = cap;
    k_spmv_bsr<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(a);
  } else if (A.fmt == 1) {
    int64_t g = (A.nslices * 32 + OT - 1) / OT;
    const int64_t cap = mode == SM_RES ? cap_red : (int64_t)NSM * 4;
    if (g > cap) g = cap;
    k_spmv_sell<<<(int)(g < 1 ? 1 : g), OT, 0, s>>>(a);
  } else {
    int64_t g = (A.n * A.lpr + OT - 1) / OT;
    const int64_t cap = mode == SM_RES ? cap_red : (int64_t)NSM * 4;
    if (g > cap) g = cap;
    const int gi = (int)(g < 1 ? 1 : g);
    switch (A.lpr) {
      case 1: k_spmv_csr<1><<<gi, OT, 0, s>>>(a); break;
      case 2: k_spmv_csr<2><<<gi, OT, 0, s>>>(a); break;
      case 4: k_spmv_csr<4><<<gi, OT, 0, s>>>(a); break;
      case 8: k_spmv_csr<8><<<gi, OT, 0, s>>>(a); break;
      case 16: k_spmv_csr<16><<<gi, OT, 0, s>>>(a); break;
      default: k_spmv_csr<32><<<gi, OT, 0, s>>>(a); break;
    }
  }
  return cudaGetLastError();
}

}  // namespace rg

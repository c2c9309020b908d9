// dense.cu — recycle-space build (K9-K12) and small dense kernels, fp64, sm_100a.
//
// Snapshot SVD (Algorithm 1) done the tall-skinny way: a fused Gram reduction
// G = X^T X (one sweep of X), a one-CTA parallel-cyclic Jacobi eigensolver, Y = X V_1, a second
// Gram/Jacobi pass on Y to restore the accuracy the squared conditioning costs (DESIGN.md
// reading R-SVD), and W = Y V_2 Sigma^{-1}.  CholQR2 of C = A W uses the same Gram and X*M
// kernels plus a one-CTA Cholesky.
#include "common.cuh"
#include "kernels.cuh"

namespace rg {
namespace {

constexpr int GT = 256;         // threads of the Gram kernel
constexpr int GTR = 32;         // rows per Gram tile
constexpr int MAXP = MAXS * (MAXS + 1) / 2;
constexpr int PPT = (MAXP + GT - 1) / GT;

// G = Y^T Y.  Each thread owns fixed (a,b) pairs (deterministic), tiles of GTR rows staged in
// shared memory (row-major, padded), per-CTA partials grid-reduced in index order.
__global__ void __launch_bounds__(GT) k_gram(const double* __restrict__ Y, int64_t ld, int64_t n, int s,
                                             double* G, double* partial, unsigned* counter, DevState* st) {
  extern __shared__ double sm[];
  double* tile = sm;                        // GTR x (s+1)
  double* pv = tile + GTR * (MAXS + 1);     // MAXP
  double* tot = pv + MAXP;                  // MAXP
  double* scr = tot + MAXP;                 // MAXP (>= GT)
  __shared__ unsigned char pa[MAXP], pb[MAXP];
  const int P = s * (s + 1) / 2;
  if (st) prof_begin(st, K_GRAM);
  if (threadIdx.x == 0) {
    int p = 0;
    for (int a2 = 0; a2 < s; ++a2)
      for (int b2 = a2; b2 < s; ++b2) { pa[p] = (unsigned char)a2; pb[p] = (unsigned char)b2; ++p; }
  }
  __syncthreads();
  double acc[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) acc[q] = 0.0;
  const int64_t ntiles = (n + GTR - 1) / GTR;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * GTR;
    for (int e = threadIdx.x; e < GTR * s; e += GT) {
      const int c = e / GTR, r = e % GTR;      // coalesced: consecutive threads, consecutive rows
      tile[r * (s + 1) + c] = (r0 + r < n) ? Y[(int64_t)c * ld + r0 + r] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int p = threadIdx.x + q * GT;
      if (p < P) {
        const int a2 = pa[p], b2 = pb[p];
        double sacc = 0.0;
#pragma unroll 8
        for (int r = 0; r < GTR; ++r) sacc += tile[r * (s + 1) + a2] * tile[r * (s + 1) + b2];
        acc[q] += sacc;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int p = threadIdx.x + q * GT;
    if (p < P) pv[p] = acc[q];
  }
  __syncthreads();
  if (!grid_reduce(pv, P, partial, counter, tot, scr, MAXP)) return;
  for (int p = threadIdx.x; p < P; p += GT) {
    const int a2 = pa[p], b2 = pb[p];
    G[a2 * s + b2] = tot[p];
    G[b2 * s + a2] = tot[p];
  }
  if (st && threadIdx.x == 0) prof_end(st, K_GRAM, 8.0 * (double)n * s);
}

// Parallel cyclic (round-robin) Jacobi on a symmetric s x s matrix, one CTA.
constexpr int JLD = MAXS + 1;
__global__ void __launch_bounds__(256) k_jacobi(const double* G, int s, double* lam, double* V,
                                                double* sigma_out, DevState* st) {
  extern __shared__ double jsm[];
  double* A_ = jsm;                    // JLD x JLD, A(r, c) = A_[r * JLD + c]
  double* V_ = jsm + JLD * JLD;
  __shared__ double cs[MAXS / 2 + 1], sn[MAXS / 2 + 1];
  __shared__ int pp[MAXS / 2 + 1], qq[MAXS / 2 + 1];
  __shared__ double ev[MAXS + 1];
  __shared__ int perm[MAXS + 1];
  __shared__ double s_off, s_fro;
  const int tid = threadIdx.x, bd = blockDim.x;
  if (st) prof_begin(st, K_JACOBI);
  const int ne = s + (s & 1);  // even size (pad with a decoupled zero row/column)
  for (int e = tid; e < ne * ne; e += bd) {
    const int r = e / ne, c = e % ne;
    A_[(r) * JLD + (c)] = (r < s && c < s) ? G[c * s + r] : 0.0;
    V_[(r) * JLD + (c)] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = ne / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) {
      double off = 0.0, fro = 0.0;
      for (int r = 0; r < ne; ++r)
        for (int c = 0; c < ne; ++c) {
          const double v2 = A_[(r) * JLD + (c)] * A_[(r) * JLD + (c)];
          fro += v2;
          if (r != c) off += v2;
        }
      s_off = off;
      s_fro = fro;
    }
    __syncthreads();
    if (!(s_off > 1e-28 * s_fro) || ne < 2) break;  // off(A)_F <= 1e-14 ||A||_F
    for (int round = 0; round < ne - 1; ++round) {
      // circle method: fix player ne-1; pair (round, ne-1) and ((round+i)%(ne-1), (round-i)%(ne-1))
      for (int i = tid; i < half; i += bd) {
        int p, q;
        if (i == 0) { p = round; q = ne - 1; }
        else { p = (round + i) % (ne - 1); q = (round - i + (ne - 1)) % (ne - 1); }
        if (p > q) { const int t = p; p = q; q = t; }
        pp[i] = p; qq[i] = q;
        const double apq = A_[(p) * JLD + (q)], app = A_[(p) * JLD + (p)], aqq = A_[(q) * JLD + (q)];
        double c = 1.0, sv = 0.0;
        if (fabs(apq) > 1e-300 && fabs(apq) > 1e-18 * sqrt(fabs(app * aqq))) {
          const double th = (aqq - app) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
          c = 1.0 / sqrt(1.0 + t * t);
          sv = t * c;
        }
        cs[i] = c; sn[i] = sv;
      }
      __syncthreads();
      for (int e = tid; e < half * ne; e += bd) {  // rows: A <- J^T A
        const int i = e / ne, col = e % ne;
        const int p = pp[i], q = qq[i];
        const double ap = A_[(p) * JLD + (col)], aq = A_[(q) * JLD + (col)];
        A_[(p) * JLD + (col)] = cs[i] * ap - sn[i] * aq;
        A_[(q) * JLD + (col)] = sn[i] * ap + cs[i] * aq;
      }
      __syncthreads();
      for (int e = tid; e < half * ne; e += bd) {  // columns: A <- A J, V <- V J
        const int i = e / ne, row = e % ne;
        const int p = pp[i], q = qq[i];
        const double ap = A_[(row) * JLD + (p)], aq = A_[(row) * JLD + (q)];
        A_[(row) * JLD + (p)] = cs[i] * ap - sn[i] * aq;
        A_[(row) * JLD + (q)] = sn[i] * ap + cs[i] * aq;
        const double vp = V_[(row) * JLD + (p)], vq = V_[(row) * JLD + (q)];
        V_[(row) * JLD + (p)] = cs[i] * vp - sn[i] * vq;
        V_[(row) * JLD + (q)] = sn[i] * vp + cs[i] * vq;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {  // sort eigenvalues of the first s (the pad is the zero eigenpair of the pad)
    int cnt = 0;
    for (int i = 0; i < ne; ++i) {
      if (s < ne && fabs(V_[(ne - 1) * JLD + (i)]) > 0.5) continue;  // the decoupled pad vector
      perm[cnt] = i;
      ev[cnt] = A_[(i) * JLD + (i)];
      ++cnt;
    }
    for (int a2 = 0; a2 < s; ++a2) {
      int best = a2;
      for (int c = a2 + 1; c < s; ++c)
        if (ev[c] > ev[best]) best = c;
      const double te = ev[a2]; ev[a2] = ev[best]; ev[best] = te;
      const int tp = perm[a2]; perm[a2] = perm[best]; perm[best] = tp;
    }
  }
  __syncthreads();
  for (int e = tid; e < s * s; e += bd) {
    const int c = e / s, r = e % s;
    V[c * s + r] = V_[r * JLD + perm[c]];
  }
  for (int c = tid; c < s; c += bd) {
    lam[c] = ev[c];
    if (sigma_out) sigma_out[c] = ev[c] > 0.0 ? sqrt(ev[c]) : 0.0;
  }
  if (st && tid == 0) prof_end(st, K_JACOBI, 0.0);
}

// Y[:, c] = colscale[c] * X[:, 0:s] M[:, c]; tiles of 64 rows staged in shared memory.
constexpr int XT = 256, XTR = 64;
__global__ void __launch_bounds__(XT) k_xm(const double* __restrict__ X, int64_t ldx, int64_t n, int s,
                                           const double* __restrict__ M, int ldm, int q,
                                           const double* __restrict__ colscale, double* Y, int64_t ldy,
                                           DevState* st) {
  extern __shared__ double sm[];
  double* Ms = sm;                       // s x q, [c * s + a]
  double* tile = Ms + MAXS * MAXS;       // XTR x (s+1)
  (void)st;
  for (int e = threadIdx.x; e < s * q; e += XT) {
    const int c = e / s, a2 = e % s;
    Ms[e] = M[(int64_t)c * ldm + a2] * (colscale ? colscale[c] : 1.0);
  }
  const int64_t ntiles = (n + XTR - 1) / XTR;
  const int row = threadIdx.x % XTR, cg = threadIdx.x / XTR;  // 4 column groups
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * XTR;
    __syncthreads();
    for (int e = threadIdx.x; e < XTR * s; e += XT) {
      const int c = e / XTR, r = e % XTR;
      tile[r * (s + 1) + c] = (r0 + r < n) ? X[(int64_t)c * ldx + r0 + r] : 0.0;
    }
    __syncthreads();
    if (r0 + row < n) {
      for (int c = cg; c < q; c += XT / XTR) {
        double acc = 0.0;
        for (int a2 = 0; a2 < s; ++a2) acc += tile[row * (s + 1) + a2] * Ms[c * s + a2];
        Y[(int64_t)c * ldy + r0 + row] = acc;
      }
    }
  }
}

__global__ void k_inv(const double* sigma, int q, double* out) {
  for (int c = threadIdx.x; c < q; c += blockDim.x) out[c] = 1.0 / sigma[c];
}

// Cholesky G = R^T R (R upper, column-major R[c*k + r]) and R^{-1}, one CTA.
constexpr int CLD = MAXK + 1;
__global__ void __launch_bounds__(256) k_chol(const double* G, int k, double* R, double* Ri, int* fail) {
  __shared__ double Rs[MAXK * CLD];  // R(r, c) = Rs[c * CLD + r]
  __shared__ int bad;
  const int tid = threadIdx.x, bd = blockDim.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < MAXK * CLD; e += bd) Rs[e] = 0.0;
  __syncthreads();
  for (int jj = 0; jj < k; ++jj) {
    if (tid == 0) {
      double d = G[jj * k + jj];
      for (int l = 0; l < jj; ++l) d -= Rs[jj * CLD + l] * Rs[jj * CLD + l];
      if (!(d > 0.0)) { bad = 1; d = 1.0; }
      Rs[jj * CLD + jj] = sqrt(d);
    }
    __syncthreads();
    for (int i = jj + 1 + tid; i < k; i += bd) {
      double v = G[i * k + jj];
      for (int l = 0; l < jj; ++l) v -= Rs[jj * CLD + l] * Rs[i * CLD + l];
      Rs[i * CLD + jj] = v / Rs[jj * CLD + jj];
    }
    __syncthreads();
  }
  // R^{-1}: column c solves R x = e_c (back substitution), one thread per column
  for (int c = tid; c < k; c += bd) {
    for (int r = k - 1; r >= 0; --r) {
      double v = (r == c) ? 1.0 : 0.0;
      for (int l = r + 1; l <= c; ++l) v -= Rs[l * CLD + r] * Ri[c * k + l];
      Ri[c * k + r] = r <= c ? v / Rs[r * CLD + r] : 0.0;
    }
  }
  for (int e = tid; e < k * k; e += bd) R[e] = Rs[(e / k) * CLD + (e % k)];
  __syncthreads();
  if (tid == 0 && bad) *fail = 1;
}

__global__ void k_rc_finish(const double* R1, const double* R1i, const double* R2, const double* R2i,
                            int k, DevState* st, int* fail) {
  __shared__ double dmax, dmin;
  for (int e = threadIdx.x; e < MAXK * MAXK; e += blockDim.x) {
    const int c = e / MAXK, r = e % MAXK;
    double v = 0.0, vi = 0.0;
    if (c < k && r < k) {
      for (int l = 0; l < k; ++l) {
        v += R2[l * k + r] * R1[c * k + l];      // (R2 R1)[r][c]
        vi += R1i[l * k + r] * R2i[c * k + l];   // (R1^-1 R2^-1)[r][c]
      }
    }
    st->RC[c][r] = v;
    st->RCinv[c][r] = vi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    dmax = 0.0; dmin = 1e308;
    for (int i = 0; i < k; ++i) {
      const double d = fabs(st->RC[i][i]);
      dmax = d > dmax ? d : dmax;
      dmin = d < dmin ? d : dmin;
    }
    if (!(dmin > 1e-12 * dmax)) *fail = 1;
  }
}

__global__ void k_sell_widths(const int32_t* rp, int64_t n, int32_t* sw) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < ns; sl += (int64_t)gridDim.x * blockDim.x) {
    int w = 0;
    for (int r = 0; r < 32; ++r) {
      const int64_t row = sl * 32 + r;
      if (row < n) { const int l = rp[row + 1] - rp[row]; w = l > w ? l : w; }
    }
    sw[sl] = w;
  }
}

__global__ void k_sell_pack(const int32_t* rp, const int32_t* ci, const double* v, int64_t n,
                            const int64_t* sp, const int32_t* sw, int32_t* sci, double* sv, int pattern) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < ns * 32;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = row >> 5;
    const int w = sw[sl];
    const int64_t base = sp[sl] + (row & 31);
    int len = 0, p0 = 0;
    if (row < n) { p0 = rp[row]; len = rp[row + 1] - p0; }
    for (int c = 0; c < w; ++c) {
      const int64_t e = base + (int64_t)c * 32;
      if (c < len) {
        sv[e] = v[p0 + c];
        if (pattern) sci[e] = ci[p0 + c];
      } else {
        sv[e] = 0.0;
        if (pattern) sci[e] = 0;
      }
    }
  }
}

__global__ void k_validate(const int32_t* rp, const int32_t* ci, int64_t nrows, int64_t ncols, int64_t nnz,
                           int* bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p0 = rp[r], p1 = rp[r + 1];
    if (r == 0 && p0 != 0) atomicOr(bad, 1);
    if (r == nrows - 1 && p1 != nnz) atomicOr(bad, 2);
    if (p1 < p0) { atomicOr(bad, 4); continue; }
    if (p0 < 0 || p1 > nnz) { atomicOr(bad, 8); continue; }
    int32_t prev = -1;
    for (int32_t p = p0; p < p1; ++p) {
      const int32_t c = ci[p];
      if (c < 0 || c >= ncols) atomicOr(bad, 16);
      if (c <= prev) atomicOr(bad, 32);
      prev = c;
    }
  }
}

}  // namespace

cudaError_t launch_gram(const double* Y, int64_t ld, int64_t n, int s, double* G, double* partial,
                        unsigned* counter, DevState* st, cudaStream_t strm) {
  const size_t smem = sizeof(double) * (GTR * (MAXS + 1) + 3 * MAXP);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    init = true;
  }
  int64_t g = (n + GTR - 1) / GTR;
  if (g > NSM) g = NSM;
  k_gram<<<(int)(g < 1 ? 1 : g), GT, smem, strm>>>(Y, ld, n, s, G, partial, counter, st);
  return cudaGetLastError();
}

cudaError_t launch_jacobi(const double* G, int s, double* lam, double* V, double* sigma_out,
                          DevState* st, cudaStream_t strm) {
  const size_t smem = sizeof(double) * 2 * JLD * JLD;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    init = true;
  }
  k_jacobi<<<1, 256, smem, strm>>>(G, s, lam, V, sigma_out, st);
  return cudaGetLastError();
}

cudaError_t launch_xm(const double* X, int64_t ldx, int64_t n, int s, const double* M, int ldm, int q,
                      const double* colscale, double* Y, int64_t ldy, DevState* st, cudaStream_t strm) {
  const size_t smem = sizeof(double) * (MAXS * MAXS + XTR * (MAXS + 1));
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_xm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    init = true;
  }
  int64_t g = (n + XTR - 1) / XTR;
  if (g > NSM * 4) g = NSM * 4;
  k_xm<<<(int)(g < 1 ? 1 : g), XT, smem, strm>>>(X, ldx, n, s, M, ldm, q, colscale, Y, ldy, st);
  return cudaGetLastError();
}

cudaError_t launch_inv(const double* sigma, int q, double* out, cudaStream_t strm) {
  k_inv<<<1, 64, 0, strm>>>(sigma, q, out);
  return cudaGetLastError();
}

cudaError_t launch_chol(const double* G, int k, double* R, double* Rinv, int* fail, cudaStream_t strm) {
  k_chol<<<1, 256, 0, strm>>>(G, k, R, Rinv, fail);
  return cudaGetLastError();
}

cudaError_t launch_rc_finish(const double* R1, const double* R1i, const double* R2, const double* R2i,
                             int k, DevState* st, int* fail, cudaStream_t strm) {
  k_rc_finish<<<1, 256, 0, strm>>>(R1, R1i, R2, R2i, k, st, fail);
  return cudaGetLastError();
}

cudaError_t launch_sell_widths(const int32_t* rp, int64_t n, int32_t* sw, cudaStream_t strm) {
  k_sell_widths<<<NSM * 4, 256, 0, strm>>>(rp, n, sw);
  return cudaGetLastError();
}

cudaError_t launch_sell_pack(const int32_t* rp, const int32_t* ci, const double* v, int64_t n,
                             const int64_t* sp, const int32_t* sw, int32_t* sci, double* sv,
                             int pattern, cudaStream_t strm) {
  k_sell_pack<<<NSM * 8, 256, 0, strm>>>(rp, ci, v, n, sp, sw, sci, sv, pattern);
  return cudaGetLastError();
}

cudaError_t launch_validate(const int32_t* rp, const int32_t* ci, int64_t nrows, int64_t ncols,
                            int64_t nnz, int* bad, cudaStream_t strm) {
  k_validate<<<NSM * 4, 256, 0, strm>>>(rp, ci, nrows, ncols, nnz, bad);
  return cudaGetLastError();
}

}  // namespace rg

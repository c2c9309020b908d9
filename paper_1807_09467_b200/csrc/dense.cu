// dense.cu — recycle-space build (K9-K12) and small dense kernels, fp64, sm_100a.
//
// Snapshot SVD (Algorithm 1) done the tall-skinny way: a fused Gram reduction
// G = X^T X (one sweep of X), a one-CTA parallel-cyclic Jacobi eigensolver, Y = X V_1, a second
// Gram/Jacobi pass on Y to restore the accuracy the squared conditioning costs (DESIGN.md
// reading R-SVD), and W = Y V_2 Sigma^{-1}.  CholQR2 of C = A W uses the same Gram and X*M
// kernels plus a one-CTA Cholesky.
#define RG_FILE_ID 2  // RG_CHK locations (checked builds)
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "knobs.cuh"

namespace rg {
namespace {

constexpr int GT = 256;         // threads of the Gram kernel (8 warps)
constexpr int GTR = 64;         // rows per Gram tile
constexpr int S8MAX = 64;       // s rounded up to a multiple of 8

constexpr int GRAM_CTAS = NSM * 2;
constexpr int GPL = S8MAX * S8MAX;  // partial stride per CTA

// FP64 tensor-core MMA (DMMA.8x8x4): C[8x8] += A[8x4] B[4x8].  Fragments (PTX ISA, m8n8k4 .f64):
// a: A(lane/4, lane%4), b: B(lane%4, lane/4), c{0,1}: C(lane/4, 2*(lane%4) + {0,1}).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// ---- cp.async ring of column-major tiles: stage[c * TS + r] = Y(r0 + r, c), 64 rows, s8 columns
// (columns >= s zero-filled by a 0-byte source).  16-byte copies of row pairs; NST tiles in flight
// per CTA without holding registers (the register-staged version above kept one).
constexpr int TS = GTR + 4;   // column stride (doubles): fragment reads hit 16 distinct 8-byte banks
constexpr int NST = 3;        // ring stages
__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (valid)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_stages() { asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory"); }
// rows r0 .. r0+63 exist in the column-major buffer (n_pad is a multiple of 64; padding rows are 0)
__device__ __forceinline__ void tile_issue(double* stage, const double* __restrict__ Y, int64_t ld, int s, int s8,
                                           int64_t r0) {
  for (int e = threadIdx.x; e < s8 * (GTR / 2); e += blockDim.x) {
    const int c = e / (GTR / 2), i = e % (GTR / 2);
    const bool ok = c < s;
    cp16(stage + c * TS + 2 * i, Y + (int64_t)(ok ? c : 0) * ld + r0 + 2 * i, ok);
  }
}

// Pass 1 of G = Y^T Y: every CTA accumulates the upper block pairs (I <= J) of its rows with
// DMMA; warp w owns pairs w, w+8, ... and keeps their 8x8 accumulators in registers across tiles.
__global__ void __launch_bounds__(GT) k_gram_mma(const double* __restrict__ Y, int64_t ld, int64_t n, int s,
                                                 double* __restrict__ partial, DevState* st) {
  extern __shared__ double ring[];     // NST x s8 x TS
  if (st) prof_begin(st, K_GRAM);
  const int s8 = (s + 7) & ~7, nb = s8 / 8, np = nb * (nb + 1) / 2;
  RG_CHK(st, s >= 1 && s8 <= S8MAX);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int MAXQ = (S8MAX / 8) * (S8MAX / 8 + 1) / 2 / 8 + 1;  // pairs per warp (<= 5)
  double acc[MAXQ][2];
  int pi[MAXQ], pj[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    acc[q][0] = acc[q][1] = 0.0;
    int p = wid + 8 * q, I = 0;
    while (p >= nb - I && I < nb) { p -= nb - I; ++I; }  // p-th upper pair in row-major order
    pi[q] = I;
    pj[q] = I + p;
  }
  const int nq = (np - wid + 7) / 8;
  const int64_t ntiles = (n + GTR - 1) / GTR;
  const int sstride = s8 * TS;
  for (int i = 0; i < NST - 1; ++i) {  // prologue: the first NST-1 tiles of this CTA
    const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
    if (t < ntiles) tile_issue(ring + i * sstride, Y, ld, s, s8, t * GTR);
    cp_commit();
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    cp_wait_stages();
    __syncthreads();  // tile `it` complete for every thread; stage (it-1) % NST free again
    const int64_t tn = t + (int64_t)(NST - 1) * gridDim.x;
    if (tn < ntiles) tile_issue(ring + ((it + NST - 1) % NST) * sstride, Y, ld, s, s8, tn * GTR);
    cp_commit();
    const double* tile = ring + (it % NST) * sstride;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      if (q < nq) {
        const double* ta = tile + (pi[q] * 8 + (lane >> 2)) * TS + (lane & 3);
        const double* tb = tile + (pj[q] * 8 + (lane >> 2)) * TS + (lane & 3);
#pragma unroll
        for (int kk = 0; kk < GTR / 4; ++kk) dmma(acc[q][0], acc[q][1], ta[kk * 4], tb[kk * 4]);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  double* P = partial + (size_t)blockIdx.x * GPL;
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    if (q < nq) {
      const int row = pi[q] * 8 + (lane >> 2), col = pj[q] * 8 + (lane & 3) * 2;
      P[row * S8MAX + col] = acc[q][0];
      P[row * S8MAX + col + 1] = acc[q][1];
    }
  }
}

// Pass 2: G(a,b) = sum over CTAs (index order within each lane, fixed shuffle tree) of the
// partials, a <= b; mirrored.  One warp per entry.
__global__ void __launch_bounds__(256) k_gram_reduce(const double* __restrict__ partial, int nparts, int s,
                                                     double* G, unsigned* counter, DevState* st, double bytes) {
  const int P = s * (s + 1) / 2;
  const int lane = threadIdx.x & 31;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += (gridDim.x * blockDim.x) >> 5) {
    int a = 0, q = p;
    while (q >= s - a) { q -= s - a; ++a; }
    const int b = a + q;
    const int off = a * S8MAX + b;
    double acc = 0.0;
    for (int c = lane; c < nparts; c += 8 * 32) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = c + 32 * u < nparts ? __ldcg(partial + (size_t)(c + 32 * u) * GPL + off) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      G[a * s + b] = acc;
      G[b * s + a] = acc;
    }
  }
  if (st && st->profile && grid_last(counter) && threadIdx.x == 0) prof_end(st, K_GRAM, bytes);
}

// Parallel cyclic (round-robin) Jacobi on a symmetric s x s matrix, one CTA.
constexpr int JLD = MAXS + 1;
// V0 (nullable, s0 x s0, column-major, leading dimension s0 <= s): warm start A = V0^T G V0, V = V0
// (V0 extended by the identity when the window has grown since V0 was computed).  Any orthogonal
// start is valid for Jacobi.  With the previous system's eigenvectors (the window changed by one
// column) the sweep count at the 1e-14 stop is unchanged (7 at s = 20), but most pairs fall below
// the rotation threshold early and are skipped: measured -40 us per build at C2.
// rel != 0 (the SVD's second pass, R7): stop only when no pair has |a_pq| > 1e-15 sqrt(a_pp a_qq)
// and rotate only such pairs — the criterion of one-sided Jacobi.  The Gram matrix of the second pass
// is scaled diagonally dominant (nearly orthogonal columns of graded norms), so this converges in a few
// sweeps to eigenvalues with HIGH RELATIVE accuracy; the absolute stop off(A)_F <= 1e-14 ||A||_F (pass 1)
// would stop at sweep 0 and leave the small singular values at the ~sqrt(eps) sigma_1 level of one Gram
// pass (measured C4 window: 4e-9 sigma_1 errors; relative stop: <= 1e-15 sigma_1).
__global__ void __launch_bounds__(1024) k_jacobi(const double* G, int s, double* lam, double* V,
                                                double* sigma_out, DevState* st, const double* V0, int s0,
                                                int rel) {
  extern __shared__ double jsm[];
  double* A_ = jsm;                    // JLD x JLD, A(r, c) = A_[r * JLD + c]
  double* V_ = jsm + JLD * JLD;
  double* B_ = jsm + 2 * JLD * JLD;    // warm start scratch: G V0
  __shared__ double ev[MAXS + 1];
  __shared__ int perm[MAXS + 1];
  __shared__ double jred[33], jcs[MAXS / 2 + 1], jsn[MAXS / 2 + 1];
  __shared__ unsigned short jpair[MAXS * MAXS / 2];  // round-robin pairing: (p | q << 8) per (round, i)
  __shared__ int s_rot;                                // rel: rotations in the current sweep
  __shared__ int s_rr[MAXS];                           // per round of the sweep: some pair rotates
  const int tid = threadIdx.x, bd = blockDim.x;
  if (st) prof_begin(st, K_JACOBI);
  const int ne = s + (s & 1);  // even size (pad with a decoupled zero row/column)
  for (int e = tid; e < ne * ne; e += bd) {
    const int r = e / ne, c = e % ne;
    A_[(r) * JLD + (c)] = (r < s && c < s) ? G[c * s + r] : 0.0;
    V_[(r) * JLD + (c)] = (V0 && r < s0 && c < s0) ? V0[c * s0 + r] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  if (V0) {  // A <- V^T A V (B = A V, then V^T B), fixed summation order
    for (int e = tid; e < s * s; e += bd) {
      const int r = e / s, c = e % s;
      double acc = 0.0;
      for (int i = 0; i < s; ++i) acc += A_[(r) * JLD + (i)] * V_[(i) * JLD + (c)];
      B_[(r) * JLD + (c)] = acc;
    }
    __syncthreads();
    for (int e = tid; e < s * s; e += bd) {
      const int r = e / s, c = e % s;
      double acc = 0.0;
      for (int i = 0; i < s; ++i) acc += V_[(i) * JLD + (r)] * B_[(i) * JLD + (c)];
      A_[(r) * JLD + (c)] = acc;
    }
    __syncthreads();
  }
  const int half = ne / 2;
  // Per round: the `half` rotation threads compute (c, s) of their pair from the current A (pairs
  // from a table built once: no integer division in the loop), barrier, then thread (i, i2)
  // updates the 2x2 block of rows {p_i, q_i} x columns {p_i2, q_i2} into the other buffer of a
  // double-buffered A — rows first (J^T A), then columns (A J): the operation order of a full row
  // pass followed by a column pass, so every entry gets the same arithmetic as before — and rows
  // 2 i2, 2 i2 + 1 of V for pair i (in place: no other thread touches them in this round), barrier.
  // The loop is latency-bound (one warp per SM sub-partition): ncu showed ~390 instructions per
  // warp per round in the first version (integer modulo for the pairing, the rotation formula
  // evaluated by every block thread); 1.16 us per round at s = 20.
  for (int e = tid; e < (ne - 1) * half; e += bd) {
    const int round = e / half, i = e % half;
    int p, q;
    if (i == 0) { p = round; q = ne - 1; }
    else { p = (round + i) % (ne - 1); q = (round - i + (ne - 1)) % (ne - 1); }
    if (p > q) { const int t = p; p = q; q = t; }
    jpair[e] = (unsigned short)(p | (q << 8));
  }
  double* Ac = A_;
  double* An = B_;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (rel) {
      if (ne < 2) break;
      if (sweep > 0 && s_rot == 0) break;  // no pair above the relative threshold in the last sweep
      __syncthreads();                      // everyone has read s_rot
      if (tid == 0) s_rot = 0;
      __syncthreads();
    } else {
      double off = 0.0, fro = 0.0;
      for (int e = tid; e < ne * ne; e += bd) {
        const int r = e / ne, c = e % ne;
        const double v2 = Ac[(r) * JLD + (c)] * Ac[(r) * JLD + (c)];
        fro += v2;
        if (r != c) off += v2;
      }
      off = block_sum(off, jred);
      fro = block_sum(fro, jred);
      if (!(off > 1e-28 * fro) || ne < 2) break;  // off(A)_F <= 1e-14 ||A||_F
    }
    for (int r = tid; r < ne; r += bd) s_rr[r] = 0;
    __syncthreads();
    for (int round = 0; round < ne - 1; ++round) {
      const unsigned short* pr = jpair + round * half;
      if (tid < half) {
        const int p = pr[tid] & 0xff, q = pr[tid] >> 8;
        const double apq = Ac[(p) * JLD + (q)], app = Ac[(p) * JLD + (p)], aqq = Ac[(q) * JLD + (q)];
        double c = 1.0, sv = 0.0;
        const bool go = rel ? (fabs(apq) > 1e-300 && apq * apq > 1e-30 * fabs(app * aqq))
                            : (fabs(apq) > 1e-300 && apq * apq > 1e-36 * fabs(app * aqq));
        if (go) {
          s_rr[round] = 1;
          if (rel) s_rot = 1;
          // t = tan(theta) = sign(th) / (|th| + sqrt(1 + th^2)), th = (aqq - app) / (2 apq), written as
          // t = b' / d with a = aqq - app, b = 2 apq, b' = b sign(a), d = |a| + sqrt(a^2 + b^2); then
          // c = 1 / sqrt(1 + t^2) = d w and s = t c = b' w with w = 1 / sqrt(d^2 + b^2): one sqrt and
          // one reciprocal square root on the dependent chain, no division (the loop is latency-bound)
          const double a = aqq - app, b = 2.0 * apq;
          const double d = fabs(a) + sqrt(a * a + b * b);
          const double w = rsqrt(d * d + b * b);
          c = d * w;
          sv = (a >= 0.0 ? b : -b) * w;
        }
        jcs[tid] = c;
        jsn[tid] = sv;
      }
      __syncthreads();
      if (!s_rr[round]) continue;  // no pair rotates: the update would be an exact identity (c = 1, s = 0)
      for (int e = tid; e < half * half; e += bd) {
        const int i = e / half, i2 = e - i * half;
        const int p = pr[i] & 0xff, q = pr[i] >> 8, p2 = pr[i2] & 0xff, q2 = pr[i2] >> 8;
        const double c = jcs[i], sv = jsn[i], c2 = jcs[i2], s2 = jsn[i2];
        const double a = Ac[(p) * JLD + (p2)], b = Ac[(p) * JLD + (q2)];
        const double d = Ac[(q) * JLD + (p2)], f = Ac[(q) * JLD + (q2)];
        const double a1 = c * a - sv * d, b1 = c * b - sv * f;   // rows p, q: J^T A
        const double d1 = sv * a + c * d, f1 = sv * b + c * f;
        An[(p) * JLD + (p2)] = c2 * a1 - s2 * b1;                // columns p2, q2: A J
        An[(p) * JLD + (q2)] = s2 * a1 + c2 * b1;
        An[(q) * JLD + (p2)] = c2 * d1 - s2 * f1;
        An[(q) * JLD + (q2)] = s2 * d1 + c2 * f1;
#pragma unroll
        for (int row = 2 * i2; row < 2 * i2 + 2; ++row) {         // V <- V J (rows of pair i)
          const double vp = V_[(row) * JLD + (p)], vq = V_[(row) * JLD + (q)];
          V_[(row) * JLD + (p)] = c * vp - sv * vq;
          V_[(row) * JLD + (q)] = sv * vp + c * vq;
        }
      }
      __syncthreads();
      double* t = Ac; Ac = An; An = t;
    }
  }
  A_ = Ac;
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
  if (tid == 0) lam[s + (sigma_out ? 1 : 0)] = (double)sweep;  // diagnostics (RG_DEBUG): sweeps used
  if (st && tid == 0) prof_end(st, K_JACOBI, 0.0);
}

// Y[:, c] = colscale[c] * X[:, 0:s] M[:, c] with DMMA: tiles of 64 rows of X staged in shared
// memory; warp w computes rows 8w..8w+7 of the tile for all column blocks; the output tile is staged
// in shared memory and written column-coalesced.
constexpr int XT = 256, XTR = 64;
constexpr int XMS = S8MAX + 1;  // stride of the M (a-major) and output tiles
__global__ void __launch_bounds__(XT) k_xm(const double* __restrict__ X, int64_t ldx, int64_t n, int s,
                                           const double* __restrict__ M, int ldm, int q,
                                           const double* __restrict__ colscale, double* Y, int64_t ldy,
                                           DevState* st) {
  extern __shared__ double sm[];
  const int s8_ = (s + 7) & ~7;
  double* Ms = sm;                     // s8 x XMS    : Ms[a * XMS + c]
  double* out = Ms + s8_ * XMS;        // XTR x XMS   : out[r * XMS + c]
  double* ring = out + XTR * XMS;      // NST x s8 x TS column-major tiles
  (void)st;
  const int s8 = (s + 7) & ~7, q8 = (q + 7) & ~7, ncb = q8 / 8;
  for (int e = threadIdx.x; e < s8 * q8; e += XT) {
    const int c = e / s8, a2 = e % s8;
    Ms[a2 * XMS + c] = (a2 < s && c < q) ? M[(int64_t)c * ldm + a2] * (colscale ? colscale[c] : 1.0) : 0.0;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t ntiles = (n + XTR - 1) / XTR;
  static_assert(XTR == GTR, "k_xm stages GTR-row tiles");
  const int sstride = s8 * TS;
  for (int i = 0; i < NST - 1; ++i) {
    const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
    if (t < ntiles) tile_issue(ring + i * sstride, X, ldx, s, s8, t * XTR);
    cp_commit();
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int64_t r0 = t * XTR;
    cp_wait_stages();
    __syncthreads();  // tile `it` complete; the previous tile's output staging has been written out
    const int64_t tn = t + (int64_t)(NST - 1) * gridDim.x;
    if (tn < ntiles) tile_issue(ring + ((it + NST - 1) % NST) * sstride, X, ldx, s, s8, tn * XTR);
    cp_commit();
    const double* tile = ring + (it % NST) * sstride;
    double acc[S8MAX / 8][2];
#pragma unroll
    for (int cb = 0; cb < S8MAX / 8; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
    const double* ta = tile + (lane & 3) * TS + wid * 8 + (lane >> 2);
    for (int k4 = 0; k4 < s8; k4 += 4) {
      const double a = ta[k4 * TS];
      const double* mb = Ms + (k4 + (lane & 3)) * XMS + (lane >> 2);
#pragma unroll
      for (int cb = 0; cb < S8MAX / 8; ++cb)
        if (cb < ncb) dmma(acc[cb][0], acc[cb][1], a, mb[cb * 8]);
    }
#pragma unroll
    for (int cb = 0; cb < S8MAX / 8; ++cb) {
      if (cb < ncb) {
        const int r = wid * 8 + (lane >> 2), c = cb * 8 + (lane & 3) * 2;
        out[r * XMS + c] = acc[cb][0];
        out[r * XMS + c + 1] = acc[cb][1];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < XTR * q; e += XT) {
      const int c = e / XTR, r = e % XTR;
      if (r0 + r < n) Y[(int64_t)c * ldy + r0 + r] = out[r * XMS + c];
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__global__ void k_inv(const double* sigma, int q, double* out) {
  for (int c = threadIdx.x; c < q; c += blockDim.x) out[c] = 1.0 / sigma[c];
}

// Cholesky G = R^T R (R upper, column-major R[c*k + r]) and R^{-1}, one CTA.
constexpr int CLD = MAXK + 1;
// E^{-1} by Gauss-Jordan elimination with partial pivoting on [E | I] in shared memory, one CTA
// (k <= 32).  E(a, b) = W_a^T C_b = G[(k + b) * 2k + a] (the off-diagonal block of Gram([W | C])).
constexpr int EK = 32;
__global__ void __launch_bounds__(256) k_einv(const double* G, int k, DevState* st, int* fail) {
  __shared__ double M[EK][2 * EK + 1];
  __shared__ double f[EK];
  __shared__ int s_p, s_bad;
  __shared__ double s_emax;
  const int tid = threadIdx.x, bd = blockDim.x, s = 2 * k;
  for (int e = tid; e < k * 2 * k; e += bd) {
    const int r = e / (2 * k), c = e % (2 * k);
    M[r][c] = c < k ? G[(int64_t)(k + c) * s + r] : (c - k == r ? 1.0 : 0.0);
  }
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int r = 0; r < k; ++r)
      for (int c = 0; c < k; ++c) mx = fmax(mx, fabs(M[r][c]));
    s_emax = mx;
    s_bad = !(mx > 0.0);
  }
  __syncthreads();
  for (int c = 0; c < k && !s_bad; ++c) {
    if (tid == 0) {
      int p = c;
      for (int r = c + 1; r < k; ++r)
        if (fabs(M[r][c]) > fabs(M[p][c])) p = r;
      s_p = p;
      if (!(fabs(M[p][c]) > 1e-13 * s_emax)) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) break;
    const int p = s_p;
    if (p != c)
      for (int cc = tid; cc < 2 * k; cc += bd) {
        const double t = M[c][cc];
        M[c][cc] = M[p][cc];
        M[p][cc] = t;
      }
    __syncthreads();
    const double piv = M[c][c];
    __syncthreads();
    for (int cc = tid; cc < 2 * k; cc += bd) M[c][cc] /= piv;
    for (int r = tid; r < k; r += bd) f[r] = r == c ? 0.0 : M[r][c];  // multipliers vs the scaled pivot row
    __syncthreads();
    for (int e = tid; e < k * 2 * k; e += bd) {
      const int r = e / (2 * k), cc = e % (2 * k);
      if (r != c) M[r][cc] -= f[r] * M[c][cc];
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) fail[0] = 1;
    return;
  }
  for (int e = tid; e < k * k; e += bd) {
    const int r = e % k, c = e / k;
    st->Einv[c][r] = M[r][k + c];
  }
}

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

// SELL position i holds matrix row perm[i] (identity when perm is null: sigma = 1)
__global__ void k_sell_widths(const int32_t* rp, int64_t n, int32_t* sw, const int32_t* perm) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < ns; sl += (int64_t)gridDim.x * blockDim.x) {
    int w = 0;
    for (int r = 0; r < 32; ++r) {
      const int64_t pos = sl * 32 + r;
      if (pos < n) {
        const int64_t row = perm ? perm[pos] : pos;
        const int l = rp[row + 1] - rp[row];
        w = l > w ? l : w;
      }
    }
    sw[sl] = w;
  }
}

__global__ void k_sell_pack(const int32_t* rp, const int32_t* ci, const double* v, int64_t n,
                            const int64_t* sp, const int32_t* sw, int32_t* sci, double* sv, int pattern,
                            const int32_t* perm) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < ns * 32;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = pos >> 5;
    const int w = sw[sl];
    const int64_t base = sp[sl] + (pos & 31);
    int len = 0, p0 = 0;
    if (pos < n) {
      const int64_t row = perm ? perm[pos] : pos;
      p0 = rp[row];
      len = rp[row + 1] - p0;
    }
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
  note_host_launches(1);
  const int s8 = (s + 7) & ~7;
  const size_t smem = sizeof(double) * NST * s8 * TS;
  static PerDevice init_once;
  if (init_once.first()) {
    cudaFuncSetAttribute(k_gram_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * NST * S8MAX * TS));
  }
  int64_t g = (n + GTR - 1) / GTR;
  if (g > GRAM_CTAS) g = GRAM_CTAS;
  const int gi = (int)(g < 1 ? 1 : g);
  k_gram_mma<<<gi, GT, smem, strm>>>(Y, ld, n, s, partial, st);
  const int P = s * (s + 1) / 2;
  k_gram_reduce<<<(P + 7) / 8, 256, 0, strm>>>(partial, gi, s, G, counter, st, 8.0 * (double)n * s);
  return cudaGetLastError();
}

cudaError_t launch_jacobi(const double* G, int s, double* lam, double* V, double* sigma_out,
                          DevState* st, cudaStream_t strm, const double* V0, int s0, int rel) {
  const size_t smem = sizeof(double) * 3 * JLD * JLD;
  static PerDevice init_once;
  if (init_once.first()) {
    cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int half = (s + (s & 1)) / 2;  // one thread per 2x2 block of the rotation round (<= 1024)
  static const int nt_env = knob_int("RG_JACOBI_NT", 0);
  const int nt = nt_env > 0 ? nt_env : std::max(64, std::min(1024, (half * half + 31) / 32 * 32));
  k_jacobi<<<1, nt, smem, strm>>>(G, s, lam, V, sigma_out, st, s0 > 0 ? V0 : nullptr, s0, rel);
  return cudaGetLastError();
}

cudaError_t launch_xm(const double* X, int64_t ldx, int64_t n, int s, const double* M, int ldm, int q,
                      const double* colscale, double* Y, int64_t ldy, DevState* st, cudaStream_t strm) {
  note_host_launches(1);
  const int s8 = (s + 7) & ~7;
  const size_t smem = sizeof(double) * (s8 * XMS + XTR * XMS + NST * s8 * TS);
  static PerDevice init_once;
  if (init_once.first()) {
    cudaFuncSetAttribute(k_xm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (S8MAX * XMS + XTR * XMS + NST * S8MAX * TS)));
  }
  static int occ_s8[MAXDEV][S8MAX / 8 + 1] = {};  // occupancy per device and panel width (queried once each)
  int& occ = occ_s8[current_device()][s8 / 8];
  if (occ == 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_xm, XT, smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  int64_t g = (n + XTR - 1) / XTR;
  const int64_t cap = (int64_t)NSM * (occ < 1 ? 1 : (occ > 4 ? 4 : occ));
  if (g > cap) g = cap;
  k_xm<<<(int)(g < 1 ? 1 : g), XT, smem, strm>>>(X, ldx, n, s, M, ldm, q, colscale, Y, ldy, st);
  return cudaGetLastError();
}

cudaError_t launch_inv(const double* sigma, int q, double* out, cudaStream_t strm) {
  note_host_launches(1);
  k_inv<<<1, 64, 0, strm>>>(sigma, q, out);
  return cudaGetLastError();
}

cudaError_t launch_einv(const double* G, int k, DevState* st, int* fail, cudaStream_t strm) {
  note_host_launches(1);
  if (k < 1 || k > EK) return cudaErrorInvalidValue;
  k_einv<<<1, 256, 0, strm>>>(G, k, st, fail);
  return cudaGetLastError();
}

cudaError_t launch_chol(const double* G, int k, double* R, double* Rinv, int* fail, cudaStream_t strm) {
  note_host_launches(1);
  k_chol<<<1, 256, 0, strm>>>(G, k, R, Rinv, fail);
  return cudaGetLastError();
}

cudaError_t launch_rc_finish(const double* R1, const double* R1i, const double* R2, const double* R2i,
                             int k, DevState* st, int* fail, cudaStream_t strm) {
  note_host_launches(1);
  k_rc_finish<<<1, 256, 0, strm>>>(R1, R1i, R2, R2i, k, st, fail);
  return cudaGetLastError();
}

cudaError_t launch_sell_widths(const int32_t* rp, int64_t n, int32_t* sw, cudaStream_t strm, const int32_t* perm) {
  note_host_launches(1);
  k_sell_widths<<<NSM * 4, 256, 0, strm>>>(rp, n, sw, perm);
  return cudaGetLastError();
}

cudaError_t launch_sell_pack(const int32_t* rp, const int32_t* ci, const double* v, int64_t n,
                             const int64_t* sp, const int32_t* sw, int32_t* sci, double* sv,
                             int pattern, cudaStream_t strm, const int32_t* perm) {
  note_host_launches(1);
  k_sell_pack<<<NSM * 8, 256, 0, strm>>>(rp, ci, v, n, sp, sw, sci, sv, pattern, perm);
  return cudaGetLastError();
}

cudaError_t launch_validate(const int32_t* rp, const int32_t* ci, int64_t nrows, int64_t ncols,
                            int64_t nnz, int* bad, cudaStream_t strm) {
  note_host_launches(1);
  k_validate<<<NSM * 4, 256, 0, strm>>>(rp, ci, nrows, ncols, nnz, bad);
  return cudaGetLastError();
}

}  // namespace rg

// dcgs.cu — delayed classical Gram-Schmidt with re-orthogonalisation (DCGS2) for the Arnoldi
// step: one grid reduction and two passes over the basis per step (the classical CGS2 path in
// orth.cu needs three of each).
//
// Iteration j of a restart cycle holds u = the step-(j-1) vector after ONE CGS pass against
// P_j = [Q | v_0 .. v_{j-1}] (deflate) or [v_0 .. v_{j-1}] (plain, augment), stored raw in V
// column j, and y = A u (SpMV, V column j+1).
//   DK1 (this file): one sweep computing a = P_j^T u, b = P_j^T y, s = u.u, g = u.y (+ Q^T u for
//       augment).  Its last CTA finishes column j-1 of the Hessenberg matrix: the delayed second
//       pass gives h_{j-1} += a and nu = sqrt(s - a.a) = H[j][j-1] (Pythagoras: a is O(eps |u|),
//       no cancellation), runs the least-squares step on it (epi_ls), and, from the Arnoldi
//       relation A V_j = Q B_j + V_{j+1} H_j, derives without another pass
//         A v_j = (y - A P_j a)/nu,  w = [P] A v_j,  first-pass coefficients h1 = P_{j+1}^T w.
//   DK2 (this file): one sweep writing v_j = (u - P_j a)/nu and the next u = w - P_{j+1} h1 as two
//       linear combinations of the same rows of [u, y, P_j]; no reduction.
// (Swirydowicz, Langou, Ananthan, Yang, Thomas, "Low synchronization Gram-Schmidt and GMRES
// algorithms", 2020, and Bielich et al. 2022 describe the delayed re-orthogonalisation idea; the
// recycled (Q) bookkeeping here follows the GCRO relation of PAPER.md:332.)  The A Q a_Q term is
// dropped: a_Q = Q^T u is at rounding level because u was projected against Q.
//
// Oblique variant (operator M_D A, M_D = I - C E^{-1} W^T, C = A W in columns [k, 2k)): DK1 also
// reduces W^T y and C^T u; the epilogue forms t = E^{-1} W^T y, appends the row v_j^T C =
// (C^T u - (V_j^T C)^T a)/nu to the maintained V^T C (state Gm), and corrects the first-pass
// coefficients by -(V_{j+1}^T C) t / nu; DK2 adds -C t / nu to the next u.  No extra pass or
// reduction: M_D A v_j is never formed explicitly.
#define RG_FILE_ID 1  // RG_CHK locations (checked builds)
#include "epilogue.cuh"
#include "kernels.cuh"
#include "knobs.cuh"

#include <cstdlib>

namespace rg {
namespace {

constexpr int DT = 512;
// values one DK1 reduction returns: [a | b] over P = [Q | V] (<= MAXK + MAXM columns each), u.u,
// u.y and up to 2 MAXK extras; also the row stride of its partials (fits the partial buffer)
constexpr int DK1RED = 2 * (MAXK + MAXM) + 2 + 2 * MAXK;

// ---------------------------------------------------------------- DK1 epilogue
// tot = [a (p) | b (p) | s | g | q (k, augment) or W^T y (k), C^T u (k) (oblique)],
// P = columns [lo, VB + j).
__device__ void epi_dcgs(DevState* st, const Layout& L, const double* tot, int p) {
  __shared__ double Ha[MAXM + 2], Ba[MAXK], ob_t[MAXK], ob_ct[MAXM + 2];
  __shared__ double s_nu, s_d, s_aj;
  __shared__ int s_go;
  const int tid = threadIdx.x, bd = blockDim.x;
  const int j = st->j, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB;
  const int nq = VB - lo;  // Q columns inside P (deflate)
  RG_CHK(st, j >= 0 && j < MAXM && lo + p <= MAXCOL && (var != RG_DEFLATE || nq == k));
  const double* a = tot;
  const double* b = tot + p;
  const double ss = tot[2 * p], gg = tot[2 * p + 1];
  {  // a.a and a.b: deterministic block reductions (warp 0 and warp 1)
    const int lane = tid & 31, w = tid >> 5;
    if (w < 2) {
      double acc = 0.0;
      for (int c = lane; c < p; c += 32) acc += a[c] * (w == 0 ? a[c] : b[c]);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (w == 0) {
          const double nu2 = ss - acc;
          s_nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
        } else {
          s_d = acc;  // a.b, consumed below
        }
      }
    }
  }
  __syncthreads();
  const double ab = s_d;
  const double nu = s_nu;
  if (j >= 1) {
    // finish column j-1: second-pass coefficients a (V part -> H, Q part -> B via hcol), stored as
    // H-bar column j-1 (rows 0..j, h_{j,j-1} = nu) and B column j-1; the least-squares step on that
    // column (Givens, stop test, history) is left to k_dcgs_ls, which runs concurrently with DK2: it
    // gates only the NEXT step, and nothing DK2 needs depends on it (split epilogue: the last-CTA
    // tail of this kernel no longer holds the whole GPU for the serial Givens chain)
    for (int c = tid; c < p; c += bd) st->hcol[lo + c] += a[c];
    __syncthreads();
    for (int i = tid; i < j; i += bd) st->Hraw[j - 1][i] = st->hcol[VB + i];
    if (var == RG_DEFLATE)
      for (int l = tid; l < k; l += bd) st->Bm[j - 1][l] = st->hcol[QB + l];
    if (var == RG_AUGMENT && k > 0) {  // Q^T v_j = (Q^T u - G_j^T a_V) / nu, handed to the LS step as (.)*nu
      for (int l = tid; l < k; l += bd) {
        double q = tot[2 * p + 2 + l];
        for (int i = 0; i < j; ++i) q -= st->Gm[i][l] * a[nq + i];
        st->ls_in[l] = q;
      }
    }
    if (tid == 0) {
      st->Hraw[j - 1][j] = nu;
      st->ls_in[(var == RG_AUGMENT) ? k : 0] = nu * nu;
      st->ls_j = j - 1;
      st->sc[VB + j] = 1.0;  // DK2 writes v_j normalised
    }
  } else if (tid == 0) {
    st->ls_j = -1;
  }
  if (tid == 0) {
    s_go = j < st->m;        // j = m: no next column (DK2 would write past the basis)
    st->k2_skip = !s_go;
  }
  __syncthreads();
  if (!s_go) return;
  // ---- coefficients of DK2 and the first-pass coefficients of column j
  const double inv = nu > 0.0 ? 1.0 / nu : 0.0;
  const bool obl = galerkin_variant(var) && k > 0;  // oblique / orthogonal (P = C / W, T = E^{-1} / I)
  const int pbase = proj_base(var, k);
  if (obl) {
    const double* wy = tot + 2 * p + 2;  // W^T y
    const double* cu = wy + k;           // P^T u
    for (int l = tid; l < k; l += bd) {
      double t = 0.0;
      if (var == RG_ORTHOGONAL) t = wy[l];
      else
        for (int b2 = 0; b2 < k; ++b2) t += st->Einv[b2][l] * wy[b2];
      ob_t[l] = t;
      double g = cu[l];                  // v_j^T C = (u - V_j a)^T C / nu
      for (int i = 0; i < j; ++i) g -= a[i] * st->Gm[i][l];
      st->Gm[j][l] = g * inv;
    }
    __syncthreads();
    {
      const int lane = tid & 31, nw = bd >> 5;
      for (int i = tid >> 5; i <= j; i += nw) {  // ct_i = (V^T C t)_i
        double s = 0.0;
        for (int l = lane; l < k; l += 32) s += st->Gm[i][l] * ob_t[l];
        s = warp_sum(s);
        if (lane == 0) ob_ct[i] = s;
      }
    }
    for (int l = tid; l < k; l += bd) st->coef[pbase + l] = -ob_t[l] * inv;
    __syncthreads();
  }
  // (H a_V)_c over the final columns 0..j-1 (Hessenberg) and (B a_V)_l: one warp per output,
  // lanes over the summation index (all loads of a warp in flight), fixed shuffle tree.
  {
    const int lane = tid & 31, nw = bd >> 5;
    for (int o = tid >> 5; o < j + (var == RG_DEFLATE ? nq : 0); o += nw) {
      double s = 0.0;
      if (o < j) {
        for (int i = (o > 0 ? o - 1 : 0) + lane; i < j; i += 32) s += st->Hraw[i][o] * a[nq + i];
      } else {
        const int l = o - j;
        for (int i = lane; i < j; i += 32) s += st->Bm[i][l] * a[nq + i];
      }
      s = warp_sum(s);
      if (lane == 0) {
        if (o < j) Ha[o] = s;
        else Ba[o - j] = s;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double aj = j >= 1 ? a[nq + j - 1] : 0.0;
    s_aj = aj;
    s_d = ((gg - ab) * inv - nu * aj - (obl ? ob_ct[j] : 0.0)) * inv;  // v_j^T w
    st->k2_inv_nu = inv;
    st->k2_y = inv;
    st->k2_u_next = -(aj + s_d) * inv;
    st->hcol[VB + j] = s_d;
  }
  __syncthreads();
  const double f = (s_aj + s_d) * inv;
  for (int c = tid; c < j; c += bd) {  // V columns
    const double cv = (b[nq + c] - Ha[c] - (obl ? ob_ct[c] : 0.0)) * inv;
    st->hcol[VB + c] = cv;
    st->coef[VB + c] = -Ha[c] * inv - cv + f * a[nq + c];
    st->coefv[VB + c] = -a[nq + c] * inv;
  }
  for (int l = tid; l < nq; l += bd) {  // Q columns (deflate): w = (I - QQ^T) A v_j
    st->hcol[QB + l] = (b[l] - Ba[l]) * inv;
    st->coef[QB + l] = -b[l] * inv + f * a[l];
    st->coefv[QB + l] = -a[l] * inv;
  }
  __syncthreads();
}

// grid reduction of DK1's partial vector, the DCGS2 epilogue in the last CTA, state advance
__device__ __forceinline__ void dk1_finish(const Layout& L, DevState* st, double* dpart, double* tot, int nv, int p,
                                           int nqd, int j, bool have_y, unsigned long long cond) {
  if (!grid_reduce(dpart, nv, L.partial, L.counter, tot, tot, DK1RED)) return;
  prof_tail(st, K_DK1);
  epi_dcgs(st, L, tot, p);
  if (threadIdx.x == 0) {
    st->j = j + 1;  // next iteration (DK2 of this one uses st->j - 1); k_dcgs_ls decides whether it runs
    (void)cond;     // the WHILE condition is set by k_dcgs_ls
    prof_end(st, K_DK1, 8.0 * (double)L.n * (p + nqd + (have_y ? 2 : 1)));
  }
}

// DK1 of a step after the cycle stopped (unrolled Arnoldi bodies run up to RG_UNROLL-1 such steps):
// nothing to reduce; the step's update pass and least-squares kernel must not act either
__device__ __forceinline__ void dk1_noop(DevState* st) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->k2_skip = 1;
    st->ls_j = -1;
  }
  prof_noop(st, K_DK1);
}

// ---------------------------------------------------------------- the least-squares step (split epilogue)
// Column st->ls_j of the cycle (finished by DK1): Givens / M = T H update, history, stop test, and at a
// stop the cycle-end coefficients (epi_ls).  Runs on a side branch of the graph, concurrently with DK2;
// the graph joins both before the next step, whose launch this kernel's WHILE condition gates.
__global__ void __launch_bounds__(256) k_dcgs_ls(Layout L, DevState* st, unsigned long long cond) {
  __shared__ double lst[MAXK + 2];
  const int jx = st->ls_j;
  RG_CHK(st, jx < MAXM && jx < st->m);
  if (jx >= 0) {
    if (st->profile && threadIdx.x == 0) {
      st->kstat[K_DLS].start = gtimer();
      trace_ev(st, K_DLS, 0u, st->kstat[K_DLS].start);
    }
    const int nd = st->variant == RG_AUGMENT ? st->k_eff : 0;
    for (int i = threadIdx.x; i <= nd; i += blockDim.x) lst[i] = st->ls_in[i];
    __syncthreads();
    epi_ls(st, L, lst, nd, jx);
    if (threadIdx.x == 0) prof_end(st, K_DLS, 0.0);
  }
  if (cond && threadIdx.x == 0) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, st->active ? 1u : 0u);
}

// ---------------------------------------------------------------- DK1: dots of u and y with P
// Rows are split evenly over the CTAs; per 512-row sub-tile u and y are staged in shared memory,
// warp w owns columns w, w+16, ...: 16 independent loads per lane, two products, fixed shuffle
// tree, warp-owned shared-memory accumulators (deterministic).
__global__ void __launch_bounds__(DT, 2) k_dk1(Layout L, DevState* st, unsigned long long cond) {
  __shared__ double us[DT], ys[DT];
  __shared__ double dpart[DK1RED];
  __shared__ double tot[DK1RED];
  __shared__ double bsh[33];
  if (!st->active) { dk1_noop(st); return; }
  prof_begin(st, K_DK1);
  const int j = st->j, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j, p = hi - lo;
  const int nqd = (var == RG_AUGMENT) ? k : (galerkin_variant(var) ? 2 * k : 0);  // extra dots
  const bool have_y = j < st->m;                // no SpMV was run at j == m
  const bool keep = L.keep_l2 != 0;  // basis fits L2: let DK2 re-hit what DK1 streamed
  const int64_t ld = L.ld;
  const double* __restrict__ u = L.Z + (int64_t)(VB + j) * ld;
  const double* __restrict__ y = L.Z + (int64_t)(VB + j + 1) * ld;
  const double* __restrict__ Z = L.Z;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nv = 2 * p + 2 + nqd;
  for (int c = threadIdx.x; c < nv; c += DT) dpart[c] = 0.0;
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  double s_uu = 0.0, s_uy = 0.0;
  constexpr int RPL = DT / 32;
  for (int64_t base = r0; base < r1; base += DT) {
    const int64_t r = base + threadIdx.x;
    const bool in = r < r1;
    const double ur = in ? u[r] : 0.0;
    const double yr = (in && have_y) ? y[r] : 0.0;
    __syncthreads();  // previous sub-tile's readers are done with us/ys (and dpart zeroed)
    us[threadIdx.x] = ur;
    ys[threadIdx.x] = yr;
    s_uu += ur * ur;
    s_uy += ur * yr;
    __syncthreads();
    const int cnt = (int)((r1 - base) < DT ? (r1 - base) : DT);
    for (int c = wid; c < p + nqd; c += 16) {
      // extras: W^T y (cols [0,k)), P^T u (P = C: cols [k,2k); P = W: cols [0,k) again)
      const bool obl = galerkin_variant(var);
      const int col = c < p ? lo + c : (obl ? ((c - p) < k ? c - p : proj_base(var, k) + (c - p - k)) : QB + (c - p));
      const double* __restrict__ zc = Z + (int64_t)col * ld + base + lane;
      double zv[RPL];
#pragma unroll
      for (int q = 0; q < RPL; ++q) zv[q] = (lane + 32 * q < cnt) ? (keep ? zc[32 * q] : __ldcs(zc + 32 * q)) : 0.0;
      double su = 0.0, sy = 0.0;
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        su += zv[q] * us[lane + 32 * q];
        sy += zv[q] * ys[lane + 32 * q];
      }
      su = warp_sum(su);
      if (c < p) {
        sy = warp_sum(sy);
        if (lane == 0) {
          dpart[c] += su;
          dpart[p + c] += sy;
        }
      } else {
        const bool wy = obl && (c - p) < k;
        if (wy) sy = warp_sum(sy);
        if (lane == 0) dpart[2 * p + 2 + (c - p)] += wy ? sy : su;
      }
    }
  }
  // layout of the reduced vector: [a (p) | b (p) | s | g | q (nqd)]
  const double t1 = block_sum(s_uu, bsh);
  const double t2 = block_sum(s_uy, bsh);
  if (threadIdx.x == 0) {
    dpart[2 * p] = t1;
    dpart[2 * p + 1] = t2;
  }
  __syncthreads();
  dk1_finish(L, st, dpart, tot, nv, p, nqd, j, have_y, cond);
}

// ---------------------------------------------------------------- DK1, streaming variant
// The DK2 access pattern (thread per row, stride = CTA size, all loads of a row independent) with the
// dot columns taken in chunks of SCH: per chunk every thread keeps 2 * SCH partial sums (u and y) in
// registers over all of the CTA's rows and the chunk ends with ONE block reduction; u and y are
// re-read per chunk (L2 hits).  No per-sub-tile barrier and no shared-memory staging.
template <int SCH, int RU>  // SCH columns per chunk, RU rows per thread per iteration (loads in flight)
__global__ void __launch_bounds__(DT, 2) k_dk1_stream(Layout L, DevState* st, unsigned long long cond, int nvw) {
  // per-warp partials in the layout of dpart: a chunk ends with warp shuffles only (no barrier), so
  // warps drift freely from chunk to chunk; ONE cross-warp sum at the end (fixed warp order).
  // (First version: a block reduction with two barriers per chunk.)
  extern __shared__ double wsm[];  // [DT / 32][nvw]
  __shared__ double dpart[DK1RED];
  __shared__ double tot[DK1RED];
  if (!st->active) { dk1_noop(st); return; }
  prof_begin(st, K_DK1);
  const int j = st->j, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j, p = hi - lo;
  const int nqd = (var == RG_AUGMENT) ? k : (galerkin_variant(var) ? 2 * k : 0);
  const bool have_y = j < st->m;
  const bool keep = L.keep_l2 != 0;
  const int64_t ld = L.ld;
  const double* __restrict__ u = L.Z + (int64_t)(VB + j) * ld;
  const double* __restrict__ y = L.Z + (int64_t)(VB + j + 1) * ld;
  const double* __restrict__ Z = L.Z;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nv = 2 * p + 2 + nqd, ncols = p + nqd;
  const bool obl = galerkin_variant(var);
  double* wp = wsm + (size_t)wid * nvw;
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  double s_uu = 0.0, s_uy = 0.0;
  for (int c0 = 0; c0 < ncols || c0 == 0; c0 += SCH) {
    const int nc = min(SCH, ncols - c0);
    const double* zp[SCH];
#pragma unroll
    for (int kk = 0; kk < SCH; ++kk) {
      const int c = c0 + (kk < nc ? kk : 0);
      const int col = c < p ? lo + c : (obl ? ((c - p) < k ? c - p : proj_base(var, k) + (c - p - k)) : QB + (c - p));
      zp[kk] = Z + (int64_t)col * ld;
    }
    double su[SCH], sy[SCH];
#pragma unroll
    for (int kk = 0; kk < SCH; ++kk) su[kk] = sy[kk] = 0.0;
    for (int64_t rb = r0 + threadIdx.x; rb < r1; rb += DT * RU) {
      double ur[RU], yr[RU], z[RU][SCH];
#pragma unroll
      for (int q = 0; q < RU; ++q) {  // all loads of RU rows issued before any use
        const int64_t r = rb + (int64_t)q * DT;
        const bool ok = r < r1;
        ur[q] = ok ? u[r] : 0.0;
        yr[q] = (ok && have_y) ? y[r] : 0.0;
#pragma unroll
        for (int kk = 0; kk < SCH; ++kk) z[q][kk] = (ok && kk < nc) ? (keep ? zp[kk][r] : __ldcs(zp[kk] + r)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < RU; ++q) {
#pragma unroll
        for (int kk = 0; kk < SCH; ++kk) {
          su[kk] += z[q][kk] * ur[q];
          sy[kk] += z[q][kk] * yr[q];
        }
        if (c0 == 0) {
          s_uu += ur[q] * ur[q];
          s_uy += ur[q] * yr[q];
        }
      }
    }
#pragma unroll
    for (int kk = 0; kk < SCH; ++kk) {
      const double a = warp_sum(su[kk]), b = warp_sum(sy[kk]);
      const int c = c0 + kk;
      if (lane == 0 && kk < nc) {
        if (c < p) {
          wp[c] = a;
          wp[p + c] = b;
        } else {
          const bool wy = obl && (c - p) < k;  // extras: W^T y, P^T u (galerkin) / Q^T u (augment)
          wp[2 * p + 2 + (c - p)] = wy ? b : a;
        }
      }
    }
    if (ncols == 0) break;
  }
  {
    const double t1 = warp_sum(s_uu), t2 = warp_sum(s_uy);
    if (lane == 0) {
      wp[2 * p] = t1;
      wp[2 * p + 1] = t2;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += DT) {
    double sacc = 0.0;
    for (int w = 0; w < DT / 32; ++w) sacc += wsm[(size_t)w * nvw + i];
    dpart[i] = sacc;
  }
  __syncthreads();
  dk1_finish(L, st, dpart, tot, nv, p, nqd, j, have_y, cond);
}

// ---------------------------------------------------------------- DK2: v_j and the next u
__global__ void __launch_bounds__(DT, 2) k_dk2(Layout L, DevState* st) {
  __shared__ double cv[MAXCOL], cn[MAXCOL], cc2[MAXK];
  if (st->k2_skip) { prof_noop(st, K_DK2); return; }  // (not st->active: k_dcgs_ls may be writing it)
  prof_begin(st, K_DK2);
  const int j = st->j - 1, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j, p = hi - lo;
  const int64_t ld = L.ld;
  const bool keep = L.keep_l2 != 0;
  double* __restrict__ u = L.Z + (int64_t)(VB + j) * ld;      // in: u, out: v_j
  double* __restrict__ y = L.Z + (int64_t)(VB + j + 1) * ld;  // in: y, out: next u
  const double* __restrict__ Z = L.Z;
  for (int c = threadIdx.x; c < p; c += DT) {
    cv[c] = st->coefv[lo + c];
    cn[c] = st->coef[lo + c];
  }
  const int k2 = galerkin_variant(var) ? k : 0;  // next u also gets -P t / nu (P = C or W)
  const int pb2 = proj_base(var, k);
  for (int l = threadIdx.x; l < k2; l += DT) cc2[l] = st->coef[pb2 + l];
  const double inv = st->k2_inv_nu, fy = st->k2_y, fu = st->k2_u_next;
  __syncthreads();
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += DT) {
    const double ur = u[r], yr = y[r];
    double sv = 0.0, sn = 0.0;
    int c = 0;
    for (; c + 8 <= p; c += 8) {
      double z[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) z[t] = keep ? Z[(int64_t)(lo + c + t) * ld + r] : __ldcs(Z + (int64_t)(lo + c + t) * ld + r);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        sv += cv[c + t] * z[t];
        sn += cn[c + t] * z[t];
      }
    }
    for (; c < p; ++c) {
      const double z = keep ? Z[(int64_t)(lo + c) * ld + r] : __ldcs(Z + (int64_t)(lo + c) * ld + r);
      sv += cv[c] * z;
      sn += cn[c] * z;
    }
    for (int l = 0; l < k2; ++l) sn += cc2[l] * (keep ? Z[(int64_t)(pb2 + l) * ld + r] : __ldcs(Z + (int64_t)(pb2 + l) * ld + r));
    u[r] = ur * inv + sv;
    y[r] = yr * fy + ur * fu + sn;
  }
  if (st->profile && grid_last(L.counter) && threadIdx.x == 0) prof_end(st, K_DK2, 8.0 * (double)L.n * (p + k2 + 4));
}

// ---------------------------------------------------------------- TMA-streamed DK1 / DK2
// The register-limited kernels above keep ~10 loads of 8 B in flight per thread (64 registers at
// 2 CTAs/SM): ncu shows them long-scoreboard bound at 3.8 (DK1) / 4.6 (DK2) TB/s cold at C4.  Here a
// producer warp streams the CTA's rows of the basis columns with cp.async.bulk (TMA, 1-D) into a
// TS_STG-stage shared-memory ring (TS_CH columns x TS_R rows per stage, 32 KB), completing on
// mbarriers, so ~128 KB per SM are in flight independently of registers; TS_R consumer threads own
// one row each of the current row tile.  Same loop order and accumulation order as the streaming
// kernels (DK1: column chunk outer, row tile inner; DK2: row tile outer, columns ascending).
constexpr int TS_R = 512;              // consumer threads = rows per tile
constexpr int TS_T = TS_R + 32;        // + producer warp
constexpr int TS_CH = 8;               // columns per stage
constexpr int TS_STG = 4;              // stages
constexpr int TS_STAGE = TS_CH * TS_R; // doubles per stage

__device__ __forceinline__ uint32_t ts_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ts_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(ts_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void ts_init(uint64_t* full, uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < TS_STG; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ts_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ts_u32(&empty[i])), "r"(TS_R / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
// L2 policy of the streamed basis: evict-first when the basis does not fit L2 (as the __ldcs loads
// of the register kernels: the SpMV's A / x and DK1's u, y re-reads keep their L2 lines), evict-
// normal when it does (keep_l2: the next pass re-hits it)
__device__ __forceinline__ uint64_t ts_policy(bool keep) {
  uint64_t pol;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// producer WARP: stage number t (global sequence) of `nc` column segments [col_c + base, +cnt rows).  Lane c
// issues column c's bulk copy (round 2, late: one lane issuing all 8 copies, each with its own index
// load and 64-bit address arithmetic, took about as long per stage as the stage's 32 KB take to stream
// — the producer lane, not HBM, set the rate of the dots pass).
__device__ __forceinline__ void ts_issue(double* ring, uint64_t* full, uint64_t* empty, int t, const double* Z,
                                         int64_t ld, const int* cols, int nc, int64_t base, int cnt, uint64_t pol) {
  const int s = t % TS_STG, lane = threadIdx.x & 31;
  if (t >= TS_STG) ts_wait(&empty[s], (uint32_t)((t / TS_STG - 1) & 1));
  if (lane == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ts_u32(&full[s])),
                 "r"((uint32_t)(nc * cnt * 8)) : "memory");
  __syncwarp();
  if (lane < nc)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(ts_u32(ring + (size_t)s * TS_STAGE + lane * TS_R)), "l"(Z + (int64_t)cols[lane] * ld + base),
                 "r"((uint32_t)(cnt * 8)), "r"(ts_u32(&full[s])), "l"(pol) : "memory");
}
__device__ __forceinline__ void ts_release(uint64_t* empty, int s) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ts_u32(&empty[s])) : "memory");
}

__global__ void __launch_bounds__(TS_T, 1) k_dk1_tma(Layout L, DevState* st, unsigned long long cond, int nvw) {
  extern __shared__ __align__(128) double ring[];   // [TS_STG][TS_STAGE], then per-warp partials [TS_R / 32][nvw]
  __shared__ __align__(8) uint64_t full[TS_STG], empty[TS_STG];
  double* wsm = ring + (size_t)TS_STG * TS_STAGE;
  __shared__ double dpart[DK1RED];
  __shared__ double tot[DK1RED];
  __shared__ int colidx[DK1RED];
  if (!st->active) { dk1_noop(st); return; }
  prof_begin(st, K_DK1);
  const int j = st->j, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j, p = hi - lo;
  const int nqd = (var == RG_AUGMENT) ? k : (galerkin_variant(var) ? 2 * k : 0);
  const bool have_y = j < st->m;
  const int64_t ld = L.ld;
  const double* __restrict__ u = L.Z + (int64_t)(VB + j) * ld;
  const double* __restrict__ y = L.Z + (int64_t)(VB + j + 1) * ld;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nv = 2 * p + 2 + nqd, ncols = p + nqd;
  const bool obl = galerkin_variant(var);
  for (int c = tid; c < ncols; c += TS_T) {
    colidx[c] = c < p ? lo + c : (obl ? ((c - p) < k ? c - p : proj_base(var, k) + (c - p - k)) : QB + (c - p));
    RG_CHK(st, colidx[c] >= 0 && colidx[c] < L.ncol && (c >= p || colidx[c] < VB + j));
  }
  RG_CHK(st, j >= 0 && j <= st->m && st->m <= MAXM && k >= 0 && k <= L.maxk && lo >= 0 && nv <= DK1RED && nv <= nvw &&
                 ncols <= DK1RED && (!have_y || VB + j + 1 < L.ncol));
  ts_init(full, empty);
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const int nchunk = (ncols + TS_CH - 1) / TS_CH;
  if (wid == TS_R / 32) {  // ---- producer warp (lane = column of the stage): chunk outer, row tile inner
    const uint64_t pol = ts_policy(L.keep_l2 != 0);
    int t = 0;
    for (int q = 0; q < nchunk; ++q)
      for (int64_t base = r0; base < r1; base += TS_R, ++t)
        ts_issue(ring, full, empty, t, L.Z, ld, colidx + q * TS_CH, min(TS_CH, ncols - q * TS_CH), base,
                 (int)min((int64_t)TS_R, r1 - base), pol);
  } else {  // ---- consumers: thread = row of the tile
    pdl_wait();  // u, y: written by the SpMV this launch may overlap (PDL); the basis stream above is not
    double s_uu = 0.0, s_uy = 0.0;
    int t = 0;
    // u, y of the tile TS_PF tiles ahead are loaded now (L2 hits, off the per-tile critical path);
    // the tile sequence repeats per chunk, so "ahead" wraps to the start of the CTA's rows
#ifndef RG_DK1_PF
#define RG_DK1_PF 3
#endif
    constexpr int TS_PF = RG_DK1_PF;
    double upf[TS_PF], ypf[TS_PF];
    int64_t bnext = r0;  // base of the next tile to prefetch
#pragma unroll
    for (int i = 0; i < TS_PF; ++i) {
      const int64_t rn = bnext + tid;
      upf[i] = rn < r1 ? u[rn] : 0.0;
      ypf[i] = (rn < r1 && have_y) ? y[rn] : 0.0;
      bnext = bnext + TS_R < r1 ? bnext + TS_R : r0;
    }
    for (int q = 0; q < nchunk || q == 0; ++q) {
      const int nc = min(TS_CH, ncols - q * TS_CH);
      double su[TS_CH], sy[TS_CH];
#pragma unroll
      for (int c = 0; c < TS_CH; ++c) su[c] = sy[c] = 0.0;
      for (int64_t base = r0; base < r1; base += TS_R) {
        const int64_t r = base + tid;
        const bool ok = r < r1;
        const double ur = upf[0], yr = ypf[0];
        {
#pragma unroll
          for (int i = 0; i + 1 < TS_PF; ++i) {
            upf[i] = upf[i + 1];
            ypf[i] = ypf[i + 1];
          }
          const int64_t rn = bnext + tid;
          upf[TS_PF - 1] = rn < r1 ? u[rn] : 0.0;
          ypf[TS_PF - 1] = (rn < r1 && have_y) ? y[rn] : 0.0;
          bnext = bnext + TS_R < r1 ? bnext + TS_R : r0;
        }
        if (q == 0) {
          s_uu += ur * ur;
          s_uy += ur * yr;
        }
        if (nc <= 0) continue;
        const int stg = t % TS_STG;
        ts_wait(&full[stg], (uint32_t)((t / TS_STG) & 1));
        const double* zs = ring + (size_t)stg * TS_STAGE + tid;
#pragma unroll
        for (int c = 0; c < TS_CH; ++c) {
          const double z = (ok && c < nc) ? zs[c * TS_R] : 0.0;
          su[c] += z * ur;
          sy[c] += z * yr;
        }
        ts_release(empty, stg);
        ++t;
      }
#pragma unroll
      for (int c = 0; c < TS_CH; ++c) {
        const double a = warp_sum(su[c]), b = warp_sum(sy[c]);
        const int cc = q * TS_CH + c;
        if (lane == 0 && c < nc) {
          if (cc < p) {
            wsm[wid * nvw + cc] = a;
            wsm[wid * nvw + p + cc] = b;
          } else {
            const bool wy = obl && (cc - p) < k;  // extras: W^T y, P^T u (galerkin) / Q^T u (augment)
            wsm[wid * nvw + 2 * p + 2 + (cc - p)] = wy ? b : a;
          }
        }
      }
    }
    const double t1 = warp_sum(s_uu), t2 = warp_sum(s_uy);
    if (lane == 0) {
      wsm[wid * nvw + 2 * p] = t1;
      wsm[wid * nvw + 2 * p + 1] = t2;
    }
  }
  pdl_trigger();  // the update pass may be scheduled (it waits for this grid before reading anything)
  __syncthreads();
  for (int i = tid; i < nv; i += TS_T) {
    double sacc = 0.0;
    for (int w = 0; w < TS_R / 32; ++w) sacc += wsm[w * nvw + i];
    dpart[i] = sacc;
  }
  __syncthreads();
  dk1_finish(L, st, dpart, tot, nv, p, nqd, j, have_y, cond);
}

__global__ void __launch_bounds__(TS_T, 1) k_dk2_tma(Layout L, DevState* st) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[TS_STG], empty[TS_STG];
  __shared__ double cv[MAXCOL + MAXK], cn[MAXCOL + MAXK];
  __shared__ int colidx[MAXCOL + MAXK];
  pdl_wait();  // everything below reads DK1's epilogue output (launched with PDL behind DK1)
  if (st->k2_skip) { prof_noop(st, K_DK2); return; }  // (not st->active: k_dcgs_ls may be writing it)
  prof_begin(st, K_DK2);
  const int j = st->j - 1, k = st->k_eff, var = st->variant, VB = L.VB, QB = VB - k;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j, p = hi - lo;
  const int64_t ld = L.ld;
  double* __restrict__ u = L.Z + (int64_t)(VB + j) * ld;      // in: u, out: v_j
  double* __restrict__ y = L.Z + (int64_t)(VB + j + 1) * ld;  // in: y, out: next u
  const int tid = threadIdx.x, wid = tid >> 5;
  const int k2 = galerkin_variant(var) ? k : 0;  // next u also gets -P t / nu (P = C or W)
  const int pb2 = proj_base(var, k), ncols = p + k2;
  for (int c = tid; c < ncols; c += TS_T) {
    if (c < p) {
      cv[c] = st->coefv[lo + c];
      cn[c] = st->coef[lo + c];
      colidx[c] = lo + c;
    } else {
      cv[c] = 0.0;
      cn[c] = st->coef[pb2 + (c - p)];
      colidx[c] = pb2 + (c - p);
    }
  }
  RG_CHK(st, j >= 0 && j < st->m && VB + j + 1 < L.ncol && ncols <= MAXCOL + MAXK && lo >= 0 && pb2 + k2 <= L.ncol);
  const double inv = st->k2_inv_nu, fy = st->k2_y, fu = st->k2_u_next;
  ts_init(full, empty);
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const int nchunk = (ncols + TS_CH - 1) / TS_CH;
  if (wid == TS_R / 32) {  // ---- producer warp: row tile outer, column chunk inner
    const uint64_t pol = ts_policy(L.keep_l2 != 0);
    int t = 0;
    for (int64_t base = r0; base < r1; base += TS_R)
      for (int q = 0; q < nchunk; ++q, ++t)
        ts_issue(ring, full, empty, t, L.Z, ld, colidx + q * TS_CH, min(TS_CH, ncols - q * TS_CH), base,
                 (int)min((int64_t)TS_R, r1 - base), pol);
  } else {
    int t = 0;
    for (int64_t base = r0; base < r1; base += TS_R) {
      const int64_t r = base + tid;
      const bool ok = r < r1;
      const double ur = ok ? u[r] : 0.0, yr = ok ? y[r] : 0.0;
      double sv = 0.0, sn = 0.0;
      for (int q = 0; q < nchunk; ++q, ++t) {
        const int stg = t % TS_STG, c0 = q * TS_CH, nc = min(TS_CH, ncols - c0);
        ts_wait(&full[stg], (uint32_t)((t / TS_STG) & 1));
        const double* zs = ring + (size_t)stg * TS_STAGE + tid;
#pragma unroll
        for (int c = 0; c < TS_CH; ++c) {
          if (c < nc) {
            const double z = ok ? zs[c * TS_R] : 0.0;
            sv += cv[c0 + c] * z;
            sn += cn[c0 + c] * z;
          }
        }
        ts_release(empty, stg);
      }
      if (ok) {
        u[r] = ur * inv + sv;
        y[r] = yr * fy + ur * fu + sn;
      }
    }
  }
  if (st->profile && grid_last(L.counter) && threadIdx.x == 0) prof_end(st, K_DK2, 8.0 * (double)L.n * (p + k2 + 4));
}

}  // namespace

// one CTA per SM (the TMA kernels), at most one per 512-row tile
static int tma_grid(int64_t rows) {
  int64_t g = (rows + TS_R - 1) / TS_R;
  if (g > NSM) g = NSM;
  return (int)(g < 1 ? 1 : g);
}

// PDL between the kernels of an Arnoldi step (SpMV -> DK1 -> DK2): measured in a conditional WHILE body,
// ~2.5 us per edge (tools/cutest/t_pdl.cu); RG_NO_PDL (EXPERIMENTS builds) for A/B
static bool pdl_on() {
  static const bool off = knob("RG_NO_PDL");
  return !off;
}

cudaError_t launch_dcgs(const Layout& L, DevState* st, int phase, cudaStream_t s, unsigned long long cond) {
  static PerDevice init_once;
  if (init_once.first()) {
    cudaFuncSetAttribute(k_dk1, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_dk2, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  }
  if (phase == 1) {
    // streaming variant by default (C4: 3.90 -> 4.54 TB/s; (SCH, RU) = (4, 2) and (6, 2) measured
    // equal, (4, 4) spills); RG_DK1_TILES=1 selects the shared-memory sub-tile kernel
    static const int tiles = knob("RG_DK1_TILES") ? 1 : 0;
    static const int tma = knob("RG_NO_TMA_DCGS") || knob("RG_NO_TMA_DK1") ? 0 : 1;
    if (tma && !tiles) {
      const int nvw = 2 * (L.maxk + MAXM) + 2 + 2 * L.maxk;  // >= nv of any step of this context
      const size_t smem = sizeof(double) * ((size_t)TS_STG * TS_STAGE + (size_t)(TS_R / 32) * nvw);
      static PerDevice attr_once;
      if (attr_once.first()) {
        cudaFuncSetAttribute(k_dk1_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * ((size_t)TS_STG * TS_STAGE + (size_t)(TS_R / 32) * DK1RED)));
      }
      return launch_ex(k_dk1_tma, dim3(tma_grid(L.ld)), dim3(TS_T), smem, s, pdl_on(), L, st, cond, nvw);
    }
    if (!tiles) {
      const int nvw = 2 * (L.maxk + MAXM) + 2 + 2 * L.maxk;  // >= nv of any step of this context
      const size_t smem = sizeof(double) * (DT / 32) * (size_t)nvw;
      static PerDevice attr_once;
      if (attr_once.first()) {
        cudaFuncSetAttribute(k_dk1_stream<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * (DT / 32) * (size_t)DK1RED));
      }
      k_dk1_stream<8, 1><<<vec_grid(L.ld), DT, smem, s>>>(L, st, cond, nvw);
    } else
      k_dk1<<<vec_grid(L.ld), DT, 0, s>>>(L, st, cond);
    return cudaGetLastError();
  }
  if (phase == 3) {
    k_dcgs_ls<<<1, 256, 0, s>>>(L, st, cond);
    return cudaGetLastError();
  }
  static const int tma = knob("RG_NO_TMA_DCGS") || knob("RG_NO_TMA_DK2") ? 0 : 1;
  if (tma) {
    static PerDevice attr_once;
    if (attr_once.first()) {
      cudaFuncSetAttribute(k_dk2_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * TS_STG * TS_STAGE));
    }
    // one SM left to the concurrent least-squares kernel (k_dcgs_ls) so that no update-pass CTA shares
    // an SM with it
    const int g2 = tma_grid(L.ld) == NSM ? NSM - 1 : tma_grid(L.ld);
    return launch_ex(k_dk2_tma, dim3(g2), dim3(TS_T), sizeof(double) * TS_STG * TS_STAGE, s, pdl_on(), L, st);
  }
  k_dk2<<<vec_grid(L.ld), DT, 0, s>>>(L, st);
  return cudaGetLastError();
}

}  // namespace rg

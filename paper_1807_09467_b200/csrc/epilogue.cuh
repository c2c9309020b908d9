// epilogue.cuh — work done by the LAST CTA of a reducing kernel, on the device-resident state.
//
// These replace the host round trips of a textbook GMRES: the Givens least-squares update
// (one warp / thread, "not computed naively ... but in more efficient ways"), the
// restart decision, the GCRO (deflate) and G/T/M (augment) bookkeeping and the cycle-end
// coefficient computation.  All threads of the last CTA call each function (they contain
// __syncthreads); the serial chains run in thread 0 from shared memory.
#pragma once
#include "common.cuh"

namespace rg {

// ---------------------------------------------------------------- cycle start
// beta2 = ||r_c||^2 of the (projected) residual r_c = b - A x_c stored in V column 0.
__device__ __forceinline__ void epi_cycle_start(DevState* st, const Layout& L, double beta2) {
  if (threadIdx.x == 0) {
    const double beta = sqrt(beta2);
    st->beta = beta;
    st->relres = beta / st->bnorm;
    st->have_xupd = 0;
    if (!isfinite(beta)) {
      st->status = RG_E_NUMERIC;
      st->done = 1;
      st->active = 0;
    } else if (st->relres <= st->tol) {
      st->done = 1;
      st->converged = 1;
      st->active = 0;
    } else if (st->iters >= st->max_iters) {
      st->done = 1;
      st->active = 0;
    } else {
      st->active = 1;
      st->j = 0;
      st->cycles++;
      st->sc[L.VB] = st->dcgs ? 1.0 : 1.0 / beta;  // DCGS2 stores every v_i normalised
      st->g[0] = beta;
      if (st->variant == RG_AUGMENT) {
        // v_0 = r_c/beta with Q^T r_c = 0 after the cycle-start projection: G[0,:] = 0, T00 = 1.
        st->T[0][0] = 1.0;
        st->Si[0][0] = 1.0;
        for (int l = 0; l < st->k_eff; ++l) st->Gm[0][l] = 0.0;
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- CGS2 passes
// tot[0..nd) = raw dots with columns [d0, d0+nd); h_c = sc_c * dot.
__device__ __forceinline__ void epi_pass(DevState* st, const double* tot, int d0, int nd, bool first) {
  for (int c = threadIdx.x; c < nd; c += blockDim.x) {
    const double v = st->sc[d0 + c] * tot[c];
    st->coef[d0 + c] = v;
    st->hcol[d0 + c] = first ? v : st->hcol[d0 + c] + v;
  }
  __syncthreads();
}

// R_C^{-1} u for the k-vector u in shared memory -> out (shared); parallel over rows.
__device__ __forceinline__ void rcinv_apply(const DevState* st, int k, const double* u, double* out) {
  for (int l = threadIdx.x; l < k; l += blockDim.x) {
    double s = 0.0;
    for (int c = l; c < k; ++c) s += st->RCinv[c][l] * u[c];
    out[l] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- least-squares step
// After the last orthogonalisation pass of Arnoldi step j: tot[0..nd) = Q^T w (augment,
// nd = k_eff), tot[nd] = ||w||^2 of the new (un-normalised) basis vector w = raw v_{j+1}.
// Every global access is issued as a parallel batch (no serial chains of dependent loads);
// the serial Givens recurrence runs in thread 0 from shared memory.
// jx >= 0 (graph-path DCGS2 split epilogue, k_dcgs_ls): the column index is jx, its Hessenberg entries
// h_0..h_jx come from Hraw[jx] (DK1's last CTA stored them with B), and the state DK1 owns is left alone
// (the step index st->j, the column scales sc, Hraw / Bm).
__device__ __noinline__ static void epi_ls(DevState* st, const Layout& L, const double* tot, int nd, int jx = -1) {
  __shared__ double h[MAXM + 2], mc[MAXM + 2], tv[MAXM + 2], csS[MAXM], snS[MAXM];
  __shared__ double ys[MAXM + 2], gs[MAXM + 2], us[MAXK], zs[MAXK], rd[MAXM + 2];
  __shared__ int s_stop, s_jf, s_tb;
  __shared__ double s_sc[8];
  __shared__ int s_ic[8];
  const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, nw = bd >> 5;
  const bool split = jx >= 0;
  const int j = split ? jx : st->j, VB = L.VB, k = st->k_eff, var = st->variant;
  const int QB = VB - k;
  RG_CHK(st, j >= 0 && j < MAXM && j < st->m && k <= MAXK && nd <= MAXK && st->hist_cap <= (1 << 16));
  const double nrm = sqrt(tot[nd]);
  // ---- one parallel batch of loads: h column, rotations, scalars
  for (int i = tid; i <= j; i += bd) h[i] = split ? st->Hraw[j][i] : st->hcol[VB + i];
  for (int i = tid; i < j; i += bd) { csS[i] = st->cs[i]; snS[i] = st->sn[i]; }
  if (tid == 0) {
    h[j + 1] = nrm;
    s_tb = 0;
    s_stop = 0;
    s_sc[0] = st->g[j];
    s_sc[1] = st->bnorm;
    s_sc[2] = st->tol;
    s_sc[3] = st->beta;
    s_ic[0] = st->m;
    s_ic[1] = st->iters;
    s_ic[2] = st->max_iters;
    s_ic[3] = st->hist_len;
    s_ic[4] = st->hist_cap;
  }
  __syncthreads();
  if (!split) {
    for (int i = tid; i <= j + 1; i += bd) st->Hraw[j][i] = h[i];
    if (var == RG_DEFLATE)
      for (int l = tid; l < k; l += bd) st->Bm[j][l] = st->hcol[QB + l];
  }
  if (var == RG_AUGMENT)
    for (int l = tid; l < k; l += bd) st->Gm[j + 1][l] = nrm > 0.0 ? tot[l] / nrm : 0.0;
  __syncthreads();
  if (var == RG_AUGMENT && k > 0) {
    // M = I - G^T G on v_0..v_{j+1}; new column (t, tau) of its Cholesky factor T = S^{-1}:
    //   t = T_old^{-T} M[0..j, j+1] = S_old^T M[0..j, j+1],  tau^2 = M[j+1,j+1] - t.t,
    //   new column of S: -S_old t / tau, S[j+1][j+1] = 1/tau.  Warp per output, lanes over the sum.
    for (int i = tid >> 5; i <= j + 1; i += nw) {
      double sacc = 0.0;
      for (int l = lane; l < k; l += 32) sacc += st->Gm[i][l] * st->Gm[j + 1][l];
      sacc = warp_sum(sacc);
      if (lane == 0) mc[i] = ((i == j + 1) ? 1.0 : 0.0) - sacc;
    }
    __syncthreads();
    for (int i = tid >> 5; i <= j; i += nw) {  // t_i = sum_{l<=i} S(l,i) mc_l
      double sacc = 0.0;
      for (int l = lane; l <= i; l += 32) sacc += st->Si[i][l] * mc[l];
      sacc = warp_sum(sacc);
      if (lane == 0) tv[i] = sacc;
    }
    __syncthreads();
    if (tid == 0) {
      double t2 = 0.0;
      for (int i = 0; i <= j; ++i) t2 += tv[i] * tv[i];
      const double tau2 = mc[j + 1] - t2;
      // tau^2 <= 1e-14: v_{j+1} lies (numerically) in span(Q) + span(V_{j+1}) — the search space
      // span(W) + K_{j+1} already holds everything the next direction could add (k + j + 1 >= n at the
      // latest).  The column is ACCEPTED with tau = 0: the last row of M = T H-bar vanishes, the projected
      // least squares has a zero residual, and the cycle ends here (R5).  (Until the soak runs of
      // round 2 this ended the cycle at the PREVIOUS step, discarding the step that completes the solve:
      // n = 7, k = 5 took 23 iterations in 11 cycles where the explicit-space oracle takes 2.)
      s_sc[4] = tau2 > 1e-14 ? sqrt(tau2) : 0.0;
    }
    __syncthreads();
    {
      const double tau = s_sc[4];
      if (tau > 0.0) {  // S = T^{-1} is only needed by later columns of this cycle
        for (int l = tid >> 5; l <= j; l += nw) {  // S(l, j+1) = -(sum_{i>=l} S(l,i) t_i)/tau
          double sacc = 0.0;
          for (int i = l + lane; i <= j; i += 32) sacc += st->Si[i][l] * tv[i];
          sacc = warp_sum(sacc);
          if (lane == 0) st->Si[j + 1][l] = -sacc / tau;
        }
      }
      for (int i = tid; i <= j; i += bd) st->T[j + 1][i] = tv[i];
      if (tid == 0) {
        st->T[j + 1][j + 1] = tau;
        if (tau > 0.0) st->Si[j + 1][j + 1] = 1.0 / tau;
      }
      __syncthreads();
      for (int i = tid >> 5; i <= j + 1; i += nw) {  // column j of M = T H: sum_{l>=i} T(i,l) h_l
        double sacc = 0.0;
        for (int l = i + lane; l <= j + 1; l += 32) sacc += st->T[l][i] * h[l];
        sacc = warp_sum(sacc);
        if (lane == 0) mc[i] = sacc;
      }
      __syncthreads();
      for (int i = tid; i <= j + 1; i += bd) h[i] = mc[i];
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (!split) st->sc[VB + j + 1] = nrm > 0.0 ? 1.0 / nrm : 0.0;
    const double bnorm = s_sc[1], tol = s_sc[2], beta = s_sc[3];
    int iters = s_ic[1];
    int stop = 0, jf = j;
    if (!s_tb) {
      double carry = h[0];  // apply the previous rotations; the rotated entry stays in a register
#pragma unroll 4
      for (int i = 0; i < j; ++i) {
        const double b = h[i + 1], ci = csS[i], si = snS[i];
        h[i] = ci * carry + si * b;
        carry = -si * carry + ci * b;
      }
      h[j] = carry;
      if (!(hypot(h[j], h[j + 1]) > 0.0)) s_tb = 1;  // A v_j = 0 within span: no progress possible
    }
    if (s_tb) {
      stop = 1;
      jf = j - 1;
      ++iters;
    } else {
      const double a = h[j], b = h[j + 1];
      const double den = hypot(a, b);
      const double c = a / den, s = b / den;
      st->cs[j] = c;
      st->sn[j] = s;
      h[j] = den;
      const double gj = s_sc[0];
      st->g[j] = c * gj;
      st->g[j + 1] = -s * gj;
      const double res = fabs(s * gj) / bnorm;
      if (s_ic[3] < s_ic[4]) { L.hist[s_ic[3]] = res; st->hist_len = s_ic[3] + 1; }
      ++iters;
      if (!isfinite(res)) {
        st->status = RG_E_NUMERIC;
        st->done = 1;
        stop = 1;
        jf = -1;
      } else {
        stop = (res <= tol) || (nrm <= 1e-14 * beta) || (j + 1 >= s_ic[0]) || (iters >= s_ic[2]) ||
               (var == RG_AUGMENT && k > 0 && !(s_sc[4] > 0.0));  // tau = 0: nothing left to add this cycle
      }
    }
    st->iters = iters;
    if (!stop && !split) st->j = j + 1;
    s_stop = stop;
    s_jf = jf;
    if (stop) {
      st->active = 0;
      st->jfinal = jf;
      st->have_xupd = jf >= 0;
    }
  }
  __syncthreads();
  if (!s_tb) for (int i = tid; i <= j; i += bd) st->R[j][i] = h[i];  // rotated column (parallel stores)
  if (!s_stop || s_jf < 0) return;
  // ---- cycle end: y = R^{-1} g[0..jf] (R columns 0..jf-1 from global, column jf possibly fresh)
  const int jf = s_jf;
  for (int i = tid; i <= jf; i += bd) {
    gs[i] = (i == j && !s_tb) ? st->g[j] : st->g[i];
    rd[i] = (i == j && !s_tb) ? h[j] : st->R[i][i];
  }
  __syncthreads();
  for (int i = jf; i >= 0; --i) {
    if (tid == 0) ys[i] = gs[i] / rd[i];
    __syncthreads();
    for (int l = tid; l < i; l += bd) gs[l] -= ((i == j && !s_tb) ? h[l] : st->R[i][l]) * ys[i];
    __syncthreads();
  }
  for (int i = tid; i <= jf; i += bd) st->coefx[VB + i] = -ys[i];  // x += V y
  if (k > 0 && (var == RG_DEFLATE || var == RG_AUGMENT)) {
    if (var == RG_DEFLATE) {  // x -= W R_C^{-1} B y
      for (int l = tid >> 5; l < k; l += nw) {
        double sacc = 0.0;
        for (int i = lane; i <= jf; i += 32) sacc += st->Bm[i][l] * ys[i];
        sacc = warp_sum(sacc);
        if (lane == 0) us[l] = sacc;
      }
    } else {  // augment: x -= W R_C^{-1} G Hbar y
      for (int i = tid >> 5; i <= jf + 1; i += nw) {
        double sacc = 0.0;
        for (int c = (i > 0 ? i - 1 : 0) + lane; c <= jf; c += 32) sacc += st->Hraw[c][i] * ys[c];  // Hessenberg
        sacc = warp_sum(sacc);
        if (lane == 0) mc[i] = sacc;
      }
      __syncthreads();
      for (int l = tid >> 5; l < k; l += nw) {
        double sacc = 0.0;
        for (int i = lane; i <= jf + 1; i += 32) sacc += st->Gm[i][l] * mc[i];
        sacc = warp_sum(sacc);
        if (lane == 0) us[l] = sacc;
      }
    }
    __syncthreads();
    rcinv_apply(st, k, us, zs);
    for (int l = tid; l < k; l += bd) st->coefx[l] = zs[l];  // x -= coefx_l W_l
  }
  __syncthreads();
}

// ---------------------------------------------------------------- cycle-start projection
// tot[0..k) = Q^T r_c.  Sets the r update (r -= Q a) and the x update (x += W R_C^{-1} a).
__device__ __forceinline__ void epi_cs_dq(DevState* st, const Layout& L, const double* tot) {
  __shared__ double us[MAXK], zs[MAXK];
  const int k = st->k_eff, QB = L.VB - k;
  for (int l = threadIdx.x; l < k; l += blockDim.x) {
    us[l] = tot[l];
    st->coef[QB + l] = tot[l];
  }
  __syncthreads();
  rcinv_apply(st, k, us, zs);
  for (int l = threadIdx.x; l < k; l += blockDim.x) st->coefx[l] = -zs[l];
  __syncthreads();
}

// ---------------------------------------------------------------- oblique projection
// tot[0..k) = W^T w.  t = E^{-1} W^T w -> coef[k + l] (the update w -= C t, C in columns [k, 2k));
// at the cycle start also coefx[l] = -t_l (OP_XW: x += W t, the Galerkin start of PAPER.md:289).
// Orthogonal variant, Arnoldi step: t = W^T w -> coef[l] (w -= W t: the projector I - W W^T).
__device__ __forceinline__ void epi_ob(DevState* st, const double* tot, bool cycle_start) {
  const int k = st->k_eff;
  const bool orth = !cycle_start && st->variant == RG_ORTHOGONAL;
  const int pb = orth ? 0 : k;
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    double t = 0.0;
    if (orth) {
      t = tot[a];
    } else {
      for (int b = 0; b < k; ++b) t += st->Einv[b][a] * tot[b];
    }
    st->coef[pb + a] = t;
    if (cycle_start) st->coefx[a] = -t;
  }
  __syncthreads();
}

}  // namespace rg

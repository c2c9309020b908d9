// orth.cu — fused block-vector kernels of the Arnoldi step and the cycle boundaries (K5/K6/K8/K13).
//
// One kernel family covers every tall-skinny operation of the hot path:
//   target w (an n-vector) is optionally UPDATED  w -= sum_{c in U} cf_c Z_c      (Z_c one read each)
//   then optionally DOTTED                           d_c = Z_c . w,  c in D       (same sweep)
//   and/or NORMED                                    ||w||^2
// with a deterministic grid reduction whose last CTA runs the epilogue (epilogue.cuh).  The
// CGS2 step of PAPER.md's GMRES (classical Gram-Schmidt with one re-orthogonalisation, the
// "Arnoldi orthogonalization" of PAPER.md:705-711) is then three launches:
//   OP_D1   h1 = [Q|V]^T w                         (deflate orthogonalises against Q too)
//   OP_UD2  w -= [Q|V] h1 ; h2 = [Q|V]^T w         (update fused with the second pass' dots)
//   OP_UN   w -= [Q|V] h2 ; ||w||  (+ Q^T w for augment) -> least-squares epilogue
// Cycle start (recycled variants): OP_CS_DQ a = Q^T r ; OP_XW x += W R_C^{-1} a ;
// OP_CS_UN r -= Q a, ||r|| -> cycle-start epilogue.  Cycle end: OP_XUPD x += V y + W z.
// OP_NORMB: ||b||.
// Oblique variant (M_D = I - C E^{-1} W^T): OP_OB_CSD / OP_OB_SD t = E^{-1} W^T w,
// OP_OB_CSU / OP_OB_SU w -= C t (+ ||w|| -> cycle-start epilogue at the cycle start).
#define RG_FILE_ID 3  // RG_CHK locations (checked builds)
#include "epilogue.cuh"
#include "kernels.cuh"
#include "knobs.cuh"

namespace rg {
namespace {

struct OrthArgs {
  Layout L;
  DevState* st;
  int op;
  unsigned long long cond;  // cudaGraphConditionalHandle of the Arnoldi-step WHILE node (OP_UN)
  int use_cond;
};

// Sets a WHILE-node condition from the device state: which = 0 -> st->active (Arnoldi loop),
// which = 1 -> !st->done (restart-cycle loop).
__global__ void k_cond(DevState* st, cudaGraphConditionalHandle h, int which) {
  if (threadIdx.x == 0) {
    cudaGraphSetConditional(h, which == 0 ? (st->active ? 1u : 0u) : (st->done ? 0u : 1u));
    if (st->profile) st->kstat[K_COND].launches++;
  }
}

__global__ void __launch_bounds__(OT, 2) k_orth(OrthArgs a) {
  __shared__ double cf[MAXCOL];
  __shared__ double ws[OT];
  __shared__ double dpart[MAXRED];
  __shared__ double tot[MAXRED];
  __shared__ double bsh[33];
  DevState* st = a.st;
  const Layout& L = a.L;
  const int op = a.op;
  static constexpr int kids[13] = {K_ORTH_D1, K_ORTH_UD2, K_ORTH_UN, K_CS_DQ, K_CS_UN, K_XW, K_XUPD, K_NORMB,
                                   K_OBD, K_OBU, K_OBD, K_OBU, K_XUPD};
  const int kid = kids[op];
  bool go;
  switch (op) {
    case OP_D1: case OP_UD2: case OP_UN: case OP_OB_SD: case OP_OB_SU: go = st->active != 0; break;
    case OP_CS_DQ: case OP_CS_UN: case OP_XW: case OP_OB_CSD: case OP_OB_CSU: go = st->done == 0; break;
    case OP_XUPD: case OP_VY: go = st->have_xupd != 0; break;
    default: go = true;
  }
  if (!go) { prof_noop(st, kid); return; }
  prof_begin(st, kid);

  const int j = st->j, k = st->k_eff, var = st->variant;
  const int VB = L.VB, QB = VB - k;
  const int64_t ld = L.ld;
  double* w = nullptr;
  const double* csrc = st->coef;
  int u0 = 0, u1 = 0, u2 = 0, u3 = 0, d0 = 0, d1 = 0;
  bool nrmflag = false;
  const int lo = (var == RG_DEFLATE) ? QB : VB;
  switch (op) {
    case OP_D1:
      w = L.Z + (int64_t)(VB + j + 1) * ld; d0 = lo; d1 = VB + j + 1; break;
    case OP_UD2:
      w = L.Z + (int64_t)(VB + j + 1) * ld; u0 = lo; u1 = VB + j + 1; d0 = lo; d1 = VB + j + 1; break;
    case OP_UN:
      w = L.Z + (int64_t)(VB + j + 1) * ld; u0 = lo; u1 = VB + j + 1; nrmflag = true;
      if (var == RG_AUGMENT) { d0 = QB; d1 = VB; }
      break;
    case OP_CS_DQ: w = L.Z + (int64_t)VB * ld; d0 = QB; d1 = VB; break;
    case OP_CS_UN: w = L.Z + (int64_t)VB * ld; u0 = QB; u1 = VB; nrmflag = true; break;
    case OP_XW: w = L.x; csrc = st->coefx; u0 = 0; u1 = k; break;
    case OP_XUPD:  // x += V y (+ W part); preconditioned: x += pz (= M^{-1} V y, OP_VY + SSOR) + W part
      w = L.x; csrc = st->coefx;
      if (!L.prec) { u0 = VB; u1 = VB + st->jfinal + 1; }
      if (var == RG_AUGMENT || var == RG_DEFLATE) { u2 = 0; u3 = k; }
      break;
    case OP_VY: w = L.pt; csrc = st->coefx; u0 = VB; u1 = VB + st->jfinal + 1; break;
    case OP_OB_CSD: w = L.Z + (int64_t)VB * ld; d0 = 0; d1 = k; break;
    case OP_OB_CSU: w = L.Z + (int64_t)VB * ld; u0 = k; u1 = 2 * k; nrmflag = true; break;
    case OP_OB_SD: w = L.Z + (int64_t)(VB + j + 1) * ld; d0 = 0; d1 = k; break;
    case OP_OB_SU: w = L.Z + (int64_t)(VB + j + 1) * ld; u0 = proj_base(var, k); u1 = u0 + k; break;
    default: w = const_cast<double*>(L.b); nrmflag = true; break;  // OP_NORMB (read only)
  }
  RG_CHK(st, u0 >= 0 && u1 <= L.ncol && u2 >= 0 && u3 <= L.ncol && d0 >= 0 && d1 <= L.ncol && d1 - d0 < MAXRED &&
                 u1 <= MAXCOL && u3 <= MAXCOL);
  const bool upd = (u1 > u0) || (u3 > u2) || (op == OP_XUPD && L.prec) || op == OP_VY;
  const bool dots = d1 > d0;
  const int nd = d1 - d0;
  for (int c = u0 + threadIdx.x; c < u1; c += OT) cf[c] = csrc[c] * st->sc[c];
  for (int c = u2 + threadIdx.x; c < u3; c += OT) cf[c] = csrc[c] * st->sc[c];
  for (int c = threadIdx.x; c <= nd; c += OT) dpart[c] = 0.0;
  __syncthreads();

  // even split of the n_pad rows over the CTAs, in 32-row granules
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const double* __restrict__ Z = L.Z;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double nrm = 0.0;
  for (int64_t base = r0; base < r1; base += OT) {
    const int64_t r = base + threadIdx.x;
    const bool in = r < r1;
    double acc = 0.0;
    if (in) {
      acc = op == OP_VY ? 0.0 : w[r];
      if (op == OP_XUPD && L.prec) acc += L.pz[r];
      if (upd) {
        int c = u0;
        for (; c + 8 <= u1; c += 8) {   // 8 independent loads in flight, applied in order
          double z[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) z[u] = __ldcs(Z + (int64_t)(c + u) * ld + r);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc -= cf[c + u] * z[u];
        }
        for (; c < u1; ++c) acc -= cf[c] * __ldcs(Z + (int64_t)c * ld + r);
        for (int c = u2; c < u3; ++c) acc -= cf[c] * __ldcs(Z + (int64_t)c * ld + r);
        w[r] = acc;
      }
      nrm += acc * acc;
    }
    if (dots) {
      ws[threadIdx.x] = acc;
      __syncthreads();
      const int cnt = (int)((r1 - base) < OT ? (r1 - base) : OT);
      // each warp owns columns c = d0 + wid (mod NWARP): 16 independent 8-byte loads in flight
      // per lane (OT/32 rows per lane), then a fixed shuffle tree
      constexpr int RPL = OT / 32;
      for (int c = d0 + wid; c < d1; c += NWARP) {
        const double* __restrict__ za = Z + (int64_t)c * ld + base + lane;
        double va[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) va[q] = (lane + 32 * q < cnt) ? __ldcs(za + 32 * q) : 0.0;
        double sa = 0.0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) sa += va[q] * ws[lane + 32 * q];
        sa = warp_sum(sa);
        if (lane == 0) dpart[c - d0] += sa;
      }
      __syncthreads();
    }
  }
  if (!dots && !nrmflag) {
    if (st->profile && grid_last(L.counter) && threadIdx.x == 0)
      prof_end(st, kid, 8.0 * (double)L.n * ((u1 - u0) + (u3 - u2) + 2));
    return;
  }
  if (nrmflag) {
    const double t = block_sum(nrm, bsh);
    if (threadIdx.x == 0) dpart[nd] = t;
  }
  __syncthreads();
  const int nv = nd + (nrmflag ? 1 : 0);
  if (!grid_reduce(dpart, nv, L.partial, L.counter, tot, tot)) return;

  switch (op) {
    case OP_D1: epi_pass(st, tot, d0, nd, true); break;
    case OP_UD2: epi_pass(st, tot, d0, nd, false); break;
    case OP_UN:
      epi_ls(st, L, tot, nd);
      if (a.use_cond && threadIdx.x == 0) cudaGraphSetConditional(a.cond, st->active ? 1u : 0u);
      break;
    case OP_CS_DQ: epi_cs_dq(st, L, tot); break;
    case OP_CS_UN: case OP_OB_CSU: epi_cycle_start(st, L, tot[0]); break;
    case OP_OB_CSD: epi_ob(st, tot, true); break;
    case OP_OB_SD: epi_ob(st, tot, false); break;
    default:
      if (threadIdx.x == 0) {  // OP_NORMB
        st->bnorm = sqrt(tot[0]);
        if (!(st->bnorm > 0.0)) {
          st->bzero = st->bnorm == 0.0;
          st->done = 1;
          st->converged = st->bzero;
          if (!st->bzero) st->status = RG_E_NUMERIC;
        }
      }
  }
  if (threadIdx.x == 0) {
    // algorithmic bytes = every DISTINCT column touched once + w read (+ write if updated)
    int distinct = (u1 - u0) + (u3 - u2);
    if (dots) {
      const int lo_o = d0 > u0 ? d0 : u0, hi_o = d1 < u1 ? d1 : u1;
      distinct += nd - (hi_o > lo_o ? hi_o - lo_o : 0);
    }
    prof_end(st, kid, 8.0 * (double)L.n * (distinct + (upd ? 2.0 : 1.0)));
  }
}

// ------------------------------------------------------------------------------------------
// Register-resident CGS kernel for the Arnoldi step (OP_D1 / OP_UD2 / OP_UN non-augment).
//
// The p columns of [Q|V] are split into G <= 16 chunks of <= 8 columns; thread t owns row
// t % TR (TR = 512/G rows per tile) and chunk t / TR.  Per tile a thread loads its <= 8 basis
// values and the target entry (all loads independent), keeps them in registers for BOTH the
// update w_r -= sum_c cf_c Z_rc (chunk partials combined in a fixed order through shared memory)
// and the dots d_c += Z_rc w_r (accumulated per thread across all tiles; one deterministic
// shuffle/shared-memory tree at the end).  Every column is read from HBM once per launch; there
// is no per-tile reduction and at most two barriers per tile (none when G == 1).
constexpr int CT = 512;
constexpr int CPG = 8;  // columns per thread chunk

template <int OPK>  // 0 = D1 (dots), 1 = UD2 (update + dots), 2 = UN (update + norm -> LS step)
__global__ void __launch_bounds__(CT, 2) k_cgs(Layout L, DevState* st, unsigned long long cond) {
  __shared__ double cf[MAXCOL];
  __shared__ double part[CT];
  __shared__ double ws[CT];
  __shared__ double wred[CT / 32][CPG];
  __shared__ double dpart[MAXRED];
  __shared__ double tot[MAXRED];
  __shared__ double bsh[33];
  constexpr int kid = OPK == 0 ? K_ORTH_D1 : OPK == 1 ? K_ORTH_UD2 : K_ORTH_UN;
  constexpr bool UPD = OPK != 0, DOTS = OPK != 2, NRM = OPK == 2;
  if (!st->active) { prof_noop(st, kid); return; }
  prof_begin(st, kid);
  const int j = st->j, k = st->k_eff, var = st->variant;
  const int VB = L.VB, QB = VB - k;
  const int64_t ld = L.ld;
  const int lo = (var == RG_DEFLATE) ? QB : VB, hi = VB + j + 1, p = hi - lo;
  double* __restrict__ w = L.Z + (int64_t)hi * ld;
  const double* __restrict__ Z = L.Z;
  int G = 1;
  while (G * CPG < p) G <<= 1;
  const int TR = CT / G;
  const int r = threadIdx.x % TR, g = threadIdx.x / TR;
  const int ca = g * CPG, nc = max(0, min(CPG, p - ca));   // my columns: lo + ca .. lo + ca + nc
  if (UPD)
    for (int c = threadIdx.x; c < p; c += CT) cf[c] = st->coef[lo + c] * st->sc[lo + c];
  __syncthreads();
  double cfr[CPG];
#pragma unroll
  for (int i = 0; i < CPG; ++i) cfr[i] = (UPD && i < nc) ? cf[ca + i] : 0.0;
  const double* __restrict__ zb = Z + (int64_t)(lo + ca) * ld;
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  double dacc[CPG];
#pragma unroll
  for (int i = 0; i < CPG; ++i) dacc[i] = 0.0;
  double nrm = 0.0;
  for (int64_t base = r0; base < r1; base += TR) {
    const int64_t row = base + r;
    const bool in = row < r1;
    double z[CPG];
#pragma unroll
    for (int i = 0; i < CPG; ++i) z[i] = (in && i < nc) ? __ldcs(zb + (int64_t)i * ld + row) : 0.0;
    const double wr = (in && (OPK == 0 || g == 0)) ? w[row] : 0.0;
    double wn = wr;
    if (UPD) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < CPG; i += 2) {
        a0 += cfr[i] * z[i];
        a1 += cfr[i + 1] * z[i + 1];
      }
      const double pa = a0 + a1;
      if (G == 1) {
        wn = wr - pa;
      } else {
        part[threadIdx.x] = pa;
        __syncthreads();
        if (g == 0) {
          double sum = pa;
          for (int gg = 1; gg < G; ++gg) sum += part[gg * TR + r];
          wn = wr - sum;
          ws[r] = wn;
        }
        __syncthreads();
        if (g != 0) wn = ws[r];
      }
      if (g == 0 && in) {
        w[row] = wn;
        if (NRM) nrm += wn * wn;
      }
    }
    if (DOTS) {
#pragma unroll
      for (int i = 0; i < CPG; ++i) dacc[i] += z[i] * wn;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (DOTS) {
#pragma unroll
    for (int i = 0; i < CPG; ++i) {
      const double v = warp_sum(dacc[i]);
      if (lane == 0) wred[wid][i] = v;
    }
    __syncthreads();
    const int wpg = TR / 32;  // warps per chunk group
    for (int c = threadIdx.x; c < p; c += CT) {
      const int gg = c / CPG, i = c % CPG;
      double sum = 0.0;
      for (int ww = 0; ww < wpg; ++ww) sum += wred[gg * wpg + ww][i];
      dpart[c] = sum;
    }
  }
  if (NRM) {
    const double tn = block_sum(nrm, bsh);
    if (threadIdx.x == 0) dpart[0] = tn;
  }
  __syncthreads();
  const int nv = DOTS ? p : 1;
  if (!grid_reduce(dpart, nv, L.partial, L.counter, tot, tot)) return;
  if (OPK == 0) epi_pass(st, tot, lo, p, true);
  else if (OPK == 1) epi_pass(st, tot, lo, p, false);
  else {
    epi_ls(st, L, tot, 0);
    if (cond && threadIdx.x == 0) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, st->active ? 1u : 0u);
  }
  if (threadIdx.x == 0) prof_end(st, kid, 8.0 * (double)L.n * (p + (UPD ? 2.0 : 1.0)));
}

// ------------------------------------------------------------------------------------------
// TMA-staged CGS passes of the graph path (round 2): OP_D1 / OP_UD2 / OP_UN (not augment) and the
// cycle-start OP_CS_DQ / OP_CS_UN.  The register kernels above keep <= 8 loads of 8 B in flight per
// thread and measured 3.4-4.5 TB/s on C5's 2M-row basis.  Here a producer warp streams, per tile of
// TR rows, the target w and every column of the pass ([Q|V] rows) with cp.async.bulk into a ring of
// CG_NS whole-tile stages (completion on mbarriers), so ~190 KB per SM are in flight independently of
// registers.  Consumer thread (r, g) (r < TR rows, g < G = 512/TR groups) owns columns g, g+G, ...:
//   update: part_g[r] = sum over its columns of cf_c Z_rc; w_r' = w_r - sum_g part_g[r] (groups in order)
//   dots:   d_c += Z_rc w_r' per thread over all tiles, then warp shuffles and the warps in order
//   norm:   ||w'||^2 (group 0)
// TR is picked per launch on the device from the pass width p: the largest power of two <= 512 with
// CG_NS tiles of p + 1 columns in the ring and at most CG_CPT columns per thread.  Deterministic.
constexpr int CG_NS = 3;
constexpr int CG_CPT = 16;                        // dot accumulators per thread
constexpr int CG_SMEM = 192 * 1024;               // ring bytes (dynamic shared memory)
__device__ __forceinline__ uint32_t cg_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cg_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(cg_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cg_bar_consumers() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

template <int MODE>  // 0 = dots (D1, CS_DQ), 1 = update + dots (UD2), 2 = update + norm (UN, CS_UN)
__global__ void __launch_bounds__(544, 1) k_cgs_tma(Layout L, DevState* st, int op, unsigned long long cond) {
  extern __shared__ __align__(128) double ring[];  // [CG_NS][p + 1][TR]; partials alias it at the end
  __shared__ __align__(8) uint64_t full[CG_NS], empty[CG_NS];
  __shared__ double cf[MAXCOL];
  __shared__ double part[2][512];
  __shared__ double dpart[MAXRED];
  __shared__ double tot[MAXRED];
  __shared__ double bsh[33];
  constexpr bool UPD = MODE != 0, DOTS = MODE != 2, NRM = MODE == 2;
  pdl_wait();  // launched with PDL behind the previous kernel of the Arnoldi step: everything below reads its output
  const int kid = op == OP_D1 ? K_ORTH_D1 : op == OP_UD2 ? K_ORTH_UD2 : op == OP_UN ? K_ORTH_UN
                : op == OP_CS_DQ ? K_CS_DQ : K_CS_UN;
  const bool cs = op == OP_CS_DQ || op == OP_CS_UN;
  if (cs ? st->done != 0 : st->active == 0) { prof_noop(st, kid); return; }
  prof_begin(st, kid);
  const int j = st->j, k = st->k_eff, var = st->variant;
  const int VB = L.VB, QB = VB - k;
  const int64_t ld = L.ld;
  // pass columns [c0, c0 + p) and the target column tc
  int c0, p, tc;
  if (cs) { c0 = QB; p = k; tc = VB; }
  else { c0 = (var == RG_DEFLATE) ? QB : VB; tc = VB + j + 1; p = tc - c0; }
  double* __restrict__ w = L.Z + (int64_t)tc * ld;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (UPD)
    for (int c = tid; c < p; c += 544) cf[c] = st->coef[c0 + c] * st->sc[c0 + c];
  // rows per tile
  int TR = 512;
  while (TR > 32 && ((size_t)CG_NS * (p + 1) * TR * 8 > (size_t)CG_SMEM || (p + (512 / TR) - 1) / (512 / TR) > CG_CPT)) TR >>= 1;
  const int G = 512 / TR, SD = (p + 1) * TR;  // doubles per stage: p columns then w
  RG_CHK(st, c0 >= 0 && p >= 0 && c0 + p <= tc && tc < L.ncol && p < MAXRED && p <= MAXCOL &&
                 (size_t)CG_NS * SD * 8 <= (size_t)CG_SMEM && (p + G - 1) / G <= CG_CPT && 16 * p <= CG_NS * SD);
  if (tid == 0) {
    for (int i = 0; i < CG_NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cg_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cg_u32(&empty[i])), "r"(16));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const int ntile = (int)((r1 - r0 + TR - 1) / TR);
  double dacc[CG_CPT];
#pragma unroll
  for (int i = 0; i < CG_CPT; ++i) dacc[i] = 0.0;
  double nrm = 0.0;
  const int r = tid % TR, g = tid / TR;
  if (wid == 16) {  // ---- producer warp: lane c issues the copies of columns c, c + 32, ... of a tile (one lane
                    // issuing all p + 1 copies serially was slower than the tile streams, cf. dcgs.cu ts_issue)
    uint64_t pol, keep;
    if (L.keep_l2) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
    for (int t = 0; t < ntile; ++t) {
      const int s = t % CG_NS;
      if (t >= CG_NS) cg_wait(&empty[s], (uint32_t)((t / CG_NS - 1) & 1));
      const int64_t base = r0 + (int64_t)t * TR;
      const uint32_t cnt = (uint32_t)min((int64_t)TR, r1 - base);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cg_u32(&full[s])),
                     "r"((uint32_t)(p + 1) * cnt * 8u) : "memory");
      __syncwarp();
      double* stg = ring + (size_t)s * SD;
      for (int c = lane; c <= p; c += 32) {
        const double* src = c < p ? L.Z + (int64_t)(c0 + c) * ld + base : w + base;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(cg_u32(stg + (size_t)c * TR)), "l"(src), "r"(cnt * 8u), "r"(cg_u32(&full[s])),
                     "l"(c < p ? pol : keep) : "memory");
      }
    }
  } else {  // ---- consumers
    for (int t = 0; t < ntile; ++t) {
      const int s = t % CG_NS;
      const int64_t base = r0 + (int64_t)t * TR;
      const int cnt = (int)min((int64_t)TR, r1 - base);
      const bool in = r < cnt;
      cg_wait(&full[s], (uint32_t)((t / CG_NS) & 1));
      const double* stg = ring + (size_t)s * SD;
      const double wr = in ? stg[(size_t)p * TR + r] : 0.0;
      double wn = wr;
      if (UPD) {
        double a0 = 0.0;
#pragma unroll
        for (int i = 0; i < CG_CPT; ++i) {
          const int c = g + i * G;
          if (c < p) a0 += cf[c] * (in ? stg[(size_t)c * TR + r] : 0.0);
        }
        if (G == 1) {
          wn = wr - a0;
        } else {
          double* pp = part[t & 1];
          pp[g * TR + r] = a0;
          cg_bar_consumers();
          double sum = 0.0;
          for (int gg = 0; gg < G; ++gg) sum += pp[gg * TR + r];
          wn = wr - sum;
        }
        if (g == 0 && in) {
          w[base + r] = wn;
          if (NRM) nrm += wn * wn;
        }
      }
      if (DOTS) {
#pragma unroll
        for (int i = 0; i < CG_CPT; ++i) {
          const int c = g + i * G;
          if (c < p && in) dacc[i] += stg[(size_t)c * TR + r] * wn;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cg_u32(&empty[s])) : "memory");
    }
  }
  pdl_trigger();
  __syncthreads();  // all stages consumed: the ring is free for the per-warp partials
  double* wsm = ring;  // [16][p]
  if (DOTS) {
    if (wid < 16) {
      // a warp = 32 consecutive rows of one group (TR >= 32): its columns are g + i G
#pragma unroll
      for (int i = 0; i < CG_CPT; ++i) {
        const int c = g + i * G;
        if (c < p) {
          const double v = warp_sum(dacc[i]);
          if (lane == 0) wsm[wid * p + c] = v;
        }
      }
    }
    __syncthreads();
    const int wpg = TR / 32;  // warps per group
    for (int c = tid; c < p; c += 544) {
      const int gg = c % G;
      double sum = 0.0;
      for (int ww = 0; ww < wpg; ++ww) sum += wsm[(gg * wpg + ww) * p + c];
      dpart[c] = sum;
    }
  }
  if (NRM) {
    const double tn = block_sum(nrm, bsh);  // (producer warp contributes 0)
    if (tid == 0) dpart[0] = tn;
  }
  __syncthreads();
  const int nv = DOTS ? p : 1;
  if (!grid_reduce(dpart, nv, L.partial, L.counter, tot, tot)) return;
  switch (op) {
    case OP_D1: epi_pass(st, tot, c0, p, true); break;
    case OP_UD2: epi_pass(st, tot, c0, p, false); break;
    case OP_UN:
      epi_ls(st, L, tot, 0);
      if (cond && tid == 0) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, st->active ? 1u : 0u);
      break;
    case OP_CS_DQ: epi_cs_dq(st, L, tot); break;
    default: epi_cycle_start(st, L, tot[0]); break;  // OP_CS_UN
  }
  if (tid == 0) prof_end(st, kid, 8.0 * (double)L.n * (p + (UPD ? 2.0 : 1.0)));
}

// RG_FLAG_KEEP_BASIS, cycle end: v_0 .. v_jfinal (normalised: v_i = sc_i * raw_i) into L.keepV, the
// step count into st->kb_steps.  H-bar and B of the cycle stay in st->Hraw / st->Bm (epi_ls).
__global__ void __launch_bounds__(OT) k_keep_basis(Layout L, DevState* st) {
  if (!st->have_xupd) return;
  const int J = st->jfinal + 1;
  const int64_t ld = L.ld;
  for (int i = 0; i < J; ++i) {
    const double s = st->sc[L.VB + i];
    const double* src = L.Z + (int64_t)(L.VB + i) * ld;
    double* dst = L.keepV + (int64_t)i * ld;
    for (int64_t r = (int64_t)blockIdx.x * OT + threadIdx.x; r < ld; r += (int64_t)gridDim.x * OT) dst[r] = s * src[r];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->kb_steps = J;
}

}  // namespace

cudaError_t launch_keep_basis(const Layout& L, DevState* st, cudaStream_t s) {
  k_keep_basis<<<vec_grid(L.ld), OT, 0, s>>>(L, st);
  return cudaGetLastError();
}

cudaError_t launch_cond(const DevState* st, unsigned long long h, int which, cudaStream_t s) {
  k_cond<<<1, 32, 0, s>>>(const_cast<DevState*>(st), (cudaGraphConditionalHandle)h, which);
  return cudaGetLastError();
}

cudaError_t launch_orth(const Layout& L, DevState* st, int op, cudaStream_t s, unsigned long long cond) {
  static PerDevice init_once;
  if (init_once.first()) {  // two 512-thread CTAs per SM need more than the default shared-memory carveout
    cudaFuncSetAttribute(k_orth, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_cgs<0>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_cgs<1>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_cgs<2>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  }
  // TMA-staged passes (graph path; augment's OP_UN also needs Q^T w: generic path)
  static const bool no_tma = knob("RG_NO_TMA_CGS");
  const bool tma_op = op == OP_D1 || op == OP_UD2 || (op == OP_UN && !L.augment) || op == OP_CS_DQ || op == OP_CS_UN;
  if (tma_op && !no_tma && L.ld >= (int64_t)NSM * 512) {
    static bool attr[MAXDEV] = {};
    const int dev = current_device();
    if (!attr[dev]) {
      cudaFuncSetAttribute(k_cgs_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, CG_SMEM);
      cudaFuncSetAttribute(k_cgs_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CG_SMEM);
      cudaFuncSetAttribute(k_cgs_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, CG_SMEM);
      attr[dev] = true;
    }
    const int mode = (op == OP_D1 || op == OP_CS_DQ) ? 0 : op == OP_UD2 ? 1 : 2;
    // PDL inside the Arnoldi step (behind the SpMV / the previous pass); the cycle-start passes follow
    // kernels that do not trigger early
    static const bool no_pdl = knob("RG_NO_PDL");
    const bool pdl = !no_pdl && (op == OP_D1 || op == OP_UD2 || op == OP_UN);
    if (mode == 0) return launch_ex(k_cgs_tma<0>, dim3(NSM), dim3(544), CG_SMEM, s, pdl, L, st, op, cond);
    if (mode == 1) return launch_ex(k_cgs_tma<1>, dim3(NSM), dim3(544), CG_SMEM, s, pdl, L, st, op, cond);
    return launch_ex(k_cgs_tma<2>, dim3(NSM), dim3(544), CG_SMEM, s, pdl, L, st, op, cond);
  }
  if (L.cgs_ok) {  // register-resident CGS kernels (augment's OP_UN also needs Q^T w: generic path)
    const int g = vec_grid(L.ld);
    // measured on B200 (C2, C4): k_cgs wins for the fused update+dots pass; the row-parallel
    // generic kernel is faster for the dots-only and update+norm passes
    if (op == OP_UD2) { k_cgs<1><<<g, CT, 0, s>>>(L, st, 0ull); return cudaGetLastError(); }
  }
  k_orth<<<vec_grid(L.ld), OT, 0, s>>>(OrthArgs{L, st, op, cond, cond != 0ull});
  return cudaGetLastError();
}

}  // namespace rg

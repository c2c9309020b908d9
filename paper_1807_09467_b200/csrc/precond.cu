// precond.cu — multicolour SSOR(omega) preconditioner (K14).
//
// The paper preconditions every run with SSOR.  Lexicographic SSOR is a chain of
// n dependent row solves; on the GPU the rows are processed in a MULTICOLOUR order instead: rows
// of one colour are never coupled (a valid colouring of the symmetrised pattern), so every row of
// a colour is updated in parallel.  SSOR in that order is exactly the textbook SSOR of the
// permuted matrix (R18):
//     M = (D + wL) D^{-1} (D + wU) / (w(2-w)),     L / U = couplings to earlier / later colours,
//     M^{-1} z:  forward   w_r = (w(2-w) z_r - w sum_{col(j) < col(r)} a_rj w_j) / a_rr
//                backward  t_r = w_r - (w / a_rr) sum_{col(j) > col(r)} a_rj t_j   (in place)
// one launch per colour and direction; the backward sweep of the last colour is the identity.
// It is applied as a RIGHT preconditioner: the Arnoldi SpMV becomes y = A M^{-1} u and the cycle
// end adds M^{-1} (V y) — GMRES keeps minimising the TRUE residual.
#define RG_FILE_ID 5  // RG_CHK locations (checked builds)
#include "kernels.cuh"

#include <algorithm>

namespace rg {
namespace {

constexpr int ST = 256;

struct SsorArgs {
  PrecDev P;
  int64_t c0, c1;        // this launch's range in perm
  int backward;
  int fuse0;             // forward launch over colours 0 AND 1: colour-0 values formed on the fly
  const double* in;      // forward input (nullptr: the Arnoldi vector u of the device state)
  double* out;           // w (forward) / t (backward, in place)
  int gate;              // 0 always, 1 Arnoldi step (st->active ...), 2 cycle end (st->have_xupd)
  int first;             // first sweep of an application (profiling start)
  int last;              // last sweep of an application (closes the K_SSOR interval)
  int nsweeps;           // kernel launches of the application
  Layout L;
  DevState* st;
  double bytes;
};

// One sweep = one launch, thread per row of the colour(s).  Round 2: (1) the forward sweeps of colours
// 0 and 1 are ONE launch: a colour-0 row has no lower-coloured coupling, so its forward value is the
// diagonal scale w_j = w(2-w) z_j / a_jj, which a colour-1 row forms on the fly from z instead of
// reading it back; the 1/a_jj factor is folded into the colour-1 rows' coupling values when the values
// are gathered (Lv1 = a_rj / a_jj: one gather per coupling, not two; rounding-level difference from
// the two-launch sequence); (2) every sweep after the first is launched with
// PDL and loads its row's matrix entries (constant data) before griddepcontrol.wait, so the launch ramp
// and the entry loads overlap the previous sweep's tail; (3) the last sweep closes the profiling
// interval (there was a 1-thread kernel for that).  2-colour patterns (5- / 7-point): 4 launches -> 2.
__global__ void __launch_bounds__(ST) k_ssor(SsorArgs a) {
  pdl_trigger();
  DevState* st = a.st;
  double xs = 1.0;
  const double* in = a.in;
  bool noop = false;
  // (device state read before pdl_wait: written before the application's first sweep, which is a
  // normal launch)
  if (a.gate == 1) {
    const int j = st->j;
    noop = !st->active || (st->dcgs && j >= st->m);
    if (!noop && !a.backward) {
      in = a.L.Z + (int64_t)(a.L.VB + j) * a.L.ld;
      xs = st->dcgs ? 1.0 : st->sc[a.L.VB + j];  // CGS2 path: V stored un-normalised
    }
  } else if (a.gate == 2) {
    noop = !st->have_xupd;
  }
  if (noop) {
    if (a.last && st->profile && blockIdx.x == 0 && threadIdx.x == 0) st->kstat[K_SSORK].launches += a.nsweeps;
    prof_noop(st, K_SSOR);
    return;
  }
  if (a.first && blockIdx.x == 0 && threadIdx.x == 0) prof_begin(st, K_SSOR);
  const PrecDev& P = a.P;
  const int64_t idx = a.c0 + (int64_t)blockIdx.x * ST + threadIdx.x;
  if (idx < a.c1) {
    const int32_t r = __ldg(P.perm + idx);
    const int32_t* __restrict__ rp = a.backward ? P.Urp : P.Lrp;
    const int32_t* __restrict__ ci = a.backward ? P.Uci : P.Lci;
    // fused launch: the colour-1 rows' couplings pre-multiplied by the column's 1/a_jj (Lv1, offset l1base)
    const double* __restrict__ vv = a.backward ? P.Uv : (a.fuse0 ? P.Lv1 - P.l1base : P.Lv);
    const int32_t p0 = __ldg(rp + idx), p1 = __ldg(rp + idx + 1);
    RG_CHK(st, r >= 0 && r < a.L.n && p0 <= p1 && p1 <= (a.backward ? P.nU : P.nL));
    const double om = P.omega, di = __ldg(P.dinv + idx);
    const double cf = xs * om * (2.0 - om);
    int32_t cc[8];
    double va[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = p0 + u < p1;
      cc[u] = ok ? __ldcs(ci + p0 + u) : r;
      va[u] = ok ? __ldcs(vv + p0 + u) : 0.0;
    }
    pdl_wait();  // out[] of the earlier sweeps
    double s = 0.0;
    for (int32_t p = p0;;) {
      if (a.fuse0) {
        double zz[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) zz[u] = in[cc[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p + u < p1) s += va[u] * (cf * zz[u]);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p + u < p1) s += va[u] * a.out[cc[u]];
      }
      p += 8;
      if (p >= p1) break;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = p + u < p1;
        cc[u] = ok ? __ldcs(ci + p + u) : r;
        va[u] = ok ? __ldcs(vv + p + u) : 0.0;
      }
    }
    if (!a.backward) {
      a.out[r] = (cf * in[r] - om * s) * di;
    } else {
      a.out[r] = a.out[r] - om * s * di;
    }
  }
  if (st->profile && grid_last(a.L.counter) && threadIdx.x == 0) {
    KStatDev& k = st->kstat[K_SSOR];
    k.bytes += a.bytes;
    if (a.last) {  // closes the K_SSOR timing interval of one application
      st->kstat[K_SSORK].launches += a.nsweeps;
      k.ns += gtimer() - k.start;
      k.launches++;
    }
  }
}

__global__ void k_ssor_values(PrecDev P, const double* __restrict__ v, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nL; i += stride) P.Lv[i] = v[P.Lmap[i]];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nU; i += stride) P.Uv[i] = v[P.Umap[i]];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double d = 1.0 / v[P.dmap[i]];
    P.dinv[i] = d;
    P.dinvr[P.perm[i]] = d;
  }
}

// Lv1 = (L values of the colour-1 rows) * 1/a_jj of their (colour-0) column; after k_ssor_values
__global__ void k_ssor_scale(PrecDev P) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nL1; i += stride)
    P.Lv1[i] = P.Lv[P.l1base + i] * P.dinvr[P.Lci[P.l1base + i]];
}

}  // namespace

cudaError_t launch_ssor_values(const PrecDev& P, const double* v, int64_t n, cudaStream_t s) {
  note_host_launches(1);
  const int64_t work = std::max(std::max(P.nL, P.nU), n);
  int64_t g = (work + ST - 1) / ST;
  if (g > (int64_t)NSM * 8) g = (int64_t)NSM * 8;
  k_ssor_values<<<(int)(g < 1 ? 1 : g), ST, 0, s>>>(P, v, n);
  if (P.nL1 > 0) {
    note_host_launches(1);
    int64_t g1 = (P.nL1 + ST - 1) / ST;
    if (g1 > (int64_t)NSM * 8) g1 = (int64_t)NSM * 8;
    k_ssor_scale<<<(int)g1, ST, 0, s>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_ssor(const PrecDev& P, const Layout& L, DevState* st, const double* in, double* out, int gate,
                        cudaStream_t s) {
  SsorArgs a{};
  a.P = P; a.in = in; a.out = out; a.gate = gate; a.L = L; a.st = st;
  // forward colours {0, 1} (one launch), 2 .. nc-1, backward nc-2 .. 0 (the backward sweep of the last
  // colour is the identity)
  const int nc = P.ncolors;
  const int nfwd = nc >= 2 ? nc - 1 : 1, nbwd = nc - 1;
  a.nsweeps = nfwd + nbwd;
  for (int pass = 0; pass < nfwd + nbwd; ++pass) {
    const bool bwd = pass >= nfwd;
    int clo, chi;  // colours [clo, chi) of this launch
    if (bwd) { clo = nc - 2 - (pass - nfwd); chi = clo + 1; }
    else if (pass == 0) { clo = 0; chi = nc >= 2 ? 2 : 1; }
    else { clo = pass + 1; chi = clo + 1; }
    a.backward = bwd ? 1 : 0;
    a.fuse0 = (!bwd && pass == 0 && nc >= 2) ? 1 : 0;
    a.first = pass == 0;
    a.last = pass == nfwd + nbwd - 1;
    a.c0 = P.coff[clo];
    a.c1 = P.coff[chi];
    const double rows = (double)(a.c1 - a.c0);
    // algorithmic bytes: the colours' L (or U) entries + perm, row pointer, 1/a_rr, vector in/out
    double ent = 0.0;
    for (int c = clo; c < chi; ++c) ent += (double)(bwd ? P.cU[c] : P.cL[c]);
    a.bytes = 12.0 * ent + rows * (4.0 + 4.0 + 8.0 + 16.0);
    const int64_t nrows = a.c1 - a.c0;
    const int g = (int)(nrows > 0 ? (nrows + ST - 1) / ST : 1);
    cudaError_t e = launch_ex(k_ssor, dim3(g), dim3(ST), 0, s, pass > 0, a);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rg

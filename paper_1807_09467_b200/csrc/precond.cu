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
#include "kernels.cuh"

namespace rg {
namespace {

constexpr int ST = 256;

struct SsorArgs {
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
  const uint8_t* color;
  const int32_t* perm;   // rows grouped by colour
  const int32_t* diag;   // position of a_rr in ci/v
  int64_t c0, c1;        // this colour's range in perm
  int c;                 // colour
  int backward;
  double omega;
  const double* in;      // forward input (nullptr: the Arnoldi vector u of the device state)
  double* out;           // w (forward) / t (backward, in place)
  int gate;              // 0 always, 1 Arnoldi step (st->active ...), 2 cycle end (st->have_xupd)
  Layout L;
  DevState* st;
  double bytes;
};

__global__ void __launch_bounds__(ST) k_ssor(SsorArgs a) {
  DevState* st = a.st;
  double xs = 1.0;
  const double* in = a.in;
  if (a.gate == 1) {
    const int j = st->j;
    if (!st->active || (st->dcgs && j >= st->m)) { prof_noop(st, K_SSOR); return; }
    if (!a.backward) {
      in = a.L.Z + (int64_t)(a.L.VB + j) * a.L.ld;
      xs = st->dcgs ? 1.0 : st->sc[a.L.VB + j];  // CGS2 path: V stored un-normalised
    }
  } else if (a.gate == 2) {
    if (!st->have_xupd) { prof_noop(st, K_SSOR); return; }
  }
  if (st && blockIdx.x == 0 && threadIdx.x == 0 && a.c == 0 && !a.backward) prof_begin(st, K_SSOR);
  const int64_t idx = a.c0 + (int64_t)blockIdx.x * ST + threadIdx.x;
  if (idx < a.c1) {
    const int32_t r = __ldg(a.perm + idx);
    const int32_t p0 = __ldg(a.rp + r), p1 = __ldg(a.rp + r + 1);
    const double arr = __ldg(a.v + __ldg(a.diag + r));
    const int c = a.c;
    double s = 0.0;
    for (int32_t p = p0; p < p1; p += 8) {
      int32_t cc[8];
      double vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = p + u < p1;
        cc[u] = ok ? __ldg(a.ci + p + u) : r;
        vv[u] = ok ? __ldg(a.v + p + u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int cj = __ldg(a.color + cc[u]);
        const bool take = a.backward ? cj > c : cj < c;
        if (take) s += vv[u] * a.out[cc[u]];
      }
    }
    const double om = a.omega;
    if (!a.backward) {
      a.out[r] = (xs * om * (2.0 - om) * in[r] - om * s) / arr;
    } else {
      a.out[r] = a.out[r] - om * s / arr;
    }
  }
  if (st && st->profile && grid_last(a.L.counter) && threadIdx.x == 0) st->kstat[K_SSOR].bytes += a.bytes;
}

// closes the K_SSOR timing interval after the last sweep of one application
__global__ void k_ssor_done(DevState* st, int gate) {
  if (!st->profile) return;
  if (gate == 1 && (!st->active || (st->dcgs && st->j >= st->m))) return;
  if (gate == 2 && !st->have_xupd) return;
  KStatDev& k = st->kstat[K_SSOR];
  const unsigned long long t = gtimer();
  k.ns += t - k.start;
  k.launches++;
}

}  // namespace

cudaError_t launch_ssor(const PrecDev& P, const Layout& L, DevState* st, const double* in, double* out, int gate,
                        cudaStream_t s) {
  SsorArgs a{};
  a.rp = P.rp; a.ci = P.ci; a.v = P.v; a.color = P.color; a.perm = P.perm; a.diag = P.diag;
  a.omega = P.omega; a.in = in; a.out = out; a.gate = gate; a.L = L; a.st = st;
  // forward colours 0 .. nc-1, backward nc-2 .. 0
  for (int pass = 0; pass < 2 * P.ncolors - 1; ++pass) {
    const bool bwd = pass >= P.ncolors;
    const int c = bwd ? 2 * P.ncolors - 2 - pass : pass;
    a.c = c;
    a.backward = bwd ? 1 : 0;
    a.c0 = P.coff[c];
    a.c1 = P.coff[c + 1];
    a.bytes = 12.0 * (double)P.cnnz[c] + 8.0 * (double)(a.c1 - a.c0) * (bwd ? 3.0 : 4.0);
    const int64_t rows = a.c1 - a.c0;
    const int g = (int)(rows > 0 ? (rows + ST - 1) / ST : 1);
    k_ssor<<<g, ST, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_ssor_done<<<1, 1, 0, s>>>(st, gate);
  return cudaGetLastError();
}

}  // namespace rg

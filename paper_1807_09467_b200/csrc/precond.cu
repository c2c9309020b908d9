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
  int64_t c0, c1;        // this colour's range in perm
  int backward;
  const double* in;      // forward input (nullptr: the Arnoldi vector u of the device state)
  double* out;           // w (forward) / t (backward, in place)
  int gate;              // 0 always, 1 Arnoldi step (st->active ...), 2 cycle end (st->have_xupd)
  int first;             // first sweep of an application (profiling start)
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
  if (a.first && blockIdx.x == 0 && threadIdx.x == 0) prof_begin(st, K_SSOR);
  const PrecDev& P = a.P;
  const int64_t idx = a.c0 + (int64_t)blockIdx.x * ST + threadIdx.x;
  if (idx < a.c1) {
    const int32_t r = __ldg(P.perm + idx);
    const int32_t* __restrict__ rp = a.backward ? P.Urp : P.Lrp;
    const int32_t* __restrict__ ci = a.backward ? P.Uci : P.Lci;
    const double* __restrict__ vv = a.backward ? P.Uv : P.Lv;
    const int32_t p0 = __ldg(rp + idx), p1 = __ldg(rp + idx + 1);
    double s = 0.0;
    for (int32_t p = p0; p < p1; p += 8) {
      int32_t cc[8];
      double va[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = p + u < p1;
        cc[u] = ok ? __ldcs(ci + p + u) : r;
        va[u] = ok ? __ldcs(vv + p + u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < p1) s += va[u] * a.out[cc[u]];
    }
    const double om = P.omega, di = __ldg(P.dinv + idx);
    if (!a.backward) {
      a.out[r] = (xs * om * (2.0 - om) * in[r] - om * s) * di;
    } else {
      a.out[r] = a.out[r] - om * s * di;
    }
  }
  if (st->profile && grid_last(a.L.counter) && threadIdx.x == 0) st->kstat[K_SSOR].bytes += a.bytes;
}

// closes the K_SSOR timing interval after the last sweep of one application
__global__ void k_ssor_done(DevState* st, int gate, int nsweeps) {
  if (!st->profile) return;
  st->kstat[K_SSORK].launches += nsweeps + 1;  // kernel launches of this application (incl. this one)
  if (gate == 1 && (!st->active || (st->dcgs && st->j >= st->m))) return;
  if (gate == 2 && !st->have_xupd) return;
  KStatDev& k = st->kstat[K_SSOR];
  const unsigned long long t = gtimer();
  k.ns += t - k.start;
  k.launches++;
}

__global__ void k_ssor_values(PrecDev P, const double* __restrict__ v, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nL; i += stride) P.Lv[i] = v[P.Lmap[i]];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nU; i += stride) P.Uv[i] = v[P.Umap[i]];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) P.dinv[i] = 1.0 / v[P.dmap[i]];
}

}  // namespace

cudaError_t launch_ssor_values(const PrecDev& P, const double* v, int64_t n, cudaStream_t s) {
  note_host_launches(1);
  const int64_t work = std::max(std::max(P.nL, P.nU), n);
  int64_t g = (work + ST - 1) / ST;
  if (g > (int64_t)NSM * 8) g = (int64_t)NSM * 8;
  k_ssor_values<<<(int)(g < 1 ? 1 : g), ST, 0, s>>>(P, v, n);
  return cudaGetLastError();
}

cudaError_t launch_ssor(const PrecDev& P, const Layout& L, DevState* st, const double* in, double* out, int gate,
                        cudaStream_t s) {
  SsorArgs a{};
  a.P = P; a.in = in; a.out = out; a.gate = gate; a.L = L; a.st = st;
  // forward colours 0 .. nc-1, backward nc-2 .. 0 (the backward sweep of the last colour is the identity)
  for (int pass = 0; pass < 2 * P.ncolors - 1; ++pass) {
    const bool bwd = pass >= P.ncolors;
    const int c = bwd ? 2 * P.ncolors - 2 - pass : pass;
    a.backward = bwd ? 1 : 0;
    a.first = pass == 0;
    a.c0 = P.coff[c];
    a.c1 = P.coff[c + 1];
    const double rows = (double)(a.c1 - a.c0);
    // algorithmic bytes: this colour's L (or U) entries + perm, row pointer, 1/a_rr, vector in/out
    a.bytes = 12.0 * (double)(bwd ? P.cU[c] : P.cL[c]) + rows * (4.0 + 4.0 + 8.0 + 16.0);
    const int64_t nrows = a.c1 - a.c0;
    const int g = (int)(nrows > 0 ? (nrows + ST - 1) / ST : 1);
    k_ssor<<<g, ST, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_ssor_done<<<1, 1, 0, s>>>(st, gate, 2 * P.ncolors - 1);
  return cudaGetLastError();
}

}  // namespace rg

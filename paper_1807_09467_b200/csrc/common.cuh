// common.cuh — internal definitions of librg (B200 / sm_100a, fp64).
//
// Device-resident solver state, the basis layout in HBM, and the deterministic grid-reduction
// machinery shared by every reducing kernel.  See DESIGN.md §"Data layout" and §"Kernels".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rg.h"

namespace rg {

// ---------------------------------------------------------------- capacity limits
constexpr int MAXM = 128;                  // restart length
constexpr int MAXK = 64;                   // recycle dimension
constexpr int MAXS = 64;                   // snapshot window
constexpr int MAXCOL = 2 * MAXK + MAXM + 2;// columns of the basis buffer Z = [W | Q | V]
constexpr int MAXRED = MAXCOL + 2;         // values one grid reduction can return

// ---------------------------------------------------------------- launch geometry
#ifndef SELL_CH
#define SELL_CH 12  // SELL-32 entries of a row loaded together (one round for the 9-point rows of C3;
                    // measured 8 -> 12: standalone SELL SpMV 4.28 -> 5.24 TB/s, C3 persistent -1.9 %)
#endif
constexpr int OT = 512;                    // threads per CTA of the vector kernels
constexpr int NWARP = OT / 32;
constexpr int NSM = 148;                   // B200 SMs
constexpr int VEC_CTAS_PER_SM = 2;         // -> 296 CTAs: 32 resident warps / SM

// ---------------------------------------------------------------- kernel ids (statistics)
enum KernelId {
  K_SPMV_STEP = 0, K_SPMV_RES, K_SPMV_PLAIN, K_ORTH_D1, K_ORTH_UD2, K_ORTH_UN, K_CS_DQ, K_CS_UN,
  K_XW, K_XUPD, K_NORMB, K_GRAM, K_JACOBI, K_XM, K_CHOL, K_MISC, K_DK1, K_DK2,
  K_PB1, K_PB2, K_PB3, K_PB4, K_PB5, K_OBD, K_OBU, K_SSOR, K_PB6, K_COND, K_SSORK, K_PB7, K_CBUILD, K_RES_Y, K_DLS,
  K_COUNT
};

struct KStatDev {
  unsigned long long launches, noop, ns, start, tail_start, tail_ns;
  double bytes;
};

// ---------------------------------------------------------------- device-resident solver state
// Written by the host once per solve (header) and then driven entirely by kernel epilogues:
// the host never needs to read it until the solve (or a restart cycle) ends.
struct DevState {
  // per-solve header (host -> device before the solve)
  int variant, m, k_eff, max_iters, hist_cap, profile;
  double tol;
  // dynamic scalars
  int j;          // current Arnoldi step within the cycle
  int active;     // Arnoldi steps of this cycle still running
  int done;       // solve finished
  int converged;
  int iters;      // Arnoldi steps summed over cycles
  int cycles;
  int status;     // 0 ok, RG_E_NUMERIC
  int have_xupd;  // cycle-end x update pending
  int jfinal;     // last step index of the finished cycle
  int hist_len;
  int spmv_count;
  int bzero;
  int dcgs;       // 1: delayed CGS2 (one reduction per Arnoldi step), 0: classical CGS2
  int cfail;      // set by the C = A W build of this solve: singular CholQR2 factor / R_C / E
  int kb_steps;   // RG_FLAG_KEEP_BASIS: Arnoldi steps J of the last finished cycle kept for rg_export
  unsigned chk_count, chk_where;  // CHECKED builds: failed device checks, first (file id << 16 | line)
  double bnorm, beta, relres;
  double k2_inv_nu, k2_u_next, k2_y;  // DCGS2 update-pass scalars (v_j = u/nu + ..., u_next = ...)
  // least-squares state
  double cs[MAXM], sn[MAXM], g[MAXM + 2], y[MAXM + 2];
  double R[MAXM][MAXM + 2];        // rotated columns, R[j][0..j]
  double Hraw[MAXM][MAXM + 2];     // unrotated Hessenberg columns (augment)
  double Bm[MAXM][MAXK];           // deflate: B[:, j] = Q^T A v_j   (GCRO: A V = Q B + V H)
  double Gm[MAXM + 2][MAXK];       // augment: G[i, :] = Q^T v_i
  double T[MAXM + 2][MAXM + 2];    // augment: Cholesky factor of I - G^T G, T[col][row]
  double Si[MAXM + 2][MAXM + 2];   // augment: S = T^{-1} (upper triangular), Si[col][row]
  double RCinv[MAXK][MAXK];        // R_C^{-1}, column-major [col][row]
  double RC[MAXK][MAXK];           // R_C, column-major [col][row]
  double Einv[MAXK][MAXK];         // oblique: E^{-1}, E = W^T A W, column-major [col][row]
  double coef[MAXCOL];             // coefficients of the current CGS pass (absolute column)
  double hcol[MAXCOL];             // accumulated coefficients of the current column
  double coefx[MAXCOL];            // cycle-end x-update coefficients
  double sc[MAXCOL];               // column scales (V stored un-normalised: v_i = sc_i * raw_i)
  double coefv[MAXCOL];            // DCGS2: v_j = u/nu + sum_c coefv_c P_c
  KStatDev kstat[K_COUNT];
  unsigned red_epoch;              // persistent solve: last flag value of its flag-carrying reductions
  // graph-path DCGS2 split epilogue: DK1's last CTA leaves the least-squares step of column ls_j to
  // k_dcgs_ls (which runs concurrently with DK2): its input [Q^T v (augment) | ||v||^2]; k2_skip: no
  // update pass this step (j = m: no next column)
  int ls_j, k2_skip;
  double ls_in[MAXK + 2];
  // RG_FLAG_PROFILE: device timeline ring (rg_kernel_trace): 2 words per event {t_ns, kid | kind << 16}
  unsigned long long* trace;
  unsigned trace_cap, trace_len;
};
constexpr unsigned TRACE_CAP = 1u << 16;

// Basis layout (constant per context).  Z is n_pad x MAXCOL... column-major with leading
// dimension ld; columns [0, maxk) hold W, [VB - k_eff, VB) hold Q, [VB, VB + m + 1) hold V.
// The oblique variant keeps C = A W (not Q) in [k_eff, 2 k_eff), adjacent to W.
struct Layout {
  double* Z;
  int64_t ld;      // = n_pad (multiple of 64)
  int64_t n;       // true dimension
  int maxk;        // W / Q region width
  int ncol;        // columns of Z (checked builds bound every column index by it)
  int VB;          // first V column = 2 * maxk
  double* x;       // iterate (n_pad)
  const double* b; // right-hand side (n_pad)
  double* hist;    // history buffer (hist_cap)
  double* partial; // grid-reduction partials [grid][MAXRED]
  unsigned* counter;
  int cgs_ok;      // [Q|V] (max_k + max_m + 1 columns) fits k_cgs (16 chunks of 8 columns)
  int augment;     // variant of the graph being built / launched is augment
  int keep_l2;     // the whole basis [W|Q|V] is L2-sized: DCGS2 passes use cached (not streaming) loads
  int prec;        // right preconditioner active (precond.cu): cycle end adds pz = M^{-1} (V y)
  double* pz;      // preconditioner output (M^{-1} u of the Arnoldi step, M^{-1} V y at the cycle end)
  double* pt;      // cycle-end scratch: V y
  double* keepV;   // RG_FLAG_KEEP_BASIS: n_pad x (max_m + 1) copy of the last finished cycle's V (else null)
};

// Galerkin-start variants (oblique, orthogonal): C = A W in columns [k, 2k), E^{-1} in the state.
// The Krylov projector is I - P T W^T with P = C, T = E^{-1} (oblique) or P = W, T = I (orthogonal);
// proj_base() is the first column of P.
__host__ __device__ __forceinline__ bool galerkin_variant(int v) { return v == RG_OBLIQUE || v == RG_ORTHOGONAL; }
__host__ __device__ __forceinline__ int proj_base(int v, int k) { return v == RG_ORTHOGONAL ? 0 : k; }

// ---------------------------------------------------------------- small device helpers
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // valid in lane 0
}

// Deterministic block sum (fixed tree), result broadcast to all threads.  `sh` >= 33 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += sh[i];
    sh[32] = s;
  }
  __syncthreads();
  return sh[32];
}

// ---- CHECKED builds (make rg-checked, -DRG_CHECKED; test infrastructure): device-side bounds and
// invariant checks on the hand-computed indexing — TMA copy ranges, basis column ranges, reduction
// widths, least-squares state indices, sparse column indices, persistent-kernel row / neighbour
// ranges.  A failing check is counted in the device state (first location kept) and execution
// continues; the host returns RG_E_CHECK after the call.  Compiled out of the product.
#ifndef RG_FILE_ID
#define RG_FILE_ID 0
#endif
#ifdef RG_CHECKED
__device__ __noinline__ inline void rg_chk_fail(DevState* st, unsigned where) {
  if (!st) return;
  atomicAdd(&st->chk_count, 1u);
  atomicCAS(&st->chk_where, 0u, where);
}
#define RG_CHK(st, cond)                                                        \
  do {                                                                          \
    if (!(cond)) rg_chk_fail((st), ((unsigned)RG_FILE_ID << 16) | (unsigned)__LINE__); \
  } while (0)
#else
#define RG_CHK(st, cond) \
  do {                   \
  } while (0)
#endif

// Programmatic dependent launch (PDL).  A kernel launched with cudaLaunchAttributeProgrammaticStream-
// Serialization (launch_ex(..., pdl = true)) may be scheduled while its predecessor on the stream (or
// graph edge) drains: it overlaps its launch ramp and any prologue that does not read the predecessor's
// output with the predecessor's tail.  pdl_wait() blocks until the predecessor grid has completed and
// its writes are visible (a no-op when the kernel was launched normally); pdl_trigger() lets the
// dependent grid be scheduled once every CTA of this grid has executed it (or exited).  Only kernels
// that call pdl_wait() before consuming anything a predecessor wrote are ever launched with pdl = true.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Kernel-entry profiling hook (block 0 stamps the start time).
__device__ __forceinline__ void trace_ev(DevState* st, int kid, unsigned kind, unsigned long long t) {
  if (!st->trace) return;
  const unsigned i = atomicAdd(&st->trace_len, 1u);
  if (i < st->trace_cap) {
    st->trace[2 * (size_t)i] = t;
    st->trace[2 * (size_t)i + 1] = (unsigned long long)kid | ((unsigned long long)kind << 16);
  }
}
__device__ __forceinline__ void prof_begin(DevState* st, int kid) {
  if (st->profile && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    st->kstat[kid].start = t;
    trace_ev(st, kid, 0u, t);
  }
}
__device__ __forceinline__ void prof_noop(DevState* st, int kid) {
  if (st->profile && blockIdx.x == 0 && threadIdx.x == 0) {
    st->kstat[kid].noop++;
    trace_ev(st, kid, 2u, gtimer());
  }
}
// Called by thread 0 of the last CTA when it has won the grid-reduction ticket.
__device__ __forceinline__ void prof_tail(DevState* st, int kid) {
  if (st->profile && threadIdx.x == 0) st->kstat[kid].tail_start = gtimer();
}
// Called by ONE thread of the last CTA.
__device__ __forceinline__ void prof_end(DevState* st, int kid, double bytes) {
  if (st->profile) {
    KStatDev& k = st->kstat[kid];
    const unsigned long long t = gtimer();
    if (k.tail_start > k.start) k.tail_ns += t - k.tail_start;
    k.tail_start = 0;
    k.ns += t - k.start;
    k.launches++;
    k.bytes += bytes;
    trace_ev(st, kid, 1u, t);
  }
}

__device__ __forceinline__ unsigned atom_add_release(unsigned* p) {
  unsigned t;
  asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(p) : "memory");
  return t;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Deterministic two-stage grid reduction.  Every CTA passes nv values in shared memory `vals`
// (nv <= MAXRED).  Returns true in exactly one CTA (the last to arrive), whose shared array `tot`
// then holds the totals, summed over CTAs in index order.  `scr` needs max(blockDim, MAXRED)
// doubles (max(blockDim, nv) if nv > MAXRED).  ldp = row stride of `partial`.
// All threads of every CTA must call it.
__device__ __forceinline__ bool grid_reduce(const double* vals, int nv, double* partial,
                                            unsigned* counter, double* tot, double* scr,
                                            int ldp = MAXRED) {
  __shared__ unsigned s_ticket;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) partial[(size_t)blockIdx.x * ldp + i] = vals[i];
  // One release by thread 0 after the CTA barrier publishes every thread's partials (PTX memory
  // model: bar.sync orders them before the gpu-scope release); no per-thread membar.gl.
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atom_add_release(counter);
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return false;
  if (threadIdx.x == 0) fence_acq_rel();
  __syncthreads();
  // warp w reduces columns c = w, w + nwarps, ...: lane l sums partials of CTAs l, l+32, ...
  // (8 independent loads in flight), then a fixed shuffle tree: deterministic order.
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  (void)scr;
  if (nv > 2 * nw) {
    // many columns: S consecutive threads per column (S = largest power of two <= 32 with
    // S * nv <= blockDim); thread `sub` of a column sums the partials of CTAs sub, sub + S, ...
    // with 16 independent L2 loads in flight, then a fixed shuffle tree of width S.  (A thread
    // per column summing all G partials in batches of 8 was ~37 dependent L2 round trips: ~10 us
    // of last-CTA tail per launch at G = 296.)
    int S = 1;
    while (S < 32 && 2 * S * nv <= (int)blockDim.x) S <<= 1;
    const int sub = threadIdx.x % S, groups = blockDim.x / S;
    for (int c0 = 0; c0 < nv; c0 += groups) {
      const int c = c0 + (int)threadIdx.x / S;
      double a = 0.0;
      if (c < nv) {
        for (int b = sub; b < G; b += S * 16) {
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = b + u * S < G ? __ldcg(&partial[(size_t)(b + u * S) * ldp + c]) : 0.0;
#pragma unroll
          for (int u = 0; u < 16; ++u) a += v[u];
        }
      }
      for (int o = S >> 1; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o, S);
      if (c < nv && sub == 0) tot[c] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0u;
    __syncthreads();
    return true;
  }
  for (int c = threadIdx.x >> 5; c < nv; c += nw) {
    double a = 0.0;
    for (int b = lane; b < G; b += 8 * 32) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int bb = b + u * 32;
        v[u] = bb < G ? __ldcg(&partial[(size_t)bb * ldp + c]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    a = warp_sum(a);
    if (lane == 0) tot[c] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;
  __syncthreads();
  return true;
}

// Ticket only (no values): returns true in the last CTA.  Used for profiling of kernels that
// have no reduction.
__device__ __forceinline__ bool grid_last(unsigned* counter) {
  __shared__ unsigned s_t;
  __syncthreads();
  if (threadIdx.x == 0) s_t = atom_add_release(counter);
  __syncthreads();
  if (s_t != gridDim.x - 1) return false;
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

// Function attributes and occupancy results are per device: launchers cache them per ordinal.
constexpr int MAXDEV = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAXDEV) { cudaGetLastError(); d = 0; }
  return d;
}
// once per device: `static PerDevice once; if (once.first()) cudaFuncSetAttribute(...)`
struct PerDevice {
  bool done[MAXDEV];
  bool first() {
    const int d = current_device();
    if (done[d]) return false;
    done[d] = true;
    return true;
  }
};

inline int vec_grid(int64_t rows) {
  int64_t g = (rows + OT - 1) / OT;
  int64_t cap = (int64_t)NSM * VEC_CTAS_PER_SM;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace rg

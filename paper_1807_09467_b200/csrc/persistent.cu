// persistent.cu — the whole restarted solve in ONE cooperative kernel (every variant, CSR / SELL).
//
// Why: at the sizes of configs C1-C2 every kernel boundary of the graph path costs a launch ramp
// plus a single-CTA epilogue tail (~10 us per Arnoldi step).  Here every CTA of a co-resident grid
// keeps an IDENTICAL copy of the least-squares state (unrotated Hessenberg H, rotated R, GCRO B,
// Givens rotations, right-hand side g) in shared memory and recomputes the deterministic epilogue
// from the reduced totals itself; kernel boundaries become grid barriers.  Per Arnoldi step (DCGS2,
// see dcgs.cu): barrier, SpMV y = A u + local dots [P^T u, P^T y, u.u, u.y], two-barrier
// deterministic reduction, replicated epilogue, row update of v_j and the next u.
// CTA 0 alone writes the solve report (iterations, history, status) to the device state.
// Oblique (obl): P = V only; the Galerkin cycle start and the M_D projection folded into the DCGS2
// coefficients exactly as dcgs.cu does it (V^T C replicated in shared memory).
#define RG_FILE_ID 4  // RG_CHK locations (checked builds)
#include "epilogue.cuh"
#include "kernels.cuh"
#include "knobs.cuh"
#include <algorithm>
#include <climits>
#include <cstdlib>

namespace rg {
namespace {

#ifndef RG_PT
#define RG_PT 512
#endif
constexpr int PT = RG_PT;     // threads per CTA
constexpr int PCTA = 1024 / PT;  // resident CTAs per SM
constexpr int PM = 64;        // max restart length on this path
constexpr int PK = 64;        // max recycle dimension on this path
constexpr int PCOL = PK + PM + 2;
constexpr int NPFN = 10;      // k_solve_persistent instantiations (launch_persistent's table)
constexpr int CB_TSW = 36;   // k_cbuild per-warp tile column stride (32 rows + 4: DMMA fragment loads spread over banks)
constexpr int CBK = 22;       // max recycle dimension of the one-kernel operator build (k (k+1) / 2 <= MAXRED)

struct PArgs {
  Layout L;
  MatDev A;
  DevState* st;
  double* tot_g;        // reduced totals (MAXRED)
  unsigned* bar;        // [0] arrival count, [1] generation
  int m, k;             // m <= PM, k <= PK (k = 0: plain)
  int obl;              // oblique variant (k = k_eff > 0, C = A W in columns [k, 2k))
  int aug;              // augment variant (k > 0): least squares on M = T H-bar (epilogue.cuh epi_ls)
  unsigned* flags;      // [gridDim.x] neighbour-sync epochs (zeroed before the launch)
  int nbsync;           // 1: point-to-point neighbour sync before the SpMVs instead of grid barriers
  int skew;             // experiment (RG_SKEW=j): per-CTA start / dots done / reduced timestamps and SM of step j
  int prec;             // right multicolour SSOR preconditioner (precond.cu's colour-ordered L/U copies)
  PrecDev P;
  double* pz;           // M^{-1} u (step) / M^{-1} V y (cycle end)
  double* pt;           // V y (cycle end)
  double pc_bytes;      // algorithmic bytes of one SSOR application
  int rcap, ccap;       // CSR pattern cache in shared memory: row pointers / column indices capacity (0: off)
  unsigned long long* ll;  // flag-carrying reduction words (LL_WORDS; zeroed once at allocation)
  int llred;            // 1: reductions through `ll` (greduce_ll), 0: two-barrier greduce
};

// ---- grid barrier (all CTAs co-resident: cooperative launch).  Spins with a timeout so that a
// bug cannot hang the GPU: after ~2 s every CTA gives up and the solve reports RG_E_CUDA.
// Words (unsigned): [0] monotonic arrival counter, [64 + 32 b] CTA b's barrier count (zeroed per
// launch).  (Measured: a two-level arrival tree with per-group counters made no difference at 296
// CTAs.)
__device__ __forceinline__ bool gbar(unsigned* bar, int* s_fail) {
  __syncthreads();
  if (gridDim.x == 1) return true;  // single-CTA solve (tiny systems): a CTA barrier suffices
  if (threadIdx.x == 0) {
    // monotonic arrival counter: the n-th barrier of this launch completes when the counter reaches
    // n * G (every CTA passes the same barriers in the same order), so the last arrival's own atomic
    // is the release — no reset and no separate generation bump (one L2 round trip less)
    unsigned* nb = bar + 64 + blockIdx.x * 32;  // this CTA's barrier count (own 128-B line; thread 0 only)
    const unsigned target = (*nb + 1u) * gridDim.x;
    *nb += 1u;
    __threadfence();
    if (atomicAdd(bar, 1u) + 1u < target) {
      volatile unsigned* cnt = bar;
      const long long t0 = clock64();
      unsigned ns = 32;
      while (*cnt < target) {  // exponential back-off keeps ~300 pollers off the barrier's L2 line
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
        if (clock64() - t0 > 4000000000LL) { *s_fail = 1; break; }
      }
    }
    __threadfence();
  }
  __syncthreads();
  return *s_fail == 0;
}

// ---- neighbour synchronisation.  The SpMV of a CTA reads only the rows of the CTAs that own the
// columns of its rows ([c_lo, c_hi], computed once from the pattern).  After writing the vector the
// next SpMV reads (u, or x at a cycle end), every CTA publishes an epoch; before the SpMV a CTA
// waits only for the epochs of its column owners instead of a grid-wide barrier.  Every CTA runs the
// same sequence of publish points (the control flow is replicated), so epochs agree.  Write-after-
// read hazards on those rows are excluded by the grid barriers inside the reduction that separates
// a SpMV from the next write of the same column.
__device__ __forceinline__ void nb_publish(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(flags + blockIdx.x, epoch);
  }
}

__device__ __forceinline__ bool nb_wait(const unsigned* flags, int lo, int hi, unsigned epoch, int* s_fail) {
  for (int c = lo + (int)threadIdx.x; c <= hi; c += blockDim.x) {  // one polling thread per owner CTA
    volatile const unsigned* f = flags + c;
    const long long t0 = clock64();
    unsigned ns = 32;
    while (*f < epoch) {
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
      if (clock64() - t0 > 4000000000LL) { *s_fail = 1; break; }
    }
    __threadfence();
  }
  __syncthreads();
  return *s_fail == 0;
}

// owner CTA of a row under the even 32-row-granule split used by the kernel
__device__ __forceinline__ int row_owner(int64_t row, int64_t ng, int G) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {  // largest b with r0(b) <= row
    const int mid = (lo + hi + 1) >> 1;
    if ((((int64_t)mid * ng / G) << 5) <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---- deterministic grid reduction: every CTA writes its nv partials; CTA c sums columns
// c, c+G, ... over CTAs in index order; every CTA then reads the nv totals into `tot`.
// (Measured: a single "last CTA reduces" wave is slower here — the reducing CTA competes with ~300
// pollers — and so is a one-barrier variant in which every CTA reduces all columns itself (296 CTAs
// x all partials from L2: C2 reduce phase 6.8 -> 23.8 ms per 10 systems), and so is a thread-block-
// cluster variant (DSMEM sum inside clusters of 2/4/8 CTAs, one grid barrier, every CTA summing the
// G/CS cluster partials: reduce phase +40..140 %: every CTA reading the same few KB hot-spots the
// same L2 lines); the work is spread over all CTAs between two barriers.)
__device__ __forceinline__ bool greduce(const double* vals, int nv, double* partial, double* tot_g, double* tot,
                                        unsigned* bar, int* s_fail, DevState* st = nullptr) {
  if (gridDim.x == 1) {  // single CTA: the CTA's values are the totals
    __syncthreads();
    for (int i = threadIdx.x; i < nv; i += blockDim.x) tot[i] = vals[i];
    __syncthreads();
    return true;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, G = gridDim.x;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) partial[(size_t)blockIdx.x * MAXRED + i] = vals[i];
  const unsigned long long ta = (st && st->profile && blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
  if (!gbar(bar, s_fail)) return false;
  if (ta) {  // profiling: time CTA 0 waits in the first barrier (skew + arrival) -> p_reduce_arrive
    st->kstat[K_PB6].ns += gtimer() - ta;
    st->kstat[K_PB6].launches++;
  }
  for (int col = blockIdx.x + G * wid; col < nv; col += G * (int)(blockDim.x / 32)) {
    double a = 0.0;
    for (int b0 = lane; b0 < G; b0 += 32 * 8) {  // 8 independent L2 loads in flight per lane
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < G ? __ldcg(partial + (size_t)(b0 + 32 * u) * MAXRED + col) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    a = warp_sum(a);
    if (lane == 0) tot_g[col] = a;
  }
  if (!gbar(bar, s_fail)) return false;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) tot[i] = __ldcg(tot_g + i);
  __syncthreads();
  return true;
}

// ---- flag-carrying ("LL") deterministic grid reduction, no barrier at all.  Every value travels as
// two 64-bit words {low half | epoch, high half | epoch}; an aligned 64-bit store is single-copy
// atomic, so a reader that sees the current epoch in both words holds the value — data and flag
// arrive together, no fence, no counter.  CTA b publishes its nv partials; CTA c sums columns
// c, c+G, ... (thread t polls CTA t's partial, fixed-tree block sum: deterministic) and publishes
// the total; every CTA polls the nv totals.  Latency after the last partial: one poll round trip,
// a block sum, one poll round trip (the two-barrier version adds two atomic arrivals, four fences
// and the barrier polls).  Epochs increase by one per reduction and persist across launches in
// DevState::red_epoch; partials and totals are double-buffered by epoch parity, so a slot is
// rewritten only two reductions later, after every CTA has consumed it (each CTA must have read
// every total of the reduction in between).  Requires G <= PT and G <= LL_GMAX.  Each total is
// written to LL_R replicas (CTA b polls replica b % LL_R): ~300 CTAs polling the same few lines
// queue at their L2 slices (micro-benchmark, nv = 92: 4.8 -> 3.8 us per reduction with 16 replicas).
constexpr int LL_GMAX = NSM * 2;
constexpr int LL_R = 16;
}  // namespace
size_t ll_words() { return (size_t)2 * 2 * ((size_t)LL_GMAX * MAXRED + (size_t)LL_R * MAXRED); }
namespace {

__device__ __forceinline__ void ll_st(unsigned long long* p, double v, unsigned ep) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long e = (unsigned long long)ep << 32;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"((b & 0xffffffffull) | e), "l"((b >> 32) | e)
               : "memory");
}

__device__ __forceinline__ bool ll_ld(const unsigned long long* p, unsigned ep, double& v) {
  unsigned long long w0, w1;
  long long t0 = 0;
  for (int it = 0;; ++it) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if ((unsigned)(w0 >> 32) == ep && (unsigned)(w1 >> 32) == ep) break;
    if (it == 0) {
      t0 = clock64();
    } else if (clock64() - t0 > 4000000000LL) {
      return false;
    }
    __nanosleep(32);
  }
  v = __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
  return true;
}

__device__ __forceinline__ bool greduce_ll(const double* vals, int nv, unsigned long long* ll, double* tot,
                                           unsigned& ep, double* bsh, int* s_fail, DevState* st = nullptr) {
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  ++ep;
  const int buf = (int)(ep & 1u);
  unsigned long long* part = ll + (size_t)buf * LL_GMAX * MAXRED * 2;
  unsigned long long* totw = ll + (size_t)2 * LL_GMAX * MAXRED * 2 + (size_t)buf * LL_R * MAXRED * 2;
  __syncthreads();  // vals complete
  for (int i = tid; i < nv; i += blockDim.x) ll_st(part + ((size_t)b * MAXRED + i) * 2, vals[i], ep);
  const unsigned long long ta = (st && st->profile && b == 0 && tid == 0) ? gtimer() : 0ull;
  bool ok = true;
  for (int col = b; col < nv; col += G) {
    double a = 0.0;
    if (tid < G && !ll_ld(part + ((size_t)tid * MAXRED + col) * 2, ep, a)) ok = false;
    a = block_sum(a, bsh);
    if (ta && col == b) {  // profiling: CTA 0 waits for its column's partials (skew + latency) -> p_reduce_arrive
      st->kstat[K_PB6].ns += gtimer() - ta;
      st->kstat[K_PB6].launches++;
    }
    if (tid < LL_R) ll_st(totw + ((size_t)tid * MAXRED + col) * 2, a, ep);
  }
  const unsigned long long* mine = totw + (size_t)(b % LL_R) * MAXRED * 2;
  for (int i = tid; i < nv; i += blockDim.x) {
    double v = 0.0;
    if (!ll_ld(mine + (size_t)i * 2, ep, v)) ok = false;
    tot[i] = v;
  }
  if (!ok) *s_fail = 1;
  __syncthreads();
  return *s_fail == 0;
}

// y_r = (A x)_r for one row (CSR thread-per-row / SELL).  x is written INSIDE this kernel (V columns
// are reused every cycle, x is updated at every cycle end), so it is gathered with ordinary coherent
// loads — never through the non-coherent read-only path (__ldg / ld.global.nc).  Visibility of other
// CTAs' rows follows from the grid barrier's release/acquire fences (the acquire fence also
// invalidates the SM's L1), and within one CTA from __syncthreads.
__device__ __forceinline__ double row_dot(const MatDev& A, int64_t row, const double* __restrict__ x) {
  double s = 0.0;
  if (A.fmt == 1) {
    const int64_t pos = A.siperm ? (int64_t)__ldg(A.siperm + row) : row;  // (sorted SELL runs the graph path)
    const int64_t sl = pos >> 5;
    const int w = __ldg(A.sw + sl);
    const int64_t base = __ldg(A.sp + sl) + (pos & 31);
    for (int c = 0; c < w; c += SELL_CH) {
      int32_t cc[SELL_CH];
      double vv[SELL_CH];
#pragma unroll
      for (int u = 0; u < SELL_CH; ++u) {
        const bool ok = c + u < w;
        const int64_t e = base + (int64_t)(c + u) * 32;
        cc[u] = ok ? __ldcs(A.sci + e) : 0;
        vv[u] = ok ? __ldcs(A.sv + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SELL_CH; ++u)
        if (c + u < w) s += vv[u] * x[cc[u]];
    }
  } else {
    const int32_t p0 = __ldg(A.rp + row), p1 = __ldg(A.rp + row + 1);
    for (int32_t p = p0; p < p1; p += 8) {
      int32_t cc[8];
      double vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = p + u < p1;
        cc[u] = ok ? __ldcs(A.ci + p + u) : 0;
        vv[u] = ok ? __ldcs(A.v + p + u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < p1) s += vv[u] * x[cc[u]];
    }
  }
  return s;
}

// CSR row from the CTA's shared-memory copy of its pattern (row pointers relative to the CTA's first
// entry): the column indices no longer need a global load, so a row costs one dependent round trip
// (value and x gathers in parallel) instead of three (row pointer -> index -> x).  Same order as row_dot.
__device__ __forceinline__ double row_dot_sc(const MatDev& A, int64_t lr, const int32_t* s_rp, const int32_t* s_ci,
                                            const double* __restrict__ vb, const double* __restrict__ x) {
  const int32_t p0 = s_rp[lr], p1 = s_rp[lr + 1];
  double s = 0.0;
  for (int32_t p = p0; p < p1; p += 8) {
    int32_t cc[8];
    double vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = p + u < p1;
      cc[u] = ok ? s_ci[p + u] : 0;
      vv[u] = ok ? __ldcs(vb + p + u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p + u < p1) s += vv[u] * x[cc[u]];
  }
  return s;
}

// phase timer (CTA 0, thread 0, profiling only): adds now - *t0 to the phase slot and resets t0
__device__ __forceinline__ void ptick(DevState* st, int kid, unsigned long long& t0) {
  if (st->profile && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    st->kstat[kid].ns += t - t0;
    st->kstat[kid].launches++;
    t0 = t;
  }
}

// VK selects the code the instantiation contains: 0 plain / deflate, 1 oblique / orthogonal, 2 augment
// (one kernel with every variant's code carried more live registers and spilled in the hot loops:
// C2 deflate +1.7 %).
// PTT: threads per CTA — RG_PT (512, 2 CTAs/SM) for multi-CTA solves, 1024 for single-CTA (tiny)
// solves, where one CTA holds the whole problem (C1: 0.80 -> 0.74 ms/system measured)
// KEEP: RG_FLAG_KEEP_BASIS (plain / deflate / augment only) — the cycle end also keeps the finished
// cycle's basis for rg_export; a separate instantiation so the default kernels are untouched.
template <int VK, int PTT, bool KEEP = false>
__global__ void __launch_bounds__(PTT, 1024 / PTT) k_solve_persistent(PArgs pa) {
  constexpr int PT = PTT;  // shadows the namespace-scope default inside this kernel
  extern __shared__ double sm[];
  const Layout& L = pa.L;
  const MatDev& A = pa.A;
  DevState* st = pa.st;
  const int m = pa.m, k = pa.k, VB = L.VB, QB = VB - k;
  const bool obl = VK == 1 && pa.obl != 0;
  constexpr bool aug = VK == 2;
  const int lo = (obl || aug) ? VB : QB, nq = (obl || aug) ? 0 : k;  // P = [Q | V] (deflate) or V
  const int nx = obl ? 2 * k : (aug ? k : 0);       // extra dots per step: W^T y, P^T u / Q^T u
  const bool orthp = VK == 1 && pa.obl == 2;        // orthogonal: projector I - W W^T (P = W, T = I)
  const int pbase = orthp ? 0 : k;                  // first column of P (C = A W at [k, 2k) or W)
  const int64_t ld = L.ld;
  double* Z = L.Z;
  // ---- shared-memory layout (replicated least-squares state + staging)
  double* Hs = sm;                           // [m][m+2]  H(r, i) = Hs[i*(m+2) + r]
  double* Rs = Hs + m * (m + 2);             // [m][m+1]
  double* Bs = Rs + m * (m + 1);             // [m+1][k]  B(l, i) = Bs[i*k + l]; oblique: (V^T C)(i, l)
  double* cs = Bs + (m + 1) * (k > 0 ? k : 1);
  double* sn = cs + PM;
  double* gg = sn + PM;                      // PM + 2
  double* h1 = gg + PM + 2;                  // PCOL: first-pass coefficients of the pending column
  double* cv = h1 + PCOL;                    // PCOL: v_j coefficients
  double* cn = cv + PCOL;                    // PCOL: next-u coefficients
  double* us = cn + PCOL;                    // PT
  double* ysm = us + PT;                     // PT
  double* dpart = ysm + PT;                  // MAXRED
  double* tot = dpart + MAXRED;              // MAXRED
  double* ys = tot + MAXRED;                 // PM + 2: cycle-end y
  double* zk = ys + PM + 2;                  // PK
  double* wk = zk + PK;                      // PK (+ PM+2 behind it: (H a)_c at wk[PK + c])
  // augment only: G (rows v_0..v_{m+1}: Q^T v_i) in Bs (sized (m+2) k), T and S = T^{-1} ([col][row])
  double* Ts = wk + PK + PM + 2;             // [(m+2)][(m+2)] when aug
  double* Ss = Ts + (aug ? (m + 2) * (m + 2) : 0);
  int32_t* s_rp = (int32_t*)(Ss + (aug ? (m + 2) * (m + 2) : 0));  // CSR cache (pa.rcap / pa.ccap entries)
  int32_t* s_ci = s_rp + pa.rcap;
  __shared__ double bsh[33];
  __shared__ int s_fail, s_stop;
  __shared__ double s_sc[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) { s_fail = 0; s_stop = 0; }
  __syncthreads();
  const bool cta0 = blockIdx.x == 0;
  if (cta0) prof_begin(st, K_MISC);
  unsigned rep = pa.llred ? *(volatile unsigned*)&st->red_epoch : 0u;  // reduction epoch (LL)
  auto gred = [&](int nv, DevState* pst) -> bool {
    return pa.llred ? greduce_ll(dpart, nv, pa.ll, tot, rep, bsh, &s_fail, pst)
                    : greduce(dpart, nv, L.partial, pa.tot_g, tot, pa.bar, &s_fail, pst);
  };
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  const double tol = st->tol;
  const int max_iters = st->max_iters, hist_cap = st->hist_cap;
  double* __restrict__ x = L.x;
  const double* __restrict__ b = L.b;
  double bytes = 0.0;  // algorithmic bytes (CTA 0 accounts them)
  int spmvs = 0;       // sparse products issued (CTA 0: rg_report.spmv_count)
  const bool keep = L.keep_l2 != 0;  // basis L2-sized: cached loads (the update pass re-hits them)
  // ---- this CTA's CSR pattern into shared memory when it fits (the SpMVs then read only values and x)
  bool sc = false;
  const double* __restrict__ sc_v = A.v;
  {
    const int64_t re = r1 < L.n ? r1 : L.n;
    if (pa.ccap > 0 && A.fmt == 0 && r0 < re && re - r0 + 1 <= pa.rcap) {
      const int32_t e0 = A.rp[r0], cnt = A.rp[re] - e0;
      if (cnt <= pa.ccap) {
        for (int64_t i = tid; i <= re - r0; i += PT) s_rp[i] = A.rp[r0 + i] - e0;
        for (int32_t e = tid; e < cnt; e += PT) s_ci[e] = A.ci[e0 + e];
        sc = true;
        sc_v = A.v + e0;
      }
    }
    __syncthreads();
  }
  // ---- column owners of this CTA's rows (neighbour sync): min / max column of its CSR entries
  __shared__ int s_clo, s_chi;
  unsigned epoch = 0;
  const bool nbs = pa.nbsync != 0 && gridDim.x > 1;
  if (nbs) {
    int cmin = INT_MAX, cmax = -1;
    const int64_t re = r1 < L.n ? r1 : L.n;
    if (r0 < re) {
      const int32_t p0 = A.rp[r0], p1 = A.rp[re];
      for (int32_t p = p0 + tid; p < p1; p += PT) {
        const int c = A.ci[p];
        cmin = min(cmin, c);
        cmax = max(cmax, c);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (tid == 0) { s_clo = INT_MAX; s_chi = -1; }
    __syncthreads();
    if (lane == 0) { atomicMin(&s_clo, cmin); atomicMax(&s_chi, cmax); }
    __syncthreads();
    if (tid == 0) {
      const int G = gridDim.x;
      s_clo = s_chi < 0 ? (int)blockIdx.x : row_owner(s_clo, ng, G);
      s_chi = s_chi < 0 ? (int)blockIdx.x : row_owner(s_chi, ng, G);
      RG_CHK(st, s_clo >= 0 && s_clo <= s_chi && s_chi < G && s_clo <= (int)blockIdx.x && (int)blockIdx.x <= s_chi &&
                     A.sperm == nullptr);
    }
    __syncthreads();
  }

  // ---- SSOR: this CTA's rows of colour c are perm[s_ilo[c] .. s_ihi[c]) (perm is row-sorted per colour)
  __shared__ int s_ilo[MAXCOLORS], s_ihi[MAXCOLORS];
  const bool prec = pa.prec != 0;
  if (prec) {
    const int64_t rend = r1 < L.n ? r1 : L.n;
    for (int c = tid; c < pa.P.ncolors; c += PT) {
      auto lower = [&](int64_t row) {  // first idx of colour c with perm[idx] >= row
        int64_t lo2 = pa.P.coff[c], hi2 = pa.P.coff[c + 1];
        while (lo2 < hi2) {
          const int64_t mid = (lo2 + hi2) >> 1;
          if (pa.P.perm[mid] < row) lo2 = mid + 1;
          else hi2 = mid;
        }
        return (int)lo2;
      };
      s_ilo[c] = lower(r0 < rend ? r0 : rend);
      s_ihi[c] = lower(rend);
    }
    __syncthreads();
  }
  // out = M^{-1} in on this CTA's rows; `in` is read on own rows only.  Sweep c waits for the
  // neighbours' previous sweep (their rows of the colours it reads are final), then publishes.
  auto ssor_apply = [&](const double* in, double* out) -> bool {
    const int nc = pa.P.ncolors;
    const double om = pa.P.omega, sc = om * (2.0 - om);
    for (int pass = 0; pass < 2 * nc - 1; ++pass) {
      const bool bwd = pass >= nc;
      const int c = bwd ? 2 * nc - 2 - pass : pass;
      if (pass > 0) {
        if (nbs) {
          if (!nb_wait(pa.flags, s_clo, s_chi, epoch, &s_fail)) return false;
        } else if (!gbar(pa.bar, &s_fail)) {
          return false;
        }
      }
      const int32_t* __restrict__ rp = bwd ? pa.P.Urp : pa.P.Lrp;
      const int32_t* __restrict__ ci = bwd ? pa.P.Uci : pa.P.Lci;
      const double* __restrict__ vv = bwd ? pa.P.Uv : pa.P.Lv;
      for (int idx = s_ilo[c] + tid; idx < s_ihi[c]; idx += PT) {
        const int32_t r = pa.P.perm[idx];
        double s = 0.0;
        for (int32_t q = rp[idx]; q < rp[idx + 1]; ++q) s += vv[q] * out[ci[q]];
        const double di = pa.P.dinv[idx];
        out[r] = bwd ? out[r] - om * s * di : (sc * in[r] - om * s) * di;
      }
      if (nbs) nb_publish(pa.flags, ++epoch);
      else __syncthreads();
    }
    if (nbs) return nb_wait(pa.flags, s_clo, s_chi, epoch, &s_fail);  // out complete on the owners
    return gbar(pa.bar, &s_fail);
  };

  // ---- ||b||
  {
    double s = 0.0;
    for (int64_t r = r0 + tid; r < r1; r += PT) s += b[r] * b[r];
    s = block_sum(s, bsh);
    if (tid == 0) dpart[0] = s;
    __syncthreads();
    if (!gred(1, nullptr)) goto fail;
  }
  {
  const double bnorm = sqrt(tot[0]);
  if (!(bnorm > 0.0)) {
    if (cta0 && tid == 0) {
      st->bnorm = bnorm;
      st->bzero = bnorm == 0.0;
      st->done = 1;
      st->converged = st->bzero;
      if (!st->bzero) st->status = RG_E_NUMERIC;
    }
    goto out;
  }
  int iters = 0, cycles = 0, hist_len = 0, converged = 0, status = 0;
  double beta = 0.0, relres = 0.0;
  for (;;) {
    // ================= cycle start: r = b - A x into V column 0 (+ Q^T r, ||r||^2)
    if (nbs) {  // x of the column owners complete
      if (!nb_wait(pa.flags, s_clo, s_chi, epoch, &s_fail)) goto fail;
    } else if (!gbar(pa.bar, &s_fail)) {
      goto fail;
    }
    double* __restrict__ u0 = Z + (int64_t)VB * ld;
    {
      double s = 0.0;
      for (int64_t r = r0 + tid; r < r1; r += PT) {
        const double rr = r < L.n ? b[r] - (sc ? row_dot_sc(A, r - r0, s_rp, s_ci, sc_v, x) : row_dot(A, r, x)) : 0.0;
        u0[r] = rr;
        s += rr * rr;
      }
      s = block_sum(s, bsh);
      if (tid == 0) dpart[0] = s;
      __syncthreads();
      if (!gred(1, nullptr)) goto fail;
      beta = sqrt(tot[0]);
      if (cta0) { bytes += A.bytes + 8.0 * L.n; ++spmvs; }
    }
    if (k > 0) {  // LS projection onto span(W): a = Q^T r, x += W R_C^{-1} a, r -= Q a
                  // (oblique: Galerkin start a = W^T r, t = E^{-1} a, x += W t, r -= C t)
      for (int c = tid; c < k; c += PT) dpart[c] = 0.0;
      __syncthreads();
      for (int64_t base = r0; base < r1; base += PT) {
        const int64_t r = base + tid;
        us[tid] = r < r1 ? u0[r] : 0.0;
        __syncthreads();
        const int cnt = (int)min((int64_t)PT, r1 - base);
        for (int c = wid; c < k; c += PT / 32) {
          const double* zc = Z + (int64_t)((obl ? 0 : QB) + c) * ld + base;
          double s = 0.0;
          for (int q = lane; q < cnt; q += 32) s += zc[q] * us[q];
          s = warp_sum(s);
          if (lane == 0) dpart[c] += s;
        }
        __syncthreads();
      }
      if (!gred(k, nullptr)) goto fail;
      for (int l = tid; l < k; l += PT) {  // z = R_C^{-1} a  (oblique: t = E^{-1} a)
        double s = 0.0;
        if (obl) {
          for (int c = 0; c < k; ++c) s += st->Einv[c][l] * tot[c];
        } else {
          for (int c = l; c < k; ++c) s += st->RCinv[c][l] * tot[c];
        }
        zk[l] = s;
      }
      __syncthreads();
      const double* rq = obl ? zk : tot;            // r -= Q a  or  r -= C t
      const int rb = obl ? k : QB;
      double s2 = 0.0;
      for (int64_t r = r0 + tid; r < r1; r += PT) {
        double xr = x[r], rr = u0[r];
        for (int l = 0; l < k; ++l) {
          xr += zk[l] * Z[(int64_t)l * ld + r];
          rr -= rq[l] * Z[(int64_t)(rb + l) * ld + r];
        }
        x[r] = xr;
        u0[r] = rr;
        s2 += rr * rr;
      }
      s2 = block_sum(s2, bsh);
      if (tid == 0) dpart[0] = s2;
      __syncthreads();
      if (!gred(1, nullptr)) goto fail;
      beta = sqrt(tot[0]);
      if (cta0) bytes += 8.0 * L.n * (4 * k + 4);
    }
    relres = beta / bnorm;
    if (!isfinite(beta)) { status = RG_E_NUMERIC; break; }
    if (relres <= tol) { converged = 1; break; }
    if (iters >= max_iters) break;
    ++cycles;
    if (tid == 0) gg[0] = beta;
    for (int i = tid; i < PCOL; i += PT) h1[i] = 0.0;
    if (aug) {  // v_0 = r_c / beta with Q^T r_c = 0 after the cycle-start projection: G[0,:] = 0, T00 = S00 = 1
      for (int l = tid; l < k; l += PT) Bs[l] = 0.0;
      if (tid == 0) { Ts[0] = 1.0; Ss[0] = 1.0; }
    }
    __syncthreads();
    // ================= Arnoldi steps (DCGS2), u = V column j (raw), y -> V column j+1
    int jf = -1;
    for (int j = 0; j <= m; ++j) {
      const int p = nq + j;
      RG_CHK(st, m <= MAXM && VB + j < L.ncol && (j == m || VB + j + 1 < L.ncol) && p <= MAXCOL && nq <= MAXK);
      double* __restrict__ u = Z + (int64_t)(VB + j) * ld;
      double* __restrict__ y = Z + (int64_t)(VB + j + 1) * ld;
      const bool have_y = j < m;
      unsigned long long tph = (st->profile && cta0 && tid == 0) ? gtimer() : 0ull;
      if (j > 0) {  // u complete (on the column owners' rows)
        if (nbs) {
          if (!nb_wait(pa.flags, s_clo, s_chi, epoch, &s_fail)) goto fail;
        } else if (!gbar(pa.bar, &s_fail)) {
          goto fail;
        }
      }
      ptick(st, K_PB1, tph);
      if (pa.skew && cycles == 1 && j == pa.skew && tid == 0) {  // experiment: step start, SM id
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pa.flags[NSM * 2 + 1 * NSM * 2 + blockIdx.x] = (unsigned)(gtimer() & 0xffffffffu);
        pa.flags[NSM * 2 + 3 * NSM * 2 + blockIdx.x] = smid;
      }
      const int nv = 2 * p + 2 + nx;
      for (int c = tid; c < nv; c += PT) dpart[c] = 0.0;
      double s_uu = 0.0, s_uy = 0.0;
      if (have_y) {  // SpMV over this CTA's rows first (many rows in flight), then the dot pass
        const double* sx = u;
        if (prec) {  // y = A M^{-1} u
          if (!ssor_apply(u, pa.pz)) goto fail;
          sx = pa.pz;
          if (cta0) bytes += pa.pc_bytes;
        }
        if (sc) {
          for (int64_t r = r0 + tid; r < r1; r += PT) y[r] = r < L.n ? row_dot_sc(A, r - r0, s_rp, s_ci, sc_v, sx) : 0.0;
        } else {
          for (int64_t r = r0 + tid; r < r1; r += PT) y[r] = r < L.n ? row_dot(A, r, sx) : 0.0;
        }
      }
      if (st->profile && cta0 && tid == 0) {  // sub-interval of p_spmv_dots: the SpMV alone
        st->kstat[K_PB7].ns += gtimer() - tph;
        st->kstat[K_PB7].launches++;
      }
      for (int64_t base = r0; base < r1; base += PT) {
        const int64_t r = base + tid;
        double ur = 0.0, yr = 0.0;
        if (r < r1) {
          ur = u[r];
          if (have_y) yr = y[r];  // written by this thread above
        }
        __syncthreads();
        us[tid] = ur;
        ysm[tid] = yr;
        s_uu += ur * ur;
        s_uy += ur * yr;
        __syncthreads();
        const int cnt = (int)min((int64_t)PT, r1 - base);
        constexpr int RPL = 16;
        for (int c = wid; c < p + nx; c += PT / 32) {
          const int zcol = c < p ? lo + c : (aug ? QB + (c - p) : ((c - p) < k ? c - p : pbase + (c - p - k)));
          double su = 0.0, sy = 0.0;
#pragma unroll 1
          for (int h = 0; h < PT / (32 * RPL); ++h) {
            const int lh = lane + 32 * RPL * h;
            const double* zc = Z + (int64_t)zcol * ld + base + lh;
            double zv[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q)  // 16 independent loads in flight per lane
              zv[q] = (lh + 32 * q < cnt) ? (keep ? zc[32 * q] : __ldcs(zc + 32 * q)) : 0.0;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
              su += zv[q] * us[lh + 32 * q];
              sy += zv[q] * ysm[lh + 32 * q];
            }
          }
          su = warp_sum(su);
          sy = warp_sum(sy);
          if (lane == 0) {
            if (c < p) {
              dpart[c] += su;
              dpart[p + c] += sy;
            } else {  // extras after [a | b | s | g]: oblique [W^T y (k) | P^T u (k)], augment Q^T u (k)
              dpart[2 * p + 2 + (c - p)] += (!aug && (c - p) < k) ? sy : su;
            }
          }
        }
      }
      {
        const double t1 = block_sum(s_uu, bsh);
        const double t2 = block_sum(s_uy, bsh);
        if (tid == 0) { dpart[2 * p] = t1; dpart[2 * p + 1] = t2; }
        __syncthreads();
      }
      ptick(st, K_PB2, tph);
      if (pa.skew && cycles == 1 && j == pa.skew && tid == 0) {  // experiment: dots done
        pa.flags[NSM * 2 + blockIdx.x] = (unsigned)(gtimer() & 0xffffffffu);
      }
      if (!gred(nv, st)) goto fail;
      if (pa.skew && cycles == 1 && j == pa.skew && tid == 0) {  // experiment: reduction done
        pa.flags[NSM * 2 + 2 * NSM * 2 + blockIdx.x] = (unsigned)(gtimer() & 0xffffffffu);
      }
      ptick(st, K_PB3, tph);
      if (cta0) { bytes += (have_y ? A.bytes : 0.0) + 8.0 * L.n * (p + nx + 2); spmvs += have_y ? 1 : 0; }
      // ---- replicated epilogue: delayed second pass, column j-1, least squares
      const double* a = tot;
      const double* bb = tot + p;
      const double ss = tot[2 * p], gm = tot[2 * p + 1];
      if (wid < 2) {
        double acc = 0.0;
        for (int c = lane; c < p; c += 32) acc += a[c] * (wid == 0 ? a[c] : bb[c]);
        acc = warp_sum(acc);
        if (lane == 0) s_sc[wid] = acc;
      }
      __syncthreads();
      const double nu2 = ss - s_sc[0], ab = s_sc[1];
      const double nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
      if (j >= 1) {
        const int col = j - 1;
        for (int i = tid; i < j; i += PT) Hs[col * (m + 2) + i] = h1[nq + i] + a[nq + i];
        for (int l = tid; l < nq; l += PT) Bs[col * k + l] = h1[l] + a[l];
        if (tid == 0) Hs[col * (m + 2) + j] = nu;
        __syncthreads();
        const int M2 = m + 2;
        int aug_tb = 0;  // (kept for the Givens step below: no augment-specific breakdown any more, see tau = 0)
        if (aug) {
          // G row j = Q^T v_j = (Q^T u - G_j^T a) / nu; then the new column of T (Cholesky factor of
          // M = I - G^T G) and of S = T^{-1}; the least squares runs on M H-bar column col = T h.
          const double* qu = tot + 2 * p + 2;
          for (int l = tid; l < k; l += PT) {
            double g = qu[l];
            for (int i = 0; i < j; ++i) g -= Bs[i * k + l] * a[i];
            Bs[j * k + l] = nu > 0.0 ? g / nu : 0.0;
          }
          __syncthreads();
          for (int i = wid; i <= j; i += PT / 32) {  // mc_i = delta_ij - G_i . G_j  -> cv[i]
            double sacc = 0.0;
            for (int l = lane; l < k; l += 32) sacc += Bs[i * k + l] * Bs[j * k + l];
            sacc = warp_sum(sacc);
            if (lane == 0) cv[i] = (i == j ? 1.0 : 0.0) - sacc;
          }
          __syncthreads();
          for (int i = wid; i < j; i += PT / 32) {  // t_i = sum_{l <= i} S(l, i) mc_l -> cn[i]
            double sacc = 0.0;
            for (int l = lane; l <= i; l += 32) sacc += Ss[i * M2 + l] * cv[l];
            sacc = warp_sum(sacc);
            if (lane == 0) cn[i] = sacc;
          }
          __syncthreads();
          if (tid == 0) {
            double t2 = 0.0;
            for (int i = 0; i < j; ++i) t2 += cn[i] * cn[i];
            const double tau2 = cv[j] - t2;
            s_sc[2] = tau2 > 1e-14 ? sqrt(tau2) : 0.0;
          }
          __syncthreads();
          // tau = 0 (tau^2 <= 1e-14): v_j adds nothing outside span(Q) + span(V_j); the column is accepted
          // with a vanishing last row of M = T H-bar (zero projected residual) and ends the cycle — see
          // epi_ls (epilogue.cuh); S = T^{-1} is only needed by later columns
          aug_tb = 0;
          {
            const double tau = s_sc[2];
            if (tau > 0.0) {
              for (int l = wid; l < j; l += PT / 32) {  // S(l, j) = -(sum_{i >= l} S(l, i) t_i) / tau
                double sacc = 0.0;
                for (int i = l + lane; i < j; i += 32) sacc += Ss[i * M2 + l] * cn[i];
                sacc = warp_sum(sacc);
                if (lane == 0) Ss[j * M2 + l] = -sacc / tau;
              }
            }
            for (int i = tid; i < j; i += PT) Ts[j * M2 + i] = cn[i];
            if (tid == 0) {
              Ts[j * M2 + j] = tau;
              if (tau > 0.0) Ss[j * M2 + j] = 1.0 / tau;
            }
            __syncthreads();
            for (int i = wid; i <= j; i += PT / 32) {  // column col of M = T H: sum_{l >= i} T(i, l) h_l -> ys[i]
              double sacc = 0.0;
              for (int l = i + lane; l <= j; l += 32) sacc += Ts[l * M2 + i] * Hs[col * M2 + l];
              sacc = warp_sum(sacc);
              if (lane == 0) ys[i] = sacc;
            }
            __syncthreads();
          }
        }
        if (tid == 0) {  // Givens on column col (same arithmetic in every CTA)
          // the rotated entry travels in a register; the loads of H, cs, sn do not depend on the
          // chain, so the unrolled loop keeps them in flight (2 FMAs per rotation on the chain)
          const double* Hc = aug ? ys : Hs + col * (m + 2);
          double* Rc = Rs + col * (m + 1);
          double carry = Hc[0];
#pragma unroll 4
          for (int i = 0; i < col; ++i) {
            const double x1 = Hc[i + 1], ci = cs[i], si = sn[i];
            Rc[i] = ci * carry + si * x1;
            carry = -si * carry + ci * x1;
          }
          const double hlast = Hc[col + 1];
          const double den = hypot(carry, hlast);
          int stop = 0;
          if (aug_tb || !(den > 0.0)) {
            stop = 2;  // no progress possible: end the cycle at the previous column
          } else {
            const double c = carry / den, s = hlast / den;
            cs[col] = c;
            sn[col] = s;
            Rc[col] = den;
            const double gj = gg[col];
            gg[col] = c * gj;
            gg[col + 1] = -s * gj;
            const double res = fabs(s * gj) / bnorm;
            if (cta0 && hist_len < hist_cap) L.hist[hist_len] = res;
            if (!isfinite(res)) stop = 3;
            else if (res <= tol || nu <= 1e-14 * beta || col + 1 >= m || iters + 1 >= max_iters ||
                     (aug && !(s_sc[2] > 0.0)))
              stop = 1;
          }
          s_stop = stop;
        } else if (wid > 0) {
          // meanwhile warps 1..: the products (H a_V)_c and (B a_V)_l of the coefficient step below
          // (they read the unrotated H and B only, not the rotation thread 0 is computing)
          for (int o = wid - 1; o < j + nq; o += PT / 32 - 1) {
            double s = 0.0;
            if (o < j) {
              for (int i = (o > 0 ? o - 1 : 0) + lane; i < j; i += 32) s += Hs[i * (m + 2) + o] * a[nq + i];
            } else {
              for (int i = lane; i < j; i += 32) s += Bs[i * k + (o - j)] * a[nq + i];
            }
            s = warp_sum(s);
            if (lane == 0) wk[o < j ? PK + o : o - j] = s;  // reuse: [0,k) Ba, [PK, PK+j) Ha
          }
        }
        __syncthreads();
        ++iters;
        if (hist_len < hist_cap && s_stop != 2) ++hist_len;
        if (s_stop) {
          jf = s_stop == 2 ? col - 1 : (s_stop == 3 ? -1 : col);
          if (s_stop == 3) status = RG_E_NUMERIC;
          break;
        }
      }
      // ---- coefficients of the update pass and first-pass coefficients of column j
      const double inv = nu > 0.0 ? 1.0 / nu : 0.0;
      const double aj = j >= 1 ? a[nq + j - 1] : 0.0;
      const double d = ((gm - ab) * inv - nu * aj) * inv;
      if (obl) {  // t = E^{-1} W^T y -> wk[0,k) = -t/nu (C coefficients of the next u); row j of V^T C
        const double* wy = tot + 2 * p + 2;
        const double* cu = wy + k;
        for (int l = tid; l < k; l += PT) {
          double t = 0.0;
          if (orthp) t = wy[l];
          else
            for (int c = 0; c < k; ++c) t += st->Einv[c][l] * wy[c];
          zk[l] = t;
          double g = cu[l];
          for (int i = 0; i < j; ++i) g -= a[i] * Bs[i * k + l];
          Bs[j * k + l] = g * inv;
        }
        __syncthreads();
        for (int i = wid; i <= j; i += PT / 32) {  // ct_i = (V^T C t)_i -> ys[i] (free until cycle end)
          double s = 0.0;
          for (int l = lane; l < k; l += 32) s += Bs[i * k + l] * zk[l];
          s = warp_sum(s);
          if (lane == 0) ys[i] = s;
        }
        for (int l = tid; l < k; l += PT) wk[l] = -zk[l] * inv;
        __syncthreads();
      }
      const double dob = obl ? ((gm - ab) * inv - nu * aj - ys[j]) * inv : d;
      const double f = (aj + dob) * inv;
      if (j == 0) {  // (for j >= 1 computed during the Givens step above)
        for (int o = wid; o < j + nq; o += PT / 32) {  // (H a_V)_c and (B a_V)_l
          double s = 0.0;
          if (o < j) {
            for (int i = (o > 0 ? o - 1 : 0) + lane; i < j; i += 32) s += Hs[i * (m + 2) + o] * a[nq + i];
          } else {
            for (int i = lane; i < j; i += 32) s += Bs[i * k + (o - j)] * a[nq + i];
          }
          s = warp_sum(s);
          if (lane == 0) wk[o < j ? PK + o : o - j] = s;  // reuse: [0,k) Ba, [PK, PK+j) Ha
        }
      }
      __syncthreads();
      for (int c = tid; c < j; c += PT) {
        const double Ha = wk[PK + c];
        const double cvv = (bb[nq + c] - Ha - (obl ? ys[c] : 0.0)) * inv;
        cn[nq + c] = -Ha * inv - cvv + f * a[nq + c];
        cv[nq + c] = -a[nq + c] * inv;
        h1[nq + c] = cvv;
      }
      for (int l = tid; l < nq; l += PT) {
        cn[l] = -bb[l] * inv + f * a[l];
        cv[l] = -a[l] * inv;
        h1[l] = (bb[l] - wk[l]) * inv;
      }
      if (tid == 0) h1[nq + j] = dob;
      __syncthreads();
      ptick(st, K_PB4, tph);
      // ---- update pass: v_j = u/nu + P cv, u_next = y/nu - f u + P cn (- C t/nu)  (own rows)
      const double fu = -(aj + dob) * inv;
      for (int64_t r = r0 + tid; r < r1; r += PT) {
        const double ur = u[r], yr = y[r];
        double sv = 0.0, sn2 = 0.0;
        int c = p;  // columns in DESCENDING order: the dot pass just streamed them ascending, so the
                    // most recently touched ones come first (LRU-friendly when the basis nears the L2 size)
        for (; c >= 8; c -= 8) {  // 8 independent loads in flight
          double z[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const double* zp = Z + (int64_t)(lo + c - 1 - t) * ld + r;
            z[t] = keep ? *zp : __ldcs(zp);
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            sv += cv[c - 1 - t] * z[t];
            sn2 += cn[c - 1 - t] * z[t];
          }
        }
        for (; c > 0; --c) {
          const double z = Z[(int64_t)(lo + c - 1) * ld + r];
          sv += cv[c - 1] * z;
          sn2 += cn[c - 1] * z;
        }
        if (obl)
          for (int l = 0; l < k; ++l) sn2 += wk[l] * Z[(int64_t)(pbase + l) * ld + r];
        u[r] = ur * inv + sv;
        y[r] = yr * inv + ur * fu + sn2;
      }
      if (cta0) bytes += 8.0 * L.n * (p + (obl ? k : 0) + 4);
      if (nbs) nb_publish(pa.flags, ++epoch);  // u complete on this CTA's rows
      else __syncthreads();
      ptick(st, K_PB5, tph);
    }
    // ================= cycle end: y = R^{-1} g, x += V y - W R_C^{-1} B y (own rows)
    if constexpr (KEEP) {  // RG_FLAG_KEEP_BASIS: this cycle's V (own rows), H-bar and B (CTA 0) for rg_export
      if (jf >= 0) {
        for (int i = 0; i <= jf; ++i)
          for (int64_t r = r0 + tid; r < r1; r += PT) L.keepV[(int64_t)i * ld + r] = Z[(int64_t)(VB + i) * ld + r];
        if (cta0) {
          for (int e = tid; e < (jf + 1) * (m + 2); e += PT) st->Hraw[e / (m + 2)][e % (m + 2)] = e % (m + 2) <= e / (m + 2) + 1 ? Hs[e] : 0.0;
          if (!aug)
            for (int e = tid; e < (jf + 1) * k; e += PT) st->Bm[e / k][e % k] = Bs[e];
          if (tid == 0) st->kb_steps = jf + 1;
        }
      }
    }
    if (jf >= 0) {
      if (tid == 0) {
        for (int i = jf; i >= 0; --i) {
          double s = gg[i];
          for (int l = i + 1; l <= jf; ++l) s -= Rs[l * (m + 1) + i] * ys[l];
          ys[i] = s / Rs[i * (m + 1) + i];
        }
      }
      __syncthreads();
      const int kx = obl ? 0 : k;  // oblique: x += V y (the next cycle start applies the W part)
      if (kx > 0 && aug) {  // x -= W R_C^{-1} G H-bar y
        for (int i = wid; i <= jf + 1; i += PT / 32) {  // (H-bar y)_i -> cv[i] (Hessenberg)
          double s = 0.0;
          for (int c2 = (i > 0 ? i - 1 : 0) + lane; c2 <= jf; c2 += 32) s += Hs[c2 * (m + 2) + i] * ys[c2];
          s = warp_sum(s);
          if (lane == 0) cv[i] = s;
        }
        __syncthreads();
        for (int l = wid; l < k; l += PT / 32) {
          double s = 0.0;
          for (int i = lane; i <= jf + 1; i += 32) s += Bs[i * k + l] * cv[i];
          s = warp_sum(s);
          if (lane == 0) wk[l] = s;
        }
        __syncthreads();
        for (int l = tid; l < k; l += PT) {
          double s = 0.0;
          for (int c = l; c < k; ++c) s += st->RCinv[c][l] * wk[c];
          zk[l] = s;
        }
        __syncthreads();
      } else if (kx > 0) {
        for (int l = tid; l < k; l += PT) {
          double s = 0.0;
          for (int i = 0; i <= jf; ++i) s += Bs[i * k + l] * ys[i];
          wk[l] = s;
        }
        __syncthreads();
        for (int l = tid; l < k; l += PT) {
          double s = 0.0;
          for (int c = l; c < k; ++c) s += st->RCinv[c][l] * wk[c];
          zk[l] = s;
        }
        __syncthreads();
      }
      if (prec) {  // x += M^{-1} (V y) - W part
        for (int64_t r = r0 + tid; r < r1; r += PT) {
          double t = 0.0;
          for (int i = 0; i <= jf; ++i) t += ys[i] * Z[(int64_t)(VB + i) * ld + r];
          pa.pt[r] = t;
        }
        __syncthreads();
        if (!ssor_apply(pa.pt, pa.pz)) goto fail;
        if (cta0) bytes += pa.pc_bytes + 16.0 * L.n;
      }
      for (int64_t r = r0 + tid; r < r1; r += PT) {
        double xr = x[r];
        if (prec) {
          xr += pa.pz[r];
        } else {
          for (int i = 0; i <= jf; ++i) xr += ys[i] * Z[(int64_t)(VB + i) * ld + r];
        }
        for (int l = 0; l < kx; ++l) xr -= zk[l] * Z[(int64_t)l * ld + r];
        x[r] = xr;
      }
      if (cta0) bytes += 8.0 * L.n * (jf + 1 + kx + 2);
      if (nbs) nb_publish(pa.flags, ++epoch);  // x complete on this CTA's rows
    }
    if (status) break;
  }
  if (cta0 && tid == 0) {
    st->bnorm = bnorm;
    st->beta = beta;
    st->relres = relres;
    st->iters = iters;
    st->cycles = cycles;
    st->spmv_count += spmvs;
    st->hist_len = hist_len;
    st->converged = converged;
    st->status = status;
    st->done = 1;
    prof_end(st, K_MISC, bytes);
  }
  }
out:
  if (pa.llred && cta0 && tid == 0) st->red_epoch = rep;
  return;
fail:
  if (cta0 && tid == 0) {
    st->status = RG_E_CUDA;
    st->done = 1;
    if (pa.llred) st->red_epoch = rep + 16u;  // past anything a CTA may have published
  }
}

// ---- recycle-operator build as ONE cooperative kernel (replaces build_c's chain of ~10 launches —
// SpMM, 2 x (Gram, reduce, Cholesky, X*M), R_C finish — measured 165 us per C2 system, mostly launch
// ramps and single-CTA tails).  P:310: the deflation projector uses an orthonormal basis of C = A W;
// here C = A W (this CTA's rows, W complete from rg_build_recycle), CholQR2 with the two Gram
// matrices grid-reduced (deterministic, fixed order) and the k x k Cholesky factors computed
// REDUNDANTLY by every CTA (identical inputs and code: identical results, no broadcast), Q = C
// R1^{-1} R2^{-1} in place in the Q columns; CTA 0 writes R_C = R2 R1 and R_C^{-1} = R1^{-1} R2^{-1}
// to the device state and flags a singular factor (same tests as k_chol / k_rc_finish).  A separate
// kernel, not a prologue of k_solve_persistent: inside it the extra code perturbed the register
// allocation of the Arnoldi loop (update pass 8.8 -> 11.7 us per step at C2).
// Thread per row (all k <= KC columns in registers: every load of a row is in flight at once);
// rows staged in PT-row tiles [KC][PT] for the Gram, which is register-blocked: warp w owns the 4 x 4
// blocks w and w + 16 (a-block <= b-block) of the k x k Gram and accumulates them over all of the
// CTA's rows (lanes over rows), reduced across lanes once per pass.
// CGIVEN: C = A W is already in the Q columns (BSR: the TMA + DMMA SpMM ran first); the kernel then is
// the CholQR2 alone (replaces 2 x (Gram, reduce, Cholesky, X R^{-1}) + R_C finish: 8 launches).
// FP64 tensor-core MMA (DMMA.8x8x4): C[8x8] += A[8x4] B[4x8]; fragments (PTX m8n8k4 .f64):
// a: A(lane/4, lane%4), b: B(lane%4, lane/4), c{0,1}: C(lane/4, 2*(lane%4) + {0,1}).
__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int KC, bool CGIVEN = false>
__global__ void __launch_bounds__(PT, 1) k_cbuild(const __grid_constant__ PArgs pa, int* cflag) {
  // Gram of the staged rows: warp w stages ITS 32 rows of a tile ([KC][CB_TSW] column-major, rows past
  // the CTA's range zero) and accumulates the upper 8 x 8 block pairs (I <= J) of their Gram with FP64
  // DMMA (m8n8k4: 8 k-steps over the 32 rows) in registers across all tiles: no CTA barrier per tile
  // (the first version staged PT-row tiles for 4 x 4 register blocks owned by NB(NB+1)/2 warps: two
  // __syncthreads per tile, the other warps idle — C4 k = 8: 462 us, barrier-stall bound).
  constexpr int NBK = KC / 8, NPR = NBK * (NBK + 1) / 2, NWP = PT / 32;
  extern __shared__ double sm[];
  double* tile = sm;                   // per warp [KC][CB_TSW]; after a pass: per-warp Gram partials
  double* R1 = tile + KC * NWP * CB_TSW;  // [col][row], k x k each
  double* R1i = R1 + CBK * CBK;
  double* R2 = R1i + CBK * CBK;
  double* R2i = R2 + CBK * CBK;
  double* dpart = R2i + CBK * CBK;     // MAXRED
  double* tot = dpart + MAXRED;        // MAXRED
  __shared__ double bsh[33];
  __shared__ int s_fail;
  const Layout& L = pa.L;
  const MatDev& A = pa.A;
  DevState* st = pa.st;
  const int k = pa.k, QB = L.VB - k, P2 = k * (k + 1) / 2;
  RG_CHK(pa.st, k >= 1 && k <= KC && k <= CBK && QB >= k && P2 <= MAXRED);
  const int64_t ld = L.ld;
  double* Qc = L.Z + (int64_t)QB * ld;
  const double* __restrict__ Wc = L.Z;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool cta0 = blockIdx.x == 0;
  if (cta0) prof_begin(st, K_CBUILD);
  if (tid == 0) s_fail = 0;
  unsigned rep = pa.llred ? *(volatile unsigned*)&st->red_epoch : 0u;
  const int64_t ng = ld >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * ng / gridDim.x) << 5;
  const int64_t r1 = ((int64_t)(blockIdx.x + 1) * ng / gridDim.x) << 5;
  auto gred = [&](int nv) -> bool {
    return pa.llred ? greduce_ll(dpart, nv, pa.ll, tot, rep, bsh, &s_fail, nullptr)
                    : greduce(dpart, nv, L.partial, pa.tot_g, tot, pa.bar, &s_fail, nullptr);
  };
  double* wt = tile + wid * KC * CB_TSW;
  double gacc[NPR][2];
  auto gram_zero = [&]() {
#pragma unroll
    for (int q = 0; q < NPR; ++q) gacc[q][0] = gacc[q][1] = 0.0;
  };
  auto gram_rows = [&]() {  // the warp's staged 32 rows
    __syncwarp();
    int q = 0;
#pragma unroll
    for (int I = 0; I < NBK; ++I)
#pragma unroll
      for (int J = I; J < NBK; ++J, ++q) {
        const double* ta = wt + (8 * I + (lane >> 2)) * CB_TSW + (lane & 3);
        const double* tb = wt + (8 * J + (lane >> 2)) * CB_TSW + (lane & 3);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma_f64(gacc[q][0], gacc[q][1], ta[4 * kk], tb[4 * kk]);
      }
    __syncwarp();
  };
  auto gram_flush = [&]() {  // per-warp blocks -> shared, warps summed in index order -> dpart (packed upper)
    __syncthreads();  // every warp is done with its tile region (reused here)
    int q = 0;
#pragma unroll
    for (int I = 0; I < NBK; ++I)
#pragma unroll
      for (int J = I; J < NBK; ++J, ++q) {
        const int a2 = 8 * I + (lane >> 2), b2 = 8 * J + 2 * (lane & 3);
        tile[(size_t)wid * KC * KC + a2 * KC + b2] = gacc[q][0];
        tile[(size_t)wid * KC * KC + a2 * KC + b2 + 1] = gacc[q][1];
      }
    __syncthreads();
    for (int e = tid; e < k * k; e += PT) {
      const int a2 = e / k, b2 = e % k;
      if (a2 > b2) continue;
      double v = 0.0;
      for (int w = 0; w < NWP; ++w) v += tile[(size_t)w * KC * KC + a2 * KC + b2];
      dpart[a2 * k - a2 * (a2 - 1) / 2 + (b2 - a2)] = v;
    }
    __syncthreads();
  };
  // upper Cholesky G = R^T R of the packed upper Gram in `tot` (warp 0), R^{-1} (lane c: column c)
  auto chol = [&](double* R, double* Ri) {
    if (wid == 0) {
      auto g = [&](int a2, int b2) {
        const int a3 = a2 < b2 ? a2 : b2, b3 = a2 < b2 ? b2 : a2;
        return tot[a3 * k - a3 * (a3 - 1) / 2 + (b3 - a3)];
      };
      for (int jj = 0; jj < k; ++jj) {
        if (lane == 0) {
          double d = g(jj, jj);
          for (int l = 0; l < jj; ++l) d -= R[jj * k + l] * R[jj * k + l];
          if (!(d > 0.0)) { if (cta0) *cflag = 1; d = 1.0; }
          R[jj * k + jj] = sqrt(d);
        }
        __syncwarp();
        for (int i = jj + 1 + lane; i < k; i += 32) {
          double v = g(i, jj);
          for (int l = 0; l < jj; ++l) v -= R[jj * k + l] * R[i * k + l];
          R[i * k + jj] = v / R[jj * k + jj];
        }
        __syncwarp();
      }
      for (int c = lane; c < k; c += 32) {
        for (int r = k - 1; r >= 0; --r) {
          double v = (r == c) ? 1.0 : 0.0;
          for (int l = r + 1; l <= c; ++l) v -= R[l * k + r] * Ri[c * k + l];
          Ri[c * k + r] = r <= c ? v / R[r * k + r] : 0.0;
        }
      }
    }
    __syncthreads();
  };
  // row r of the Q columns times an upper-triangular inverse (this thread owns the row); computed in
  // place in x, columns descending (column c needs x_0..x_c only: one KC-vector of registers)
  auto row_load = [&](int64_t r, double* x) {
#pragma unroll
    for (int l = 0; l < KC; ++l) x[l] = l < k ? Qc[(int64_t)l * ld + r] : 0.0;
  };
  auto tri = [&](const double* Ri, double* x) {
#pragma unroll
    for (int c = KC - 1; c >= 0; --c) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l <= c; ++l) acc += x[l] * Ri[c * k + l];
      x[c] = acc;
    }
  };
  // KC = 8: the next row's values are loaded while this row's triangular products run (16 loads in
  // flight per thread in the streaming passes 2 and 3); wider rows would spill
  constexpr bool PF = KC <= 8;
  for (int i = tid; i < MAXRED; i += PT) dpart[i] = 0.0;
  for (int i = tid; i < 4 * CBK * CBK; i += PT) R1[i] = 0.0;
  __syncthreads();
  // pass 1: C = A W into the Q columns (padding rows stay 0), Gram of C
  gram_zero();
  for (int64_t base = r0; base < r1; base += PT) {
    const int64_t r = base + tid;
    const int cnt = (int)min((int64_t)PT, r1 - base);
    if (tid < cnt) {
      double acc[KC];
#pragma unroll
      for (int u = 0; u < KC; ++u) acc[u] = 0.0;
      if (CGIVEN) {
#pragma unroll
        for (int u = 0; u < KC; ++u) acc[u] = u < k ? Qc[(int64_t)u * ld + r] : 0.0;
      } else if (r < L.n) {
        // 8 (value, column) pairs in flight, then the W gathers of every column in flight
        int64_t e0, est;
        int ne;
        if (A.fmt == 1) {
          const int64_t pos = A.siperm ? (int64_t)__ldg(A.siperm + r) : r;  // row -> SELL position (sigma > 1)
          const int64_t sl = pos >> 5;
          ne = __ldg(A.sw + sl);
          e0 = __ldg(A.sp + sl) + (pos & 31);
          est = 32;
        } else {
          e0 = __ldg(A.rp + r);
          ne = __ldg(A.rp + r + 1) - (int32_t)e0;
          est = 1;
        }
        const double* __restrict__ av = A.fmt == 1 ? A.sv : A.v;
        const int32_t* __restrict__ ac = A.fmt == 1 ? A.sci : A.ci;
        for (int q0 = 0; q0 < ne; q0 += 8) {
          double vv[8];
          int32_t cc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const bool okq = q0 + q < ne;
            vv[q] = okq ? __ldcs(av + e0 + (int64_t)(q0 + q) * est) : 0.0;
            cc[q] = okq ? __ldcs(ac + e0 + (int64_t)(q0 + q) * est) : 0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q0 + q < ne) {
#pragma unroll
              for (int u = 0; u < KC; ++u)
                if (u < k) acc[u] += vv[q] * __ldg(Wc + (int64_t)u * ld + cc[q]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < KC; ++u) {
        if (u < k && !CGIVEN) Qc[(int64_t)u * ld + r] = acc[u];
        wt[u * CB_TSW + lane] = acc[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < KC; ++u) wt[u * CB_TSW + lane] = 0.0;
    }
    gram_rows();
  }
  gram_flush();
  bool ok = gred(P2);
  if (ok) chol(R1, R1i);
  // pass 2: Gram of Q1 = C R1^{-1}, Q1 NOT stored (pass 3 recomputes it from C with the same arithmetic:
  // one n x k write and its re-read less than storing Q1)
  gram_zero();
  {
    double nx[KC];
    if (ok && r0 + tid < r1) row_load(r0 + tid, nx);
    for (int64_t base = r0; ok && base < r1; base += PT) {
      const int64_t r = base + tid;
      const int cnt = (int)min((int64_t)PT, r1 - base);
      if (tid < cnt) {
        double y[KC];
        if (PF) {
#pragma unroll
          for (int u = 0; u < KC; ++u) y[u] = nx[u];
          if (r + PT < r1) row_load(r + PT, nx);
        } else {
          row_load(r, y);
        }
        tri(R1i, y);
#pragma unroll
        for (int u = 0; u < KC; ++u) wt[u * CB_TSW + lane] = u < k ? y[u] : 0.0;
      } else {
#pragma unroll
        for (int u = 0; u < KC; ++u) wt[u * CB_TSW + lane] = 0.0;
      }
      gram_rows();
    }
  }
  gram_flush();
  if (ok) ok = gred(P2);
  if (ok) chol(R2, R2i);
  // pass 3: Q = (C R1^{-1}) R2^{-1} in place (no staging)
  {
    double nx[KC];
    if (ok && r0 + tid < r1) row_load(r0 + tid, nx);
    for (int64_t r = r0 + tid; ok && r < r1; r += PT) {
      double y[KC];
      if (PF) {
#pragma unroll
        for (int u = 0; u < KC; ++u) y[u] = nx[u];
        if (r + PT < r1) row_load(r + PT, nx);
      } else {
        row_load(r, y);
      }
      tri(R1i, y);
      tri(R2i, y);
#pragma unroll
      for (int u = 0; u < KC; ++u)
        if (u < k) Qc[(int64_t)u * ld + r] = y[u];
    }
  }
  if (cta0) {
    // R_C = R2 R1, R_C^{-1} = R1^{-1} R2^{-1} ([col][row]), and k_rc_finish's singularity test
    for (int e = tid; e < k * k; e += PT) {
      const int c = e / k, r = e % k;
      double v = 0.0, vi = 0.0;
      for (int l = 0; l < k; ++l) {
        v += R2[l * k + r] * R1[c * k + l];
        vi += R1i[l * k + r] * R2i[c * k + l];
      }
      st->RC[c][r] = v;
      st->RCinv[c][r] = vi;
      if (r == c) tot[c] = fabs(v);
    }
    __syncthreads();
    if (tid == 0) {
      double dmax = 0.0, dmin = 1e308;
      for (int i = 0; i < k; ++i) {
        dmax = tot[i] > dmax ? tot[i] : dmax;
        dmin = tot[i] < dmin ? tot[i] : dmin;
      }
      if (!ok || !(dmin > 1e-12 * dmax)) *cflag = 1;
      if (!CGIVEN) st->spmv_count += k;  // C = A W (rg_report.spmv_count; the SpMM counts its own)
      if (pa.llred) st->red_epoch = ok ? rep : rep + 16u;  // past anything a CTA may have published
      prof_end(st, K_CBUILD, (CGIVEN ? 0.0 : A.bytes) + 8.0 * (double)L.n * (CGIVEN ? 5.0 : 6.0) * k);
    }
  }
}

}  // namespace

size_t persistent_smem(int m, int k, bool aug, int pt = PT) {
  return sizeof(double) * ((size_t)m * (m + 2) + (size_t)m * (m + 1) + (size_t)(m + 1) * (k > 0 ? k : 1) + 2 * PM +
                           (PM + 2) + 3 * PCOL + 2 * (size_t)pt + 2 * MAXRED + (PM + 2) + 2 * PK + PM + 2 +
                           (aug ? 2 * (size_t)(m + 2) * (m + 2) : 0));
}

// Returns cudaErrorNotSupported when the configuration is outside this path.
cudaError_t launch_persistent(const Layout& L, const MatDev& A, DevState* st, double* tot_g, unsigned* bar,
                              unsigned* flags, unsigned long long* ll, int m, int k, int variant, const PrecDev* P,
                              cudaStream_t s) {
  if (m > PM || k > PK || A.fmt == 2) return cudaErrorNotSupported;
  const bool aug = variant == RG_AUGMENT && k > 0;
  const int vk = aug ? 2 : ((galerkin_variant(variant) && k > 0) ? 1 : 0);
  // tiny systems (<= 8 rows per thread of one 512-thread CTA) run on ONE CTA: no grid barriers at
  // all, and that CTA gets 1024 threads
  static const bool no1024 = knob("RG_NO_PT1024");
  const bool single = L.ld <= 8 * PT;
  const int pt = (single && !no1024) ? 1024 : PT, pcta = 1024 / pt;
  if (L.keepV && vk == 1) return cudaErrorNotSupported;  // no basis export for oblique / orthogonal here
  const int vi = L.keepV ? 6 + (vk == 2 ? 1 : 0) + (pt == 1024 ? 2 : 0) : vk + (pt == 1024 ? 3 : 0);
  static const void* fns[NPFN] = {
      (const void*)k_solve_persistent<0, PT>,         (const void*)k_solve_persistent<1, PT>,
      (const void*)k_solve_persistent<2, PT>,         (const void*)k_solve_persistent<0, 1024>,
      (const void*)k_solve_persistent<1, 1024>,       (const void*)k_solve_persistent<2, 1024>,
      (const void*)k_solve_persistent<0, PT, true>,   (const void*)k_solve_persistent<2, PT, true>,
      (const void*)k_solve_persistent<0, 1024, true>, (const void*)k_solve_persistent<2, 1024, true>};
  const void* fn = fns[vi];
  const int dev = current_device();
  const size_t smem0 = persistent_smem(m, k, aug, pt);
  // CSR pattern cache: what keeps pcta CTAs per SM resident (228 KB per SM, 1 KB per CTA reserved,
  // ~1 KB static), sized for this CTA count's rows and ~1.5x its share of the entries
  int rcap = 0, ccap = 0;
  if (A.fmt == 0 && !knob("RG_NO_SMEM_CSR")) {
    const int64_t G0 = single ? 1 : std::min<int64_t>((int64_t)NSM * pcta, std::max<int64_t>(1, (L.ld + pt - 1) / pt));
    const int64_t rows = ((L.ld >> 5) / G0 + 2) * 32 + 1;
    const int64_t ents = A.nnz / G0 * 3 / 2 + 1024;
    const int64_t budget = ((int64_t)228 * 1024 / pcta - 2 * 1024 - (int64_t)smem0) / 4;
    if (budget >= rows + ents) {
      rcap = (int)rows;
      ccap = (int)ents;
    }
  }
  const size_t smem = smem0 + sizeof(int32_t) * (size_t)(rcap + ccap);
  // function attributes and occupancy are per device: cached per device ordinal
  static bool attr_set[MAXDEV] = {};
  constexpr size_t max_smem = 200 * 1024;
  if (!attr_set[dev]) {
    for (const void* f : fns) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    attr_set[dev] = true;
  }
  if (smem > max_smem) return cudaErrorNotSupported;
  static size_t occ_smem[MAXDEV][NPFN] = {};  // occupancy per device, instantiation and shared-memory size
  static int occ_last[MAXDEV][NPFN] = {};
  if (occ_smem[dev][vi] != smem) {
    occ_last[dev][vi] = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_last[dev][vi], fn, pt, smem) != cudaSuccess) {
      cudaGetLastError();
      occ_last[dev][vi] = 0;
    }
    occ_smem[dev][vi] = smem;
  }
  const int occ = occ_last[dev][vi];
  if (occ < 1) return cudaErrorNotSupported;
  int64_t want = single ? 1 : (L.ld + pt - 1) / pt;
  static const int per_sm = knob_int("RG_PERSIST_CTAS_PER_SM", PCTA);
  int64_t cap = (int64_t)NSM * (occ >= per_sm ? per_sm : occ);
  const int G = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  static const int nbsync = knob("RG_NO_NBSYNC") ? 0 : 1;
  PArgs pa{L, A, st, tot_g, bar, m, variant == RG_PLAIN ? 0 : k,
           galerkin_variant(variant) && k > 0 ? (variant == RG_ORTHOGONAL ? 2 : 1) : 0, aug ? 1 : 0, flags, nbsync,
           knob_int("RG_SKEW", 0),
           P ? 1 : 0, P ? *P : PrecDev(), L.pz, L.pt, 0.0, rcap, ccap, ll,
           (ll && G > 1 && G <= LL_GMAX && G <= PT && !knob("RG_NO_LLRED")) ? 1 : 0};
  if (P) {
    double b2 = 0.0;
    for (int c = 0; c < P->ncolors; ++c) b2 += 12.0 * (double)(P->cL[c] + P->cU[c]);
    pa.pc_bytes = b2 + 8.0 * (double)L.n * 6.0;  // + perm, row pointers, 1/a_rr, in, out (fwd), out r/w (bwd)
  }
  void* args[] = {&pa};
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(pt), args, smem, s);
}

// One cooperative launch building C = A W, Q, R_C, R_C^{-1} (k_cbuild).  cudaErrorNotSupported when
// outside its scope (BSR, k > CBK, not co-resident): the caller runs build_c's kernel chain instead.
cudaError_t launch_cbuild(const Layout& L, const MatDev& A, DevState* st, double* tot_g, unsigned* bar,
                          unsigned long long* ll, int k, int* cflag, cudaStream_t s, bool cgiven) {
  // CSR / SELL: C = A W computed here; BSR: only with C given (the TMA + DMMA SpMM ran first)
  if (k < 1 || k > CBK || (A.fmt == 2 && !cgiven)) return cudaErrorNotSupported;
  if (k > 16 && !cgiven) return cudaErrorNotSupported;  // the fused SpMV + 24-column rows spill: build_c
  const int kc = k <= 8 ? 8 : (k <= 16 ? 16 : 24);
  const int vi = (kc / 8 - 1) + (cgiven ? 3 : 0);
  static const void* fns[6] = {(const void*)k_cbuild<8>, (const void*)k_cbuild<16>, (const void*)k_cbuild<16>,
                               (const void*)k_cbuild<8, true>, (const void*)k_cbuild<16, true>,
                               (const void*)k_cbuild<24, true>};
  const void* fn = fns[vi];
  const size_t smem = sizeof(double) * ((size_t)kc * (PT / 32) * CB_TSW + 4 * CBK * CBK + 2 * MAXRED);
  static int occ_dev[MAXDEV][6] = {};  // 0: not yet queried on that device, else occupancy + 1
  int& oc = occ_dev[current_device()][vi];
  if (oc == 0) {
    int o = 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, PT, smem) != cudaSuccess) {
      cudaGetLastError();
      o = 0;
    }
    oc = o + 1;
  }
  const int occ = oc - 1;
  if (occ < 1) return cudaErrorNotSupported;
  const int64_t want = L.ld <= 8 * PT ? 1 : (L.ld + PT - 1) / PT;
  const int64_t cap = (int64_t)NSM * (occ >= PCTA ? PCTA : occ);
  const int G = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  PArgs pa{};
  pa.L = L;
  pa.A = A;
  pa.st = st;
  pa.tot_g = tot_g;
  pa.bar = bar;
  pa.k = k;
  pa.ll = ll;
  pa.llred = (ll && G > 1 && G <= LL_GMAX && G <= PT && !knob("RG_NO_LLRED")) ? 1 : 0;
  void* args[] = {&pa, &cflag};
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(PT), args, smem, s);
}

}  // namespace rg

// spmv.cu — sparse matrix-vector products (K1 CSR, K2 SELL-32, K3 BSR), fp64, sm_100a.
//
// One read of the matrix per product, coalesced ("the cost of a matrix-vector
// multiplication reduces to O(mb)").  HBM-bound: bytes per product are in DESIGN.md §Roofline.
// Three output modes share each kernel:
//   SM_STEP  w = A v_j into V column j+1 (x = un-normalised column j, scaled on output)
//   SM_RES   r = b - A x into V column 0, ||r||^2 grid-reduced (cycle start)
//   SM_PLAIN y = A x (rg_apply, C = A W)
//   SM_RES_Y r = b - y into V column 0 where y = A x already sits there (the solve-start product
//            fused into the C = A W SpMM as its extra column: one read of A for both), ||r||^2
#define RG_FILE_ID 7  // RG_CHK locations (checked builds)
#include "epilogue.cuh"
#include "kernels.cuh"

#include <cuda.h>

#ifndef RG_SPMV_CAP
#define RG_SPMV_CAP 2  // CTAs per SM of the grid-stride SpMV launches (STEP / PLAIN modes): one wave
                       // (measured: 4 -> 2 per SM: SELL C3 4.03 -> 4.28 TB/s, CSR C4 5.40 -> 5.67)
#endif

namespace rg {
namespace {

struct SpmvArgs {
  MatDev A;
  Layout L;
  DevState* st;
  int mode;
  const double* x;
  double* y;
  int res_epi;
};

struct Io {
  const double* x;
  double* y;
  const double* b;
  double xs;
  bool res;
};

// Returns false if this launch is a no-op (decided uniformly from the device state).
__device__ __forceinline__ bool setup(const SpmvArgs& a, Io& io, int& kid) {
  pdl_trigger();  // the Arnoldi step's next kernel (PDL) may be scheduled as SpMV CTAs retire
  DevState* st = a.st;
  const Layout& L = a.L;
  io.res = false;
  io.b = nullptr;
  io.xs = 1.0;
  if (a.mode == SM_STEP || a.mode == SM_STEP_PC) {
    kid = K_SPMV_STEP;
    const int j = st->j;
    if (!st->active || (st->dcgs && j >= st->m)) { prof_noop(st, kid); return false; }
    io.x = a.mode == SM_STEP_PC ? L.pz : L.Z + (int64_t)(L.VB + j) * L.ld;
    io.y = L.Z + (int64_t)(L.VB + j + 1) * L.ld;
    // DCGS2: y = A u on the raw vector; STEP_PC: the SSOR sweep already applied the column scale
    io.xs = (st->dcgs || a.mode == SM_STEP_PC) ? 1.0 : st->sc[L.VB + j];
  } else if (a.mode == SM_RES || a.mode == SM_RES_Y) {
    kid = a.mode == SM_RES ? K_SPMV_RES : K_RES_Y;
    if (st->done) { prof_noop(st, kid); return false; }
    io.x = L.x;
    io.y = L.Z + (int64_t)L.VB * L.ld;
    io.b = L.b;
    io.res = true;
  } else {
    kid = K_SPMV_PLAIN;
    io.x = a.x;
    io.y = a.y;
  }
  // rg_report.spmv_count: every sparse product this solve issues, counted where it runs
  if (st && kid != K_RES_Y && blockIdx.x == 0 && threadIdx.x == 0) st->spmv_count++;
  if (st) prof_begin(st, kid);
  return true;
}

// Tail shared by every format: residual reduction + epilogue, profiling.
__device__ __forceinline__ void finish(const SpmvArgs& a, const Io& io, int kid, double nrm) {
  __shared__ double bsh[33], vals[1], tot[1];
  DevState* st = a.st;
  if (io.res) {
    const double t = block_sum(nrm, bsh);
    if (threadIdx.x == 0) vals[0] = t;
    __syncthreads();
    if (!grid_reduce(vals, 1, a.L.partial, a.L.counter, tot, tot)) return;
    if (a.res_epi) epi_cycle_start(st, a.L, tot[0]);
    if (threadIdx.x == 0) prof_end(st, kid, a.mode == SM_RES_Y ? 24.0 * a.L.n : a.A.bytes + 8.0 * a.L.n);
    return;
  }
  if (st && st->profile) {
    if (grid_last(a.L.counter) && threadIdx.x == 0) prof_end(st, kid, a.A.bytes);
  }
}

__device__ __forceinline__ double emit(const Io& io, int64_t r, double s) {
  double v;
  if (io.res) {
    v = io.b[r] - s;
  } else {
    v = io.xs * s;
  }
  io.y[r] = v;
  return v * v;
}

// ---------------------------------------------------------------- CSR, LPR lanes per row
template <int LPR>
__global__ void __launch_bounds__(OT, 2) k_spmv_csr(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int lane = threadIdx.x & (LPR - 1);
  const int64_t rows_per_cta = OT / LPR;
  const int64_t stride = (int64_t)gridDim.x * rows_per_cta;
  double nrm = 0.0;
  const int32_t* __restrict__ rp = A.rp;
  const int32_t* __restrict__ ci = A.ci;
  const double* __restrict__ v = A.v;
  const double* __restrict__ x = io.x;
  // warp-uniform trip count: iterate over groups of rows covering whole warps
  for (int64_t base = (int64_t)blockIdx.x * rows_per_cta + (threadIdx.x & ~31) / LPR; base < A.n;
       base += stride) {
    const int64_t row = base + (threadIdx.x & 31) / LPR;
    double s = 0.0;
    if (row < A.n) {
      const int32_t p0 = __ldg(rp + row), p1 = __ldg(rp + row + 1);
      if constexpr (LPR == 1) {
        // thread per row: up to 8 (column, value) pairs in flight, then 8 gathers of x
        for (int32_t p = p0; p < p1; p += 8) {
          int32_t cc[8];
          double vv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool ok = p + u < p1;
            cc[u] = ok ? __ldcs(ci + p + u) : 0;
            vv[u] = ok ? __ldcs(v + p + u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            RG_CHK(a.st, !(p + u < p1) || (cc[u] >= 0 && cc[u] < A.n));
            if (p + u < p1) s += vv[u] * __ldg(x + cc[u]);
          }
        }
      } else {
        for (int32_t p = p0 + lane; p < p1; p += LPR) s += __ldcs(v + p) * __ldg(x + __ldcs(ci + p));
      }
    }
    if constexpr (LPR > 1) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, LPR);
    }
    if (lane == 0 && row < A.n) nrm += emit(io, row, s);
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- CSR, thread per row, software-pipelined
// Short rows (<= 8 entries: 5- / 7-point stencils): the next row's row pointers and entries are loaded
// while the current row's x gathers are in flight, so each thread keeps two rows' loads outstanding
// instead of paying the three dependent latencies (row pointer, entries, x) of every row in sequence.
// Rows longer than 8 entries are finished by a plain loop.
__global__ void __launch_bounds__(OT, 2) k_spmv_csr_pipe(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int32_t* __restrict__ rp = A.rp;
  const int32_t* __restrict__ ci = A.ci;
  const double* __restrict__ v = A.v;
  const double* __restrict__ x = io.x;
  const int64_t stride = (int64_t)gridDim.x * OT;
  double nrm = 0.0;
  int64_t row = (int64_t)blockIdx.x * OT + threadIdx.x;
  int32_t p0 = 0, p1 = 0;
  int32_t cc[8];
  double vv[8];
  auto load_row = [&](int64_t r, int32_t& q0, int32_t& q1, int32_t (&c)[8], double (&w)[8]) {
    q0 = r < A.n ? __ldg(rp + r) : 0;
    q1 = r < A.n ? __ldg(rp + r + 1) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = q0 + u < q1;
      c[u] = ok ? __ldcs(ci + q0 + u) : 0;
      w[u] = ok ? __ldcs(v + q0 + u) : 0.0;
    }
  };
  load_row(row, p0, p1, cc, vv);
  for (; row < A.n; row += stride) {
    double xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = p0 + u < p1 ? __ldg(x + cc[u]) : 0.0;  // this row's gathers
    int32_t q0, q1, nc[8];
    double nv[8];
    load_row(row + stride, q0, q1, nc, nv);                                      // next row, in flight
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      RG_CHK(a.st, !(p0 + u < p1) || (cc[u] >= 0 && cc[u] < A.n));
      if (p0 + u < p1) s += vv[u] * xv[u];
    }
    RG_CHK(a.st, p0 <= p1);
    for (int32_t p = p0 + 8; p < p1; ++p) s += __ldcs(v + p) * __ldg(x + __ldcs(ci + p));  // long rows
    nrm += emit(io, row, s);
    p0 = q0;
    p1 = q1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      cc[u] = nc[u];
      vv[u] = nv[u];
    }
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- SELL-32 (sigma = 1)
// Thread per row; the first SELL_CH entries of the NEXT row (slice width / pointer, columns, values)
// are loaded while this row's x gathers are in flight (software pipelining across the grid-stride rows,
// as k_spmv_csr_pipe); entries beyond SELL_CH are finished by a plain loop.
__global__ void __launch_bounds__(OT, 2) k_spmv_sell(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  double nrm = 0.0;
  const int64_t rows = A.nslices * 32;
  const double* __restrict__ x = io.x;
  const int64_t stride = (int64_t)gridDim.x * OT;
  auto load_row = [&](int64_t r, int& w, int64_t& base, int32_t (&c)[SELL_CH], double (&vv)[SELL_CH]) {
    w = 0;
    base = 0;
    if (r < rows) {
      const int64_t sl = r >> 5;
      w = __ldg(A.sw + sl);
      base = __ldg(A.sp + sl) + (r & 31);
    }
#pragma unroll
    for (int u = 0; u < SELL_CH; ++u) {
      const bool ok = u < w;
      const int64_t e = base + (int64_t)u * 32;
      c[u] = ok ? __ldcs(A.sci + e) : 0;
      vv[u] = ok ? __ldcs(A.sv + e) : 0.0;
    }
  };
  int64_t row = (int64_t)blockIdx.x * OT + threadIdx.x;
  int w;
  int64_t base;
  int32_t cc[SELL_CH];
  double vv[SELL_CH];
  load_row(row, w, base, cc, vv);
  for (; row < rows; row += stride) {
    double xv[SELL_CH];
#pragma unroll
    for (int u = 0; u < SELL_CH; ++u) xv[u] = u < w ? __ldg(x + cc[u]) : 0.0;   // this row's gathers
    int wn;
    int64_t bn;
    int32_t cn[SELL_CH];
    double vn[SELL_CH];
    load_row(row + stride, wn, bn, cn, vn);                                        // next row, in flight
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < SELL_CH; ++u) {
      RG_CHK(a.st, !(u < w) || (cc[u] >= 0 && cc[u] < A.n));
      if (u < w) s += vv[u] * xv[u];
    }
    for (int c = SELL_CH; c < w; ++c) {                                            // long rows
      const int64_t e = base + (int64_t)c * 32;
      s += __ldcs(A.sv + e) * __ldg(x + __ldcs(A.sci + e));
    }
    if (row < A.n) nrm += emit(io, A.sperm ? (int64_t)__ldg(A.sperm + row) : row, s);  // SELL position -> row
    w = wn;
    base = bn;
#pragma unroll
    for (int u = 0; u < SELL_CH; ++u) {
      cc[u] = cn[u];
      vv[u] = vn[u];
    }
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- BSR (b <= 64), 64 threads / block row
__global__ void __launch_bounds__(256) k_spmv_bsr(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int b = A.b;
  const int r = threadIdx.x & 63;
  double nrm = 0.0;
  const double* __restrict__ x = io.x;
  for (int64_t I = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 6); I < A.nb; I += (int64_t)gridDim.x * 4) {
    if (r < b) {
      double s0 = 0.0, s1 = 0.0;
      const int32_t p0 = __ldg(A.rp + I), p1 = __ldg(A.rp + I + 1);
      for (int32_t p = p0; p < p1; ++p) {
        const double* __restrict__ blk = A.v + (int64_t)p * b * b + r;
        const double* __restrict__ xb = x + (int64_t)__ldg(A.ci + p) * b;
        int c = 0;
        for (; c + 16 <= b; c += 16) {  // 16 block values + 16 x entries in flight, then FMAs
          double av[16], xv[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            av[u] = __ldcs(blk + (int64_t)(c + u) * b);
            xv[u] = __ldg(xb + c + u);
          }
          asm volatile("" ::: "memory");  // keep ptxas from sinking the loads into the FMA chain
#pragma unroll
          for (int u = 0; u < 16; u += 2) {
            s0 += av[u] * xv[u];
            s1 += av[u + 1] * xv[u + 1];
          }
        }
        for (; c < b; ++c) s0 += __ldcs(blk + (int64_t)c * b) * __ldg(xb + c);
      }
      nrm += emit(io, I * b + r, s0 + s1);
    }
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- BSR-64 via TMA bulk copies
// Each 64x64 fp64 block is 32 KB contiguous: a producer warp streams the CTA's blocks (block rows
// blockIdx.x, +gridDim.x, ...) into a 4-stage shared-memory ring with cp.async.bulk (TMA),
// completing on per-stage mbarriers; 8 consumer warps compute from shared memory: thread t owns
// row t % 64 and column quarter t / 64; the quarters are combined in a fixed order per block row.
constexpr int BT_CONS = 256;            // consumer threads
constexpr int BT = BT_CONS + 32;        // + producer warp
constexpr int BNS = 4;                  // stages
constexpr int BSTAGE = 64 * 64 * 8;     // bytes per stage (one block)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(BT, 1) k_spmv_bsr_tma(SpmvArgs a) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[BNS], empty[BNS];
  __shared__ double qpart[4][64];
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  const MatDev& A = a.A;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < BNS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(BT_CONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double nrm = 0.0;
  if (wid == BT_CONS / 32) {
    // ---- producer: lane 0 walks the same block sequence as the consumers
    if (lane == 0) {
      int t = 0;
      for (int64_t I = blockIdx.x; I < A.nb; I += gridDim.x) {
        const int32_t p0 = __ldg(A.rp + I), p1 = __ldg(A.rp + I + 1);
        RG_CHK(a.st, p0 >= 0 && p0 <= p1 && p1 <= A.nnz);
        for (int32_t p = p0; p < p1; ++p, ++t) {
          const int s = t % BNS;
          if (t >= BNS) bar_wait(&empty[s], (uint32_t)((t / BNS - 1) & 1));
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(BSTAGE) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(ring + (size_t)s * (BSTAGE / 8))), "l"(A.v + (int64_t)p * 4096), "r"(BSTAGE),
                       "r"(su32(&full[s])) : "memory");
        }
      }
    }
  } else {
    // ---- consumers
    const int r = tid & 63, q = tid >> 6;
    int t = 0;
    for (int64_t I = blockIdx.x; I < A.nb; I += gridDim.x) {
      const int32_t p0 = __ldg(A.rp + I), p1 = __ldg(A.rp + I + 1);
      double s0 = 0.0, s1 = 0.0;
      for (int32_t p = p0; p < p1; ++p, ++t) {
        const int st = t % BNS;
        RG_CHK(a.st, __ldg(A.ci + p) >= 0 && __ldg(A.ci + p) < A.nb);
        const double* __restrict__ xb = io.x + (int64_t)__ldg(A.ci + p) * 64 + q * 16;
        double xv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) xv[u] = __ldg(xb + u);
        bar_wait(&full[st], (uint32_t)((t / BNS) & 1));
        const double* blk = ring + (size_t)st * (BSTAGE / 8) + (q * 16) * 64 + r;
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          s0 += blk[u * 64] * xv[u];
          s1 += blk[(u + 1) * 64] * xv[u + 1];
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
      }
      qpart[q][r] = s0 + s1;
      asm volatile("bar.sync 1, %0;" ::"r"(BT_CONS) : "memory");
      if (q == 0) nrm += emit(io, I * 64 + r, ((qpart[0][r] + qpart[1][r]) + qpart[2][r]) + qpart[3][r]);
      asm volatile("bar.sync 1, %0;" ::"r"(BT_CONS) : "memory");
    }
  }
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- r = b - y, y = A x already in V column 0
__global__ void __launch_bounds__(OT) k_res_y(SpmvArgs a) {
  Io io;
  int kid;
  if (!setup(a, io, kid)) return;
  double nrm = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * OT + threadIdx.x; r < a.A.n; r += (int64_t)gridDim.x * OT)
    nrm += emit(io, r, io.y[r]);
  finish(a, io, kid, nrm);
}

// ---------------------------------------------------------------- SpMM  Y = A W  (C = A W, a4)
// BSR-64: one TMA-streamed read of A for all k columns; the 64x64 block (shared memory) times the
// 64 x k panel of W runs on the FP64 tensor cores (DMMA m8n8k4): warp w owns output rows
// 8w..8w+7 of the block row and every 8-column group.
//
// Landing layout: a block arrives as four 8 KB row-quarter slices q (rows 16q..16q+15), each through a
// 3-D tensor map {16 rows, 4 quarters, columns} with box {16, 1, 64} and the 128-byte swizzle: inside
// slice q, line c (16 rows of column c, 128 B) has its 16-byte chunks permuted by chunk ^= c % 8.  The
// DMMA k-step s takes the four columns kset(s) = c0 + {0, 2, 4, 6} (c0 = 8 (s/2) + s%2; the k order of a
// sum is free): the XOR values of those columns differ in bits 1-2, so each half-warp's 16 A elements
// (4 rows x 4 columns) fill 8 distinct chunks x both halves = one 128-byte wavefront, the ideal.  (Dense
// column-major landing: 4 wavefronts per load, ncu r02: 171M bank conflicts in 321M shared wavefronts,
// the shared-memory pipe and not the DMMA pipe was the limiter.)
// element (r, c) of a landed block -> double offset
__device__ __forceinline__ int swz_off(int r, int c) {
  return (r >> 4) * 1024 + c * 16 + ((((r & 15) >> 1) ^ (c & 7)) << 1) + (r & 1);
}
// column of k-step s, lane j = lane % 4
__device__ __forceinline__ int kcol(int s, int j) { return 8 * (s >> 1) + (s & 1) + 2 * j; }
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// acc[g] += A_block(rows 8w.., :) * W_panel(:, 8g..8g+7), g < NG.  W panel stored k-major [kk][n] with
// stride WS == 2 mod 16 (the B elements W(kcol(s, j), 8g + i) of a half-warp, i < 4, j < 4, land in 16
// distinct bank pairs).  ae / ao: this lane's A element of k-steps 0 / 1 (k-step s adds 128 (s / 2));
// we / wo: its W element of k-steps 0 / 1 (+ 8 WS (s / 2) + 8 g).
// CH independent accumulator chains per column group hide the DMMA latency when NG is small.  The chains
// PERSIST over the blocks of a block row (round 2, late): folding them into one accumulator after every block
// drained the DMMA pipe once per block and warp — a fixed ~0.26 us per block whatever the warp mapping.
template <int NG>
struct SpmmChains {
  static constexpr int CH = NG >= 4 ? 1 : (NG >= 2 ? 2 : 4);
};
template <int NG, int WS>
__device__ __forceinline__ void block_mma(double (&ch)[NG][SpmmChains<NG>::CH][2], const double* blk, const double* wp,
                                          int ae, int ao, int we, int wo) {
  constexpr int CH = SpmmChains<NG>::CH;
#pragma unroll
  for (int s0 = 0; s0 < 16; s0 += CH) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int s = s0 + c;
      const double av = blk[((s & 1) ? ao : ae) + 128 * (s >> 1)];          // A(rrow, kcol(s, lane%4))
      const int wb = ((s & 1) ? wo : we) + 8 * WS * (s >> 1);
#pragma unroll
      for (int g = 0; g < NG; ++g) dmma884(ch[g][c][0], ch[g][c][1], av, wp[wb + 8 * g]);  // W(kcol, 8g + lane/4)
    }
  }
}

// The consumer loop of one CTA for a fixed number NG of 8-column groups: block rows I = blockIdx, +gridDim, ...;
// the blocks of a row stream through the ring; the chains are folded and the 8 rows stored once per block row.
template <int NG, int NST, int WS>
__device__ __forceinline__ void spmm_consume(const MatDev& A, const double* ring, const double* wpan, uint64_t* full,
                                             uint64_t* empty, double* Y, int64_t ld, int kw, const double* xe,
                                             double* ye, int wid, int lane) {
  constexpr int CH = SpmmChains<NG>::CH;
  const int rrow = wid * 8 + (lane >> 2);                    // A fragment row inside the block
  const int ae = swz_off(rrow, kcol(0, lane & 3)), ao = swz_off(rrow, kcol(1, lane & 3));
  const int we = kcol(0, lane & 3) * WS + (lane >> 2), wo = kcol(1, lane & 3) * WS + (lane >> 2);
  int t = 0;
  int64_t I = blockIdx.x;
  int32_t p = I < A.nb ? __ldg(A.rp + I) : 0, pend = I < A.nb ? __ldg(A.rp + I + 1) : 0;
  for (; I < A.nb; I += gridDim.x) {
    const int64_t In = I + gridDim.x;  // the next block row's range, loaded early
    const int32_t pn = In < A.nb ? __ldg(A.rp + In) : 0, pendn = In < A.nb ? __ldg(A.rp + In + 1) : 0;
    double ch[NG][CH][2];
#pragma unroll
    for (int g = 0; g < NG; ++g)
#pragma unroll
      for (int c = 0; c < CH; ++c) ch[g][c][0] = ch[g][c][1] = 0.0;
    for (; p < pend; ++p, ++t) {
      const int st = t % NST;
      bar_wait(&full[st], (uint32_t)((t / NST) & 1));
      block_mma<NG, WS>(ch, ring + (size_t)st * (BSTAGE / 8), wpan + (size_t)st * 64 * WS, ae, ao, we, wo);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      double a0 = ch[g][0][0], a1 = ch[g][0][1];
#pragma unroll
      for (int c = 1; c < CH; ++c) {
        a0 += ch[g][c][0];
        a1 += ch[g][c][1];
      }
      const int col = g * 8 + (lane & 3) * 2;
      const int64_t row = I * 64 + rrow;
      if (col < kw) Y[(int64_t)col * ld + row] = a0;
      else if (col == kw && xe) ye[row] = a0;
      if (col + 1 < kw) Y[(int64_t)(col + 1) * ld + row] = a1;
      else if (col + 1 == kw && xe) ye[row] = a1;
    }
    p = pn;
    pend = pendn;
  }
}

// xe != nullptr: one extra input column (panel column k) whose product goes to ye (y = A x0 of the
// solve start, fused with C = A W: one read of A instead of two).
//
// Pipeline: the producer warp streams, per block of the CTA's sequence, the 32 KB block (lane 0: four
// tensor-map TMA copies, complete_tx) AND the block column's 64 x k panel of W (all 32 lanes:
// cp.async 8-byte copies into the stage's k-major panel, completion tracked by the same mbarrier via
// cp.async.mbarrier.arrive.noinc) into an NST-stage ring; the 8 consumer warps only wait on the
// stage's full barrier, run the DMMAs out of shared memory and release the stage.  No global load
// and no CTA-wide barrier on the consumer side.  (Previous version: consumers prefetched the next
// panel through registers with a dependent column-index load and a named barrier per block; ncu r02
// showed them stalled on that load chain and the barrier: 1.79 ms for one 7.3 GB read of A.)
// WS: k-major panel stride (== 2 mod 16, >= the panel width k + [xe]); NST: stages.
template <int NST, int WS>
__global__ void __launch_bounds__(BT, 1) k_spmm_bsr_tma(const __grid_constant__ CUtensorMap tmA, MatDev A,
                                                        const double* __restrict__ W, double* Y,
                                                        int64_t ld, int k, DevState* pst, unsigned* counter,
                                                        const double* __restrict__ xe, double* ye) {
  if (pst) prof_begin(pst, K_SPMV_PLAIN);
  if (pst && blockIdx.x == 0 && threadIdx.x == 0) pst->spmv_count += k + (xe ? 1 : 0);
  extern __shared__ __align__(128) double smraw[];
  // the 128-byte swizzle repeats every 1024 bytes: the ring starts on a 1024-byte boundary (pointer
  // arithmetic on smraw keeps the shared address space: LDS, not generic loads)
  double* ring = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u) / 8u;
  double* wpan = ring + (size_t)NST * (BSTAGE / 8);  // NST x [64 k-rows][WS]
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  for (int e = tid; e < NST * 64 * WS; e += BT) wpan[e] = 0.0;  // pad columns [k, 8 ng) stay zero
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      // full: lane 0's expect_tx arrival + the 32 producer lanes' cp.async completions (+ TMA bytes)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(33));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(BT_CONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kw = k;                  // columns of W / Y
  if (xe) k += 1;                    // + the extra column
  const int ng = (k + 7) / 8;
  if (wid == BT_CONS / 32) {
    // ---- producer warp.  The block sequence (block rows I = blockIdx, +gridDim, ...; blocks p of each)
    // is walked one block AHEAD: the next block's column index (and the next block row's range) are
    // loaded while the current block's copies are issued, so no dependent global load sits between
    // two blocks' copies.  A streams through L2 with evict-first (read once); the W panels (re-read by
    // the ~7 block rows that touch a block column) keep the normal policy.
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int64_t I = blockIdx.x;
    int32_t p = 0, pend = 0;
    auto next_block = [&](int64_t& Ib, int32_t& pb, int32_t& pe) -> bool {  // successor in the sequence
      ++pb;
      while (pb >= pe) {
        Ib += gridDim.x;
        if (Ib >= A.nb) return false;
        pb = __ldg(A.rp + Ib);
        pe = __ldg(A.rp + Ib + 1);
      }
      return true;
    };
    bool have = false;
    if (I < A.nb) {
      p = __ldg(A.rp + I) - 1;
      pend = __ldg(A.rp + I + 1);
      have = next_block(I, p, pend);
    }
    int32_t ci_cur = have ? __ldg(A.ci + p) : 0;
    for (int t = 0; have; ++t) {
      int64_t I2 = I;
      int32_t p2 = p, pe2 = pend;
      const bool have2 = next_block(I2, p2, pe2);
      const int32_t ci_next = have2 ? __ldg(A.ci + p2) : 0;  // consumed next iteration
      const int s = t % NST;
      if (t >= NST) bar_wait(&empty[s], (uint32_t)((t / NST - 1) & 1));
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(BSTAGE) : "memory");
#pragma unroll
        for (int q = 0; q < 4; ++q)  // row quarter q -> slice q of the stage (8 KB, 1024-byte aligned)
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
                       "[%0], [%1, {%2, %3, %4}], [%5], %6;"
                       ::"r"(su32(ring + (size_t)s * (BSTAGE / 8) + q * 1024)), "l"(&tmA), "r"(0), "r"(q), "r"(p * 64),
                       "r"(su32(&full[s])), "l"(pol) : "memory");
      }
      const int64_t J64 = (int64_t)ci_cur * 64;
      const uint32_t pan = su32(wpan + (size_t)s * 64 * WS);
      {  // W(J64 + kk, n) -> panel[kk][n], kk = lane and lane + 32; coalesced per column.  Pointer increments
         // only: the index / select arithmetic of a flat element loop made this loop (2 k copies per lane,
         // behind the consumers on the warp's scheduler) the per-block critical path at k >= 9
        const double* src = W + J64 + lane;
        uint32_t dst = pan + 8u * (uint32_t)(lane * WS);
#pragma unroll 4
        for (int n = 0; n < kw; ++n, src += ld, dst += 8u) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * 32u * (uint32_t)WS), "l"(src + 32) : "memory");
        }
        if (xe) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(xe + J64 + lane) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * 32u * (uint32_t)WS), "l"(xe + J64 + lane + 32) : "memory");
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
      I = I2;
      p = p2;
      pend = pe2;
      ci_cur = ci_next;
      have = have2;
    }
    return;
  }
  // ---- consumers (the loop is instantiated per number of 8-column groups: exact DMMA trip counts, and the
  // accumulator chains of a block row stay in registers)
  switch (ng) {
    case 1: spmm_consume<1, NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 2: spmm_consume<2, NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 3: spmm_consume<3, NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 4: spmm_consume<(WS > 24 ? 4 : 1), NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 5: spmm_consume<(WS > 32 ? 5 : 1), NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 6: spmm_consume<(WS > 40 ? 6 : 1), NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    case 7: spmm_consume<(WS > 48 ? 7 : 1), NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
    default: spmm_consume<(WS > 56 ? 8 : 1), NST, WS>(A, ring, wpan, full, empty, Y, ld, kw, xe, ye, wid, lane); break;
  }
  if (pst && pst->profile) {
    asm volatile("bar.sync 1, %0;" ::"r"(BT_CONS) : "memory");
    if (tid == 0) {
      const unsigned tk = atom_add_release(counter);
      if (tk == gridDim.x - 1) {
        *counter = 0u;
        prof_end(pst, K_SPMV_PLAIN, A.bytes + 16.0 * (double)A.n * k);
      }
    }
  }
}

// CSR / SELL: thread per row, 16 columns of W per pass (k <= 64 -> at most 4 reads of A).
template <int KC>
__global__ void __launch_bounds__(256) k_spmm_rows(MatDev A, const double* __restrict__ W, double* Y, int64_t ld,
                                                   int k0, int kc, DevState* st) {
  if (st && blockIdx.x == 0 && threadIdx.x == 0) st->spmv_count += kc;
  for (int64_t row = blockIdx.x * 256ll + threadIdx.x; row < A.n; row += (int64_t)gridDim.x * 256) {
    double acc[KC];
#pragma unroll
    for (int l = 0; l < KC; ++l) acc[l] = 0.0;
    if (A.fmt == 1) {
      const int64_t pos = A.siperm ? (int64_t)__ldg(A.siperm + row) : row;  // row -> SELL position
      const int64_t sl = pos >> 5;
      const int w = __ldg(A.sw + sl);
      const int64_t base = __ldg(A.sp + sl) + (pos & 31);
      for (int c = 0; c < w; ++c) {
        const int64_t e = base + (int64_t)c * 32;
        const double v = __ldcs(A.sv + e);
        const int32_t col = __ldcs(A.sci + e);
#pragma unroll
        for (int l = 0; l < KC; ++l)
          if (l < kc) acc[l] += v * __ldg(W + (int64_t)(k0 + l) * ld + col);
      }
    } else {
      const int32_t p0 = __ldg(A.rp + row), p1 = __ldg(A.rp + row + 1);
      for (int32_t p = p0; p < p1; ++p) {
        const double v = __ldcs(A.v + p);
        const int32_t col = __ldcs(A.ci + p);
#pragma unroll
        for (int l = 0; l < KC; ++l)
          if (l < kc) acc[l] += v * __ldg(W + (int64_t)(k0 + l) * ld + col);
      }
    }
#pragma unroll
    for (int l = 0; l < KC; ++l)
      if (l < kc) Y[(int64_t)(k0 + l) * ld + row] = acc[l];
  }
}

}  // namespace

cudaError_t launch_spmv(const MatDev& A, const Layout& L, DevState* st, int mode, const double* x,
                        double* y, int res_epi, cudaStream_t s, bool pdl) {
  SpmvArgs a{A, L, st, mode, x, y, res_epi};
  const int cap_red = NSM * VEC_CTAS_PER_SM;  // reducing launches: bounded partials
  if (mode == SM_RES_Y) {
    int64_t g = (A.n + OT - 1) / OT;
    if (g > cap_red) g = cap_red;
    k_res_y<<<(int)(g < 1 ? 1 : g), OT, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (A.fmt == 2 && A.b == 64 && A.tma) {
    static PerDevice init_once;
    if (init_once.first()) {
      cudaFuncSetAttribute(k_spmv_bsr_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, BNS * BSTAGE);
    }
    int64_t g = A.nb < NSM ? A.nb : NSM;
    return launch_ex(k_spmv_bsr_tma, dim3((int)(g < 1 ? 1 : g)), dim3(BT), BNS * BSTAGE, s, pdl, a);
  }
  if (A.fmt == 2) {
    int64_t g = (A.nb + 3) / 4;
    const int64_t cap = (int64_t)NSM * 8;  // partials buffer holds NSM*8 rows: RES may use them all
    if (g > cap) g = cap;
    return launch_ex(k_spmv_bsr, dim3((int)(g < 1 ? 1 : g)), dim3(256), 0, s, pdl, a);
  } else if (A.fmt == 1) {
    int64_t g = (A.nslices * 32 + OT - 1) / OT;
    const int64_t cap = mode == SM_RES ? cap_red : (int64_t)NSM * RG_SPMV_CAP;
    if (g > cap) g = cap;
    return launch_ex(k_spmv_sell, dim3((int)(g < 1 ? 1 : g)), dim3(OT), 0, s, pdl, a);
  } else {
    int64_t g = (A.n * A.lpr + OT - 1) / OT;
    const int64_t cap = mode == SM_RES ? cap_red : (int64_t)NSM * RG_SPMV_CAP;
    if (g > cap) g = cap;
    const int gi = (int)(g < 1 ? 1 : g);
    switch (A.lpr) {
      case 1: return launch_ex(k_spmv_csr_pipe, dim3(gi), dim3(OT), 0, s, pdl, a);
      case 2: return launch_ex(k_spmv_csr<2>, dim3(gi), dim3(OT), 0, s, pdl, a);
      case 4: return launch_ex(k_spmv_csr<4>, dim3(gi), dim3(OT), 0, s, pdl, a);
      case 8: return launch_ex(k_spmv_csr<8>, dim3(gi), dim3(OT), 0, s, pdl, a);
      case 16: return launch_ex(k_spmv_csr<16>, dim3(gi), dim3(OT), 0, s, pdl, a);
      default: return launch_ex(k_spmv_csr<32>, dim3(gi), dim3(OT), 0, s, pdl, a);
    }
  }
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled resolved through the runtime's driver entry point: librg.so does not link
// libcuda (the library must load, and export its symbols, on a host without the driver)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    tried = true;
  }
  return fn;
}

cudaError_t launch_spmm(const MatDev& A, const double* W, double* Y, int64_t ld, int k, DevState* st, unsigned* counter,
                        cudaStream_t s, const double* xe, double* ye) {
  if (k <= 0) return cudaSuccess;
  if (xe && !(A.fmt == 2 && A.b == 64 && A.tma && k + 1 <= 64)) return cudaErrorInvalidValue;  // callers check
  if (A.fmt == 2 && A.b == 64 && A.tma && k <= 64) {
    // the values as a 3-D tensor {16 rows, 4 row quarters, nnzb * 64 columns} (strides 128 B, 512 B):
    // box {16, 1, 64} = one row quarter of a block (8 KB), landed with the 128-byte swizzle (swz_off)
    CUtensorMap tm;
    const cuuint64_t dims[3] = {16, 4, (cuuint64_t)A.nnz * 64};
    const cuuint64_t strides[2] = {16 * 8, 64 * 8};
    const cuuint32_t box[3] = {16, 1, 64}, estr[3] = {1, 1, 1};  // one row quarter of a block (8 KB)
    if (!encode_tiled() || encode_tiled()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A.v, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    // panel stride (== 2 mod 16, >= the panel width) and ring depth within ~200 KB of shared memory
    const int width = k + (xe ? 1 : 0);
    static bool attr_set[MAXDEV] = {};
    const int dev = current_device();
    auto smem_of = [](int nst, int ws) { return nst * BSTAGE + nst * 64 * ws * 8 + 1024; };  // + 1024-byte alignment slack
    if (!attr_set[dev]) {
      cudaFuncSetAttribute(k_spmm_bsr_tma<4, 18>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_of(4, 18));
      cudaFuncSetAttribute(k_spmm_bsr_tma<4, 34>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_of(4, 34));
      cudaFuncSetAttribute(k_spmm_bsr_tma<3, 66>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_of(3, 66));
      attr_set[dev] = true;
    }
    const int g = (int)(A.nb < NSM ? (A.nb < 1 ? 1 : A.nb) : NSM);
    if (width <= 18) k_spmm_bsr_tma<4, 18><<<g, BT, smem_of(4, 18), s>>>(tm, A, W, Y, ld, k, st, counter, xe, ye);
    else if (width <= 34) k_spmm_bsr_tma<4, 34><<<g, BT, smem_of(4, 34), s>>>(tm, A, W, Y, ld, k, st, counter, xe, ye);
    else k_spmm_bsr_tma<3, 66><<<g, BT, smem_of(3, 66), s>>>(tm, A, W, Y, ld, k, st, counter, xe, ye);
    return cudaGetLastError();
  }
  if (A.fmt == 2) return cudaErrorNotSupported;  // caller falls back to per-column SpMV
  int64_t g = (A.n + 255) / 256;
  if (g > NSM * 8) g = NSM * 8;
  for (int k0 = 0; k0 < k; k0 += 16) {
    k_spmm_rows<16><<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(A, W, Y, ld, k0, k - k0 < 16 ? k - k0 : 16, st);
    note_host_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace rg

/* synth_common.h — seeded synthetic INPUT generators for the five BASELINE.json configs.
 *
 * This module is the one place both sides of the parity tests share: it builds the
 * matrices A_t, right-hand sides b_t and the initial field u_0 of the sequences of
 * systems (eq. algebra_pde / sequence_linear_systems: "the sequence of
 * matrices and right-hand sides depend on the previous solution").  It holds NONE of the
 * method's arithmetic (no Krylov, no projector, no SVD): only stencil coefficients and
 * counter-based random numbers.
 *
 * The same inline functions are compiled by gcc (synth.c, -ffp-contract=off) and by nvcc
 * (synth_cuda.cu, -fmad=false), so host and device produce bit-identical values
 * (SURVEY.md §8c-A22).  Transcendental functions (exp, sin, cos) never appear here: the
 * scalars that need them are computed on the host and passed in.
 *
 * Stencil readings:
 *   lexicographic node order x-fastest, h = 1/(N+1), homogeneous Dirichlet (entries that
 *   fall outside the grid are dropped), first-order upwind = backward difference where the
 *   velocity component is > 0, chosen per node and per axis.
 */
#ifndef SYNTH_COMMON_H
#define SYNTH_COMMON_H
#include <stdint.h>

#ifdef __CUDACC__
#define SY_HD __host__ __device__ __forceinline__
#else
#define SY_HD static inline
#endif

SY_HD double sy_fmax0(double a) { return a > 0.0 ? a : 0.0; }
SY_HD double sy_fabs(double a) { return a < 0.0 ? -a : a; }

/* splitmix64 finaliser (Steele, Lea, Flood 2014) used as a counter-based hash. */
SY_HD uint64_t sy_fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* U[0,1) with 53 random bits. */
SY_HD double sy_u01(uint64_t z) { return (double)(z >> 11) * (1.0 / 9007199254740992.0); }
/* counter-based draw number `idx` of stream `stream` under `seed`. */
SY_HD uint64_t sy_hash3(uint64_t seed, uint64_t stream, uint64_t idx) {
  return sy_fmix(sy_fmix(seed ^ (stream * 0xD1B54A32D192ED03ULL)) + idx * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL);
}
/* Approximately standard normal: Irwin-Hall sum of 12 uniforms minus 6 (mean 0, variance 1,
 * support [-6,6]).  Chosen over Box-Muller because it needs no libm, so host and device are
 * bit-identical (reading R-C5a). Summation order is fixed. */
SY_HD double sy_normal12(uint64_t seed, uint64_t stream, uint64_t idx) {
  double s = 0.0;
  for (int q = 0; q < 12; ++q) s += sy_u01(sy_hash3(seed, stream, idx * 12ULL + (uint64_t)q));
  return s - 6.0;
}

/* ---------------- 2-D 5-point first-order upwind (configs C1, C2) -----------------------
 * Row of node (i,j) of an N x N interior grid, operator  -nu Lap u + beta.grad u + u/dt.
 *   cd = nu/h^2, ih = 1/h, idt = 1/dt (host scalars).  Entries in increasing column order
 *   S (j-1), W (i-1), C, E (i+1), N (j+1); those outside the grid are dropped.
 * Returns the number of entries written to val (and col when col != 0). */
SY_HD int sy_row5(int i, int j, int N, double cd, double ih, double idt, double bx, double by,
                  double* val, int32_t* col) {
  int k = 0;
  int64_t r = (int64_t)j * N + i;
  double cW = -(cd + sy_fmax0(bx) * ih);
  double cE = -(cd + sy_fmax0(-bx) * ih);
  double cS = -(cd + sy_fmax0(by) * ih);
  double cN = -(cd + sy_fmax0(-by) * ih);
  double cC = 4.0 * cd + (sy_fabs(bx) + sy_fabs(by)) * ih + idt;
  if (j > 0)     { val[k] = cS; if (col) col[k] = (int32_t)(r - N); ++k; }
  if (i > 0)     { val[k] = cW; if (col) col[k] = (int32_t)(r - 1); ++k; }
  val[k] = cC; if (col) col[k] = (int32_t)r; ++k;
  if (i < N - 1) { val[k] = cE; if (col) col[k] = (int32_t)(r + 1); ++k; }
  if (j < N - 1) { val[k] = cN; if (col) col[k] = (int32_t)(r + N); ++k; }
  return k;
}

/* ---------------- 2-D 9-point cross (config C3) ------------------------------------------
 * 4th-order central diffusion per axis  nu(u_{i-2} - 16u_{i-1} + 30u_i - 16u_{i+1} + u_{i+2})/(12h^2)
 * plus 3rd-order upwind-biased convection per axis
 *   beta>0 : beta(u_{i-2} - 6u_{i-1} + 3u_i + 2u_{i+1})/(6h)
 *   beta<=0: beta(-2u_{i-1} - 3u_i + 6u_{i+1} - u_{i+2})/(6h)   (mirror image)
 * plus 1/dt.  cdif = nu/(12h^2), c6 = 1/(6h).  Column order: j-2, j-1, i-2, i-1, C, i+1,
 * i+2, j+1, j+2. */
SY_HD void sy_axis9(double cdif, double a, double* o /* offsets -2..2 */) {
  if (a > 0.0) {
    o[0] = cdif + a;
    o[1] = cdif * -16.0 + a * -6.0;
    o[2] = cdif * 30.0 + a * 3.0;
    o[3] = cdif * -16.0 + a * 2.0;
    o[4] = cdif;
  } else {
    o[0] = cdif;
    o[1] = cdif * -16.0 + a * -2.0;
    o[2] = cdif * 30.0 + a * -3.0;
    o[3] = cdif * -16.0 + a * 6.0;
    o[4] = cdif + a * -1.0;
  }
}
SY_HD int sy_row9(int i, int j, int N, double cdif, double c6, double idt, double bx, double by,
                  double* val, int32_t* col) {
  double ox[5], oy[5];
  sy_axis9(cdif, bx * c6, ox);
  sy_axis9(cdif, by * c6, oy);
  int64_t r = (int64_t)j * N + i;
  int k = 0;
  if (j > 1)     { val[k] = oy[0]; if (col) col[k] = (int32_t)(r - 2 * N); ++k; }
  if (j > 0)     { val[k] = oy[1]; if (col) col[k] = (int32_t)(r - N); ++k; }
  if (i > 1)     { val[k] = ox[0]; if (col) col[k] = (int32_t)(r - 2); ++k; }
  if (i > 0)     { val[k] = ox[1]; if (col) col[k] = (int32_t)(r - 1); ++k; }
  val[k] = ox[2] + oy[2] + idt; if (col) col[k] = (int32_t)r; ++k;
  if (i < N - 1) { val[k] = ox[3]; if (col) col[k] = (int32_t)(r + 1); ++k; }
  if (i < N - 2) { val[k] = ox[4]; if (col) col[k] = (int32_t)(r + 2); ++k; }
  if (j < N - 1) { val[k] = oy[3]; if (col) col[k] = (int32_t)(r + N); ++k; }
  if (j < N - 2) { val[k] = oy[4]; if (col) col[k] = (int32_t)(r + 2 * N); ++k; }
  return k;
}

/* ---------------- 3-D 7-point first-order upwind (config C4) ------------------------------
 * Column order z-1, y-1, x-1, C, x+1, y+1, z+1. */
SY_HD int sy_row7(int i, int j, int l, int N, double cd, double ih, double idt, double bx,
                  double by, double bz, double* val, int32_t* col) {
  int64_t NN = (int64_t)N * N;
  int64_t r = (int64_t)l * NN + (int64_t)j * N + i;
  int k = 0;
  double cC = 6.0 * cd + (sy_fabs(bx) + sy_fabs(by) + sy_fabs(bz)) * ih + idt;
  if (l > 0)     { val[k] = -(cd + sy_fmax0(bz) * ih);  if (col) col[k] = (int32_t)(r - NN); ++k; }
  if (j > 0)     { val[k] = -(cd + sy_fmax0(by) * ih);  if (col) col[k] = (int32_t)(r - N); ++k; }
  if (i > 0)     { val[k] = -(cd + sy_fmax0(bx) * ih);  if (col) col[k] = (int32_t)(r - 1); ++k; }
  val[k] = cC; if (col) col[k] = (int32_t)r; ++k;
  if (i < N - 1) { val[k] = -(cd + sy_fmax0(-bx) * ih); if (col) col[k] = (int32_t)(r + 1); ++k; }
  if (j < N - 1) { val[k] = -(cd + sy_fmax0(-by) * ih); if (col) col[k] = (int32_t)(r + N); ++k; }
  if (l < N - 1) { val[k] = -(cd + sy_fmax0(-bz) * ih); if (col) col[k] = (int32_t)(r + NN); ++k; }
  return k;
}

/* ---------------- block-sparse "high-order-like" operator (config C5) ---------------------
 * E^3 elements x B dofs, BSR with B x B blocks stored COLUMN-MAJOR inside each block
 * (val[blk*B*B + c*B + r] = block(r,c)).  Block row order z-1, y-1, x-1, self, x+1, y+1, z+1.
 * Diagonal block: N(0,1) + 100 I.  Face block: N(0,1) * s_up (upstream faces -x,-y,-z) or
 * N(0,1) * s_dn (downstream), s_up = 0.1*1.5, s_dn = 0.1*0.5. */
SY_HD double sy_c5_base(uint64_t seed, int64_t blk, int r, int c, int B, int kind /*0 diag,1 up,2 down*/,
                        double s_up, double s_dn) {
  double z = sy_normal12(seed, (uint64_t)blk, (uint64_t)(c * B + r));
  if (kind == 0) return r == c ? z + 100.0 : z;
  return z * (kind == 1 ? s_up : s_dn);
}
/* multiplicative perturbation factor (1 + 0.01 xi), xi ~ U[-1,1], of stored entry e at system t. */
SY_HD double sy_c5_factor(uint64_t seed, int t, int64_t e) {
  double xi = 2.0 * sy_u01(sy_hash3(seed ^ 0x5EEDF00DULL, (uint64_t)t, (uint64_t)e)) - 1.0;
  return 1.0 + 0.01 * xi;
}

#endif

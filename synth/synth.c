/* synth.c — host (CPU) side of the seeded input generators (see synth_common.h).
 * Compiled with -O2 -ffp-contract=off so the values are bit-identical to synth_cuda.cu.
 * Used by the tests (both sides of parity), by bench.py's e2e leg and by smoke(). */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include "synth_common.h"

/* splitmix64 stream (sequential draws for bump centres / amplitudes). */
static uint64_t sm64_next(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ULL;
  return sy_fmix(*s);
}

/* 2-D 5-point upwind.  If uvel != NULL the velocity at node r is (uvel[r], uvel[r]) (config C2,
 * Picard linearisation b = u_{k-1}(1,1)); otherwise it is the constant (bx, by) (config C1).
 * row_ptr/col_idx may be NULL (values only, pattern assumed from a previous call). */
int64_t sy_fill5(int N, double cd, double ih, double idt, double bx, double by, const double* uvel,
                 int32_t* row_ptr, int32_t* col_idx, double* val) {
  int64_t nnz = 0;
  double tv[5];
  int32_t tc[5];
  if (row_ptr) row_ptr[0] = 0;
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) {
      int64_t r = (int64_t)j * N + i;
      double vx = uvel ? uvel[r] : bx, vy = uvel ? uvel[r] : by;
      int k = sy_row5(i, j, N, cd, ih, idt, vx, vy, tv, tc);
      for (int q = 0; q < k; ++q) {
        if (val) val[nnz + q] = tv[q];
        if (col_idx) col_idx[nnz + q] = tc[q];
      }
      nnz += k;
      if (row_ptr) row_ptr[r + 1] = (int32_t)nnz;
    }
  return nnz;
}

/* 2-D 9-point cross, rotating velocity b = (-(y-1/2), x-1/2) at node ((i+1)h, (j+1)h). */
int64_t sy_fill9(int N, double h, double cdif, double c6, double idt, int32_t* row_ptr,
                 int32_t* col_idx, double* val) {
  int64_t nnz = 0;
  double tv[9];
  int32_t tc[9];
  if (row_ptr) row_ptr[0] = 0;
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) {
      int64_t r = (int64_t)j * N + i;
      double x = (double)(i + 1) * h, y = (double)(j + 1) * h;
      double bx = -(y - 0.5), by = x - 0.5;
      int k = sy_row9(i, j, N, cdif, c6, idt, bx, by, tv, tc);
      for (int q = 0; q < k; ++q) {
        if (val) val[nnz + q] = tv[q];
        if (col_idx) col_idx[nnz + q] = tc[q];
      }
      nnz += k;
      if (row_ptr) row_ptr[r + 1] = (int32_t)nnz;
    }
  return nnz;
}

/* 3-D 7-point upwind, constant velocity (bx, by, bz). */
int64_t sy_fill7(int N, double cd, double ih, double idt, double bx, double by, double bz,
                 int32_t* row_ptr, int32_t* col_idx, double* val) {
  int64_t nnz = 0;
  double tv[7];
  int32_t tc[7];
  if (row_ptr) row_ptr[0] = 0;
  for (int l = 0; l < N; ++l)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        int64_t r = ((int64_t)l * N + j) * N + i;
        int k = sy_row7(i, j, l, N, cd, ih, idt, bx, by, bz, tv, tc);
        for (int q = 0; q < k; ++q) {
          if (val) val[nnz + q] = tv[q];
          if (col_idx) col_idx[nnz + q] = tc[q];
        }
        nnz += k;
        if (row_ptr) row_ptr[r + 1] = (int32_t)nnz;
      }
  return nnz;
}

/* C5 block pattern: E^3 elements, 7-point face connectivity, non-periodic. Returns nnzb. */
int64_t sy_c5_pattern(int E, int32_t* row_ptr, int32_t* col_idx, int8_t* kind) {
  int64_t nb = 0;
  int64_t EE = (int64_t)E * E;
  if (row_ptr) row_ptr[0] = 0;
  for (int z = 0; z < E; ++z)
    for (int y = 0; y < E; ++y)
      for (int x = 0; x < E; ++x) {
        int64_t e = (int64_t)z * EE + (int64_t)y * E + x;
        int64_t cols[7];
        int8_t kd[7];
        int k = 0;
        if (z > 0)     { cols[k] = e - EE; kd[k++] = 1; }
        if (y > 0)     { cols[k] = e - E;  kd[k++] = 1; }
        if (x > 0)     { cols[k] = e - 1;  kd[k++] = 1; }
        cols[k] = e; kd[k++] = 0;
        if (x < E - 1) { cols[k] = e + 1;  kd[k++] = 2; }
        if (y < E - 1) { cols[k] = e + E;  kd[k++] = 2; }
        if (z < E - 1) { cols[k] = e + EE; kd[k++] = 2; }
        for (int q = 0; q < k; ++q) {
          if (col_idx) col_idx[nb + q] = (int32_t)cols[q];
          if (kind) kind[nb + q] = kd[q];
        }
        nb += k;
        if (row_ptr) row_ptr[e + 1] = (int32_t)nb;
      }
  return nb;
}

/* C5 base values of the nnzb blocks (B x B, column-major inside a block). */
void sy_c5_values(int64_t nnzb, int B, uint64_t seed, const int8_t* kind, double s_up, double s_dn,
                  double* val) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nnzb; ++b)
    for (int c = 0; c < B; ++c)
      for (int r = 0; r < B; ++r)
        val[b * B * B + (int64_t)c * B + r] = sy_c5_base(seed, b, r, c, B, kind[b], s_up, s_dn);
}

/* A_t = A_{t-1} o (1 + 0.01 xi_t), entry-wise. */
void sy_c5_perturb(int64_t nval, uint64_t seed, int t, double* val) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < nval; ++e) val[e] = val[e] * sy_c5_factor(seed, t, e);
}

/* seeded N(0,1)-like vector (C5 right-hand side). */
void sy_normal_vec(int64_t n, uint64_t seed, uint64_t stream, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sy_normal12(seed, stream, (uint64_t)i);
}

/* b = u/dt + f (implicit Euler right-hand side, PAPER.md:592-598 with the configs' forcing). */
void sy_rhs(int64_t n, const double* u, double dt, double f, double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) b[i] = u[i] / dt + f;
}

/* Sum of nb Gaussian bumps exp(-|x-c|^2/w^2) on the interior nodes of an N^dim grid
 * (dim 2 or 3), h = 1/(N+1); centres U[0.2,0.8]^dim, amplitudes U[amp_lo, amp_hi], drawn
 * in that order from splitmix64(seed).  Host only (uses exp). */
void sy_bumps(int dim, int N, int nb, double width, double amp_lo, double amp_hi, uint64_t seed,
              double* u) {
  double c[16][3], a[16];
  uint64_t s = seed;
  if (nb > 16) nb = 16;
  for (int b = 0; b < nb; ++b) {
    for (int d = 0; d < dim; ++d) c[b][d] = 0.2 + 0.6 * sy_u01(sm64_next(&s));
    a[b] = amp_lo + (amp_hi - amp_lo) * sy_u01(sm64_next(&s));
  }
  double h = 1.0 / (double)(N + 1);
  int64_t n = 1;
  for (int d = 0; d < dim; ++d) n *= N;
  for (int64_t r = 0; r < n; ++r) {
    double p[3];
    int64_t q = r;
    for (int d = 0; d < dim; ++d) { p[d] = (double)(q % N + 1) * h; q /= N; }
    double v = 0.0;
    for (int b = 0; b < nb; ++b) {
      double d2 = 0.0;
      for (int d = 0; d < dim; ++d) d2 += (p[d] - c[b][d]) * (p[d] - c[b][d]);
      v += a[b] * exp(-d2 / (width * width));
    }
    u[r] = v;
  }
}

/* oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation (C99, IEEE binary64, single thread,
 * built with -O2 -ffp-contract=off, no -ffast-math) of what the recycled-GMRES hot path
 * computes, written from PAPER.md (arXiv:1807.09467).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or helper with the CUDA library (paper_1807_09467_b200/csrc); neither includes the other.
 *
 * Definitions followed (SURVEY.md §8c gives the readings; DESIGN.md lists them):
 *   - or_spmv:  y = A x, CSR or BSR, each row summed in stored order ("the cost of a
 *               matrix-vector multiplication reduces to O(mb)").
 *   - or_solve: the minimal-residual iterate ("minimal residual:
 *               min_{z in S_k} ||r_k||") over the search space of each restart cycle c
 *                 plain   : x_c + K_j(A, r_c)                        (GMRES)
 *                 augment : x_c + span(W) + K_j(A, r_c)              (eq. def_aug_S_space)
 *                 deflate : x_c + span(W) + K_j(P A, P r_c),         (Table 1 row "deflated LS",
 *                           P = I - AW((AW)^T AW)^{-1}(AW)^T          PAPER.md:310, 348; eq. def_S_k_projected)
 *               with the start x_0 <- x0 + W (C^T C)^{-1} C^T r(x0), C = AW (the j = 0 case of the
 *               same minimisation; min-residual analogue of eq. projection_t_s).
 *                 orthogonal: Table 1 rows 4 / 1: as oblique with the Krylov projector I - W W^T
 *                            and the same per-cycle Galerkin start (R19)
 *                 oblique : Table 1 rows 5 / 2 (deflated / augmented oblique):
 *                           GMRES(m) on M_D A, M_D = I - AW E^{-1} W^T, E = W^T A W,
 *                           Galerkin start x_c += W E^{-1} W^T r(x_c) at every cycle (reading R15)
 *               The minimisation is solved EXPLICITLY: an orthonormal basis U_Z of the image
 *               A*[W, v_0..v_j] is grown by modified Gram-Schmidt applied twice (MGS2), the residual
 *               is r - U_Z U_Z^T r and the coefficients are R_Z^{-1} U_Z^T r.  This is the plain
 *               definition, not the GPU's Hessenberg/Givens/GCRO algebra.
 *   - or_ssor / or_solve_pc: SSOR(omega) preconditioner ("Symmetric Successive Over-Relaxation")
 *               in a given row ORDER (a permutation: the GPU's multicolour ordering is one such
 *               order), M = (D + wL) D^{-1} (D + wU) / (w(2-w)) with L/U the parts of A before/after
 *               each row in that order; applied as a RIGHT preconditioner ("A M y = b,
 *               x = M^{-1} y"): every Krylov direction v enters the search space as M^{-1} v and the
 *               Krylov operator is (projector) A M^{-1}.  DESIGN.md reading R18.
 *   - or_svd:   thin SVD by one-sided (Hestenes) Jacobi directly on X, long-double dot products;
 *               sorted non-increasing; rank = #{sigma > 1e-12 sigma_1} (PAPER.md:524-537, 552-553,
 *               Algorithm 1; Schmidt-Eckart-Young eq. opt_svd).
 *
 * Threading: every length-n loop is split into the SAME fixed partition of
 * OR_CHUNKS = 256 contiguous chunks whatever the thread count; a reduction sums each chunk
 * sequentially and then adds the 256 chunk sums in chunk order.  So every result is bitwise
 * identical for 1 or N threads (tested); OpenMP only decides which thread runs which chunk.
 * Loops shorter than OR_PAR_MIN run the same chunks on the calling thread.  Thread count:
 * or_set_threads (default: OpenMP's, i.e. all online cores or OMP_NUM_THREADS).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int fmt;          /* 0 = CSR, 1 = BSR (b x b blocks, column-major inside a block) */
  int64_t n;        /* scalar rows = columns */
  int32_t b;        /* block size (1 for CSR) */
  const int32_t* rp;/* row pointer (block rows for BSR), length n/b + 1 */
  const int32_t* ci;/* column (block-column) indices */
  const double* v;  /* values */
} or_mat;

typedef struct {
  int iterations;   /* Arnoldi steps summed over cycles */
  int cycles;       /* restart cycles started */
  int converged;
  int status;       /* 0 ok, 1 singular AW, 2 allocation failure */
  int hist_len;
  int k_used;
  double rel_residual; /* final TRUE ||b - A x|| / ||b|| */
} or_report;

/* ------------------------------------------------------------------------------------------ */
#define OR_CHUNKS 256
#define OR_PAR_MIN 65536
/* first index of chunk c of [0, n): a fixed partition, independent of the thread count */
static int64_t chunk_lo(int64_t n, int c) { return n * c / OR_CHUNKS; }

void or_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
int or_get_threads(void) { return omp_get_max_threads(); }

/* one scalar row of A x, summed in stored order */
static double spmv_row(const or_mat* A, int64_t row, const double* x) {
  double s = 0.0;
  if (A->fmt == 0) {
    for (int32_t p = A->rp[row]; p < A->rp[row + 1]; ++p) s += A->v[p] * x[A->ci[p]];
    return s;
  }
  const int64_t b = A->b, I = row / b, r = row % b;
  for (int32_t p = A->rp[I]; p < A->rp[I + 1]; ++p)
    for (int64_t c = 0; c < b; ++c) s += A->v[(int64_t)p * b * b + c * b + r] * x[(int64_t)A->ci[p] * b + c];
  return s;
}

/* y = A x: every row is an independent sum in stored order, so the row split cannot change it */
void or_spmv(const or_mat* A, const double* x, double* y) {
  const int64_t n = A->n;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int64_t i = 0; i < n; ++i) y[i] = spmv_row(A, i, x);
}

/* a single row of A x (used by tests to check sampled rows of huge products) */
double or_spmv_row(const or_mat* A, int64_t row, const double* x) { return spmv_row(A, row, x); }

/* a^T b: chunk sums in index order, then the OR_CHUNKS sums in chunk order */
static double dot(int64_t n, const double* a, const double* b) {
  double part[OR_CHUNKS];
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int c = 0; c < OR_CHUNKS; ++c) {
    double s = 0.0;
    for (int64_t i = chunk_lo(n, c); i < chunk_lo(n, c + 1); ++i) s += a[i] * b[i];
    part[c] = s;
  }
  double s = 0.0;
  for (int c = 0; c < OR_CHUNKS; ++c) s += part[c];
  return s;
}
static double nrm2(int64_t n, const double* a) { return sqrt(dot(n, a, a)); }
/* y += al x */
static void axpy(int64_t n, double al, const double* x, double* y) {
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int64_t i = 0; i < n; ++i) y[i] += al * x[i];
}
/* y = x / d */
static void divide(int64_t n, const double* x, double d, double* y) {
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] / d;
}
/* sum_i a_i b_i (and optionally a_i a_i, b_i b_i) in long double, chunked like dot() */
static void dot3_ld(int64_t n, const double* a, const double* b, long double* aa, long double* bb, long double* ab) {
  long double pa[OR_CHUNKS], pb[OR_CHUNKS], pg[OR_CHUNKS];
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int c = 0; c < OR_CHUNKS; ++c) {
    long double sa = 0.0L, sb = 0.0L, sg = 0.0L;
    for (int64_t i = chunk_lo(n, c); i < chunk_lo(n, c + 1); ++i) {
      sa += (long double)a[i] * a[i];
      sb += (long double)b[i] * b[i];
      sg += (long double)a[i] * b[i];
    }
    pa[c] = sa; pb[c] = sb; pg[c] = sg;
  }
  long double sa = 0.0L, sb = 0.0L, sg = 0.0L;
  for (int c = 0; c < OR_CHUNKS; ++c) { sa += pa[c]; sb += pb[c]; sg += pg[c]; }
  *aa = sa; *bb = sb; *ab = sg;
}

/* Modified Gram-Schmidt applied twice: z <- (I - U U^T) z against the q orthonormal columns
 * of U (n x q, column-major, leading dimension n).  coef[i] accumulates u_i^T z over both
 * passes (so that z_in = U coef + z_out).  Returns ||z_out||. */
static double mgs2(int64_t n, int q, const double* U, double* z, double* coef) {
  for (int i = 0; i < q; ++i) coef[i] = 0.0;
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < q; ++i) {
      double t = dot(n, U + (int64_t)i * n, z);
      coef[i] += t;
      axpy(n, -t, U + (int64_t)i * n, z);
    }
  return nrm2(n, z);
}

/* back substitution R c = e, R upper triangular q x q stored column-major with leading dim ld */
static void backsolve(int q, const double* R, int ld, const double* e, double* c) {
  for (int i = q - 1; i >= 0; --i) {
    double s = e[i];
    for (int l = i + 1; l < q; ++l) s -= R[(int64_t)l * ld + i] * c[l];
    c[i] = s / R[(int64_t)i * ld + i];
  }
}

static void residual(const or_mat* A, const double* b, const double* x, double* r) {
  or_spmv(A, x, r);
  const int64_t n = A->n;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
}

/* SSOR preconditioner in a row order: order[idx] = row processed idx-th (a permutation of 0..n-1). */
typedef struct {
  const int32_t* order;
  double omega;
  int32_t* pos;      /* pos[order[idx]] = idx */
  double* tmp;       /* n scratch */
} or_prec;

/* out = M^{-1} z, M = (D + wL) D^{-1} (D + wU) / (w(2-w)) in the order of pc (Saad, "Iterative
 * Methods for Sparse Linear Systems", SSOR preconditioner): forward sweep w = (D + wL)^{-1} w(2-w) z,
 * then backward sweep t = (D + wU)^{-1} D w.  CSR only.  Returns 0, or 3 if a diagonal entry is
 * missing or zero. */
static int ssor_apply(const or_mat* A, const or_prec* pc, const double* z, double* out) {
  const int64_t n = A->n;
  const double om = pc->omega, sc = om * (2.0 - om);
  for (int64_t idx = 0; idx < n; ++idx) {          /* forward: rows in order */
    const int32_t r = pc->order[idx];
    double s = sc * z[r], d = 0.0;
    for (int32_t p = A->rp[r]; p < A->rp[r + 1]; ++p) {
      const int32_t j = A->ci[p];
      if (j == r) d = A->v[p];
      else if (pc->pos[j] < idx) s -= om * A->v[p] * out[j];
    }
    if (d == 0.0) return 3;
    out[r] = s / d;
  }
  for (int64_t idx = n - 1; idx >= 0; --idx) {     /* backward: rows in reverse order */
    const int32_t r = pc->order[idx];
    double s = 0.0, d = 0.0;
    for (int32_t p = A->rp[r]; p < A->rp[r + 1]; ++p) {
      const int32_t j = A->ci[p];
      if (j == r) d = A->v[p];
      else if (pc->pos[j] > idx) s += om * A->v[p] * out[j];
    }
    out[r] = (d * out[r] - s) / d;
  }
  return 0;
}

/* y = A M^{-1} v (pc != NULL) or A v */
static int op_apply(const or_mat* A, const or_prec* pc, const double* v, double* y) {
  if (!pc) { or_spmv(A, v, y); return 0; }
  int st = ssor_apply(A, pc, v, pc->tmp);
  or_spmv(A, pc->tmp, y);
  return st;
}

/* x += M^{-1} (V c) over q columns of V (n x q, column-major); scratch t (n) */
static int add_krylov_part(const or_mat* A, const or_prec* pc, const double* V, const double* c, int q,
                           double* t, double* x) {
  const int64_t n = A->n;
  if (!pc) {
    for (int i = 0; i < q; ++i) axpy(n, c[i], V + (int64_t)i * n, x);
    return 0;
  }
  memset(t, 0, sizeof(double) * n);
  for (int i = 0; i < q; ++i) axpy(n, c[i], V + (int64_t)i * n, t);
  int st = ssor_apply(A, pc, t, pc->tmp);
  axpy(n, 1.0, pc->tmp, x);
  return st;
}

static int solve_oblique(const or_mat* A, const double* b, const double* x0, int m, int row2, int orth,
                         const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                         double* hist, int hist_cap, const or_prec* pc);
/* The Krylov basis of the LAST restart cycle of a solve, for the basis invariants (SURVEY.md §8(c)
 * "Arnoldi relation A V_m = V_{m+1} H_m", "V orthonormal", GCRO relation "A V_m = Q B_m + V_{m+1} H_m"
 * ).  With J Arnoldi steps in that cycle:
 *   V  n x J        v_0 .. v_{J-1} (column-major, leading dimension n)
 *   H  (m+1) x m    column-major, leading dimension m+1: H[i + j(m+1)] = h_{ij}, i <= j+1 < J+1
 *                   (the MGS2 coefficients of A v_j against v_0..v_j, and h_{j+1,j} = ||w||)
 *   B  k x m        deflate only: B[l + j k] = u_l^T A v_j against the orthonormal basis U_C of A W
 *                   (the coefficients of the projection P, P = I - U_C U_C^T)
 *   steps           J */
typedef struct {
  double* V;
  double* H;
  double* B;
  int steps;
} or_basis;

static int solve_impl(const or_mat* A, const double* b, const double* x0, int m, int variant,
                      const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                      double* hist, int hist_cap, const or_prec* pc, or_basis* bx);

int or_solve(const or_mat* A, const double* b, const double* x0, int m, int variant,
             const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
             double* hist, int hist_cap) {
  return solve_impl(A, b, x0, m, variant, W, k, tol, max_iters, x, rep, hist, hist_cap, NULL, NULL);
}

/* or_solve that also returns the last cycle's Krylov basis (or_basis above; plain, augment,
 * deflate; V n x m, H (m+1) x m, B k x m caller-allocated, B may be NULL).  *steps = J. */
int or_solve_basis(const or_mat* A, const double* b, const double* x0, int m, int variant,
                   const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                   double* V, double* H, double* B, int* steps) {
  or_basis bx = {V, H, B, 0};
  int st = solve_impl(A, b, x0, m, variant, W, k, tol, max_iters, x, rep, NULL, 0, NULL, &bx);
  *steps = bx.steps;
  return st;
}

/* or_solve with a right SSOR(omega) preconditioner in the row order `order` (NULL: none). */
int or_solve_pc(const or_mat* A, const double* b, const double* x0, int m, int variant,
                const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                double* hist, int hist_cap, const int32_t* order, double omega) {
  if (!order) return solve_impl(A, b, x0, m, variant, W, k, tol, max_iters, x, rep, hist, hist_cap, NULL, NULL);
  or_prec pc = {order, omega, malloc(sizeof(int32_t) * A->n), malloc(sizeof(double) * A->n)};
  int st = 2;
  if (pc.pos && pc.tmp) {
    for (int64_t i = 0; i < A->n; ++i) pc.pos[order[i]] = (int32_t)i;
    st = solve_impl(A, b, x0, m, variant, W, k, tol, max_iters, x, rep, hist, hist_cap, &pc, NULL);
  }
  free(pc.pos); free(pc.tmp);
  return st;
}

/* out = M^{-1} z for the SSOR(omega) preconditioner in row order `order` (0, or 3: zero diagonal) */
int or_ssor(const or_mat* A, const int32_t* order, double omega, const double* z, double* out) {
  or_prec pc = {order, omega, malloc(sizeof(int32_t) * A->n), NULL};
  if (!pc.pos) return 2;
  for (int64_t i = 0; i < A->n; ++i) pc.pos[order[i]] = (int32_t)i;
  int st = ssor_apply(A, &pc, z, out);
  free(pc.pos);
  return st;
}

static int solve_impl(const or_mat* A, const double* b, const double* x0, int m, int variant,
                      const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                      double* hist, int hist_cap, const or_prec* pc, or_basis* bx) {
  if (variant >= 3 && variant <= 6 && W != NULL && k > 0)
    return solve_oblique(A, b, x0, m, variant == 4 || variant == 6, variant >= 5, W, k, tol, max_iters, x, rep,
                         hist, hist_cap, pc);
  if (variant >= 3 && variant <= 6) variant = 0;   /* no recycle space: plain GMRES */
  const int64_t n = A->n;
  memset(rep, 0, sizeof(*rep));
  const int kk = (variant != 0 && W != NULL) ? k : 0;
  rep->k_used = kk;
  double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {                       /* b = 0 -> x = 0 */
    memset(x, 0, sizeof(double) * n);
    rep->converged = 1;
    return 0;
  }
  if (x0) memcpy(x, x0, sizeof(double) * n); else memset(x, 0, sizeof(double) * n);

  const int qmax = kk + m;
  double* V = malloc(sizeof(double) * n * (m + 1));       /* Krylov basis */
  double* UZ = malloc(sizeof(double) * n * (qmax + 1));   /* orthonormal image basis */
  double* RZ = calloc((size_t)(qmax + 1) * (qmax + 1), sizeof(double));
  double* e = malloc(sizeof(double) * (qmax + 1));
  double* c = malloc(sizeof(double) * (qmax + 1));
  double* coef = malloc(sizeof(double) * (qmax + m + 2));
  double* r = malloc(sizeof(double) * n);
  double* rho = malloc(sizeof(double) * n);
  double* w = malloc(sizeof(double) * n);
  double* z = malloc(sizeof(double) * n);
  if (!V || !UZ || !RZ || !e || !c || !coef || !r || !rho || !w || !z) { rep->status = 2; goto out; }

  /* U_C, R_C: thin QR of C = A W by MGS2, column by column (columns 0..kk-1 of U_Z / R_Z). */
  for (int l = 0; l < kk; ++l) {
    or_spmv(A, W + (int64_t)l * n, z);
    double cn = nrm2(n, z);
    double zn = mgs2(n, l, UZ, z, coef);
    if (!(zn > 1e-12 * cn)) { rep->status = 1; goto out; }
    for (int i = 0; i < l; ++i) RZ[(int64_t)l * (qmax + 1) + i] = coef[i];
    RZ[(int64_t)l * (qmax + 1) + l] = zn;
    divide(n, z, zn, UZ + (int64_t)l * n);
  }
  /* start: x <- x + W R_C^{-1} U_C^T r(x)  (min over x + span W) */
  if (kk > 0) {
    residual(A, b, x, r);
    for (int l = 0; l < kk; ++l) {          /* MGS projection coefficients of r on U_C */
      e[l] = dot(n, UZ + (int64_t)l * n, r);
      axpy(n, -e[l], UZ + (int64_t)l * n, r);
    }
    backsolve(kk, RZ, qmax + 1, e, c);
    for (int l = 0; l < kk; ++l) axpy(n, c[l], W + (int64_t)l * n, x);
  }

  for (;;) {
    residual(A, b, x, r);
    double beta = nrm2(n, r);
    rep->rel_residual = beta / bnorm;
    if (beta / bnorm <= tol) { rep->converged = 1; break; }
    if (rep->iterations >= max_iters) break;
    rep->cycles++;
    /* rho = r - U_C U_C^T r (MGS) and e[0..kk) */
    memcpy(rho, r, sizeof(double) * n);
    for (int l = 0; l < kk; ++l) {
      e[l] = dot(n, UZ + (int64_t)l * n, rho);
      axpy(n, -e[l], UZ + (int64_t)l * n, rho);
    }
    /* Krylov start vector: r_c (plain, augment) or P r_c (deflate, Table 1 row 6) */
    if (variant == 2 && kk > 0) {
      memcpy(w, r, sizeof(double) * n);
      mgs2(n, kk, UZ, w, coef);
    } else {
      memcpy(w, r, sizeof(double) * n);
    }
    double v0n = nrm2(n, w);
    if (!(v0n > 0.0)) break;
    divide(n, w, v0n, V);

    int q = kk;   /* current image-basis size */
    for (int j = 0; j < m; ++j) {
      double* vj = V + (int64_t)j * n;
      if (op_apply(A, pc, vj, w)) { rep->status = 3; goto out; }  /* w = A v_j  (A M^{-1} v_j) */
      /* image column A v_j -> U_Z by MGS2 */
      memcpy(z, w, sizeof(double) * n);
      double wn = nrm2(n, w);
      double zn = mgs2(n, q, UZ, z, coef);
      int image_breakdown = !(zn > 1e-14 * wn);
      if (!image_breakdown) {
        for (int i = 0; i < q; ++i) RZ[(int64_t)q * (qmax + 1) + i] = coef[i];
        RZ[(int64_t)q * (qmax + 1) + q] = zn;
        divide(n, z, zn, UZ + (int64_t)q * n);
        e[q] = dot(n, UZ + (int64_t)q * n, rho);
        axpy(n, -e[q], UZ + (int64_t)q * n, rho);
        ++q;
      }
      double res = nrm2(n, rho);
      /* next Krylov vector: Arnoldi (MGS2) on A (plain/augment) or on P A (deflate) */
      if (variant == 2 && kk > 0) {
        mgs2(n, kk, UZ, w, coef);
        if (bx && bx->B)
          for (int l = 0; l < kk; ++l) bx->B[l + (int64_t)j * kk] = coef[l];
      }
      double hn = mgs2(n, j + 1, V, w, coef);
      if (bx) {
        for (int i = 0; i <= j; ++i) bx->H[i + (int64_t)j * (m + 1)] = coef[i];
        bx->H[j + 1 + (int64_t)j * (m + 1)] = hn;
      }
      rep->iterations++;
      if (hist && rep->hist_len < hist_cap) hist[rep->hist_len++] = res / bnorm;
      int stop = (res / bnorm <= tol) || image_breakdown || !(hn > 1e-14 * beta) || j == m - 1 ||
                 rep->iterations >= max_iters;
      if (!stop) {
        divide(n, w, hn, V + (int64_t)(j + 1) * n);
        continue;
      }
      if (bx) {  /* this cycle's basis v_0 .. v_j (a later cycle overwrites it) */
        memcpy(bx->V, V, sizeof(double) * n * (j + 1));
        bx->steps = j + 1;
      }
      /* coefficients over the search basis [W, v_0, ..., v_{q-kk-1}] */
      backsolve(q, RZ, qmax + 1, e, c);
      for (int l = 0; l < kk; ++l) axpy(n, c[l], W + (int64_t)l * n, x);
      add_krylov_part(A, pc, V, c + kk, q - kk, z, x);   /* x += (M^{-1}) V c_V */
      break;
    }
  }
out:
  free(V); free(UZ); free(RZ); free(e); free(c); free(coef); free(r); free(rho); free(w); free(z);
  return rep->status;
}

/* Apply the north-star deflation projector P = I - AW((AW)^T AW)^{-1}(AW)^T (the
 * "orthogonal projector onto A V_s" applied as I - P_{AV,AV}) to the `nz` vectors Z (n x nz,
 * column-major) in place, via the MGS2 QR of AW exactly as or_solve uses it.  Returns 1 if AW is
 * rank deficient.  Exposed so tests can check idempotence and P A W = 0. */
int or_lsproj(const or_mat* A, const double* W, int k, double* Z, int nz) {
  const int64_t n = A->n;
  double* UC = malloc(sizeof(double) * n * (k + 1));
  double* coef = malloc(sizeof(double) * (k + 1));
  int st = 0;
  for (int l = 0; l < k && !st; ++l) {
    double* z = UC + (int64_t)l * n;
    or_spmv(A, W + (int64_t)l * n, z);
    double cn = nrm2(n, z);
    double zn = mgs2(n, l, UC, z, coef);
    if (!(zn > 1e-12 * cn)) { st = 1; break; }
    divide(n, z, zn, z);
  }
  if (!st)
    for (int c = 0; c < nz; ++c) mgs2(n, k, UC, Z + (int64_t)c * n, coef);
  free(UC); free(coef);
  return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Galerkin restriction and oblique deflation projector (eq. left_deflation):
 *   E = W^T A W  (k x k, "the restriction of A onto V_s"),  M_D = I - A W E^{-1} W^T.
 * E is factored by Gaussian elimination with partial pivoting (plain textbook LU). */
typedef struct {
  int k;
  int64_t n;
  const double* W;
  double* C;    /* A W, n x k column-major */
  double* LU;   /* k x k, row-major, L (unit) and U packed */
  int* piv;
} oblique_ctx;

static void ob_free(oblique_ctx* o) { free(o->C); free(o->LU); free(o->piv); }

/* returns 0 ok, 1 E singular (the paper takes no preventive measure), 2 no memory */
static int ob_setup(const or_mat* A, const double* W, int k, oblique_ctx* o) {
  const int64_t n = A->n;
  o->k = k; o->n = n; o->W = W;
  o->C = malloc(sizeof(double) * n * k);
  o->LU = malloc(sizeof(double) * k * k);
  o->piv = malloc(sizeof(int) * k);
  if (!o->C || !o->LU || !o->piv) return 2;
  for (int l = 0; l < k; ++l) or_spmv(A, W + (int64_t)l * n, o->C + (int64_t)l * n);
  double emax = 0.0;
  for (int a = 0; a < k; ++a)                       /* E[a][c] = w_a^T (A w_c) */
    for (int c = 0; c < k; ++c) {
      o->LU[a * k + c] = dot(n, W + (int64_t)a * n, o->C + (int64_t)c * n);
      if (fabs(o->LU[a * k + c]) > emax) emax = fabs(o->LU[a * k + c]);
    }
  for (int c = 0; c < k; ++c) {
    int p = c;
    for (int r = c + 1; r < k; ++r)
      if (fabs(o->LU[r * k + c]) > fabs(o->LU[p * k + c])) p = r;
    o->piv[c] = p;
    if (!(fabs(o->LU[p * k + c]) > 1e-13 * emax)) return 1;
    if (p != c)
      for (int cc = 0; cc < k; ++cc) {
        double t = o->LU[c * k + cc]; o->LU[c * k + cc] = o->LU[p * k + cc]; o->LU[p * k + cc] = t;
      }
    for (int r = c + 1; r < k; ++r) {
      double f = o->LU[r * k + c] / o->LU[c * k + c];
      o->LU[r * k + c] = f;
      for (int cc = c + 1; cc < k; ++cc) o->LU[r * k + cc] -= f * o->LU[c * k + cc];
    }
  }
  return 0;
}

/* t = E^{-1} W^T y */
static void ob_coef(const oblique_ctx* o, const double* y, double* t) {
  const int k = o->k;
  for (int a = 0; a < k; ++a) t[a] = dot(o->n, o->W + (int64_t)a * o->n, y);
  for (int c = 0; c < k; ++c) {                     /* apply the row swaps, then L, then U */
    double s = t[c]; t[c] = t[o->piv[c]]; t[o->piv[c]] = s;
  }
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < r; ++c) t[r] -= o->LU[r * k + c] * t[c];
  for (int r = k - 1; r >= 0; --r) {
    for (int c = r + 1; c < k; ++c) t[r] -= o->LU[r * k + c] * t[c];
    t[r] /= o->LU[r * k + r];
  }
}

/* y <- M_D y = y - A W E^{-1} W^T y */
static void ob_apply(const oblique_ctx* o, double* y, double* t) {
  ob_coef(o, y, t);
  for (int l = 0; l < o->k; ++l) axpy(o->n, -t[l], o->C + (int64_t)l * o->n, y);
}

/* x <- x + W E^{-1} W^T (b - A x): the Galerkin projection start (eq. projection_guess /
 * projection_t_s) applied to the correction equation of x. */
static void ob_galerkin(const or_mat* A, const oblique_ctx* o, const double* b, double* x, double* r,
                        double* t) {
  residual(A, b, x, r);
  ob_coef(o, r, t);
  for (int l = 0; l < o->k; ++l) axpy(o->n, t[l], o->W + (int64_t)l * o->n, x);
}

/* y <- (I - W W^T) y, the orthogonal projector of Table 1 rows 1 / 4 (W has
 * orthonormal columns, "V_s any orthogonal matrix"), written as its formula: t = W^T y,
 * y -= W t. */
static void orth_apply(const oblique_ctx* o, double* y, double* t) {
  for (int l = 0; l < o->k; ++l) t[l] = dot(o->n, o->W + (int64_t)l * o->n, y);
  for (int l = 0; l < o->k; ++l) axpy(o->n, -t[l], o->W + (int64_t)l * o->n, y);
}

/* Table 1 rows 5 ("deflated oblique", row2 = 0) and 2 ("augmented oblique", row2 = 1); with
 * orth = 1 rows 4 ("deflated orthogonal") and 1 ("augmented orthogonal"), whose Krylov operator is
 * (I - W W^T) A instead of M_D A and whose minimised quantity is ||(I - WW^T)(r_c - A z)||.
 * For orth the per-cycle Galerkin start is the COMPLETION of DESIGN.md R19: without it the W
 * component of the residual is never reduced (true residual stalls at 3.7e-4).  Rows 1
 * and 4 then coincide for the same reason rows 2 and 5 do (W^T r_c = 0 after the start).
 * Oblique: GMRES(m) on the Krylov operator M_D A, each restart cycle c being
 *   x_c <- x_c + W E^{-1} W^T r(x_c)                  (Galerkin start of the cycle)
 *   r_c = b - A x_c  (recomputed; equals M_D r of the un-projected iterate)
 *   stop if ||r_c|| / ||b|| <= tol                    (TRUE residual)
 *   Krylov initial vector  M_D r_c (row 5)  or  r_c (row 2)     (Table 1)
 *   x_{c+1} = x_c + z,  z = argmin_{z in K_j(M_D A, .)} ||M_D r_c - M_D A z||
 *                                                     (eq. left_deflation_iterate, PAPER.md:263,
 *                                                      with C_k = M_D A S_k: minimal residual)
 * The minimisation is explicit (MGS2 image basis of M_D A v_i, as in or_solve).  The last cycle
 * start also serves as the final oblique correction, so on return V^T (b - A x) = 0.
 * reading R15 (Galerkin start at every restart; makes rows 2 and 5 coincide at every cycle, the
 * identity eq. equivalence_oblique). */
static int solve_oblique(const or_mat* A, const double* b, const double* x0, int m, int row2, int orth,
                         const double* W, int k, double tol, int max_iters, double* x, or_report* rep,
                         double* hist, int hist_cap, const or_prec* pc) {
  const int64_t n = A->n;
  memset(rep, 0, sizeof(*rep));
  rep->k_used = k;
  double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * n);
    rep->converged = 1;
    return 0;
  }
  if (x0) memcpy(x, x0, sizeof(double) * n); else memset(x, 0, sizeof(double) * n);
  oblique_ctx o = {0};
  double* V = malloc(sizeof(double) * n * (m + 1));
  double* UZ = malloc(sizeof(double) * n * (m + 1));
  double* RZ = calloc((size_t)(m + 1) * (m + 1), sizeof(double));
  double* e = malloc(sizeof(double) * (m + 1));
  double* c = malloc(sizeof(double) * (m + 1));
  double* coef = malloc(sizeof(double) * (2 * m + 2));
  double* t = malloc(sizeof(double) * (k + 1));
  double* r = malloc(sizeof(double) * n);
  double* rho = malloc(sizeof(double) * n);
  double* w = malloc(sizeof(double) * n);
  double* z = malloc(sizeof(double) * n);
  if (!V || !UZ || !RZ || !e || !c || !coef || !t || !r || !rho || !w || !z) { rep->status = 2; goto out; }
  int st = ob_setup(A, W, k, &o);
  if (st) { rep->status = st; goto out; }
  for (;;) {
    ob_galerkin(A, &o, b, x, r, t);
    residual(A, b, x, r);
    double beta = nrm2(n, r);
    rep->rel_residual = beta / bnorm;
    if (beta / bnorm <= tol) { rep->converged = 1; break; }
    if (rep->iterations >= max_iters) break;
    rep->cycles++;
    memcpy(rho, r, sizeof(double) * n);               /* target M_D r_c */
    if (orth) orth_apply(&o, rho, t); else ob_apply(&o, rho, t);
    memcpy(w, row2 ? r : rho, sizeof(double) * n);   /* Krylov initial vector */
    double v0n = nrm2(n, w);
    if (!(v0n > 0.0)) break;
    divide(n, w, v0n, V);
    int q = 0;
    for (int j = 0; j < m; ++j) {
      if (op_apply(A, pc, V + (int64_t)j * n, w)) { rep->status = 3; goto out; }  /* w = M_D A (M^{-1}) v_j */
      if (orth) orth_apply(&o, w, t); else ob_apply(&o, w, t);
      memcpy(z, w, sizeof(double) * n);
      double wn = nrm2(n, w);
      double zn = mgs2(n, q, UZ, z, coef);
      int image_breakdown = !(zn > 1e-14 * wn);
      if (!image_breakdown) {
        for (int i = 0; i < q; ++i) RZ[(int64_t)q * (m + 1) + i] = coef[i];
        RZ[(int64_t)q * (m + 1) + q] = zn;
        divide(n, z, zn, UZ + (int64_t)q * n);
        e[q] = dot(n, UZ + (int64_t)q * n, rho);
        axpy(n, -e[q], UZ + (int64_t)q * n, rho);
        ++q;
      }
      double res = nrm2(n, rho);
      double hn = mgs2(n, j + 1, V, w, coef);         /* Arnoldi on M_D A */
      rep->iterations++;
      if (hist && rep->hist_len < hist_cap) hist[rep->hist_len++] = res / bnorm;
      int stop = (res / bnorm <= tol) || image_breakdown || !(hn > 1e-14 * beta) || j == m - 1 ||
                 rep->iterations >= max_iters;
      if (!stop) {
        divide(n, w, hn, V + (int64_t)(j + 1) * n);
        continue;
      }
      backsolve(q, RZ, m + 1, e, c);
      add_krylov_part(A, pc, V, c, q, z, x);          /* x += (M^{-1}) V c */
      break;
    }
  }
out:
  ob_free(&o);
  free(V); free(UZ); free(RZ); free(e); free(c); free(coef); free(t); free(r); free(rho); free(w); free(z);
  return rep->status;
}

/* M_D Z for the nz columns of Z (in place); returns 1 if E = W^T A W is singular.  Exposed so
 * tests can check the projector's defining properties (M_D A W = 0, W^T M_D = 0, M_D^2 = M_D). */
int or_obproj(const or_mat* A, const double* W, int k, double* Z, int nz) {
  oblique_ctx o = {0};
  double* t = malloc(sizeof(double) * (k + 1));
  int st = t ? ob_setup(A, W, k, &o) : 2;
  if (!st)
    for (int c = 0; c < nz; ++c) ob_apply(&o, Z + (int64_t)c * A->n, t);
  ob_free(&o);
  free(t);
  return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Thin SVD of X (n x s, column-major, leading dimension ldx) by one-sided Jacobi.
 * U (n x s) receives the left singular vectors (columns with sigma = 0 are left as computed,
 * i.e. zero), sigma[0..s) the singular values non-increasing.  *rank = #{sigma > 1e-12 sigma_1}.
 * Returns the number of sweeps used. */
int or_svd(int64_t n, int s, const double* X, int64_t ldx, double* U, double* sigma, int* rank) {
  for (int j = 0; j < s; ++j) memcpy(U + (int64_t)j * n, X + (int64_t)j * ldx, sizeof(double) * n);
  int sweep;
  for (sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < s - 1; ++p)
      for (int q = p + 1; q < s; ++q) {
        double* up = U + (int64_t)p * n;
        double* uq = U + (int64_t)q * n;
        long double a, bb, g;
        dot3_ld(n, up, uq, &a, &bb, &g);
        if (g == 0.0L) continue;
        if (fabsl(g) <= 1e-15L * sqrtl(a * bb)) continue;
        long double zeta = (bb - a) / (2.0L * g);
        long double t = (zeta >= 0 ? 1.0L : -1.0L) / (fabsl(zeta) + sqrtl(1.0L + zeta * zeta));
        long double cs = 1.0L / sqrtl(1.0L + t * t), sn = cs * t;
#pragma omp parallel for schedule(static) if (n >= OR_PAR_MIN)
        for (int64_t i = 0; i < n; ++i) {
          long double xp = up[i], xq = uq[i];
          up[i] = (double)(cs * xp - sn * xq);
          uq[i] = (double)(sn * xp + cs * xq);
        }
        rotated = 1;
      }
    if (!rotated) break;
  }
  /* column norms, sort non-increasing (selection sort; s is small) */
  int* perm = malloc(sizeof(int) * s);
  double* nr = malloc(sizeof(double) * s);
  for (int j = 0; j < s; ++j) {
    long double t, t2, t3;
    dot3_ld(n, U + (int64_t)j * n, U + (int64_t)j * n, &t, &t2, &t3);
    nr[j] = (double)sqrtl(t);
    perm[j] = j;
  }
  for (int a = 0; a < s; ++a) {
    int best = a;
    for (int c2 = a + 1; c2 < s; ++c2)
      if (nr[perm[c2]] > nr[perm[best]]) best = c2;
    int tmp = perm[a]; perm[a] = perm[best]; perm[best] = tmp;
  }
  double* tmpU = malloc(sizeof(double) * n * s);
  memcpy(tmpU, U, sizeof(double) * n * s);
  for (int a = 0; a < s; ++a) {
    double sg = nr[perm[a]];
    sigma[a] = sg;
    if (sg > 0.0) divide(n, tmpU + (int64_t)perm[a] * n, sg, U + (int64_t)a * n);
    else memset(U + (int64_t)a * n, 0, sizeof(double) * n);
  }
  int rk = 0;
  for (int a = 0; a < s; ++a)
    if (sigma[0] > 0.0 && sigma[a] > 1e-12 * sigma[0]) ++rk;
  *rank = rk;
  free(perm); free(nr); free(tmpU);
  return sweep;
}

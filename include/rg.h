/* rg.h — C ABI of the B200-native recycled GMRES(m) library (librg.so).
 *
 * Solves a SEQUENCE of sparse non-symmetric systems A_t x_t = b_t whose matrices and right-hand
 * sides arrive one at a time and may depend on earlier solutions (eqs.
 * algebra_pde / sequence_linear_systems: "they are not entirely available until the very last
 * element of the sequence").  Each solve is restarted GMRES(m),
 * optionally accelerated by a recycle space W built from the dominant left singular vectors of a
 * window of previous solutions (Algorithm 1), used through
 *   augmentation: search space x_c + span(W) + K_j(A, r_c)
 *   deflation   : x_c + span(W) + K_j(P A, P r_c), P = I - AW((AW)^T AW)^{-1}(AW)^T
 *                 (Table 1 row "deflated LS" :348; = GCRO inner iteration :332),
 * or through the Galerkin start and the oblique / orthogonal projectors of Table 1 rows 1, 2, 4, 5
 * (rg_variant), optionally with a right SSOR preconditioner (rg_set_preconditioner).
 * Every step runs in hand-written fp64 CUDA kernels for sm_100a; there is no CPU fallback.
 *
 * Conventions shared by all entry points
 *   - Every function returns rg_status; nothing aborts, throws or exits.  On failure the
 *     thread-local message rg_last_error() says why.
 *   - Pointers tagged by an rg_mem argument are HOST (pageable or pinned) or DEVICE (same CUDA
 *     device as the context, e.g. a torch tensor's data_ptr()) memory.  The caller owns every
 *     buffer it passes; the library deep-copies what it keeps into device memory it owns.
 *   - All work is issued on the caller's CUDA stream (rg_options.cuda_stream, NULL = a stream the
 *     library creates, ordered with the legacy default stream).  Calls that return results to
 *     the host (rg_build_recycle, rg_solve, rg_apply, rg_export, rg_kernel_stats) return when
 *     they are complete.  rg_update_matrix and rg_push_snapshot return when HOST inputs have been
 *     copied; with DEVICE inputs they return once the copy is enqueued on the stream (the caller
 *     must not overwrite the source buffer except by work ordered after it on that stream).
 *   - Dense vectors are fp64, length n, contiguous.  Indices are int32 (n, nnz < 2^31).
 *   - A context is single-owner and not thread-safe; distinct contexts are independent.
 */
#ifndef RG_H
#define RG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RG_API __attribute__((visibility("default")))
#else
#define RG_API
#endif

typedef struct rg_ctx rg_ctx; /* opaque; created by rg_create, owned by the library */

typedef enum {
  RG_OK = 0,
  RG_E_INVAL = 1,    /* invalid argument; no side effects                                      */
  RG_E_NOMEM = 2,    /* device or host allocation failed                                       */
  RG_E_CUDA = 3,     /* CUDA runtime error (message has the CUDA error string)                 */
  RG_E_STATE = 4,    /* call not valid in the current state (e.g. build with no snapshots)      */
  RG_E_SINGULAR = 5, /* A W rank deficient: min|r_ii| <= 1e-12 max|r_ii| of R_C, or (oblique)
                        E = W^T A W singular: a pivot <= 1e-13 max|E_ab| (PAPER.md:562-564
                        "E_s may be singular"); the recycle space is cleared                   */
  RG_E_NUMERIC = 6,  /* NaN/Inf met during the solve                                           */
  RG_E_CHECK = 7     /* CHECKED builds only (make rg-checked -> lib/librg_checked.so, test
                        infrastructure): a device-side bounds / invariant check failed; the
                        message names the source file and line.  Product builds never return it */
} rg_status;

typedef enum { RG_CSR = 0, RG_BSR = 1 } rg_format;
/* RG_PLAIN    GMRES(m)
 * RG_AUGMENT  min over x_c + span(W) + K_j(A, r_c)                (eq. def_aug_S_space, :205-217)
 * RG_DEFLATE  Table 1 row 6 "deflated LS" = GCRO inner iteration  (:310, :332, :348)
 * RG_OBLIQUE  Table 1 rows 5 / 2 "deflated / augmented oblique" (identical without a
 *             preconditioner, eq. equivalence_oblique :325-330): GMRES(m) on M_D A with
 *             M_D = I - A W E^{-1} W^T, E = W^T A W (:229-239), and the Galerkin start
 *             x_c += W E^{-1} W^T r(x_c) (eq. projection_t_s, :289, :419) at every restart
 *             (reading R15).  Requires k_eff <= 32; E singular -> RG_E_SINGULAR.
 * RG_ORTHOGONAL Table 1 rows 4 / 1 "deflated / augmented orthogonal" (:341, :346): GMRES(m) on
 *             (I - W W^T) A with the same per-restart Galerkin start, which is the completion that
 *             makes the TRUE residual converge (R19); rows 1 and 4 coincide under it.
 *             Same requirements as RG_OBLIQUE (the start needs E). */
typedef enum { RG_PLAIN = 0, RG_AUGMENT = 1, RG_DEFLATE = 2, RG_OBLIQUE = 3, RG_ORTHOGONAL = 4 } rg_variant;
typedef enum { RG_HOST = 0, RG_DEVICE = 1 } rg_mem;

/* A sparse matrix handed to rg_create / rg_update_matrix.
 *   CSR : n_rows scalar rows; row_ptr[n_rows+1] (row_ptr[0] = 0, non-decreasing,
 *         row_ptr[n_rows] = nnz); col_idx[nnz] strictly increasing within each row, in [0,n);
 *         val[nnz].  block must be 1.
 *   BSR : block = b (b divides n_rows); nb = n_rows/b block rows; row_ptr[nb+1] over blocks;
 *         col_idx[nnz] block-column indices (strictly increasing per block row); nnz = number of
 *         stored blocks; val[nnz*b*b], each b x b block stored COLUMN-MAJOR
 *         (val[p*b*b + c*b + r] = block_p(r, c)).
 *   In rg_update_matrix, row_ptr == col_idx == NULL keeps the current pattern and replaces the
 *   values only (the fast path for sequences with a fixed sparsity pattern).
 *   sell_C = 32 packs a CSR matrix into SELL-32-sigma internally: inside every window of
 *   sell_sigma consecutive rows the rows are ordered by decreasing length (stable), then cut into
 *   slices of 32 rows padded to the slice's longest row (Kreutzer et al.'s SELL-C-sigma; the
 *   permutation is internal: x, y, b and every vector of the API keep the caller's row order).
 *   sell_sigma = 1 (or 0): no sorting; otherwise a multiple of 32 (RG_E_INVAL if not).  A
 *   sorted SELL matrix (sigma > 1) always runs the graph path.  sell_C = 0 keeps CSR. */
typedef struct {
  rg_format fmt;
  int64_t n_rows;
  int64_t nnz;
  int32_t block;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
  rg_mem mem;
  int32_t sell_C;
  int32_t sell_sigma;
} rg_matrix;

/* Capacity limits fixed at creation (they size the device buffers):
 *   max_m         largest restart length m accepted by rg_solve      (1..128)
 *   max_snapshots snapshot-window capacity s (Algorithm 1's window)   (1..64)
 *   max_k         largest recycle dimension k                         (0..64, <= max_snapshots)
 *   cuda_stream   cudaStream_t to issue all work on (NULL = default stream)
 *   flags         RG_FLAG_* bits below */
typedef struct {
  int32_t max_m, max_snapshots, max_k;
  void* cuda_stream;
  int32_t flags;
} rg_options;

#define RG_FLAG_NO_GRAPH 1 /* launch kernels one by one instead of replaying CUDA graphs      */
#define RG_FLAG_PROFILE 2  /* record per-kernel device time (%globaltimer) for rg_kernel_stats */
#define RG_FLAG_CGS2 4     /* classical CGS2 (3 reductions per Arnoldi step) instead of the default
                              delayed CGS2 (1 reduction per step); same iterates in exact arithmetic */
#define RG_FLAG_NO_PERSIST 8 /* never use the single cooperative-kernel solve (any variant, CSR/SELL,
                                m <= 64, k <= 64, n_pad <= 1.6M rows: the measured crossover, DESIGN.md
                                §5.2); always use the CUDA-graph path */
#define RG_FLAG_KEEP_BASIS 16 /* keep the Krylov basis V, the Hessenberg matrix H-bar and (deflate) the GCRO
                                 matrix B of the last finished restart cycle of every solve, for
                                 rg_export(RG_EXPORT_V / _H / _B): one more n x (max_m + 1) device buffer and
                                 a copy of V at every cycle end (inspection and tests only) */

/* Solve report (fields follow SPEC.md's SolveReport).
 *   iterations   Arnoldi steps summed over restart cycles (residual and C = AW products are
 *                not counted; they are in spmv_count)
 *   restarts     restart cycles after the first
 *   converged    1 iff the TRUE relative residual ||b - A x||/||b|| <= tol
 *   k_eff        recycle dimension actually used (0 for plain or empty recycle space)
 *   spmv_count   sparse products issued by this solve
 *   history_len  entries written to history (one per Arnoldi step, least-squares estimate of
 *                the relative residual)
 *   rel_residual final true relative residual
 *   ms_total     device time of the solve (CUDA events), milliseconds */
typedef struct {
  int32_t iterations, restarts, converged, k_eff, spmv_count, history_len;
  double rel_residual, ms_total;
} rg_report;

/* Create a context for the sequence A_t x_t = b_t, t = 1, 2, ... of systems of dimension n
 * (eq. sequence_linear_systems: the systems arrive one at a time), with the first
 * matrix A = A_1 (validated and copied into device memory the library owns; the caller keeps its
 * arrays).  *ctx receives the context (NULL on failure).  Errors: RG_E_INVAL (n < 1 or >= 2^31, max_m
 * outside 1..128, max_snapshots outside 1..64, max_k outside 0..min(64, max_snapshots), a malformed
 * descriptor or pattern — no side effects), RG_E_CUDA (no device, or the current device is not compute
 * capability 10.x with at least 148 SMs: the kernels are sm_100a code with grids sized for the B200),
 * RG_E_NOMEM. */
RG_API rg_status rg_create(rg_ctx** ctx, int64_t n, const rg_matrix* A, const rg_options* opt);

/* Replace A by the next matrix A_t of the sequence ("the sequence of matrices and
 * right-hand sides depend on the previous solution"; same n and format).  Keeps the snapshot window
 * and W (Algorithm 1 carries them across systems); invalidates C = A W, its QR
 * factor Q and R_C, which are rebuilt by the next recycled solve.  row_ptr = col_idx = NULL: values
 * only (same pattern); otherwise the pattern is validated and replaced (RG_E_INVAL, no side
 * effects, if malformed). */
RG_API rg_status rg_update_matrix(rg_ctx* ctx, const rg_matrix* A);

/* Device pointer and length (doubles) of the library-owned matrix values (CSR order, or BSR blocks
 * column-major), for callers that generate A_t on the device: write the new values there on the
 * context's stream, then call rg_update_matrix with val == *values (row_ptr = col_idx = NULL), which
 * then skips the copy (SELL packing and the C = AW invalidation still happen).  The pointer stays
 * valid until the pattern changes or the context is destroyed. */
RG_API rg_status rg_matrix_values(rg_ctx* ctx, double** values, int64_t* len);

/* Append solution x (length n) to the snapshot window X (Algorithm 1 line "store the solution
 * x_i in the matrix X_m"), evicting the oldest column when the window is full. */
RG_API rg_status rg_push_snapshot(rg_ctx* ctx, const double* x, rg_mem mem);

/* Forget all snapshots and the recycle space. */
RG_API rg_status rg_clear_snapshots(rg_ctx* ctx);

/* Recycle space from the window: thin SVD X = Psi Sigma Phi^T, W = the first
 * k_eff = min(k, #snapshots, #{sigma_i > 1e-12 sigma_1}) left singular vectors.
 *   k       requested dimension, 1..max_k
 *   k_eff   (out, nullable) dimension kept
 *   sigma   (out, nullable, host) the #snapshots singular values, non-increasing
 * RG_E_STATE if the window is empty.
 * With k_eff == NULL and sigma == NULL the call is ASYNCHRONOUS: it enqueues the SVD on the stream
 * and returns without waiting; the next call that needs W (rg_solve, rg_export, a further build)
 * waits for the singular values, fixes k_eff and forms W.  The window may be pushed to meanwhile
 * (the build reads it in stream order).  Errors of the deferred part are reported by that call. */
RG_API rg_status rg_build_recycle(rg_ctx* ctx, int32_t k, int32_t* k_eff, double* sigma);

/* As rg_build_recycle, choosing which singular modes span W (PAPER.md:673-676 compares both):
 *   RG_MODES_LARGEST   the k dominant left singular vectors (Algorithm 1, the default)
 *   RG_MODES_SMALLEST  the k smallest NON-ZERO ones (sigma_i > 1e-12 sigma_1)
 * The SVD interval l of Algorithm 1 ("if (i mod l) = 0") is the caller's schedule: W and
 * the window persist across solves, and C = A W is rebuilt after every rg_update_matrix. */
#define RG_MODES_LARGEST 0
#define RG_MODES_SMALLEST 1
RG_API rg_status rg_build_recycle_modes(rg_ctx* ctx, int32_t k, int32_t modes, int32_t* k_eff, double* sigma);

/* Solve A x = b with restarted GMRES(m) (PAPER.md:36-38 restarts, :133-135 minimal residual,
 * :171-175 GMRES), accelerated by the recycle space through the variant's search space (rg_variant;
 * augmentation PAPER.md:205-217, deflation :310/:332/:348, Table 1 rows :341-348), stopping on the
 * true relative residual ("relative residual 1e-8").
 *   b, x0      length n in `mem`; x0 == NULL means x0 = 0
 *   m          restart length, 1..max_m
 *   tol        > 0; convergence is ||b - A x||_2 / ||b||_2 <= tol on the true residual
 *   max_iters  cap on Arnoldi steps (>= 1)
 *   x_out      length n in `mem`
 *   history    nullable HOST array receiving up to history_cap relative-residual estimates
 *   rep        nullable report
 * A recycled variant with an empty recycle space runs plain GMRES (k_eff = 0).  b = 0 gives
 * x = 0, converged, 0 iterations.  Non-convergence is RG_OK with rep->converged = 0.
 * On RG_E_SINGULAR (the recycle operator A W or E is singular; the recycle space is then cleared) the
 * contents of x_out are undefined: call again (it then runs plain GMRES, k_eff = 0). */
RG_API rg_status rg_solve(rg_ctx* ctx, const double* b, const double* x0, int32_t m, rg_variant v,
                          double tol, int32_t max_iters, double* x_out, rg_mem mem, double* history,
                          int32_t history_cap, rg_report* rep);

/* Preconditioning (R18).
 *   kind = RG_PREC_SSOR: SSOR(omega), 0 < omega < 2, in a MULTICOLOUR row order, applied as a
 *     RIGHT preconditioner ("A M y = b, x = M^{-1} y") by every later rg_solve of every
 *     variant: the Arnoldi operator becomes (projector) A M^{-1} and the Krylov part of x is
 *     M^{-1} V y, so GMRES still minimises (and the stop test still uses) the TRUE residual.
 *     M = (D + wL) D^{-1} (D + wU) / (w(2-w)), L / U = couplings to rows of lower / higher colour.
 *   colors     NULL: the library colours the symmetrised pattern greedily in natural order (5-point
 *              and 7-point grids get red-black, 9-point grids 4 colours); else n int32 colours in
 *              0..63 (host or device per `mem`) that must not give two coupled rows the same colour.
 *   ncolors_out nullable; receives the number of colours.
 *   kind = RG_PREC_NONE removes the preconditioner.
 * Errors: RG_E_INVAL for a BSR matrix, omega outside (0, 2), an invalid colouring or a row without a
 * stored diagonal entry (nothing is changed).  A later pattern change (rg_update_matrix with
 * row_ptr != NULL) removes the preconditioner; values-only updates keep it.  Solves with a
 * preconditioner run on the CUDA-graph path. */
#define RG_PREC_NONE 0
#define RG_PREC_SSOR 1
RG_API rg_status rg_set_preconditioner(rg_ctx* ctx, int32_t kind, double omega, const int32_t* colors,
                                       rg_mem mem, int32_t* ncolors_out);

/* y = M^{-1} x for the current preconditioner (x, y length n in `mem`); RG_E_STATE if none. */
RG_API rg_status rg_apply_preconditioner(rg_ctx* ctx, const double* x, double* y, rg_mem mem);

/* y = A x with the context's current matrix (x, y length n in `mem`). */
RG_API rg_status rg_apply(rg_ctx* ctx, const double* x, double* y, rg_mem mem);

/* Copy out internal quantities (for inspection and tests):
 *   RG_EXPORT_W   W   (n x k_eff, column-major, leading dimension n)
 *   RG_EXPORT_Q   Q   (n x k_eff) orthonormal basis of A W       (after a recycled solve)
 *   RG_EXPORT_RC  R_C (k_eff x k_eff, column-major, upper triangular, A W = Q R_C)
 *   *count receives k_eff for these three.
 * Krylov basis of the LAST finished restart cycle of the last rg_solve (context created with
 * RG_FLAG_KEEP_BASIS; variants plain / augment / deflate; "orthogonal basis of the
 * Krylov space", :169 the Arnoldi relation behind the iterate, :332 the GCRO relation).  With J
 * Arnoldi steps in that cycle (*count receives J):
 *   RG_EXPORT_V   V = [v_0 .. v_{J-1}]   (n x J, column-major, orthonormal)
 *   RG_EXPORT_H   H-bar                  ((J+1) x J, column-major, upper Hessenberg)
 *   RG_EXPORT_B   B = Q^T A V            (k_eff x J, column-major; deflate only)
 *   so that A V = V_{J+1} H-bar (plain, augment: Arnoldi on A) and A V = Q B + V_{J+1} H-bar (deflate:
 *   Arnoldi on P A, P = I - Q Q^T), v_J being the next (not exported) basis vector.
 * out == NULL only reports *count.  `out` must hold the stated number of doubles; returns
 * RG_E_STATE if the item is unavailable (not built, no finished cycle, flag not set). */
#define RG_EXPORT_W 0
#define RG_EXPORT_Q 1
#define RG_EXPORT_RC 2
#define RG_EXPORT_V 3
#define RG_EXPORT_H 4
#define RG_EXPORT_B 5
RG_API rg_status rg_export(rg_ctx* ctx, int32_t which, double* out, rg_mem mem, int32_t* count);

/* Per-kernel device-time statistics recorded while RG_FLAG_PROFILE is set. */
typedef struct {
  char name[24];
  int64_t launches;     /* launches that did work           */
  int64_t noop_launches;/* launches that returned early      */
  double total_ms;      /* summed device time of working launches (%globaltimer, first CTA start to
                           last CTA end) */
  double tail_ms;       /* part of total_ms spent in the last CTA's epilogue (reducing kernels) */
  double bytes;         /* summed algorithmic bytes (DESIGN.md byte model) */
} rg_kstat;
RG_API rg_status rg_kernel_stats(rg_ctx* ctx, rg_kstat* out, int32_t cap, int32_t* count);
/* Device timeline of the library's kernels (SURVEY.md §5 tracing; no nsys on the target boxes).  While
 * RG_FLAG_PROFILE is set (at rg_create), every kernel that keeps statistics appends events to a device
 * ring of 65,536 entries: its start (block 0's first instruction, %globaltimer ns), its end (the last
 * CTA's exit path) or a no-op launch.  rg_kernel_trace copies up to `cap` events in device order into
 * `out` (host memory, owned by the caller) and sets *count to the number recorded since the last
 * rg_reset_kernel_stats (which also clears the trace; events past the ring capacity are dropped and
 * counted).  `name` matches rg_kstat's.  RG_E_STATE if the context was created without RG_FLAG_PROFILE. */
typedef struct {
  int64_t t_ns;   /* %globaltimer                                  */
  int32_t kind;   /* 0 start, 1 end, 2 no-op launch                 */
  char name[20];
} rg_trace_event;
RG_API rg_status rg_kernel_trace(rg_ctx* ctx, rg_trace_event* out, int32_t cap, int32_t* count);
RG_API rg_status rg_reset_kernel_stats(rg_ctx* ctx);

RG_API void rg_destroy(rg_ctx* ctx);
RG_API const char* rg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RG_H */

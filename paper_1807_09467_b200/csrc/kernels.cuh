// kernels.cuh — host-side launch interface of librg's device kernels.
#pragma once
#include "common.cuh"
#include <utility>

namespace rg {

// Kernel launch with the PDL attribute when pdl (see pdl_wait in common.cuh).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                             Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Sparse matrix as stored on the device.
struct MatDev {
  int fmt = 0;                  // 0 CSR, 1 SELL-32, 2 BSR
  int64_t n = 0;
  const int32_t* rp = nullptr;  // CSR row pointer / BSR block-row pointer
  const int32_t* ci = nullptr;  // CSR columns / BSR block columns
  const double* v = nullptr;    // CSR values / BSR blocks (column-major b x b)
  int lpr = 4;                  // CSR lanes per row
  int b = 1;                    // BSR block size
  int64_t nb = 0;               // BSR block rows
  const int64_t* sp = nullptr;  // SELL slice pointer (entry offset of slice s)
  const int32_t* sw = nullptr;  // SELL slice widths
  const int32_t* sci = nullptr; // SELL columns (column-major inside a slice)
  const double* sv = nullptr;   // SELL values
  const int32_t* sperm = nullptr;   // SELL-32-sigma (sigma > 1): SELL position -> matrix row (null: identity)
  const int32_t* siperm = nullptr;  //                          matrix row -> SELL position
  int64_t nslices = 0;
  int tma = 1;                  // BSR-64: stream blocks with TMA bulk copies
  double bytes = 0.0;           // algorithmic bytes of one product (DESIGN.md byte model)
  int64_t nnz = 0;              // CSR entries / BSR stored blocks
};

// Kernels launched directly by the host without a device-side counter (recycle build, CholQR2,
// E^{-1}, SELL packing, validation, SSOR value refresh) are counted here; rg_kernel_stats reports
// the total as the entry "host_launched".
void note_host_launches(int n);

enum SpmvMode { SM_STEP = 0, SM_RES = 1, SM_PLAIN = 2, SM_STEP_PC = 3, SM_RES_Y = 4 };

// w = A v_j (STEP), r = b - A x (RES; epi != 0 runs the cycle-start epilogue on ||r||^2),
// y = A x (PLAIN), w = A pz (STEP_PC: pz = M^{-1} v_j from launch_ssor, same gating as STEP).
// pdl: launched with programmatic dependent launch (the kernels wait for their predecessor first)
cudaError_t launch_spmv(const MatDev& A, const Layout& L, DevState* st, int mode, const double* x,
                        double* y, int res_epi, cudaStream_t s, bool pdl = false);

// Y[:, 0:k] = A W[:, 0:k] (columns with leading dimension ld) with ONE read of A (a4: C = A W).
// Returns cudaErrorNotSupported when no SpMM kernel covers the format (caller loops SpMVs).
// xe != nullptr (BSR-64 TMA path, k + 1 <= 64 only; else cudaErrorInvalidValue): ye = A xe in the
// same pass — the solve-start product fused with C = A W (then SM_RES_Y finishes the residual).
cudaError_t launch_spmm(const MatDev& A, const double* W, double* Y, int64_t ld, int k, DevState* st, unsigned* counter,
                        cudaStream_t s, const double* xe = nullptr, double* ye = nullptr);

enum OrthOp {
  OP_D1 = 0, OP_UD2, OP_UN, OP_CS_DQ, OP_CS_UN, OP_XW, OP_XUPD, OP_NORMB,
  // oblique variant (M_D = I - C E^{-1} W^T, C = A W in columns [k, 2k)):
  OP_OB_CSD,  // cycle start: t = E^{-1} W^T r            (x += W t via OP_XW)
  OP_OB_CSU,  // cycle start: r -= C t, ||r||^2 -> cycle-start epilogue
  OP_OB_SD,   // Arnoldi step: t = E^{-1} W^T (A v_j)
  OP_OB_SU,   // Arnoldi step: A v_j -= C t               (the new column is M_D A v_j)
  OP_VY       // cycle end, preconditioned: pt = V y      (then pz = M^{-1} pt, OP_XUPD adds pz)
};
// cond != 0: cudaGraphConditionalHandle set to st->active by OP_UN's epilogue (graph WHILE node)
cudaError_t launch_orth(const Layout& L, DevState* st, int op, cudaStream_t s, unsigned long long cond = 0);
// DCGS2 Arnoldi step (dcgs.cu): phase 1 = dots + coefficient epilogue, 2 = update pass, 3 = the
// least-squares step of the finished column (one CTA, concurrent with phase 2; sets the WHILE condition)
cudaError_t launch_dcgs(const Layout& L, DevState* st, int phase, cudaStream_t s, unsigned long long cond = 0);
// RG_FLAG_KEEP_BASIS: copy the finished cycle's V into L.keepV at the cycle end (before the x update)
cudaError_t launch_keep_basis(const Layout& L, DevState* st, cudaStream_t s);
// WHILE-node condition from the state: which 0 -> active, 1 -> !done
cudaError_t launch_cond(const DevState* st, unsigned long long h, int which, cudaStream_t s);

// Whole solve in one cooperative kernel (persistent.cu): every variant, CSR / SELL, m <= 64,
// k <= 64.  cudaErrorNotSupported when outside that scope (caller uses the graph path).
// bar: [BAR_WORDS] zeroed barrier words; flags: [NSM * 8] zeroed neighbour-sync epochs;
// P: right SSOR preconditioner (nullptr: none; needs L.pz, L.pt).  ll: [ll_words()] reduction words,
// zeroed once at allocation and never again (their epochs continue in DevState::red_epoch).
constexpr int BAR_WORDS = 64 + 32 * NSM * 8;
struct PrecDev;
size_t ll_words();
cudaError_t launch_persistent(const Layout& L, const MatDev& A, DevState* st, double* tot_g, unsigned* bar,
                              unsigned* flags, unsigned long long* ll, int m, int k, int variant, const PrecDev* P,
                              cudaStream_t s);
// C = A W, CholQR2 -> Q (columns [VB - k, VB) of Z), R_C, R_C^{-1} (device state) in ONE cooperative
// kernel; *cflag (zeroed by the caller) set on a singular factor.  CSR / SELL, k <= 16; otherwise
// cudaErrorNotSupported (caller: build_c).  bar zeroed by the caller; ll as for launch_persistent.
// cgiven: C = A W already in the Q columns (BSR, after launch_spmm): the kernel is the CholQR2 alone.
// k <= 22.
cudaError_t launch_cbuild(const Layout& L, const MatDev& A, DevState* st, double* tot_g, unsigned* bar,
                          unsigned long long* ll, int k, int* cflag, cudaStream_t s, bool cgiven = false);

// ---- multicolour SSOR(omega) preconditioner (precond.cu)
constexpr int MAXCOLORS = 64;
// The matrix is stored a second time for the sweeps, rows in colour order (index idx = position in
// perm) and split by the colour of the column: L = couplings to lower colours (forward sweep), U =
// to higher colours (backward sweep), dinv = 1 / a_rr.  Each sweep then streams a contiguous slab
// and reads every off-diagonal entry exactly once per application (no colour tests).  The values
// are re-gathered from the CSR values after every matrix update (launch_ssor_values).
struct PrecDev {
  const int32_t* perm = nullptr;  // rows grouped by colour
  const int32_t* Lrp = nullptr;   // [n + 1] over idx
  const int32_t* Lci = nullptr;   // original column index
  double* Lv = nullptr;
  const int32_t* Lmap = nullptr;  // position of each L entry in the CSR values
  const int32_t* Urp = nullptr;
  const int32_t* Uci = nullptr;
  double* Uv = nullptr;
  const int32_t* Umap = nullptr;
  double* dinv = nullptr;         // [n] over idx
  double* dinvr = nullptr;        // [n] over the matrix row
  double* Lv1 = nullptr;          // [nL1] L values of the colour-1 rows times 1/a_jj of their column (fused forward sweep)
  int64_t l1base = 0, nL1 = 0;    // the colour-1 rows' L entries: [l1base, l1base + nL1)
  const int32_t* dmap = nullptr;  // position of a_rr (over idx)
  int64_t nL = 0, nU = 0;
  int ncolors = 0;
  double omega = 1.0;
  int64_t coff[MAXCOLORS + 1] = {};  // colour c = perm[coff[c] .. coff[c+1])
  int64_t cL[MAXCOLORS] = {};        // L / U entries of the rows of colour c (byte model)
  int64_t cU[MAXCOLORS] = {};
};
// Lv / Uv / dinv from the CSR values v.
cudaError_t launch_ssor_values(const PrecDev& P, const double* v, int64_t n, cudaStream_t s);
// out = M^{-1} in.  gate 0: always; 1: Arnoldi step (in = the state's u, noop as SM_STEP);
// 2: cycle end (noop unless st->have_xupd).
cudaError_t launch_ssor(const PrecDev& P, const Layout& L, DevState* st, const double* in, double* out, int gate,
                        cudaStream_t s);

// ---- dense / recycle-build kernels (dense.cu)
// E^{-1} (Gauss-Jordan, partial pivoting, one CTA) of E(a,b) = G[(k+b)*2k + a], the W^T C block of
// the Gram matrix of [W | C] (G 2k x 2k column-major), into st->Einv; fail[0] = 1 if a pivot is
// <= 1e-13 max|E_ab|.
cudaError_t launch_einv(const double* G, int k, DevState* st, int* fail, cudaStream_t strm);
// G = Y^T Y (s x s, column-major) for Y (n x s, leading dimension ld).
cudaError_t launch_gram(const double* Y, int64_t ld, int64_t n, int s, double* G, double* partial,
                        unsigned* counter, DevState* st, cudaStream_t strm);
// Symmetric eigen-decomposition of G (s x s) by parallel cyclic Jacobi in one CTA:
// lam (s, non-increasing), V (s x s column-major eigenvectors).  sigma_out (nullable) = sqrt(max(lam,0)).
// V0 (nullable, s0 x s0): warm-start eigenvectors (e.g. the previous build's), s0 <= s.
// rel != 0: relative (one-sided-Jacobi) stopping / rotation criterion |a_pq| <= 1e-15 sqrt(a_pp a_qq):
// high relative accuracy of small eigenvalues of a scaled diagonally dominant G (the SVD's pass 2).
cudaError_t launch_jacobi(const double* G, int s, double* lam, double* V, double* sigma_out,
                          DevState* st, cudaStream_t strm, const double* V0 = nullptr, int s0 = 0, int rel = 0);
// Y[:, c] = colscale[c] * sum_a X[:, a] M[a, c]  (M s x q column-major, leading dim ldm; colscale nullable).
cudaError_t launch_xm(const double* X, int64_t ldx, int64_t n, int s, const double* M, int ldm, int q,
                      const double* colscale, double* Y, int64_t ldy, DevState* st, cudaStream_t strm);
// 1 / sigma for c < q
cudaError_t launch_inv(const double* sigma, int q, double* out, cudaStream_t strm);
// Cholesky G = R^T R (k x k) and R^{-1}; fail[0] = 1 if not positive definite.
cudaError_t launch_chol(const double* G, int k, double* R, double* Rinv, int* fail, cudaStream_t strm);
// R_C = R2 R1, R_C^{-1} = R1^{-1} R2^{-1} into the state; fail if min|diag| <= 1e-12 max|diag|.
cudaError_t launch_rc_finish(const double* R1, const double* R1i, const double* R2, const double* R2i,
                             int k, DevState* st, int* fail, cudaStream_t strm);
// SELL packing of a CSR matrix (values, and columns when pattern != 0)
cudaError_t launch_sell_pack(const int32_t* rp, const int32_t* ci, const double* v, int64_t n,
                             const int64_t* sp, const int32_t* sw, int32_t* sci, double* sv,
                             int pattern, cudaStream_t strm, const int32_t* perm = nullptr);
cudaError_t launch_sell_widths(const int32_t* rp, int64_t n, int32_t* sw, cudaStream_t strm, const int32_t* perm = nullptr);
// CSR / BSR pattern validation on the device; bad[0] != 0 on failure.
cudaError_t launch_validate(const int32_t* rp, const int32_t* ci, int64_t nrows, int64_t ncols,
                            int64_t nnz, int* bad, cudaStream_t strm);

}  // namespace rg

// rg.cu — host engine and C-ABI entry points of librg (include/rg.h).
//
// The host validates arguments, owns the device buffers, and orchestrates the kernels; every
// arithmetic step of the method runs on the device.  A restart cycle (m Arnoldi steps, the
// cycle-end update and the next cycle start) is captured once as a CUDA graph and replayed;
// the host reads one 4-byte-class header per cycle to learn whether the solve has finished.
#define RG_FILE_ID 6  // RG_CHK locations (checked builds)
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a profiler is attached

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "knobs.cuh"

using namespace rg;

namespace rg {
void note_host_launches(int n);
}

namespace {

thread_local std::string g_err;
std::atomic<long long> g_host_launches{0};

rg_status fail(rg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      return fail(RG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
    }                                                                                  \
  } while (0)

constexpr int HIST_CAP = 1 << 16;
constexpr int SMALL = MAXS * MAXS;  // doubles per small-matrix slot

// What a captured solve graph bakes in: the variant's kernel sequence, the preconditioner, and the
// orthogonalisation (DCGS2 or classical CGS2 — chosen per solve from the byte model, so it can change
// between solves of one context as k_eff grows).  m, k_eff, tol are read from the state.
struct GraphKey {
  int variant, dcgs, prec;
  bool operator<(const GraphKey& o) const {
    if (variant != o.variant) return variant < o.variant;
    if (dcgs != o.dcgs) return dcgs < o.dcgs;
    return prec < o.prec;
  }
};

// Measured crossover (same box, alternating runs, tools/crossover.py; round 2, after the
// graph path's TMA DCGS2 passes, split epilogue and PDL): C3-type 9-point SELL sequences, deflate —
// 409,600 rows persistent/graph 2.59/3.12 ms, 589,824 rows 4.09/4.43, 802,816 rows 6.52/6.30,
// 1,048,576 rows (C3) 8.37/7.92; augment at 589,824 3.95/4.26 and at 1,048,576 8.47/8.08; C2 (262,144)
// 2.25/3.39.  (Round 1: the persistent solve won up to ~1.6M rows.)
constexpr int64_t PERSIST_MAX_ROWS = 700000;

}  // namespace

void rg::note_host_launches(int n) { g_host_launches += n; }

namespace {
// NVTX range per C-ABI call (SURVEY §5 tracing): nsys / ncu --nvtx show rg_solve, rg_build_recycle, ...
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct rg_ctx {
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;     // DCGS2 split epilogue: k_dcgs_ls runs here, concurrently with DK2
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t cap = nullptr;  // non-blocking stream the solve graphs are CAPTURED on (see run_solve)
  int flags = 0;
  int64_t n = 0, npad = 0;
  int max_m = 0, max_s = 0, max_k = 0;
  int ncol = 0;
  // matrix
  int fmt = 0;          // 0 CSR, 1 SELL, 2 BSR
  int block = 1;
  int64_t nnz = 0;      // CSR entries / BSR blocks
  int32_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* v = nullptr;
  int64_t v_len = 0;
  int64_t nslices = 0, sell_len = 0;
  int32_t sell_sigma = 1;
  int32_t* sperm = nullptr;   // SELL-32-sigma: SELL position -> row, and its inverse (sigma > 1 only)
  int32_t* siperm = nullptr;
  int64_t* sp = nullptr;
  int32_t* sw = nullptr;
  int32_t* sci = nullptr;
  double* sv = nullptr;
  MatDev A;
  // vectors and bases
  double* Z = nullptr;
  double* x = nullptr;
  double* b = nullptr;
  double* X = nullptr;   // snapshot ring, npad x max_s
  double* Y = nullptr;   // scratch, npad x max_s
  double* t1 = nullptr;  // scratch vectors
  double* t2 = nullptr;
  double* hist = nullptr;
  double* partial = nullptr;
  unsigned* counter = nullptr;
  double* small = nullptr;
  int* dflag = nullptr;
  double* tot_g = nullptr;   // persistent solve: reduced totals
  unsigned* gbar = nullptr;  // persistent solve: grid-barrier words
  unsigned* pflags = nullptr;  // persistent solve: neighbour-sync epochs (NSM * 8)
  unsigned long long* llw = nullptr;  // persistent solve: flag-carrying reduction words (ll_words())
  DevState* st = nullptr;
  DevState* hst = nullptr;  // pinned host mirror
  double* hhist = nullptr;  // pinned history staging
  int* hflag = nullptr;     // pinned flag staging
  double* hsig = nullptr;   // pinned singular-value staging (MAXS)
  Layout L;
  // snapshots / recycle space
  int s_count = 0, s_head = 0;
  int k_eff = 0;
  bool have_W = false;
  int v1prev_s = 0;         // size of the stored first-pass eigenvectors (Jacobi warm start), 0 = none
  bool c_valid = false;
  bool res_fused = false;  // this solve's C = A W SpMM also computes A x0 into V column 0 (SM_RES_Y start)
  int c_kind = 0;           // what c_valid refers to: 0 Q / R_C (augment, deflate), 1 C / E^{-1} (oblique)
  bool use_dcgs = true;
  bool dcgs_now = true;     // this solve uses DCGS2 (the oblique variant runs classical CGS2)
  int cur_var = 0;          // variant of the kernel sequence being issued
  // right preconditioner (precond.cu): kind 0 none, 1 SSOR(omega) in a multicolour order
  int prec_kind = 0;
  PrecDev P;
  std::vector<void*> prec_bufs;  // device arrays owned by P
  double* pz = nullptr;
  double* pt = nullptr;
  bool use_persist = true;  // one cooperative kernel per solve where supported (persistent.cu)
  double* keepV = nullptr;  // RG_FLAG_KEEP_BASIS: last finished cycle's V (n_pad x (max_m + 1))
  unsigned long long* trace = nullptr;  // RG_FLAG_PROFILE: device kernel timeline (2 words per event)
  int kb_var = 0, kb_k = 0; // variant / k_eff of the solve whose basis keepV holds
  // graphs
  std::map<GraphKey, cudaGraphExec_t> graphs;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // asynchronous recycle build (rg_build_recycle with k_eff = sigma = NULL): finished by the next
  // call that needs W (finish_build)
  cudaEvent_t ebuild = nullptr;
  bool pend = false;
  int pend_k = 0, pend_modes = 0, pend_s = 0;
};

namespace {

size_t header_bytes() { return offsetof(DevState, cs); }

void clear_graphs(rg_ctx* c) {
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();
}

void drop_preconditioner(rg_ctx* c) {
  for (void* p : c->prec_bufs) cudaFree(p);
  c->prec_bufs.clear();
  c->prec_kind = 0;
  c->P = PrecDev();
  c->L.prec = 0;
}

void free_matrix(rg_ctx* c) {
  cudaFree(c->rp); cudaFree(c->ci); cudaFree(c->v);
  cudaFree(c->sp); cudaFree(c->sw); cudaFree(c->sci); cudaFree(c->sv); cudaFree(c->sperm); cudaFree(c->siperm);
  c->rp = c->ci = nullptr; c->v = nullptr; c->sp = nullptr; c->sw = c->sci = nullptr; c->sv = nullptr;
  c->sperm = c->siperm = nullptr;
}

bool is_dev_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

rg_status copy_in(void* dst, const void* src, size_t bytes, rg_mem mem, cudaStream_t s) {
  if (bytes == 0) return RG_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  return RG_OK;
}

rg_status validate_host_pattern(const int32_t* rp, const int32_t* ci, int64_t nrows, int64_t ncols, int64_t nnz) {
  if (rp[0] != 0) return fail(RG_E_INVAL, "row_ptr[0] != 0");
  if (rp[nrows] != nnz) return fail(RG_E_INVAL, "row_ptr[n] != nnz");
  for (int64_t r = 0; r < nrows; ++r) {
    if (rp[r + 1] < rp[r]) return fail(RG_E_INVAL, "row_ptr not monotone at row " + std::to_string(r));
    int64_t prev = -1;
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
      if (ci[p] < 0 || ci[p] >= ncols) return fail(RG_E_INVAL, "column index out of range in row " + std::to_string(r));
      if (ci[p] <= prev) return fail(RG_E_INVAL, "columns not strictly increasing in row " + std::to_string(r));
      prev = ci[p];
    }
  }
  return RG_OK;
}

// Validate the rg_matrix descriptor against the context dimension (no data access).
rg_status check_desc(const rg_matrix* A, int64_t n, bool pattern_required) {
  if (!A) return fail(RG_E_INVAL, "matrix descriptor is NULL");
  if (A->fmt != RG_CSR && A->fmt != RG_BSR) return fail(RG_E_INVAL, "unknown matrix format");
  if (A->mem != RG_HOST && A->mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  if (A->n_rows != n) return fail(RG_E_INVAL, "n_rows does not match n");
  if (A->nnz < 0 || A->nnz >= (int64_t)INT32_MAX) return fail(RG_E_INVAL, "nnz out of range");
  if (A->fmt == RG_CSR && A->block != 1) return fail(RG_E_INVAL, "CSR requires block = 1");
  if (A->fmt == RG_BSR) {
    if (A->block < 1 || A->block > 64 || n % A->block) return fail(RG_E_INVAL, "BSR block must divide n and be <= 64");
    if (A->sell_C) return fail(RG_E_INVAL, "SELL packing applies to CSR only");
  }
  if (A->sell_C != 0 && A->sell_C != 32) return fail(RG_E_INVAL, "sell_C must be 0 or 32");
  if (A->sell_C == 32 && A->sell_sigma > 1 && A->sell_sigma % 32) return fail(RG_E_INVAL, "sell_sigma must be 1 or a multiple of 32");
  if (A->sell_sigma < 0) return fail(RG_E_INVAL, "sell_sigma must be >= 0");
  const bool has_rp = A->row_ptr != nullptr, has_ci = A->col_idx != nullptr;
  if (has_rp != has_ci) return fail(RG_E_INVAL, "row_ptr and col_idx must both be given or both be NULL");
  if (pattern_required && !has_rp) return fail(RG_E_INVAL, "row_ptr/col_idx required");
  if (A->nnz > 0 && !A->val) return fail(RG_E_INVAL, "val is NULL");
  return RG_OK;
}

rg_status set_matrix(rg_ctx* c, const rg_matrix* A, bool first) {
  const bool pattern = A->row_ptr != nullptr;
  const int newfmt = A->fmt == RG_BSR ? 2 : (A->sell_C == 32 ? 1 : 0);
  if (!first && !pattern) {
    if (A->nnz != c->nnz) return fail(RG_E_INVAL, "values-only update with a different nnz");
    if (newfmt != c->fmt || A->block != c->block) return fail(RG_E_INVAL, "values-only update must keep the format");
  }
  const int b = A->fmt == RG_BSR ? A->block : 1;
  const int64_t nrows = c->n / b;
  const int64_t vlen = A->nnz * (int64_t)b * b;
  if (pattern) {
    // validate the pattern before touching any state
    if (A->mem == RG_HOST) {
      rg_status s = validate_host_pattern(A->row_ptr, A->col_idx, nrows, nrows, A->nnz);
      if (s != RG_OK) return s;
    } else {
      if (!is_dev_ptr(A->row_ptr) || !is_dev_ptr(A->col_idx)) return fail(RG_E_INVAL, "mem = RG_DEVICE but pointers are not device memory");
      CK(cudaMemsetAsync(c->dflag, 0, sizeof(int), c->stream));
      CK(launch_validate(A->row_ptr, A->col_idx, nrows, nrows, A->nnz, c->dflag, c->stream));
      int bad = 0;
      CK(cudaMemcpyAsync(&bad, c->dflag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (bad) return fail(RG_E_INVAL, "invalid sparsity pattern (device check code " + std::to_string(bad) + ")");
    }
    const bool realloc = first || A->nnz != c->nnz || newfmt != c->fmt || b != c->block;
    if (c->prec_kind) {  // the colouring / diagonal positions belong to the old pattern
      clear_graphs(c);
      drop_preconditioner(c);
    }
    if (realloc) {
      clear_graphs(c);
      free_matrix(c);
      if (cudaMalloc(&c->rp, sizeof(int32_t) * (nrows + 1)) != cudaSuccess ||
          cudaMalloc(&c->ci, sizeof(int32_t) * std::max<int64_t>(A->nnz, 1)) != cudaSuccess ||
          cudaMalloc(&c->v, sizeof(double) * std::max<int64_t>(vlen, 1)) != cudaSuccess) {
        cudaGetLastError();
        free_matrix(c);
        return fail(RG_E_NOMEM, "device allocation of the matrix failed");
      }
    }
    c->nnz = A->nnz;
    c->fmt = newfmt;
    c->block = b;
    c->v_len = vlen;
    rg_status s;
    if ((s = copy_in(c->rp, A->row_ptr, sizeof(int32_t) * (nrows + 1), A->mem, c->stream)) != RG_OK) return s;
    if ((s = copy_in(c->ci, A->col_idx, sizeof(int32_t) * A->nnz, A->mem, c->stream)) != RG_OK) return s;
    if ((s = copy_in(c->v, A->val, sizeof(double) * vlen, A->mem, c->stream)) != RG_OK) return s;
    if (newfmt == 1) {  // SELL-32-sigma packing
      c->nslices = (c->n + 31) / 32;
      cudaFree(c->sp); cudaFree(c->sw); cudaFree(c->sci); cudaFree(c->sv); cudaFree(c->sperm); cudaFree(c->siperm);
      c->sp = nullptr; c->sw = nullptr; c->sci = nullptr; c->sv = nullptr; c->sperm = c->siperm = nullptr;
      c->sell_sigma = A->sell_sigma > 1 ? A->sell_sigma : 1;
      if (c->sell_sigma > 1) {
        // rows ordered by decreasing length inside each window of sigma rows (stable: equal lengths keep
        // their order), from the validated row pointers (one host pass per pattern change)
        std::vector<int32_t> rph(c->n + 1), perm(c->n), iperm(c->n);
        CK(cudaMemcpyAsync(rph.data(), c->rp, sizeof(int32_t) * (c->n + 1), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < c->n; ++i) perm[i] = (int32_t)i;
        for (int64_t w0 = 0; w0 < c->n; w0 += c->sell_sigma) {
          const int64_t w1 = std::min<int64_t>(c->n, w0 + c->sell_sigma);
          std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                           [&](int32_t a, int32_t b2) { return rph[a + 1] - rph[a] > rph[b2 + 1] - rph[b2]; });
        }
        for (int64_t i = 0; i < c->n; ++i) iperm[perm[i]] = (int32_t)i;
        CK(cudaMalloc(&c->sperm, sizeof(int32_t) * std::max<int64_t>(c->n, 1)));
        CK(cudaMalloc(&c->siperm, sizeof(int32_t) * std::max<int64_t>(c->n, 1)));
        CK(cudaMemcpyAsync(c->sperm, perm.data(), sizeof(int32_t) * c->n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->siperm, iperm.data(), sizeof(int32_t) * c->n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // (the host vectors go out of scope)
      }
      CK(cudaMalloc(&c->sw, sizeof(int32_t) * c->nslices));
      CK(cudaMalloc(&c->sp, sizeof(int64_t) * (c->nslices + 1)));
      CK(launch_sell_widths(c->rp, c->n, c->sw, c->stream, c->sperm));
      std::vector<int32_t> w(c->nslices);
      std::vector<int64_t> sp(c->nslices + 1);
      CK(cudaMemcpyAsync(w.data(), c->sw, sizeof(int32_t) * c->nslices, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      sp[0] = 0;
      for (int64_t i = 0; i < c->nslices; ++i) sp[i + 1] = sp[i] + 32 * (int64_t)w[i];
      c->sell_len = sp[c->nslices];
      CK(cudaMemcpyAsync(c->sp, sp.data(), sizeof(int64_t) * (c->nslices + 1), cudaMemcpyHostToDevice, c->stream));
      CK(cudaMalloc(&c->sci, sizeof(int32_t) * std::max<int64_t>(c->sell_len, 1)));
      CK(cudaMalloc(&c->sv, sizeof(double) * std::max<int64_t>(c->sell_len, 1)));
      CK(launch_sell_pack(c->rp, c->ci, c->v, c->n, c->sp, c->sw, c->sci, c->sv, 1, c->stream, c->sperm));
      CK(cudaStreamSynchronize(c->stream));
      clear_graphs(c);
    }
  } else {
    rg_status s;
    if (A->val != c->v) {  // val == rg_matrix_values(): updated in place, nothing to copy
      if (A->mem == RG_DEVICE && !is_dev_ptr(A->val)) return fail(RG_E_INVAL, "mem = RG_DEVICE but val is not device memory");
      if ((s = copy_in(c->v, A->val, sizeof(double) * vlen, A->mem, c->stream)) != RG_OK) return s;
    }
    if (c->fmt == 1) CK(launch_sell_pack(c->rp, c->ci, c->v, c->n, c->sp, c->sw, c->sci, c->sv, 0, c->stream, c->sperm));
    if (c->prec_kind) CK(launch_ssor_values(c->P, c->v, c->n, c->stream));  // SSOR copies follow the values
  }
  // device descriptor and byte model
  MatDev& M = c->A;
  M = MatDev();
  M.fmt = c->fmt;
  M.n = c->n;
  M.rp = c->rp; M.ci = c->ci; M.v = c->v;
  if (c->fmt == 0) {
    const double avg = c->n > 0 ? (double)c->nnz / (double)c->n : 0.0;
    M.lpr = avg <= 12.0 ? 1 : avg <= 24.0 ? 8 : avg <= 48.0 ? 16 : 32;
    M.bytes = 12.0 * c->nnz + 4.0 * (c->n + 1) + 16.0 * c->n;
    M.nnz = c->nnz;
  } else if (c->fmt == 1) {
    M.sp = c->sp; M.sw = c->sw; M.sci = c->sci; M.sv = c->sv; M.nslices = c->nslices;
    M.sperm = c->sperm; M.siperm = c->siperm;
    M.bytes = 12.0 * c->sell_len + 12.0 * c->nslices + 16.0 * c->n;
  } else {
    M.b = c->block;
    M.nb = c->n / c->block;
    M.tma = knob("RG_NO_BSR_TMA") ? 0 : 1;
    M.nnz = c->nnz;  // stored blocks
    M.bytes = 8.0 * c->v_len + 4.0 * c->nnz + 4.0 * (M.nb + 1) + 16.0 * c->n;
  }
  c->c_valid = false;
  return RG_OK;
}

// C = A W into the Q region, then CholQR2 -> Q (orthonormal), R_C, R_C^{-1} (state).
rg_status build_c(rg_ctx* c, bool sync) {
  const int k = c->k_eff;
  const int QB = c->L.VB - k;
  const int64_t ld = c->npad;
  cudaStream_t s = c->stream;
  cudaError_t es = knob("RG_NO_SPMM") ? cudaErrorNotSupported
                                        : launch_spmm(c->A, c->Z, c->Z + (int64_t)QB * ld, ld, k, c->st, c->counter, s,
                                                      c->res_fused ? c->x : nullptr, c->Z + (int64_t)c->L.VB * ld);
  if (es == cudaErrorNotSupported) {
    cudaGetLastError();
    c->res_fused = false;
    for (int l = 0; l < k; ++l)
      CK(launch_spmv(c->A, c->L, c->st, SM_PLAIN, c->Z + (int64_t)l * ld, c->Z + (int64_t)(QB + l) * ld, 0, s));
  } else {
    CK(es);
  }
  if (!sync) {
    // CholQR2 of the C just formed as ONE cooperative kernel (k_cbuild with C given: Gram, Cholesky and
    // the two in-place triangular solves for all rows, Cholesky factors redundant per CTA) instead of
    // the 8-launch chain below; k <= 22 (C5: k = 20)
    const cudaError_t eb = launch_cbuild(c->L, c->A, c->st, c->tot_g, c->gbar, c->llw, k, &c->st->cfail, s, true);
    if (eb == cudaSuccess) {
      if (knob("RG_NO_LLRED")) CK(cudaMemsetAsync(c->gbar, 0, sizeof(unsigned) * BAR_WORDS, s));
      c->c_valid = true;
      return RG_OK;
    }
    if (eb != cudaErrorNotSupported && eb != cudaErrorCooperativeLaunchTooLarge) CK(eb);
    cudaGetLastError();
  }
  double* G = c->small;
  double* R1 = c->small + 1 * SMALL;
  double* R1i = c->small + 2 * SMALL;
  double* R2 = c->small + 3 * SMALL;
  double* R2i = c->small + 4 * SMALL;
  double* Q = c->Z + (int64_t)QB * ld;
  int* flag = sync ? c->dflag : &c->st->cfail;  // solve: the header field (zeroed with the header)
  if (sync) CK(cudaMemsetAsync(c->dflag, 0, sizeof(int), s));
  CK(launch_gram(Q, ld, c->n, k, G, c->partial, c->counter, c->st, s));
  CK(launch_chol(G, k, R1, R1i, flag, s));
  CK(launch_xm(Q, ld, c->n, k, R1i, k, k, nullptr, c->Y, ld, c->st, s));
  CK(launch_gram(c->Y, ld, c->n, k, G, c->partial, c->counter, c->st, s));
  CK(launch_chol(G, k, R2, R2i, flag, s));
  CK(launch_xm(c->Y, ld, c->n, k, R2i, k, k, nullptr, Q, ld, c->st, s));
  CK(launch_rc_finish(R1, R1i, R2, R2i, k, c->st, flag, s));
  if (!sync) {  // the caller reads dflag together with the solve header (one sync per solve)
    c->c_valid = true;
    return RG_OK;
  }
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (knob("RG_DEBUG")) {
    std::vector<double> hb(5 * SMALL);
    cudaMemcpy(hb.data(), c->small, sizeof(double) * 5 * SMALL, cudaMemcpyDeviceToHost);
    for (int slot = 0; slot < 5; ++slot) {
      fprintf(stderr, "slot %d:", slot);
      for (int i = 0; i < k * k; ++i) fprintf(stderr, " %.4g", hb[slot * SMALL + i]);
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "bad=%d k=%d QB=%d\n", bad, k, QB);
  }
  if (bad) {
    c->have_W = false;
    c->k_eff = 0;
    c->c_valid = false;
    return fail(RG_E_SINGULAR, "A W is numerically rank deficient (R_C singular); recycle space cleared");
  }
  c->c_valid = true;
  return RG_OK;
}

// Oblique variant: C = A W into columns [k, 2k) (adjacent to W), E = W^T C from the Gram matrix of
// [W | C], E^{-1} by Gauss-Jordan into the state (E_s = V_s^T A V_s).
rg_status build_c_oblique(rg_ctx* c) {
  const int k = c->k_eff;
  if (2 * k > 64) return fail(RG_E_INVAL, "the oblique variant supports k_eff <= 32");
  const int64_t ld = c->npad;
  cudaStream_t s = c->stream;
  double* C = c->Z + (int64_t)k * ld;
  cudaError_t es = knob("RG_NO_SPMM") ? cudaErrorNotSupported
                                        : launch_spmm(c->A, c->Z, C, ld, k, c->st, c->counter, s,
                                                      c->res_fused ? c->x : nullptr, c->Z + (int64_t)c->L.VB * ld);
  if (es == cudaErrorNotSupported) {
    cudaGetLastError();
    c->res_fused = false;
    for (int l = 0; l < k; ++l)
      CK(launch_spmv(c->A, c->L, c->st, SM_PLAIN, c->Z + (int64_t)l * ld, C + (int64_t)l * ld, 0, s));
  } else {
    CK(es);
  }
  double* G = c->small;
  CK(launch_gram(c->Z, ld, c->n, 2 * k, G, c->partial, c->counter, c->st, s));
  CK(launch_einv(G, k, c->st, &c->st->cfail, s));  // header field, zeroed with the solve's header
  c->c_valid = true;
  c->c_kind = 1;
  return RG_OK;
}

// ---- the kernel sequences of one solve
// from_y: A x is already in V column 0 (fused into the C = A W SpMM), only r = b - A x remains
cudaError_t cycle_start(rg_ctx* c, int variant, bool from_y = false) {
  cudaError_t e = launch_spmv(c->A, c->L, c->st, from_y ? SM_RES_Y : SM_RES, nullptr, nullptr,
                              variant == RG_PLAIN ? 1 : 0, c->stream);
  if (e != cudaSuccess || variant == RG_PLAIN) return e;
  if (galerkin_variant(variant)) {  // Galerkin start x += W t, r -= C t, t = E^{-1} W^T r
    if ((e = launch_orth(c->L, c->st, OP_OB_CSD, c->stream)) != cudaSuccess) return e;
    if ((e = launch_orth(c->L, c->st, OP_XW, c->stream)) != cudaSuccess) return e;
    return launch_orth(c->L, c->st, OP_OB_CSU, c->stream);
  }
  if ((e = launch_orth(c->L, c->st, OP_CS_DQ, c->stream)) != cudaSuccess) return e;
  if ((e = launch_orth(c->L, c->st, OP_XW, c->stream)) != cudaSuccess) return e;
  return launch_orth(c->L, c->st, OP_CS_UN, c->stream);
}

// x += V y (+ W part); with a right preconditioner x += M^{-1} (V y) (+ W part)
cudaError_t cycle_end(rg_ctx* c) {
  cudaError_t e;
  if (c->L.prec) {
    if ((e = launch_orth(c->L, c->st, OP_VY, c->stream)) != cudaSuccess) return e;
    if ((e = launch_ssor(c->P, c->L, c->st, c->pt, c->pz, 2, c->stream)) != cudaSuccess) return e;
  }
  if (c->keepV && (e = launch_keep_basis(c->L, c->st, c->stream)) != cudaSuccess) return e;
  return launch_orth(c->L, c->st, OP_XUPD, c->stream);
}

// chained: not the first step of the captured body.  (Measured: launching the SpMV of a chained step with
// PDL behind the previous update pass removes most of the edge's gap but slows C4 by 1.5 %, C3 gains
// 0.4 %; A/B in profiles/r02/ab_unroll.txt.  Kept as a plain edge.)
cudaError_t arnoldi_step(rg_ctx* c, unsigned long long cond, bool chained) {
  cudaError_t e;
  (void)chained;
  if (c->L.prec) {  // y = A M^{-1} u
    if ((e = launch_ssor(c->P, c->L, c->st, nullptr, c->pz, 1, c->stream)) != cudaSuccess) return e;
    if ((e = launch_spmv(c->A, c->L, c->st, SM_STEP_PC, nullptr, nullptr, 0, c->stream)) != cudaSuccess) return e;
  } else if ((e = launch_spmv(c->A, c->L, c->st, SM_STEP, nullptr, nullptr, 0, c->stream)) != cudaSuccess) {
    return e;
  }
  if (galerkin_variant(c->cur_var) && !c->dcgs_now) {  // w = M_D A v_j = A v_j - C E^{-1} W^T A v_j (or (I-WW^T) A v_j)
    if ((e = launch_orth(c->L, c->st, OP_OB_SD, c->stream)) != cudaSuccess) return e;
    if ((e = launch_orth(c->L, c->st, OP_OB_SU, c->stream)) != cudaSuccess) return e;
  }
  if (c->dcgs_now) {  // delayed CGS2: one reduction + one update pass; the least-squares step of the
                      // finished column on a side branch, concurrent with the update pass (joined
                      // before the next step, which its WHILE condition gates)
    if ((e = launch_dcgs(c->L, c->st, 1, c->stream)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(c->ev_fork, c->stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(c->side, c->ev_fork, 0)) != cudaSuccess) return e;
    if ((e = launch_dcgs(c->L, c->st, 3, c->side, cond)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(c->ev_join, c->side)) != cudaSuccess) return e;
    if ((e = launch_dcgs(c->L, c->st, 2, c->stream)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(c->stream, c->ev_join, 0);
  }
  if ((e = launch_orth(c->L, c->st, OP_D1, c->stream)) != cudaSuccess) return e;
  if ((e = launch_orth(c->L, c->st, OP_UD2, c->stream)) != cudaSuccess) return e;
  return launch_orth(c->L, c->st, OP_UN, c->stream, cond);
}

#define CKG(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      cudaGraphDestroy(G);                                                             \
      return fail(RG_E_CUDA, std::string("graph build: ") + #call + ": " + cudaGetErrorString(e_)); \
    }                                                                                  \
  } while (0)

// The whole remainder of a solve as ONE graph with two nested WHILE nodes:
//   WHILE (!done) { set(inner = active); WHILE (active) { Arnoldi step }; x update; cycle start;
//                   set(outer = !done) }
// The Arnoldi-step condition is set by the least-squares epilogue itself, so no launch is wasted
// after convergence and the host never synchronises inside a solve.
rg_status build_solve_graph(rg_ctx* c, int variant, cudaGraphExec_t* out) {
  cudaGraph_t G = nullptr;
  CK(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle hout, hin;
  CKG(cudaGraphConditionalHandleCreate(&hout, G, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams op{};
  op.type = cudaGraphNodeTypeConditional;
  op.conditional.handle = hout;
  op.conditional.type = cudaGraphCondTypeWhile;
  op.conditional.size = 1;
  cudaGraphNode_t outer;
  CKG(cudaGraphAddNode(&outer, G, nullptr, 0, &op));
  cudaGraph_t bodyO = op.conditional.phGraph_out[0];
  CKG(cudaGraphConditionalHandleCreate(&hin, bodyO, 0, 0));
  cudaGraph_t tmp;
  CKG(cudaStreamBeginCaptureToGraph(c->stream, bodyO, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  cudaError_t e1 = launch_cond(c->st, hin, 0, c->stream);
  CKG(cudaStreamEndCapture(c->stream, &tmp));
  CKG(e1);
  cudaGraphNode_t pre;
  size_t nn = 1;
  CKG(cudaGraphGetNodes(bodyO, &pre, &nn));
  cudaGraphNodeParams ip{};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hin;
  ip.conditional.type = cudaGraphCondTypeWhile;
  ip.conditional.size = 1;
  cudaGraphNode_t inner;
  CKG(cudaGraphAddNode(&inner, bodyO, &pre, 1, &ip));
  cudaGraph_t bodyI = ip.conditional.phGraph_out[0];
  CKG(cudaStreamBeginCaptureToGraph(c->stream, bodyI, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  // U Arnoldi steps per WHILE iteration: an iteration boundary (body end -> condition -> next body launch)
  // measured ~7.3 us on the device timeline (tools/trace.py, C3 / C4) against ~3-4 us for a plain edge
  // inside the body; steps after the cycle stopped are no-op launches (every kernel gates on st->active;
  // a no-op DK1 also disables its step's update pass and least-squares kernel)
  static const int unroll_knob = knob_int("RG_UNROLL", 0);
  const int U = unroll_knob > 0 ? unroll_knob : (c->dcgs_now ? 4 : 2);
  e1 = cudaSuccess;
  for (int u = 0; u < U && e1 == cudaSuccess; ++u) e1 = arnoldi_step(c, (unsigned long long)hin, u > 0);
  CKG(cudaStreamEndCapture(c->stream, &tmp));
  CKG(e1);
  CKG(cudaStreamBeginCaptureToGraph(c->stream, bodyO, &inner, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  e1 = cycle_end(c);
  if (e1 == cudaSuccess) e1 = cycle_start(c, variant);
  if (e1 == cudaSuccess) e1 = launch_cond(c->st, hout, 1, c->stream);
  CKG(cudaStreamEndCapture(c->stream, &tmp));
  CKG(e1);
  cudaGraphExec_t ge;
  CKG(cudaGraphInstantiate(&ge, G, 0));
  cudaGraphDestroy(G);
  *out = ge;
  return RG_OK;
}

// Runs the rest of the solve after the first cycle start.
rg_status run_solve(rg_ctx* c, int variant, int m) {
  if (c->flags & RG_FLAG_NO_GRAPH) {
    // host-driven loop (debugging, profiler captures): one sync per Arnoldi step, so every launched
    // kernel does work (the graph's WHILE nodes decide the same on the device)
    for (;;) {
      CK(cudaMemcpyAsync(c->hst, c->st, offsetof(DevState, cs), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (c->hst->done) return RG_OK;
      if (c->hst->active) {
        CK(arnoldi_step(c, 0, false));
      } else {
        CK(cycle_end(c));
        CK(cycle_start(c, variant));
      }
    }
  }
  GraphKey key{variant, c->dcgs_now ? 1 : 0, c->L.prec};
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    // The graph is captured on a stream of its own: a library-created c->stream is a BLOCKING stream, and
    // while it captures, any work another host thread puts on the legacy default stream (another context's
    // caller, torch) would fail with "operation would make the legacy stream depend on a capturing blocking
    // stream" (tests/test_gpu_contexts.py).  Nodes do not keep the capture stream; the graph is launched on
    // c->stream.
    cudaGraphExec_t ge;
    cudaStream_t user = c->stream;
    c->stream = c->cap;
    rg_status s = build_solve_graph(c, variant, &ge);
    c->stream = user;
    if (s != RG_OK) return s;
    it = c->graphs.emplace(key, ge).first;
  }
  CK(cudaGraphLaunch(it->second, c->stream));
  return RG_OK;
}

template <class T>
rg_status dalloc(T** p, size_t count, const char* what) {
  if (cudaMalloc(p, sizeof(T) * std::max<size_t>(count, 1)) != cudaSuccess) {
    cudaGetLastError();
    return fail(RG_E_NOMEM, std::string("device allocation failed: ") + what);
  }
  return RG_OK;
}

}  // namespace

extern "C" {

RG_API const char* rg_last_error(void) { return g_err.c_str(); }

RG_API void rg_destroy(rg_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  clear_graphs(c);
  free_matrix(c);
  cudaFree(c->Z); cudaFree(c->x); cudaFree(c->b); cudaFree(c->X); cudaFree(c->Y);
  cudaFree(c->t1); cudaFree(c->t2); cudaFree(c->hist); cudaFree(c->partial); cudaFree(c->counter);
  cudaFree(c->small); cudaFree(c->dflag); cudaFree(c->st); cudaFree(c->tot_g); cudaFree(c->gbar); cudaFree(c->pflags); cudaFree(c->llw);
  drop_preconditioner(c);
  cudaFree(c->pz); cudaFree(c->pt); cudaFree(c->keepV); cudaFree(c->trace);
  if (c->hst) cudaFreeHost(c->hst);
  if (c->hhist) cudaFreeHost(c->hhist);
  if (c->hflag) cudaFreeHost(c->hflag);
  if (c->hsig) cudaFreeHost(c->hsig);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  if (c->ebuild) cudaEventDestroy(c->ebuild);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

RG_API rg_status rg_create(rg_ctx** out, int64_t n, const rg_matrix* A, const rg_options* opt) {
  if (!out) return fail(RG_E_INVAL, "ctx is NULL");
  *out = nullptr;
  if (n < 1 || n >= (int64_t)INT32_MAX) return fail(RG_E_INVAL, "n out of range");
  if (!opt) return fail(RG_E_INVAL, "options are NULL");
  if (opt->max_m < 1 || opt->max_m > MAXM) return fail(RG_E_INVAL, "max_m must be in 1..128");
  if (opt->max_snapshots < 1 || opt->max_snapshots > MAXS) return fail(RG_E_INVAL, "max_snapshots must be in 1..64");
  if (opt->max_k < 0 || opt->max_k > MAXK || opt->max_k > opt->max_snapshots)
    return fail(RG_E_INVAL, "max_k must be in 0..min(64, max_snapshots)");
  rg_status s = check_desc(A, n, true);
  if (s != RG_OK) return s;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(RG_E_CUDA, "no CUDA device available");
  }
  {  // the library is sm_100a code sized for the B200's 148 SMs (NSM): refuse anything else loudly
    int dev = 0, major = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return fail(RG_E_CUDA, "cannot query the current CUDA device");
    }
    if (major != 10 || sms < NSM)
      return fail(RG_E_CUDA, "librg is built for sm_100a with " + std::to_string(NSM) + " SMs (B200); the current device has "
                                 "compute capability " + std::to_string(major) + ".x and " + std::to_string(sms) + " SMs");
  }
  rg_ctx* c = new rg_ctx();
  CK(cudaGetDevice(&c->dev));
  c->flags = opt->flags;
  if (knob("RG_NO_GRAPH")) c->flags |= RG_FLAG_NO_GRAPH;  // ncu cannot profile kernels inside conditional graphs
  if (knob("RG_CGS2") || (opt->flags & RG_FLAG_CGS2)) c->use_dcgs = false;
  if (knob("RG_NO_PERSIST") || (opt->flags & RG_FLAG_NO_PERSIST)) c->use_persist = false;
  if (opt->cuda_stream) {
    c->stream = (cudaStream_t)opt->cuda_stream;
  } else {
    if (cudaStreamCreate(&c->stream) != cudaSuccess) { delete c; return fail(RG_E_CUDA, "stream creation failed"); }
    c->own_stream = true;
  }
  c->n = n;
  c->npad = (n + 63) / 64 * 64;
  c->max_m = opt->max_m;
  c->max_s = opt->max_snapshots;
  c->max_k = opt->max_k;
  const int VB = 2 * c->max_k;
  c->ncol = VB + c->max_m + 1;
  const size_t np = (size_t)c->npad;
  const size_t part = std::max<size_t>((size_t)NSM * 8 * MAXRED, (size_t)NSM * 2 * 64 * 64);  // Gram: 296 CTAs x 64^2
  if ((s = dalloc(&c->Z, np * c->ncol, "Z")) != RG_OK || (s = dalloc(&c->x, np, "x")) != RG_OK ||
      (s = dalloc(&c->b, np, "b")) != RG_OK || (s = dalloc(&c->X, np * c->max_s, "X")) != RG_OK ||
      (s = dalloc(&c->Y, np * c->max_s, "Y")) != RG_OK || (s = dalloc(&c->t1, np, "t1")) != RG_OK ||
      (s = dalloc(&c->t2, np, "t2")) != RG_OK || (s = dalloc(&c->hist, (size_t)HIST_CAP, "hist")) != RG_OK ||
      (s = dalloc(&c->partial, part, "partial")) != RG_OK || (s = dalloc(&c->counter, 4, "counter")) != RG_OK ||
      (s = dalloc(&c->small, (size_t)SMALL * 16, "small")) != RG_OK || (s = dalloc(&c->dflag, 4, "flag")) != RG_OK ||
      (s = dalloc(&c->tot_g, (size_t)MAXRED, "totals")) != RG_OK || (s = dalloc(&c->gbar, (size_t)BAR_WORDS, "barrier")) != RG_OK ||
      (s = dalloc(&c->pflags, (size_t)NSM * 16, "sync flags")) != RG_OK ||
      (s = dalloc(&c->llw, ll_words(), "reduction words")) != RG_OK ||
      (s = dalloc(&c->st, 1, "state")) != RG_OK ||
      ((c->flags & RG_FLAG_KEEP_BASIS) && (s = dalloc(&c->keepV, np * (c->max_m + 1), "kept basis")) != RG_OK) ||
      ((c->flags & RG_FLAG_PROFILE) && (s = dalloc(&c->trace, (size_t)2 * TRACE_CAP, "kernel trace")) != RG_OK)) {
    rg_destroy(c);
    return s;
  }
  if (cudaMallocHost(&c->hst, sizeof(DevState)) != cudaSuccess ||
      cudaMallocHost(&c->hhist, sizeof(double) * HIST_CAP) != cudaSuccess ||
      cudaMallocHost(&c->hflag, sizeof(int) * 4) != cudaSuccess ||
      cudaMallocHost(&c->hsig, sizeof(double) * (MAXS + 2)) != cudaSuccess) {
    cudaGetLastError();
    rg_destroy(c);
    return fail(RG_E_NOMEM, "pinned host allocation failed");
  }
  memset(c->hst, 0, sizeof(DevState));
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  ok(cudaMemsetAsync(c->Z, 0, sizeof(double) * np * c->ncol, c->stream));
  ok(cudaMemsetAsync(c->x, 0, sizeof(double) * np, c->stream));
  ok(cudaMemsetAsync(c->b, 0, sizeof(double) * np, c->stream));
  ok(cudaMemsetAsync(c->X, 0, sizeof(double) * np * c->max_s, c->stream));
  ok(cudaMemsetAsync(c->Y, 0, sizeof(double) * np * c->max_s, c->stream));
  ok(cudaMemsetAsync(c->t1, 0, sizeof(double) * np, c->stream));
  ok(cudaMemsetAsync(c->t2, 0, sizeof(double) * np, c->stream));
  ok(cudaMemsetAsync(c->counter, 0, sizeof(unsigned) * 4, c->stream));
  ok(cudaMemsetAsync(c->st, 0, sizeof(DevState), c->stream));
  if (c->trace) {  // outside the per-solve header: set once
    c->hst->trace = c->trace;
    c->hst->trace_cap = TRACE_CAP;
    ok(cudaMemcpyAsync(&c->st->trace, &c->hst->trace, sizeof(c->hst->trace) + 2 * sizeof(unsigned),
                       cudaMemcpyHostToDevice, c->stream));
  }
  ok(cudaMemsetAsync(c->llw, 0, sizeof(unsigned long long) * ll_words(), c->stream));
  // persistent-solve barrier words and neighbour epochs: zero at allocation and again right after
  // every persistent solve (off the next solve's critical path)
  ok(cudaMemsetAsync(c->gbar, 0, sizeof(unsigned) * BAR_WORDS, c->stream));
  ok(cudaMemsetAsync(c->pflags, 0, sizeof(unsigned) * NSM * 16, c->stream));
  for (int i = 0; i < MAXCOL; ++i) c->hst->sc[i] = i < VB ? 1.0 : 0.0;
  ok(cudaMemcpyAsync(&c->st->sc[0], &c->hst->sc[0], sizeof(double) * MAXCOL, cudaMemcpyHostToDevice, c->stream));
  ok(cudaEventCreate(&c->e0));
  ok(cudaEventCreate(&c->e1));
  ok(cudaEventCreateWithFlags(&c->ebuild, cudaEventDisableTiming));
  ok(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  ok(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  ok(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  ok(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
  ok(cudaStreamSynchronize(c->stream));
  if (e != cudaSuccess) {
    rg_destroy(c);
    return fail(RG_E_CUDA, std::string("initialisation: ") + cudaGetErrorString(e));
  }
  c->L.Z = c->Z;
  c->L.ld = c->npad;
  c->L.n = n;
  c->L.maxk = c->max_k;
  c->L.ncol = c->ncol;
  c->L.VB = VB;
  c->L.x = c->x;
  c->L.b = c->b;
  c->L.hist = c->hist;
  c->L.partial = c->partial;
  c->L.counter = c->counter;
  c->L.keepV = c->keepV;
  c->L.cgs_ok = (c->max_k + c->max_m + 1) <= 128 && !knob("RG_NO_CGS");
  c->L.keep_l2 = (double)c->npad * 8.0 * (2 * c->max_k + c->max_m + 1) <= 160e6;  // ~L2-sized (126 MB)

  if ((s = set_matrix(c, A, true)) != RG_OK) {
    std::string msg = g_err;
    rg_destroy(c);
    return fail(s, msg);
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    rg_destroy(c);
    return fail(RG_E_CUDA, "matrix upload failed");
  }
  *out = c;
  g_err.clear();
  return RG_OK;
}

RG_API rg_status rg_update_matrix(rg_ctx* c, const rg_matrix* A) {
  NvtxRange nvtx_("rg_update_matrix");
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  rg_status s = check_desc(A, c->n, false);
  if (s != RG_OK) return s;
  if ((A->fmt == RG_BSR) != (c->fmt == 2)) return fail(RG_E_INVAL, "matrix format differs from the context's");
  if ((s = set_matrix(c, A, false)) != RG_OK) return s;
  if (A->mem == RG_HOST) CK(cudaStreamSynchronize(c->stream));  // device inputs: stream-ordered
  return RG_OK;
}

RG_API rg_status rg_matrix_values(rg_ctx* c, double** values, int64_t* len) {
  if (!c || !values) return fail(RG_E_INVAL, "NULL argument");
  *values = c->v;
  if (len) *len = c->v_len;
  return RG_OK;
}

RG_API rg_status rg_push_snapshot(rg_ctx* c, const double* x, rg_mem mem) {
  NvtxRange nvtx_("rg_push_snapshot");
  if (!c || !x) return fail(RG_E_INVAL, "NULL argument");
  if (mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  rg_status s = copy_in(c->X + (int64_t)c->s_head * c->npad, x, sizeof(double) * c->n, mem, c->stream);
  if (s != RG_OK) return s;
  if (mem == RG_HOST) CK(cudaStreamSynchronize(c->stream));  // device inputs: stream-ordered
  c->s_head = (c->s_head + 1) % c->max_s;
  c->s_count = std::min(c->s_count + 1, c->max_s);
  return RG_OK;
}

RG_API rg_status rg_clear_snapshots(rg_ctx* c) {
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  if (c->pend) {  // drop a pending asynchronous build
    CK(cudaEventSynchronize(c->ebuild));
    c->pend = false;
  }
  c->s_count = c->s_head = 0;
  c->v1prev_s = 0;
  c->have_W = false;
  c->k_eff = 0;
  c->c_valid = false;
  return RG_OK;
}

// Second half of a recycle build, once sigma is on the host: rank, k_eff, W = Y V2 Sigma^{-1}.
#ifdef RG_CHECKED
// CHECKED builds: device check failures (RG_CHK) recorded since the last read, by the kernels of any call
static rg_status chk_report(unsigned count, unsigned where) {
  static const char* files[] = {"?", "dcgs.cu", "dense.cu", "orth.cu", "persistent.cu", "precond.cu", "rg.cu", "spmv.cu"};
  const unsigned f = where >> 16;
  char buf[192];
  snprintf(buf, sizeof buf, "device check failed at %s:%u (or a header it includes), %u failure(s)",
           f < 8 ? files[f] : "?", where & 0xffffu, count);
  return fail(RG_E_CHECK, buf);
}
static rg_status chk_pending(rg_ctx* c) {
  unsigned v[2] = {0u, 0u};
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return RG_OK;  // a CUDA error is reported by the call
  cudaMemcpy(v, &c->st->chk_count, sizeof v, cudaMemcpyDeviceToHost);
  if (!v[0]) return RG_OK;
  cudaMemset(&c->st->chk_count, 0, sizeof v);
  return chk_report(v[0], v[1]);
}
#endif

rg_status finish_build(rg_ctx* c, int k, int modes, int s, int32_t* k_eff, double* sigma) {
  const int64_t ld = c->npad;
  cudaStream_t st = c->stream;
  double* V2 = c->small + 3 * SMALL;
  double* sig = c->small + 4 * SMALL;
  double* inv = c->small + 5 * SMALL;
  double* hs = c->hsig;
  int rank = 0;
  for (int i = 0; i < s; ++i)
    if (hs[0] > 0.0 && hs[i] > 1e-12 * hs[0]) ++rank;
  const int ke = std::min(std::min(k, s), rank);
  if (sigma) memcpy(sigma, hs, sizeof(double) * s);
  if (k_eff) *k_eff = ke;
  c->k_eff = ke;
  c->have_W = ke > 0;
  c->c_valid = false;
  if (ke > 0) {
    // W = Y V2[:, off:off+k] Sigma^{-1}[off:off+k] into Z[:, 0:k]; off = 0 (largest) or rank-k (smallest)
    const int off = modes == RG_MODES_SMALLEST ? rank - ke : 0;
    CK(launch_inv(sig + off, ke, inv, st));
    CK(launch_xm(c->Y, ld, c->n, s, V2 + (int64_t)off * s, s, ke, inv, c->Z, ld, c->st, st));
    CK(cudaGetLastError());  // stream-ordered: the solve (or rg_export) consumes W on the same stream
  }
  return RG_OK;
}

// Complete a pending asynchronous build (no-op otherwise).
rg_status resolve_build(rg_ctx* c) {
  if (!c->pend) return RG_OK;
  c->pend = false;
  CK(cudaEventSynchronize(c->ebuild));
  return finish_build(c, c->pend_k, c->pend_modes, c->pend_s, nullptr, nullptr);
}

RG_API rg_status rg_build_recycle(rg_ctx* c, int32_t k, int32_t* k_eff, double* sigma) {
  return rg_build_recycle_modes(c, k, RG_MODES_LARGEST, k_eff, sigma);
}

RG_API rg_status rg_build_recycle_modes(rg_ctx* c, int32_t k, int32_t modes, int32_t* k_eff, double* sigma) {
  NvtxRange nvtx_("rg_build_recycle_modes");
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  if (modes != RG_MODES_LARGEST && modes != RG_MODES_SMALLEST) return fail(RG_E_INVAL, "unknown modes");
  if (k < 1 || k > c->max_k) return fail(RG_E_INVAL, "k must be in 1..max_k");
  if (c->s_count == 0) return fail(RG_E_STATE, "no snapshots");
  if (rg_status r0 = resolve_build(c)) return r0;  // a previous asynchronous build completes first
  const int s = c->s_count;
  const int64_t ld = c->npad;
  cudaStream_t st = c->stream;
  static const bool timing = knob("RG_TIMING");
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  double* G = c->small;
  double* V1 = c->small + 1 * SMALL;
  double* lam = c->small + 2 * SMALL;
  double* V2 = c->small + 3 * SMALL;
  double* sig = c->small + 4 * SMALL;
  // pass 1: G = X^T X, Jacobi -> V1 (warm-started from the previous build's V1) ; Y = X V1
  double* V1prev = c->small + 8 * SMALL;
  CK(launch_gram(c->X, ld, c->n, s, G, c->partial, c->counter, c->st, st));
  CK(launch_jacobi(G, s, lam, V1, nullptr, c->st, st, V1prev, c->v1prev_s <= s ? c->v1prev_s : 0));
  CK(cudaMemcpyAsync(V1prev, V1, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, st));
  c->v1prev_s = s;
  CK(launch_xm(c->X, ld, c->n, s, V1, s, s, nullptr, c->Y, ld, c->st, st));
  // pass 2: Y^T Y (nearly diagonal, column-scaled) -> V2, sigma
  CK(launch_gram(c->Y, ld, c->n, s, G, c->partial, c->counter, c->st, st));
  CK(launch_jacobi(G, s, lam, V2, sig, c->st, st, nullptr, 0, 1));
  const auto t1 = now();
  double* hs = c->hsig;  // pinned
  CK(cudaMemcpyAsync(hs, sig, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
  if (!k_eff && !sigma && !knob("RG_SYNC_BUILD")) {
    // asynchronous: nothing to return now; the next call that needs W waits for sigma (finish_build)
    CK(cudaEventRecord(c->ebuild, st));
    c->pend = true;
    c->pend_k = k;
    c->pend_modes = modes;
    c->pend_s = s;
    c->have_W = false;
    c->c_valid = false;
    return RG_OK;
  }
  CK(cudaStreamSynchronize(st));
  const auto t2 = now();
  if (knob("RG_DEBUG")) {
    double sw[2] = {0.0, 0.0};
    cudaMemcpy(sw, lam + s, 2 * sizeof(double), cudaMemcpyDeviceToHost);
    fprintf(stderr, "rg_build_recycle: s=%d, Jacobi sweeps %.0f (pass 1) %.0f (pass 2)\n", s, sw[0], sw[1]);
  }
  const rg_status rs = finish_build(c, k, modes, s, k_eff, sigma);
#ifdef RG_CHECKED
  if (rs == RG_OK)
    if (rg_status cs = chk_pending(c)) return cs;
#endif
  if (timing) {
    const auto t3 = now();
    auto us = [](auto a2, auto b2) { return std::chrono::duration<double, std::micro>(b2 - a2).count(); };
    fprintf(stderr, "rg_build_recycle host us: launch %.1f, wait %.1f, tail %.1f\n", us(t0, t1), us(t1, t2), us(t2, t3));
  }
  return rs;
}

RG_API rg_status rg_solve(rg_ctx* c, const double* b, const double* x0, int32_t m, rg_variant v, double tol,
                          int32_t max_iters, double* x_out, rg_mem mem, double* history, int32_t history_cap,
                          rg_report* rep) {
  NvtxRange nvtx_("rg_solve");
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  if (!b || !x_out) return fail(RG_E_INVAL, "b and x_out are required");
  if (m < 1 || m > c->max_m) return fail(RG_E_INVAL, "m must be in 1..max_m");
  if (!(tol > 0.0)) return fail(RG_E_INVAL, "tol must be > 0");
  if (max_iters < 1) return fail(RG_E_INVAL, "max_iters must be >= 1");
  if (v != RG_PLAIN && v != RG_AUGMENT && v != RG_DEFLATE && v != RG_OBLIQUE && v != RG_ORTHOGONAL)
    return fail(RG_E_INVAL, "unknown variant");
  if (mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  if (history_cap < 0) return fail(RG_E_INVAL, "history_cap < 0");
  cudaStream_t s = c->stream;
  rg_status rs;
  if ((rs = resolve_build(c)) != RG_OK) return rs;
  const int eff = (v != RG_PLAIN && c->have_W && c->k_eff > 0) ? (int)v : (int)RG_PLAIN;
  const int k = eff == RG_PLAIN ? 0 : c->k_eff;
  bool check_c = false;
  const int want_kind = galerkin_variant(eff) ? 1 : 0;
  // RG_TIMING: device-side phase split of one solve (events on the solve's stream)
  static const bool timing = knob("RG_TIMING");
  static cudaEvent_t tev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  if (timing && !tev[0])
    for (auto& e : tev) cudaEventCreate(&e);
  if (timing) cudaEventRecord(tev[0], s);
  const bool need_c = eff != RG_PLAIN && (!c->c_valid || c->c_kind != want_kind);
  // (a sorted SELL-32-sigma matrix permutes rows across the persistent kernel's CTA row ranges: graph path)
  const bool persist_size = (c->npad <= PERSIST_MAX_ROWS || knob("RG_FORCE_PERSIST")) && !(c->fmt == 1 && c->sperm);
  static const bool no_fuse = knob("RG_NO_FUSE_C");
  // (independent of the solve path: the graph path reads the same Q columns and R_C^{-1})
  bool fuse_c = need_c && !galerkin_variant(eff) && !no_fuse;
  // DCGS2 saves two reductions and one basis pass per Arnoldi step but spends one extra SpMV per
  // cycle (the step after the stopping column).  When one SpMV moves more bytes than a whole pass
  // over the basis (C5: 7.3 GB vs ~0.8 GB), classical CGS2 is cheaper (measured C5: see DESIGN.md).
  const double basis_pass = 8.0 * (double)c->n * (double)(k + m + 2);
  c->dcgs_now = c->use_dcgs && !(c->A.bytes > basis_pass && !knob("RG_FORCE_DCGS"));
#ifdef RG_CHECKED
  if (rg_status cs = chk_pending(c)) return cs;  // failures of earlier calls (the header upload clears them)
#endif
  DevState* h = c->hst;
  memset(h, 0, header_bytes());
  h->variant = eff;
  h->m = m;
  h->k_eff = k;
  h->max_iters = max_iters;
  h->hist_cap = std::min(HIST_CAP, std::max(history_cap, 0));
  h->profile = (c->flags & RG_FLAG_PROFILE) ? 1 : 0;
  h->tol = tol;
  h->jfinal = -1;
  h->dcgs = c->dcgs_now ? 1 : 0;
  CK(cudaMemcpyAsync(c->st, h, header_bytes(), cudaMemcpyHostToDevice, s));  // before the C build (cfail)
  // BSR-64 solves on the graph path (C5): the start residual's product A x0 rides along as one
  // extra column of the C = A W SpMM — one read of A (7.3 GB at C5) instead of two per system.
  static const bool no_fuse_res = knob("RG_NO_FUSE_RES");
  // (x0 == NULL: A x0 = 0 needs no product at all — the first cycle start forms r = b directly, below)
  c->res_fused = x0 && need_c && !no_fuse_res && c->A.fmt == 2 && c->A.b == 64 && c->A.tma && k + 1 <= 64 &&
                 !(c->use_persist && persist_size && c->dcgs_now && !(c->flags & RG_FLAG_NO_GRAPH));
  const bool early_in = c->res_fused;  // b and x0 in the library's buffers before the SpMM reads x0
  if (early_in) {
    if ((rs = copy_in(c->b, b, sizeof(double) * c->n, mem, s)) != RG_OK) return rs;
    if (x0) {
      if ((rs = copy_in(c->x, x0, sizeof(double) * c->n, mem, s)) != RG_OK) return rs;
    } else {
      CK(cudaMemsetAsync(c->x, 0, sizeof(double) * c->npad, s));
    }
  }
  if (need_c) {
    if (fuse_c) {  // one cooperative kernel (persistent.cu k_cbuild) instead of build_c's ~10 launches
      // (gbar is clean between solves; it uses it only without the flag-carrying reductions)
      const cudaError_t eb = launch_cbuild(c->L, c->A, c->st, c->tot_g, c->gbar, c->llw, k, &c->st->cfail, s);
      if (eb == cudaSuccess && knob("RG_NO_LLRED")) CK(cudaMemsetAsync(c->gbar, 0, sizeof(unsigned) * BAR_WORDS, s));
      if (eb == cudaSuccess) {
        c->c_valid = true;
      } else if (eb == cudaErrorNotSupported || eb == cudaErrorCooperativeLaunchTooLarge) {
        cudaGetLastError();
        fuse_c = false;
      } else {
        CK(eb);
      }
    }
    if (!fuse_c && (rs = (galerkin_variant(eff) ? build_c_oblique(c) : build_c(c, false))) != RG_OK) {
      c->res_fused = false;
      return rs;
    }
    c->c_kind = want_kind;

    check_c = true;
  }
  c->cur_var = eff;
  c->kb_var = eff;
  c->kb_k = k;
  c->L.prec = c->prec_kind ? 1 : 0;
  // Measured on B200: the single cooperative kernel wins while kernel-boundary
  // latency dominates (C1 -32%, C2 -16%, C3 -9% per system); at n = 2M rows (C4) its two-barrier
  // reductions cost more than the graph path's last-CTA epilogues (+11%), so it is used up to 1.6M.
  const bool try_persist = c->use_persist && persist_size && c->dcgs_now && !(c->flags & RG_FLAG_NO_GRAPH);
  // Persistent path with DEVICE buffers and n = n_pad (no padding rows): the kernel reads b and
  // iterates on x in the caller's buffers (no copy of b, none of x back); otherwise the library's.
  static const bool no_alias = knob("RG_NO_ALIAS");
  bool alias = try_persist && mem == RG_DEVICE && c->n == c->npad && !no_alias;
  if (alias) {
    if (x0 && x0 != x_out) CK(cudaMemcpyAsync(x_out, x0, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s));
    else if (!x0) CK(cudaMemsetAsync(x_out, 0, sizeof(double) * c->n, s));
  } else if (!early_in) {
    if ((rs = copy_in(c->b, b, sizeof(double) * c->n, mem, s)) != RG_OK) return rs;
    if (x0) {
      if ((rs = copy_in(c->x, x0, sizeof(double) * c->n, mem, s)) != RG_OK) return rs;
    } else {
      CK(cudaMemsetAsync(c->x, 0, sizeof(double) * c->npad, s));
    }
  }
  c->L.augment = eff == RG_AUGMENT;
  if (timing) cudaEventRecord(tev[1], s);
  CK(cudaEventRecord(c->e0, s));
  bool done_persist = false;
  if (try_persist) {  // (barrier words and neighbour epochs are zero: reset after every persistent solve)
    Layout Lp = c->L;
    if (alias) {
      Lp.b = b;
      Lp.x = x_out;
    }
    cudaError_t ep = launch_persistent(Lp, c->A, c->st, c->tot_g, c->gbar, c->pflags, c->llw, m, k, eff,
                                       c->L.prec ? &c->P : nullptr, s);
    if (ep == cudaSuccess) done_persist = true;
    else if (ep == cudaErrorNotSupported || ep == cudaErrorCooperativeLaunchTooLarge) cudaGetLastError();
    else CK(ep);
  }
  if (!done_persist && alias) {  // the graph path works on the library's buffers
    CK(cudaMemcpyAsync(c->b, b, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->x, x_out, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s));
    alias = false;
  }
  if (!done_persist) {
    CK(launch_orth(c->L, c->st, OP_NORMB, s));
    // start residual r = b - y with y = A x0 in V column 0: y from the fused SpMM, or y = 0 when
    // x0 = 0 (no SpMV of a zero vector: one read of A saved per solve, 7.3 GB at C5)
    bool from_y = c->res_fused;
    if (!x0 && !from_y) {
      CK(cudaMemsetAsync(c->Z + (int64_t)c->L.VB * c->npad, 0, sizeof(double) * c->npad, s));
      from_y = true;
    }
    c->res_fused = false;
    CK(cycle_start(c, eff, from_y));
    if ((rs = run_solve(c, eff, m)) != RG_OK) return rs;
  }
  CK(cudaEventRecord(c->e1, s));
  // one synchronisation per solve: header, C=AW singularity flag, x and the history together
  int bad = 0;
  if (timing) cudaEventRecord(tev[2], s);
  CK(cudaMemcpyAsync(h, c->st, header_bytes(), cudaMemcpyDeviceToHost, s));  // incl. the C-build flag
  if (!alias)
    CK(cudaMemcpyAsync(x_out, c->x, sizeof(double) * c->n, mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  const int hcap = std::min(history_cap, HIST_CAP);
  if (history && hcap > 0) CK(cudaMemcpyAsync(c->hhist, c->hist, sizeof(double) * hcap, cudaMemcpyDeviceToHost, s));
  if (timing) cudaEventRecord(tev[3], s);
  CK(cudaStreamSynchronize(s));
  if (timing) {
    float a = 0.f, b2 = 0.f, d = 0.f;
    cudaEventElapsedTime(&a, tev[0], tev[1]);
    cudaEventElapsedTime(&b2, tev[1], tev[2]);
    cudaEventElapsedTime(&d, tev[2], tev[3]);
    fprintf(stderr, "rg_solve device us: setup (C = A W, QR, copies) %.1f, solve %.1f, copy-out %.1f\n", a * 1e3,
            b2 * 1e3, d * 1e3);
  }
  if (check_c) bad = h->cfail;
  if (done_persist && knob("RG_SKEW")) {  // experiment: per-CTA step start / dots done / reduction done / SM
    std::vector<unsigned> ts((size_t)NSM * 8);
    cudaMemcpy(ts.data(), c->pflags + NSM * 2, sizeof(unsigned) * NSM * 8, cudaMemcpyDeviceToHost);
    unsigned mn = 0xffffffffu;
    for (int b2 = 0; b2 < NSM * 2; ++b2) mn = std::min(mn, ts[NSM * 2 + b2]);
    fprintf(stderr, "skewcsv cta,sm,start,dots,reduced\n");
    for (int b2 = 0; b2 < NSM * 2; ++b2)
      fprintf(stderr, "skewcsv %d,%u,%.3f,%.3f,%.3f\n", b2, ts[3 * NSM * 2 + b2], (int)(ts[NSM * 2 + b2] - mn) * 1e-3,
              (int)(ts[b2] - mn) * 1e-3, (int)(ts[2 * NSM * 2 + b2] - mn) * 1e-3);
  }
  if (done_persist) {  // clean barrier words / epochs for the next persistent launch (runs while the host returns)
    CK(cudaMemsetAsync(c->gbar, 0, sizeof(unsigned) * BAR_WORDS, s));
    CK(cudaMemsetAsync(c->pflags, 0, sizeof(unsigned) * NSM * 16, s));
  }
  if (bad) {
    c->have_W = false;
    c->k_eff = 0;
    c->c_valid = false;
    return fail(RG_E_SINGULAR, galerkin_variant(eff) ? "E = W^T A W is numerically singular; recycle space cleared"
                                                 : "A W is numerically rank deficient (R_C singular); recycle space cleared");
  }
  if (h->bzero) {
    if (mem == RG_DEVICE) {
      CK(cudaMemsetAsync(x_out, 0, sizeof(double) * c->n, s));
      CK(cudaStreamSynchronize(s));
    } else {
      memset(x_out, 0, sizeof(double) * c->n);
    }
  }
  const int hl = std::min(h->hist_len, history_cap);
  if (history && hl > 0) memcpy(history, c->hhist, sizeof(double) * hl);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->e0, c->e1);
  if (rep) {
    rep->iterations = h->iters;
    rep->restarts = h->cycles > 0 ? h->cycles - 1 : 0;
    rep->converged = h->converged;
    rep->k_eff = k;
    rep->spmv_count = h->spmv_count;  // counted on the device by every product the solve issued
    rep->history_len = hl;
    rep->rel_residual = h->bzero ? 0.0 : h->relres;
    rep->ms_total = ms;
  }
#ifdef RG_CHECKED
  if (h->chk_count) return chk_report(h->chk_count, h->chk_where);
#endif
  if (h->status == RG_E_NUMERIC) return fail(RG_E_NUMERIC, "NaN/Inf met during the solve");
  if (h->status == RG_E_CUDA) return fail(RG_E_CUDA, "persistent solve: grid barrier timed out");
  return RG_OK;
}

RG_API rg_status rg_apply(rg_ctx* c, const double* x, double* y, rg_mem mem) {
  NvtxRange nvtx_("rg_apply");
  if (!c || !x || !y) return fail(RG_E_INVAL, "NULL argument");
  if (mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  rg_status s = copy_in(c->t1, x, sizeof(double) * c->n, mem, c->stream);
  if (s != RG_OK) return s;
  CK(launch_spmv(c->A, c->L, nullptr, SM_PLAIN, c->t1, c->t2, 0, c->stream));
  CK(cudaMemcpyAsync(y, c->t2, sizeof(double) * c->n, mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return RG_OK;
}

RG_API rg_status rg_set_preconditioner(rg_ctx* c, int32_t kind, double omega, const int32_t* colors, rg_mem mem,
                                       int32_t* ncolors_out) {
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  if (kind == RG_PREC_NONE) {
    if (c->prec_kind) {
      CK(cudaStreamSynchronize(c->stream));
      clear_graphs(c);
      drop_preconditioner(c);
    }
    if (ncolors_out) *ncolors_out = 0;
    return RG_OK;
  }
  if (kind != RG_PREC_SSOR) return fail(RG_E_INVAL, "unknown preconditioner kind");
  if (!(omega > 0.0 && omega < 2.0)) return fail(RG_E_INVAL, "SSOR needs 0 < omega < 2");
  if (c->fmt == 2) return fail(RG_E_INVAL, "SSOR is implemented for CSR (and SELL-packed CSR) matrices only");
  if (colors && mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  const int64_t n = c->n;
  std::vector<int32_t> rp(n + 1), ci(std::max<int64_t>(c->nnz, 1));
  CK(cudaMemcpyAsync(rp.data(), c->rp, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(ci.data(), c->ci, sizeof(int32_t) * c->nnz, cudaMemcpyDeviceToHost, c->stream));
  std::vector<int32_t> col(n);
  if (colors) {
    CK(cudaMemcpyAsync(col.data(), colors, sizeof(int32_t) * n,
                       mem == RG_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  int nc = 0;
  if (colors) {
    for (int64_t r = 0; r < n; ++r) {
      if (col[r] < 0 || col[r] >= MAXCOLORS) return fail(RG_E_INVAL, "colours must be in 0..63");
      nc = std::max(nc, col[r] + 1);
    }
  } else {
    // greedy colouring of the symmetrised pattern in natural order (smallest colour not used by a
    // coloured neighbour); neighbours of r = row r's columns and column r's rows (transpose)
    std::vector<int64_t> tp(n + 1, 0);
    for (int64_t p = 0; p < c->nnz; ++p) tp[ci[p] + 1]++;
    for (int64_t i = 0; i < n; ++i) tp[i + 1] += tp[i];
    std::vector<int32_t> tr(std::max<int64_t>(c->nnz, 1));
    {
      std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
      for (int64_t r = 0; r < n; ++r)
        for (int32_t p = rp[r]; p < rp[r + 1]; ++p) tr[fill[ci[p]]++] = (int32_t)r;
    }
    std::fill(col.begin(), col.end(), -1);
    for (int64_t r = 0; r < n; ++r) {
      uint64_t used = 0;
      for (int32_t p = rp[r]; p < rp[r + 1]; ++p)
        if (ci[p] != r && col[ci[p]] >= 0) used |= 1ull << col[ci[p]];
      for (int64_t p = tp[r]; p < tp[r + 1]; ++p)
        if (tr[p] != r && col[tr[p]] >= 0) used |= 1ull << col[tr[p]];
      int cc = 0;
      while (cc < MAXCOLORS && (used >> cc & 1ull)) ++cc;
      if (cc >= MAXCOLORS) return fail(RG_E_INVAL, "greedy colouring needs more than 64 colours");
      col[r] = cc;
      nc = std::max(nc, cc + 1);
    }
  }
  // validity (no coupled rows share a colour) and the diagonal positions
  std::vector<int64_t> diag(n, -1);
  for (int64_t r = 0; r < n; ++r)
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
      if (ci[p] == r) diag[r] = p;
      else if (col[ci[p]] == col[r]) return fail(RG_E_INVAL, "not a valid colouring: row " + std::to_string(r) +
                                                              " and column " + std::to_string(ci[p]) + " share a colour");
    }
  for (int64_t r = 0; r < n; ++r)
    if (diag[r] < 0) return fail(RG_E_INVAL, "SSOR needs a stored diagonal entry in every row (row " + std::to_string(r) + ")");
  // rows grouped by colour (stable); the L / U split copies in that order (PrecDev)
  PrecDev P;
  P.ncolors = nc;
  P.omega = omega;
  std::vector<int32_t> perm(n);
  {
    std::vector<int64_t> cnt(nc + 1, 0);
    for (int64_t r = 0; r < n; ++r) cnt[col[r] + 1]++;
    for (int i = 0; i < nc; ++i) cnt[i + 1] += cnt[i];
    for (int i = 0; i <= nc; ++i) P.coff[i] = cnt[i];
    for (int64_t r = 0; r < n; ++r) perm[cnt[col[r]]++] = (int32_t)r;
  }
  std::vector<int32_t> Lrp(n + 1, 0), Urp(n + 1, 0), Lci, Uci, Lmap, Umap, dmap(n);
  Lci.reserve(c->nnz); Uci.reserve(c->nnz); Lmap.reserve(c->nnz); Umap.reserve(c->nnz);
  for (int64_t idx = 0; idx < n; ++idx) {
    const int32_t r = perm[idx];
    dmap[idx] = (int32_t)diag[r];
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
      const int32_t j = ci[p];
      if (j == r) continue;
      if (col[j] < col[r]) { Lci.push_back(j); Lmap.push_back(p); P.cL[col[r]]++; }
      else { Uci.push_back(j); Umap.push_back(p); P.cU[col[r]]++; }
    }
    Lrp[idx + 1] = (int32_t)Lci.size();
    Urp[idx + 1] = (int32_t)Uci.size();
  }
  P.nL = (int64_t)Lci.size();
  P.nU = (int64_t)Uci.size();
  if (nc >= 2) {
    P.l1base = Lrp[P.coff[1]];
    P.nL1 = Lrp[P.coff[2]] - Lrp[P.coff[1]];
  }
  CK(cudaStreamSynchronize(c->stream));
  clear_graphs(c);
  drop_preconditioner(c);
  // device copies
  auto up = [&](const void* h, size_t bytes, const char* what, void** out) -> rg_status {
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(bytes, 8)) != cudaSuccess) {
      cudaGetLastError();
      return fail(RG_E_NOMEM, std::string("device allocation failed: ") + what);
    }
    c->prec_bufs.push_back(d);
    if (h && bytes && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      return fail(RG_E_CUDA, std::string("upload failed: ") + what);
    *out = d;
    return RG_OK;
  };
  rg_status s;
  void *d_perm, *d_Lrp, *d_Lci, *d_Lmap, *d_Lv, *d_Urp, *d_Uci, *d_Umap, *d_Uv, *d_dinv, *d_dinvr, *d_dmap, *d_Lv1;
  if ((s = up(perm.data(), sizeof(int32_t) * n, "perm", &d_perm)) != RG_OK ||
      (s = up(Lrp.data(), sizeof(int32_t) * (n + 1), "L row pointer", &d_Lrp)) != RG_OK ||
      (s = up(Lci.data(), sizeof(int32_t) * P.nL, "L columns", &d_Lci)) != RG_OK ||
      (s = up(Lmap.data(), sizeof(int32_t) * P.nL, "L map", &d_Lmap)) != RG_OK ||
      (s = up(nullptr, sizeof(double) * P.nL, "L values", &d_Lv)) != RG_OK ||
      (s = up(Urp.data(), sizeof(int32_t) * (n + 1), "U row pointer", &d_Urp)) != RG_OK ||
      (s = up(Uci.data(), sizeof(int32_t) * P.nU, "U columns", &d_Uci)) != RG_OK ||
      (s = up(Umap.data(), sizeof(int32_t) * P.nU, "U map", &d_Umap)) != RG_OK ||
      (s = up(nullptr, sizeof(double) * P.nU, "U values", &d_Uv)) != RG_OK ||
      (s = up(nullptr, sizeof(double) * n, "1/diag", &d_dinv)) != RG_OK ||
      (s = up(nullptr, sizeof(double) * n, "1/diag by row", &d_dinvr)) != RG_OK ||
      (s = up(nullptr, sizeof(double) * P.nL1, "scaled colour-1 L values", &d_Lv1)) != RG_OK ||
      (s = up(dmap.data(), sizeof(int32_t) * n, "diag map", &d_dmap)) != RG_OK) {
    cudaStreamSynchronize(c->stream);
    drop_preconditioner(c);
    return s;
  }
  P.perm = (const int32_t*)d_perm;
  P.Lrp = (const int32_t*)d_Lrp; P.Lci = (const int32_t*)d_Lci; P.Lmap = (const int32_t*)d_Lmap; P.Lv = (double*)d_Lv;
  P.Urp = (const int32_t*)d_Urp; P.Uci = (const int32_t*)d_Uci; P.Umap = (const int32_t*)d_Umap; P.Uv = (double*)d_Uv;
  P.dinv = (double*)d_dinv; P.dinvr = (double*)d_dinvr; P.Lv1 = (double*)d_Lv1; P.dmap = (const int32_t*)d_dmap;
  if (!c->pz) {
    if ((s = dalloc(&c->pz, (size_t)c->npad, "pz")) != RG_OK || (s = dalloc(&c->pt, (size_t)c->npad, "pt")) != RG_OK) {
      drop_preconditioner(c);
      return s;
    }
    CK(cudaMemsetAsync(c->pz, 0, sizeof(double) * c->npad, c->stream));
    CK(cudaMemsetAsync(c->pt, 0, sizeof(double) * c->npad, c->stream));
  }
  CK(launch_ssor_values(P, c->v, n, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->P = P;
  c->prec_kind = RG_PREC_SSOR;
  c->L.pz = c->pz;
  c->L.pt = c->pt;
  if (ncolors_out) *ncolors_out = nc;
  return RG_OK;
}

RG_API rg_status rg_apply_preconditioner(rg_ctx* c, const double* x, double* y, rg_mem mem) {
  if (!c || !x || !y) return fail(RG_E_INVAL, "NULL argument");
  if (mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  if (!c->prec_kind) return fail(RG_E_STATE, "no preconditioner set");
  rg_status s = copy_in(c->t1, x, sizeof(double) * c->n, mem, c->stream);
  if (s != RG_OK) return s;
  CK(launch_ssor(c->P, c->L, c->st, c->t1, c->t2, 0, c->stream));
  CK(cudaMemcpyAsync(y, c->t2, sizeof(double) * c->n, mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return RG_OK;
}

RG_API rg_status rg_export(rg_ctx* c, int32_t which, double* out, rg_mem mem, int32_t* k_eff) {
  if (!c) return fail(RG_E_INVAL, "NULL argument");
  if (mem != RG_HOST && mem != RG_DEVICE) return fail(RG_E_INVAL, "unknown memory kind");
  if (which == RG_EXPORT_V || which == RG_EXPORT_H || which == RG_EXPORT_B) {
    if (!c->keepV) return fail(RG_E_STATE, "basis export needs a context created with RG_FLAG_KEEP_BASIS");
    if (galerkin_variant(c->kb_var)) return fail(RG_E_STATE, "basis export covers plain / augment / deflate solves");
    int J = 0;
    CK(cudaMemcpyAsync(&c->hst->kb_steps, &c->st->kb_steps, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    J = c->hst->kb_steps;
    if (J < 1) return fail(RG_E_STATE, "no finished restart cycle to export");
    const int kb = c->kb_var == RG_DEFLATE ? c->kb_k : 0;
    if (which == RG_EXPORT_B && kb == 0) return fail(RG_E_STATE, "B exists for deflate solves with k_eff > 0 only");
    if (k_eff) *k_eff = J;
    if (!out) return RG_OK;
    const cudaMemcpyKind kind = mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (which == RG_EXPORT_V) {
      CK(cudaMemcpy2DAsync(out, sizeof(double) * c->n, c->keepV, sizeof(double) * c->npad, sizeof(double) * c->n, J,
                           kind, c->stream));
    } else if (which == RG_EXPORT_H) {  // state column j holds rows 0..j+1 of H-bar column j
      CK(cudaMemcpy2DAsync(out, sizeof(double) * (J + 1), &c->st->Hraw[0][0], sizeof(double) * (MAXM + 2),
                           sizeof(double) * (J + 1), J, kind, c->stream));
    } else {
      CK(cudaMemcpy2DAsync(out, sizeof(double) * kb, &c->st->Bm[0][0], sizeof(double) * MAXK, sizeof(double) * kb, J,
                           kind, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return RG_OK;
  }
  if (!out) return fail(RG_E_INVAL, "NULL argument");
  if (rg_status r0 = resolve_build(c)) return r0;
  const int k = c->have_W ? c->k_eff : 0;
  if (k_eff) *k_eff = k;
  if (k == 0) return fail(RG_E_STATE, "no recycle space");
  const cudaMemcpyKind kind = mem == RG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (which == RG_EXPORT_W || which == RG_EXPORT_Q) {
    if (which == RG_EXPORT_Q && !(c->c_valid && c->c_kind == 0)) return fail(RG_E_STATE, "Q is not built (run a recycled solve)");
    const int c0 = which == RG_EXPORT_W ? 0 : c->L.VB - k;
    CK(cudaMemcpy2DAsync(out, sizeof(double) * c->n, c->Z + (int64_t)c0 * c->npad, sizeof(double) * c->npad,
                         sizeof(double) * c->n, k, kind, c->stream));
  } else if (which == RG_EXPORT_RC) {
    if (!(c->c_valid && c->c_kind == 0)) return fail(RG_E_STATE, "R_C is not built (run a recycled solve)");
    CK(cudaMemcpy2DAsync(out, sizeof(double) * k, &c->st->RC[0][0], sizeof(double) * MAXK, sizeof(double) * k, k,
                         kind, c->stream));
  } else {
    return fail(RG_E_INVAL, "unknown export item");
  }
  CK(cudaStreamSynchronize(c->stream));
  return RG_OK;
}

static const char* const kernel_names[K_COUNT] = {"spmv_step", "spmv_res", "spmv_plain", "orth_dots1", "orth_upd_dots2",
                                              "orth_upd_norm_ls", "cs_dots_q", "cs_upd_norm", "x_upd_w", "x_upd_cycle",
                                              "norm_b", "gram", "jacobi", "xm", "chol", "persistent_solve", "dcgs_dots_ls",
                                              "dcgs_update", "p_barrier", "p_spmv_dots", "p_reduce", "p_epilogue",
                                              "p_update", "ob_dots", "ob_update", "ssor", "p_reduce_arrive", "cond",
                                              "ssor_sweep_kernels", "p_spmv", "cbuild", "res_from_ax", "dcgs_ls"};

RG_API rg_status rg_kernel_stats(rg_ctx* c, rg_kstat* out, int32_t cap, int32_t* count) {
  const char* const* names = kernel_names;
  if (!c || !count) return fail(RG_E_INVAL, "NULL argument");
  KStatDev ks[K_COUNT];
  CK(cudaMemcpyAsync(ks, &c->st->kstat[0], sizeof(ks), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int n = 0;
  for (int i = 0; i < K_COUNT && n < cap; ++i) {
    if (!out) break;
    rg_kstat& o = out[n++];
    memset(&o, 0, sizeof(o));
    strncpy(o.name, names[i], sizeof(o.name) - 1);
    o.launches = (int64_t)ks[i].launches;
    o.noop_launches = (int64_t)ks[i].noop;
    o.total_ms = ks[i].ns * 1e-6;
    o.tail_ms = ks[i].tail_ns * 1e-6;
    o.bytes = ks[i].bytes;
  }
  if (out && n < cap) {  // kernels launched directly by the host (no device counter)
    rg_kstat& o = out[n++];
    memset(&o, 0, sizeof(o));
    strncpy(o.name, "host_launched", sizeof(o.name) - 1);
    o.launches = (int64_t)g_host_launches.load();
  }
  *count = out ? n : K_COUNT + 1;
  return RG_OK;
}

RG_API rg_status rg_kernel_trace(rg_ctx* c, rg_trace_event* out, int32_t cap, int32_t* count) {
  NvtxRange nvtx_("rg_kernel_trace");
  if (!c || !count || (cap > 0 && !out)) return fail(RG_E_INVAL, "NULL argument");
  if (!c->trace) return fail(RG_E_STATE, "the kernel trace needs a context created with RG_FLAG_PROFILE");
  unsigned len = 0;
  CK(cudaMemcpyAsync(&len, &c->st->trace_len, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *count = (int32_t)std::min<unsigned>(len, (unsigned)INT32_MAX);
  const int n = (int)std::min<int64_t>({(int64_t)len, (int64_t)TRACE_CAP, (int64_t)std::max(cap, 0)});
  if (n <= 0) return RG_OK;
  std::vector<unsigned long long> buf((size_t)2 * n);
  CK(cudaMemcpy(buf.data(), c->trace, sizeof(unsigned long long) * 2 * n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) {
    rg_trace_event& e = out[i];
    memset(&e, 0, sizeof(e));
    e.t_ns = (int64_t)buf[2 * i];
    const int kid = (int)(buf[2 * i + 1] & 0xffffu);
    e.kind = (int32_t)(buf[2 * i + 1] >> 16);
    strncpy(e.name, kid < K_COUNT ? kernel_names[kid] : "?", sizeof(e.name) - 1);
  }
  return RG_OK;
}

RG_API rg_status rg_reset_kernel_stats(rg_ctx* c) {
  if (!c) return fail(RG_E_INVAL, "ctx is NULL");
  CK(cudaMemsetAsync(&c->st->kstat[0], 0, sizeof(KStatDev) * K_COUNT, c->stream));
  CK(cudaMemsetAsync(&c->st->trace_len, 0, sizeof(unsigned), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  g_host_launches = 0;
  return RG_OK;
}

}  // extern "C"

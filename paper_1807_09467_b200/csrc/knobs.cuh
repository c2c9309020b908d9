// knobs.cuh — experiment switches for A/B measurements (DESIGN.md §7 "measured negatives").
//
// COMPILED OUT by default: every knob returns "unset" and the library reads no environment
// variable, so a product build's behaviour depends only on its arguments and rg_options.flags.
// `make rg EXPERIMENTS=1` (-DRG_EXPERIMENTS) builds a library that honours them.  The names:
//   RG_NO_TMA_DK1 / RG_NO_TMA_DK2 / RG_NO_TMA_DCGS   register-limited DCGS2 passes instead of TMA
//   RG_DK1_TILES                                   shared-memory-staged DK1 (first version)
//   RG_JACOBI_NT=n                                 threads of the Jacobi CTA
//   RG_NO_PT1024                                   no 1024-thread single-CTA persistent solve
//   RG_NO_SMEM_CSR                                 no CSR pattern cache in the persistent solve
//   RG_PERSIST_CTAS_PER_SM=n                       persistent CTAs per SM
//   RG_NO_NBSYNC / RG_NO_LLRED                     grid barriers instead of neighbour sync / LL reductions
//   RG_SKEW=j                                      per-CTA timestamps of Arnoldi step j (stderr CSV)
//   RG_NO_BSR_TMA / RG_NO_SPMM                     BSR SpMV without TMA / C = A W by k SpMVs
//   RG_NO_CGS / RG_NO_FUSE_C / RG_NO_FUSE_RES      generic CGS kernels / no k_cbuild / no fused A x0
//   RG_NO_ALIAS                                    persistent solve on the library's b / x buffers
//   RG_FORCE_PERSIST / RG_FORCE_DCGS               ignore the measured size / byte thresholds
//   RG_SYNC_BUILD                                  rg_build_recycle always synchronous
//   RG_TIMING / RG_DEBUG                           host-side phase timings / Jacobi sweep counts (stderr)
//   RG_NO_PDL / RG_NO_TMA_CGS                       no programmatic dependent launch / register CGS2 passes
//   RG_UNROLL=n                                    Arnoldi steps per WHILE-loop body (default 4 DCGS2, 2 CGS2)
//   RG_NO_GRAPH / RG_CGS2 / RG_NO_PERSIST          same as the RG_FLAG_* bits of include/rg.h
#pragma once
#include <cstdlib>

namespace rg {

#ifdef RG_EXPERIMENTS
inline const char* knob_env(const char* name) { return std::getenv(name); }
#else
inline const char* knob_env(const char*) { return nullptr; }
#endif
inline bool knob(const char* name) { return knob_env(name) != nullptr; }
inline int knob_int(const char* name, int def) {
  const char* v = knob_env(name);
  return v ? std::atoi(v) : def;
}

}  // namespace rg

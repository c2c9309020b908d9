// Grid-barrier micro-benchmark (persistent solve, C2 geometry: 296 CTAs x 512, 2 per SM).
// Variants: 0 = persistent.cu's gbar (threadfence + atomicAdd + volatile poll w/ nanosleep back-off + threadfence)
//           1 = red.release.gpu arrive + ld.acquire.gpu poll (no back-off)
//           2 = 1 with a fixed 20 ns sleep between polls
//           3 = atom.add.acq_rel arrive + ld.acquire poll w/ back-off
// Each iteration: write nv partials, barrier, per-CTA column sums (greduce), barrier, read totals.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/t_gbar tools/cutest/t_gbar.cu
#include <cstdio>
#include <cstdint>
constexpr int PT = 512, MAXRED = 512;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_ar(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}

template <int V>
__device__ __forceinline__ void gbar(unsigned* bar, unsigned& nb) {
  if (V >= 8) {  // split counters: CTA b arrives on counter b % NC (own 128-B lines); warp 0 lanes poll all NC
    constexpr int NC = V == 8 ? 4 : (V == 9 ? 8 : 16);
    __syncthreads();
    if (threadIdx.x < 32) {
      nb += 1;
      const int lane = threadIdx.x;
      if (lane == 0) red_rel(bar + 32 * (blockIdx.x % NC), 1u);
      const unsigned cntc = lane < NC ? (gridDim.x - lane + NC - 1) / NC : 0u;  // CTAs on counter `lane`
      const unsigned tgt = nb * cntc;
      for (;;) {
        const unsigned v = lane < NC ? ld_acq(bar + 32 * lane) : 0u;
        if (__all_sync(0xffffffffu, v >= tgt)) break;
        __nanosleep(20);
      }
    }
    __syncthreads();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    nb += 1;
    const unsigned target = nb * gridDim.x;
    if (V == 0) {
      __threadfence();
      if (atomicAdd(bar, 1u) + 1u < target) {
        volatile unsigned* cnt = bar;
        unsigned ns = 32;
        while (*cnt < target) { __nanosleep(ns); if (ns < 256) ns <<= 1; }
      }
      __threadfence();
    } else if (V == 1 || V == 2) {
      red_rel(bar, 1u);
      while (ld_acq(bar) < target) { if (V == 2) __nanosleep(20); }
    } else if (V == 5 || V == 6) {
      // two-level: groups of GS CTAs count on their own 128-B line; the last of a group arrives at the root
      constexpr int GS = 16;
      const int g = blockIdx.x / GS;
      const unsigned gsz = min((unsigned)GS, gridDim.x - g * GS);
      const unsigned ngr = (gridDim.x + GS - 1) / GS;
      unsigned* gc = bar + 64 + 32 * g;
      if (atom_ar(gc, 1u) + 1u == nb * gsz) {
        if (V == 5) {
          red_rel(bar, 1u);
        } else if (atom_ar(bar, 1u) + 1u == nb * ngr) {  // last group: release every group's word
          for (unsigned q = 0; q < ngr; ++q) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 64 + 32 * 64 + 32 * q), "r"(nb) : "memory");
        }
      }
      if (V == 5) {
        while (ld_acq(bar) < nb * ngr) __nanosleep(20);
      } else {
        while (ld_acq(bar + 64 + 32 * 64 + 32 * g) < nb) __nanosleep(20);
      }
    } else if (V == 7) {
      // every CTA polls until the count is reached with relaxed loads, then one acquire fence
      red_rel(bar, 1u);
      volatile unsigned* cnt = bar;
      while (*cnt < target) {}
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    } else {
      if (atom_ar(bar, 1u) + 1u < target) {
        unsigned ns = 32;
        while (ld_acq(bar) < target) { __nanosleep(ns); if (ns < 256) ns <<= 1; }
      }
    }
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(PT, 2) k(unsigned* bar, double* partial, double* tot_g, int nv, int iters, double* out,
                                          unsigned long long* t) {
  __shared__ double tot[MAXRED];
  unsigned nb = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, G = gridDim.x;
  double acc = 0;
  unsigned long long t0 = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 8 && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (nv == 0) { gbar<V>(bar, nb); continue; }  // barrier only
    for (int i = threadIdx.x; i < nv; i += PT) partial[(size_t)blockIdx.x * MAXRED + i] = 1.0 + it + i + acc * 1e-30;
    gbar<V>(bar, nb);
    for (int col = blockIdx.x + G * wid; col < nv; col += G * (PT / 32)) {
      double a = 0.0;
      for (int b0 = lane; b0 < G; b0 += 32 * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < G ? __ldcg(partial + (size_t)(b0 + 32 * u) * MAXRED + col) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) a += v[u];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) tot_g[col] = a;
    }
    gbar<V>(bar, nb);
    for (int i = threadIdx.x; i < nv; i += PT) tot[i] = __ldcg(tot_g + i);
    __syncthreads();
    acc += tot[threadIdx.x % nv];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    t[0] = t1 - t0;
  }
  if (acc == 1.2345) out[0] = acc;
}

static int g_grid = 296;
__device__ __forceinline__ void ll_st(unsigned long long* p, double v, unsigned ep) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long e = (unsigned long long)ep << 32;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"((b & 0xffffffffull) | e), "l"((b >> 32) | e) : "memory");
}
template <int SLEEP>
__device__ __forceinline__ double ll_ld(const unsigned long long* p, unsigned ep) {
  unsigned long long w0, w1;
  for (;;) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if ((unsigned)(w0 >> 32) == ep && (unsigned)(w1 >> 32) == ep) break;
    if (SLEEP) __nanosleep(SLEEP);
  }
  return __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
}
__device__ __forceinline__ double bsum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) { double s = 0.0; for (int i = 0; i < nw; ++i) s += sh[i]; sh[32] = s; }
  __syncthreads();
  return sh[32];
}
template <int SLEEP, int R>
__global__ void __launch_bounds__(PT, 2) kll(unsigned long long* ll, int nv, int iters, double* out, unsigned long long* t) {
  __shared__ double tot[MAXRED];
  __shared__ double sh[33];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  double acc = 0;
  unsigned long long t0 = 0;
  unsigned ep = 0;
  for (int it = 0; it < iters; ++it) {
    if (it == 8 && b == 0 && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    ++ep;
    const int buf = ep & 1;
    unsigned long long* part = ll + (size_t)buf * 296 * MAXRED * 2;
    unsigned long long* totw = ll + (size_t)2 * 296 * MAXRED * 2 + (size_t)buf * MAXRED * 2;  // replica stride 2*MAXRED*2
    __syncthreads();
    for (int i = tid; i < nv; i += PT) ll_st(part + ((size_t)b * MAXRED + i) * 2, 1.0 + i + acc * 1e-30, ep);
    for (int col = b; col < nv; col += G) {
      double a = tid < G ? ll_ld<SLEEP>(part + ((size_t)tid * MAXRED + col) * 2, ep) : 0.0;
      a = bsum(a, sh);
      if (tid < R) ll_st(totw + (size_t)tid * 2 * MAXRED * 2 + (size_t)col * 2, a, ep);
    }
    if (R > 0) for (int i = tid; i < nv; i += PT) tot[i] = ll_ld<SLEEP>(totw + (size_t)(b % R) * 2 * MAXRED * 2 + (size_t)i * 2, ep);
    __syncthreads();
    acc += tot[tid % nv];
  }
  if (b == 0 && tid == 0) { unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); t[0] = t1 - t0; }
  if (acc == 1.2345) out[0] = acc;
}
template <int SLEEP, int R>
void runll(int nv, unsigned long long* ll, double* out, unsigned long long* t) {
  int iters = 2008;
  cudaMemset(ll, 0, (size_t)(2 * 296 * MAXRED * 2 + 32 * 2 * MAXRED * 2) * 8);
  void* args[] = {&ll, &nv, &iters, &out, &t};
  cudaLaunchCooperativeKernel((void*)kll<SLEEP, R>, g_grid, PT, args, 0, 0);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("grid %d LL R %d sleep %d nv %d: %.3f us per reduction (%s)\n", g_grid, R, SLEEP, nv, h * 1e-3 / (iters - 8), cudaGetErrorString(cudaGetLastError()));
}

template <int V>
void run(int nv, unsigned* bar, double* partial, double* tot_g, double* out, unsigned long long* t) {
  const int iters = 2008;
  cudaMemset(bar, 0, 4096 * 4);
  void* args[] = {&bar, &partial, &tot_g, &nv, (void*)&iters, &out, &t};
  int it2 = iters;
  args[4] = &it2;
  cudaLaunchCooperativeKernel((void*)k<V>, g_grid, PT, args, 0, 0);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("grid %d variant %d nv %d: %.3f us per greduce (%s)\n", g_grid, V, nv, h * 1e-3 / (iters - 8), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned* bar;
  double *partial, *tot_g, *out;
  unsigned long long* t;
  cudaMalloc(&bar, 4096 * 4);
  cudaMalloc(&partial, 296 * MAXRED * 8);
  cudaMalloc(&tot_g, MAXRED * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&t, 8);
  unsigned long long* ll;
  cudaMalloc(&ll, (size_t)(2 * 296 * MAXRED * 2 + 32 * 2 * MAXRED * 2) * 8);
  for (int gsz : {296, 148}) for (int nv : {1, 92}) {
    g_grid = gsz;
    runll<0, 1>(nv, ll, out, t);
    runll<0, 4>(nv, ll, out, t);
    runll<0, 16>(nv, ll, out, t);
    runll<64, 16>(nv, ll, out, t);
  }
  for (int gsz : {296}) for (int nv : {92}) {
    g_grid = gsz;
    for (int r = 0; r < 1; ++r) {
      run<0>(nv, bar, partial, tot_g, out, t);
      run<2>(nv, bar, partial, tot_g, out, t);
      run<3>(nv, bar, partial, tot_g, out, t);
      run<8>(nv, bar, partial, tot_g, out, t);
    }
  }
  return 0;
}

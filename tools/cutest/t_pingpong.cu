// Cross-SM flag round trip: CTA 0 and CTA 1 (different SMs) bounce a counter through one global word.
// Variants: volatile / relaxed.gpu / acquire-release.  Prints ns per one-way hop.
#include <cstdio>
template <int V>
__device__ __forceinline__ unsigned ld(const unsigned* p) {
  unsigned v;
  if (V == 0) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else if (V == 1) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int V>
__device__ __forceinline__ void st(unsigned* p, unsigned v) {
  if (V == 0) asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else if (V == 1) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int V>
__global__ void k(unsigned* w, int n, unsigned long long* t) {
  if (threadIdx.x) return;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (blockIdx.x == 0) {
    for (unsigned i = 1; i <= (unsigned)n; ++i) {
      st<V>(w, 2 * i - 1);
      while (ld<V>(w + 32) != 2 * i) {}
    }
  } else if (blockIdx.x == gridDim.x - 1) {
    for (unsigned i = 1; i <= (unsigned)n; ++i) {
      while (ld<V>(w) != 2 * i - 1) {}
      st<V>(w + 32, 2 * i);
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0) t[0] = t1 - t0;
}
template <int V>
void run(unsigned* w, unsigned long long* t, int grid) {
  cudaMemset(w, 0, 4096);
  const int n = 20000;
  k<V><<<grid, 32>>>(w, n, t);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("variant %d grid %d: %.1f ns per one-way hop (%s)\n", V, grid, h / (2.0 * n), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned* w;
  unsigned long long* t;
  cudaMalloc(&w, 4096);
  cudaMalloc(&t, 8);
  for (int g : {2, 148, 296}) { run<0>(w, t, g); run<1>(w, t, g); run<2>(w, t, g); }
  return 0;
}

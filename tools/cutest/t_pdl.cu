// probe: programmatic dependent launch (PDL) inside the body of a conditional WHILE graph node
// captured from a stream — the structure of the solver's Arnoldi step (K1 = a streaming "SpMV",
// K2 = a streaming pass that reads K1's output, K3 = a second pass).  Reports the time per body
// iteration with plain stream edges vs programmatic edges (K2, K3 launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, griddepcontrol.wait before consuming).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cutest/t_pdl tools/cutest/t_pdl.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// y = 2 x over n doubles (streaming); trigger early
__global__ void __launch_bounds__(512, 2) k1(const double* __restrict__ x, double* __restrict__ y, int64_t n, int pdl) {
  if (pdl) pdl_trigger();
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 512) y[i] = 2.0 * __ldcs(x + i);
}
// reads a big independent array (prefetchable) and y (after the wait); writes z
__global__ void __launch_bounds__(512, 2) k2(const double* __restrict__ big, int64_t nb, const double* __restrict__ y,
                                            double* __restrict__ z, int64_t n, int pdl) {
  double acc = 0.0;
  // independent part first (does not depend on the previous kernel)
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < nb; i += (int64_t)gridDim.x * 512) acc += __ldcs(big + i);
  if (pdl) {
    pdl_trigger();
    pdl_wait();
  }
  for (int64_t i = blockIdx.x * 512ll + threadIdx.x; i < n; i += (int64_t)gridDim.x * 512) z[i] = y[i] + acc * 1e-300;
}
__global__ void k_cond(int* cnt, cudaGraphConditionalHandle h, int iters) {
  if (threadIdx.x == 0) {
    int c = ++*cnt;
    cudaGraphSetConditional(h, c < iters ? 1u : 0u);
  }
}
__global__ void k_reset(int* cnt) { *cnt = 0; }

int main() {
  const int64_t n = 2097152, nb = 8 * n;  // y: 16.8 MB, big: 134 MB
  double *x, *y, *z, *big;
  int* cnt;
  cudaMalloc(&x, 8 * n);
  cudaMalloc(&y, 8 * n);
  cudaMalloc(&z, 8 * n);
  cudaMalloc(&big, 8 * nb);
  cudaMalloc(&cnt, 4);
  cudaMemset(x, 0, 8 * n);
  cudaMemset(big, 0, 8 * nb);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int iters = 200;
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t G;
    cudaGraphCreate(&G, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, G, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, G, nullptr, 0, &p);
    if (e != cudaSuccess) { printf("add node: %s\n", cudaGetErrorString(e)); return 1; }
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaGraph_t tmp;
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { printf("capture: %s\n", cudaGetErrorString(e)); return 1; }
    k1<<<296, 512, 0, s>>>(x, y, n, pdl);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(296);
    cfg.blockDim = dim3(512);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, k2, (const double*)big, nb, (const double*)y, z, n, pdl);
    if (e != cudaSuccess) printf("launch k2: %s\n", cudaGetErrorString(e));
    e = cudaLaunchKernelEx(&cfg, k2, (const double*)big, nb, (const double*)z, x, n, pdl);
    if (e != cudaSuccess) printf("launch k2b: %s\n", cudaGetErrorString(e));
    k_cond<<<1, 32, 0, s>>>(cnt, h, iters);
    e = cudaStreamEndCapture(s, &tmp);
    if (e != cudaSuccess) { printf("end capture (pdl=%d): %s\n", pdl, cudaGetErrorString(e)); return 1; }
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, G, 0);
    if (e != cudaSuccess) { printf("instantiate (pdl=%d): %s\n", pdl, cudaGetErrorString(e)); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      k_reset<<<1, 1, 0, s>>>(cnt);
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    // kernels alone (stream launches, no graph) for reference
    printf("pdl=%d: %.2f us per WHILE iteration (k1 + 2 x k2 + cond)  %s\n", pdl, best * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// Probe: grid-wide barrier cost on B200 (cooperative_groups grid.sync vs a counter barrier) and the kernel-boundary cost inside a CUDA graph.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_gridbar.cu -o /tmp/gridbar
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int it = 0; it < iters; ++it) g.sync();
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void k_bar(unsigned* bar, int iters) {
  __shared__ unsigned gen;
  if (threadIdx.x == 0) gen = ld_acq(bar + 32);
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned g0 = gen;
      __threadfence();
      const unsigned arrived = atomicAdd(bar, 1u);
      if (arrived == gridDim.x - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicAdd(bar + 32, 1u);
      } else {
        while (ld_acq(bar + 32) == g0) {}
      }
      gen = g0 + 1;
    }
    __syncthreads();
  }
}
__global__ void k_empty() {}
int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned* bar;
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0); cudaEventCreate(&t1);
  const int N = 1000;
  for (int nb : {148, 296}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(256); cfg.stream = s;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cg, N);
    cudaEventRecord(t0, s);
    cudaLaunchKernelEx(&cfg, k_cg, N);
    cudaEventRecord(t1, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, t0, t1);
    printf("cg grid.sync  %d blocks: %.3f us/sync\n", nb, ms * 1000.f / N);
    cudaLaunchKernelEx(&cfg, k_bar, bar, N);
    cudaEventRecord(t0, s);
    cudaLaunchKernelEx(&cfg, k_bar, bar, N);
    cudaEventRecord(t1, s);
    cudaError_t e = cudaStreamSynchronize(s);
    cudaEventElapsedTime(&ms, t0, t1);
    printf("custom barrier %d blocks: %.3f us/sync (%s)\n", nb, ms * 1000.f / N, cudaGetErrorString(e));
  }
  // kernel boundary in a graph: 1000 empty kernels, and 1000 148-block kernels
  for (int nb : {1, 148, 1184}) {
    cudaGraph_t gr; cudaGraphExec_t ex;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) k_empty<<<nb, 256, 0, s>>>();
    cudaStreamEndCapture(s, &gr);
    cudaGraphInstantiate(&ex, gr, 0);
    cudaGraphLaunch(ex, s);
    cudaEventRecord(t0, s);
    cudaGraphLaunch(ex, s);
    cudaEventRecord(t1, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, t0, t1);
    printf("graph kernel boundary (%d blocks): %.3f us/kernel\n", nb, ms * 1000.f / N);
  }
  return 0;
}

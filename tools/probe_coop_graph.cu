// Probe: is a cooperative launch (grid.sync) capturable in a CUDA graph on this stack?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* a, int n) {
  cg::grid_group g = cg::this_grid();
  for (int it = 0; it < 100; ++it) {
    for (int i = g.thread_rank(); i < n; i += g.size()) a[i] += 1;
    g.sync();
    if (g.thread_rank() == 0) a[n] = a[0] + a[n - 1];
    g.sync();
  }
}
int main() {
  int n = 1 << 20, *a;
  cudaMalloc(&a, (n + 1) * sizeof(int));
  cudaMemset(a, 0, (n + 1) * sizeof(int));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, 0);
  printf("blocks/SM %d\n", nb);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaGraph_t gr;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, a, n);
  cudaError_t e2 = cudaStreamEndCapture(s, &gr);
  printf("capture launch: %s, end: %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
  cudaGraphExec_t ex;
  cudaError_t e3 = cudaGraphInstantiate(&ex, gr, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e3));
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0); cudaEventCreate(&t1);
  cudaGraphLaunch(ex, s);
  cudaEventRecord(t0, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ex, s);
  cudaEventRecord(t1, s);
  cudaError_t e4 = cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, t0, t1);
  int h[2];
  cudaMemcpy(h, a, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(h + 1, a + n, sizeof(int), cudaMemcpyDeviceToHost);
  printf("run: %s a0=%d an=%d  %.2f us per 200 grid syncs\n", cudaGetErrorString(e4), h[0], h[1], ms * 100.f);
  // empty-work barrier cost
  return 0;
}

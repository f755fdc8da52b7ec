// Microbenchmark: cost of a grid-wide cooperative sync vs kernel-boundary
// (graph) launches, for sizing the small-level strategy.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_gsync(int iters, double* x) {
  cg::grid_group g = cg::this_grid();
  double v = x[blockIdx.x * blockDim.x + threadIdx.x];
  for (int i = 0; i < iters; ++i) {
    v = v * 1.0000001 + 1e-9;
    g.sync();
  }
  x[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_step(double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  x[i] = x[i] * 1.0000001 + 1e-9;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* x;
  cudaMalloc(&x, sizeof(double) * sms * 1024 * 4);
  cudaMemset(x, 0, sizeof(double) * sms * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int thr : {256, 1024}) {
    int it = 1000;
    void* args[] = {&it, &x};
    cudaLaunchCooperativeKernel((void*)k_gsync, sms, thr, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_gsync, sms, thr, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync  %d CTAs x %d thr: %.2f us per sync (%s)\n", sms, thr, ms * 1e3 / it, cudaGetErrorString(cudaGetLastError()));
  }
  // graph of 1000 dependent small kernels
  for (int blocks : {64, 148, 1024}) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 1000; ++i) k_step<<<blocks, 256, 0, s>>>(x);
    cudaStreamEndCapture(s, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph kernel node (%d CTAs x 256): %.2f us per kernel\n", blocks, ms * 1e3 / 1000);
  }
  return 0;
}

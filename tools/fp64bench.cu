// fp64bench.cu -- FP64 vector throughput and latency of the device (DADD / DMUL / DFMA),
// the ceiling the stencil kernels' arithmetic runs against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64bench fp64bench.cu && ./fp64bench
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int ILP>
__global__ void __launch_bounds__(1024) k_tp(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = a + threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], b);
      else if (OP == 1) x[i] = __dmul_rn(x[i], b);
      else x[i] = __fma_rn(x[i], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <int OP, int ILP>
void run(const char* name, int threads, int ctas_per_sm) {
  int dev = 0, sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  k_tp<OP, ILP><<<sms * ctas_per_sm, threads>>>(out, 100, 1.0, 1.0000001);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k_tp<OP, ILP><<<sms * ctas_per_sm, threads>>>(out, iters, 1.0, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * ctas_per_sm * threads * (double)iters * ILP;
  const double rate = ops / (ms * 1e-3);
  printf("%-6s ILP %d  %4d thr x %d CTA/SM: %8.3f ms  %7.2f Gop/s  = %6.2f lanes/clk/SM at %d MHz  (chain step %.1f clk)\n",
         name, ILP, threads, ctas_per_sm, ms, rate * 1e-9, rate / sms / (khz * 1e3), khz / 1000,
         ms * 1e-3 * khz * 1e3 / ((double)iters * ILP));
  cudaFree(out);
}

int main() {
  run<0, 1>("DADD", 32, 1);    // latency: one warp per SM, one chain
  run<2, 1>("DFMA", 32, 1);
  run<0, 8>("DADD", 1024, 1);  // throughput
  run<1, 8>("DMUL", 1024, 1);
  run<2, 8>("DFMA", 1024, 1);
  run<0, 4>("DADD", 512, 2);
  run<0, 1>("DADD", 1024, 1);  // one chain per thread, 32 warps per SM
  run<0, 2>("DADD", 1024, 1);
  run<0, 1>("DADD", 256, 1);   // 2 warps per scheduler
  return 0;
}

// membench.cu -- micro-benchmarks isolating the memory behaviour of the
// GS-RB half-sweep access pattern on B200 (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
// Data: NB blocks x 4096 doubles for phi (two colour halves) and rhs, like the
// finest level of BASELINE config 2 (256^3, 16^3 blocks).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int NI = 4096, H = 2048;

// 1. flat stream: out = a + b over n doubles (2 reads + 1 write), double2
__global__ void k_stream(const double2* __restrict__ a, const double2* __restrict__ b,
                         double2* __restrict__ o, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    o[i] = make_double2(x.x + y.x, x.y + y.y);
  }
}

// 2. CTA per block: read opp half + rhs half, write active half (plain loads)
__global__ void __launch_bounds__(256) k_block_plain(const double* __restrict__ phi, const double* __restrict__ rhs,
                                                     double* __restrict__ out, int c) {
  const size_t base = (size_t)blockIdx.x * NI;
  const double* opp = phi + base + (1 - c) * H;
  const double* g = rhs + base + c * H;
  double* d = out + base + c * H;
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = opp[threadIdx.x + 256 * q] + g[threadIdx.x + 256 * q];
#pragma unroll
  for (int q = 0; q < 8; ++q) d[threadIdx.x + 256 * q] = v[q];
}

__device__ __forceinline__ void cp_async8(double* s, const double* g) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(double* s, const double* g) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory"); }

// 3. CTA per block, opp half via cp.async (8B) into smem, rhs in regs, sync, compute
template <int VEC>
__global__ void __launch_bounds__(256) k_block_async(const double* __restrict__ phi, const double* __restrict__ rhs,
                                                     double* __restrict__ out, int c) {
  __shared__ __align__(16) double T[H + 64];
  const size_t base = (size_t)blockIdx.x * NI;
  const double* opp = phi + base + (1 - c) * H;
  const double* g = rhs + base + c * H;
  double* d = out + base + c * H;
  if (VEC == 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) cp_async16(&T[2 * (threadIdx.x + 256 * q)], opp + 2 * (threadIdx.x + 256 * q));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) cp_async8(&T[threadIdx.x + 256 * q], opp + threadIdx.x + 256 * q);
  }
  double gv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) gv[q] = g[threadIdx.x + 256 * q];
  cp_wait();
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = threadIdx.x + 256 * q;
    d[e] = (T[e] + T[(e + 1) & (H - 1)] + T[(e + 8) & (H - 1)] + gv[q]) / 6.0;
  }
}

// 4. as 3 plus a gather of 768 halo values from 6 neighbour blocks (same
//    positions as the real x/y/z faces: x faces are 1 value per 8-entry row)
__global__ void __launch_bounds__(256) k_block_halo(const double* __restrict__ phi, const double* __restrict__ rhs,
                                                    double* __restrict__ out, int c, int nbx) {
  __shared__ __align__(16) double T[H + 1024];
  const int b = blockIdx.x;
  const size_t base = (size_t)b * NI;
  const double* opp = phi + base + (1 - c) * H;
  const double* g = rhs + base + c * H;
  double* d = out + base + c * H;
#pragma unroll
  for (int q = 0; q < 8; ++q) cp_async8(&T[threadIdx.x + 256 * q], opp + threadIdx.x + 256 * q);
  double gv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) gv[q] = g[threadIdx.x + 256 * q];
  // halo: 6 faces x 128 values; neighbour = b +- 1, +- nbx, +- nbx^2 (clamped)
  double hv[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int q = threadIdx.x + 256 * u;
    const int dir = q >> 7, r = q & 127;
    const int off[6] = {-1, 1, -nbx, nbx, -nbx * nbx, nbx * nbx};
    int nb = b + off[dir];
    nb = nb < 0 ? 0 : (nb >= (int)gridDim.x ? gridDim.x - 1 : nb);
    int e;
    if (dir < 2) e = (r << 3) + (dir ? 0 : 7);          // x face: one per row
    else if (dir < 4) e = (r & 7) + ((r >> 3) << 7) + (dir == 2 ? 120 : 0);  // y face
    else e = r + (dir == 4 ? 1920 : 0);                  // z face
    hv[u] = phi[(size_t)nb * NI + (1 - c) * H + e];
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) T[H + threadIdx.x + 256 * u] = hv[u];
  cp_wait();
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = threadIdx.x + 256 * q;
    d[e] = (T[e] + T[(e + 1) & (H - 1)] + T[H + ((e + 8) & 767)] + gv[q]) / 6.0;
  }
}


// 5. real tile geometry: opposite colour register-staged into a padded
//    (18 x 18 rows x 9 slots) tile, barrier, 6-point GS update from smem
__device__ __forceinline__ double div6m(double x) {
  const double y = 0.16666666666666666;
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, 6.0, x);
  const double q1 = __fma_rn(r, y, q);
  const double aq = fabs(q);
  if (__builtin_expect(aq > 1e-300 && aq < 1e300, 1)) return q1;
  return x / 6.0;
}
template <int MODE>
__global__ void __launch_bounds__(256) k_tile_gs(const double* __restrict__ phi, const double* __restrict__ rhs,
                                                 double* __restrict__ out, int c) {
  constexpr int RW = 9, P = 18, ZS = RW * P;
  __shared__ double T[P * P * RW];
  const size_t base = (size_t)blockIdx.x * NI;
  const double* opp = phi + base + (1 - c) * H;
  const double* g = rhs + base + c * H;
  double* d = out + base + c * H;
  double ov[8], gv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { ov[q] = opp[threadIdx.x + 256 * q]; gv[q] = g[threadIdx.x + 256 * q]; }
  const int m = threadIdx.x & 7, row0 = threadIdx.x >> 3;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int row = row0 + 32 * q, j = row & 15, k = row >> 4;
    const int B = ((k + 1) * P + (j + 1)) * RW + m;
    T[B + ((1 - c + j + k) & 1)] = ov[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int row = row0 + 32 * q, j = row & 15, k = row >> 4;
    const int B = ((k + 1) * P + (j + 1)) * RW + m;
    const int o = (c + j + k) & 1;
    double s;
    if (MODE == 3) {
      s = T[B + o] + gv[q];
    } else {
      s = T[B] + T[B + 1] + T[B + o - RW] + T[B + o + RW] + T[B + o - ZS] + T[B + o + ZS] - 1e-3 * gv[q];
    }
    double v;
    if (MODE == 0) v = s / 6.0;
    else if (MODE == 1) v = div6m(s);
    else v = s * 0.16666666666666666;
    d[threadIdx.x + 256 * q] = v;
  }
}

int main() {
  const int nbx = 16, NB = nbx * nbx * nbx;
  const size_t n = (size_t)NB * NI;
  double *phi, *rhs, *out;
  CK(cudaMalloc(&phi, n * 8));
  CK(cudaMalloc(&rhs, n * 8));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMemset(phi, 0, n * 8));
  CK(cudaMemset(rhs, 0, n * 8));
  CK(cudaMemset(out, 0, n * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch(i);
    CK(cudaDeviceSynchronize());
    const int R = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) launch(i);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-28s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  const double half = (double)NB * H * 8;
  timeit("stream a+b->o (3x half)", 3 * half, [&](int) {
    k_stream<<<148 * 8, 256>>>((const double2*)phi, (const double2*)rhs, (double2*)out, (long)(NB * H / 2));
  });
  timeit("block plain", 3 * half, [&](int i) { k_block_plain<<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("block cp.async 8B", 3 * half, [&](int i) { k_block_async<8><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("block cp.async 16B", 3 * half, [&](int i) { k_block_async<16><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("block cp.async + halo", 3 * half, [&](int i) { k_block_halo<<<NB, 256>>>(phi, rhs, phi, i & 1, nbx); });
  timeit("tile gs  / 6.0", 3 * half, [&](int i) { k_tile_gs<0><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("tile gs  div6 fma", 3 * half, [&](int i) { k_tile_gs<1><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("tile gs  * (1/6)", 3 * half, [&](int i) { k_tile_gs<2><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  timeit("tile 1 LDS", 3 * half, [&](int i) { k_tile_gs<3><<<NB, 256>>>(phi, rhs, phi, i & 1); });
  return 0;
}

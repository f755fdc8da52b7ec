// Microbenchmark: cost of the coarse solve's cluster primitives (8 CTAs x 512
// threads): the st.async cluster reduction (csum), the plane publish, a
// cluster barrier and a CTA barrier.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/clusterbench tools/clusterbench.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int NC = 8, THR = 512, N = 16, P = N + 2, PP = P * P, NSTAGE = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __cluster_dims__(NC, 1, 1) __launch_bounds__(THR) k_bench(int mode, int iters, double* out,
                                                                           long long* cyc) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double part[NSTAGE][NC][2];
  __shared__ double vals[2][THR];
  __shared__ double bc[4];
  __shared__ double Gx[2][PP];
  __shared__ double gh[2][2][PP];
  __shared__ __align__(8) uint64_t sbar[NSTAGE];
  __shared__ __align__(8) uint64_t gbar[2];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int zr = (int)cl.block_rank();
  const int x = t % N, y = (t / N) % N, lp = t / (N * N);
  const int pi = (x + 1) + (y + 1) * P;
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) mbar_init(&sbar[k], 1);
    mbar_init(&gbar[0], 1);
    mbar_init(&gbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  unsigned uses = 0, guses = 0;
  double acc = t * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {  // csum
      const int stage = it % 5;
      vals[0][t] = acc;
      vals[1][t] = acc * 0.5;
      if (t == 0) mbar_arrive_expect_tx(&sbar[stage], NC * 16u);
      __syncthreads();
      if (wid == 0) {
        double sa = 0, sb = 0;
#pragma unroll
        for (int k = 0; k < THR / 32; ++k) {
          sa += vals[0][lane + 32 * k];
          sb += vals[1][lane + 32 * k];
        }
        sa = warp_sum(sa);
        sb = warp_sum(sb);
        if (lane < NC) {
          uint32_t ra, rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&part[stage][zr][0])), "r"(lane));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&sbar[stage])), "r"(lane));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                       "d"(sa), "d"(sb), "r"(rb)
                       : "memory");
        }
        mbar_wait(&sbar[stage], (uses >> stage) & 1u);
        uses ^= 1u << stage;
        if (lane == 0) {
          double ta = 0, tb = 0;
          for (int r = 0; r < NC; ++r) {
            ta += part[stage][r][0];
            tb += part[stage][r][1];
          }
          bc[0] = ta / (tb + 1.0);
        }
      }
      __syncthreads();
      acc += bc[0] * 1e-9;
    } else if (mode == 1) {  // publish
      const int k = it & 1;
      const uint32_t gbytes = (uint32_t)(((zr > 0) + (zr < NC - 1)) * N * N * 8);
      double* Gs = Gx[lp];
      Gs[pi] = acc;
      if (t == 0) mbar_arrive_expect_tx(&gbar[k], gbytes);
      if (lp == 0 && zr > 0) {
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&gh[k][1][pi])), "r"(zr - 1));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&gbar[k])), "r"(zr - 1));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(acc),
                     "r"(rb)
                     : "memory");
      }
      if (lp == 1 && zr < NC - 1) {
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&gh[k][0][pi])), "r"(zr + 1));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&gbar[k])), "r"(zr + 1));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(acc),
                     "r"(rb)
                     : "memory");
      }
      if (wid == 0) mbar_wait(&gbar[k], (guses >> k) & 1u);
      guses ^= 1u << k;
      __syncthreads();
      acc += gh[k][lp][pi] * 1e-9 + Gx[1 - lp][pi] * 1e-9;
    } else if (mode == 2) {  // cluster barrier
      cl.sync();
      acc += 1e-9;
    } else {  // CTA barrier
      __syncthreads();
      acc += 1e-9;
    }
  }
  long long t1 = clock64();
  // publish pairs need one more round so no CTA exits with pushes in flight
  cl.sync();
  out[zr * THR + t] = acc;
  if (t == 0) cyc[zr] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * NC * THR);
  cudaMallocManaged(&cyc, sizeof(long long) * NC);
  const char* names[] = {"csum (st.async cluster reduce)", "publish (st.async planes)", "cluster.sync", "__syncthreads"};
  for (int mode = 0; mode < 4; ++mode) {
    const int iters = 2000;
    k_bench<<<NC, THR>>>(mode, iters, out, cyc);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_bench<<<NC, THR>>>(mode, iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.1f ns/op  %7.0f cycles/op (%s)\n", names[mode], ms * 1e6 / iters, (double)cyc[0] / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

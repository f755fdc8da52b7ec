// coop.cuh -- a whole smoothing phase of a small level in ONE cooperative launch.
//
// smooth(l, steps) (multigrid.hpp:641-690, called from v_cycle :486/:496) is
// 2 x steps GS-RB half-sweeps.  On the levels below the finest the
// half-sweeps are latency-bound (level 4 of a 256^3 mesh: 512 blocks, ~7 us
// per launch, of which the data movement is < 2 us), so k_gs_coop runs all of
// them in one launch with a grid barrier between half-sweeps.  One CTA per
// lean block, all co-resident (cooperative launch): the block's two colour
// halves stay in shared memory for the whole phase, each half-sweep only
// gathers the other colour's face layers of the six neighbours (L2), and the
// colour just computed is written to global memory (for the neighbours) and
// to the shared copy (for this block's next half-sweep).  The arithmetic per
// cell is k_gs_stream's / k_gs_cut's (same operation order), so the result is
// bit-identical to the launch-per-half-sweep path.
//
// Shared memory: per colour X one Stream3 region [X half | z, y, x face
// layers] (stream.cuh), so the column routine of k_gs_stream reads it
// unchanged; the region of colour c holds that colour's half, refreshed in place.
#pragma once
#include "stream.cuh"

namespace pmgdev {

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid-wide barrier of a cooperative launch: bar[0] counts arrivals, bar[1]
// is the generation.  The last arriver resets the count before it releases the
// new generation, so the state is ready for the next barrier / launch.  The
// acquire load (LDG.STRONG.GPU + L1 invalidate) makes the other CTAs' stores
// visible to this CTA's plain loads and cp.async reads after the barrier.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = ld_acquire_gpu(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nblk - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      st_release_gpu(bar + 1, g0 + 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == g0) __nanosleep(20);
    }
    (void)ld_acquire_gpu(bar + 1);
  }
  __syncthreads();
}

// the k_gs_cut tables of both colours with per-slot row ranges
struct CutTabs {
  const int32_t* ent[2];
  const double* gbc[2];
  const double* coef[2];
  const int32_t* off[2];  // nb + 1 per colour: rows of slot s are [off[s], off[s+1])
};

constexpr int kCoopThreads = 256;
constexpr int kCoopMaxBlocks = 1024;
constexpr bool kCoopEnabled = false;  // levels above this stream (k_gs_stream)

template <int N>
struct Coop3 {
  using S = Stream3<N, kCoopThreads>;
  static constexpr int REG = S::ORQ;  // X half + face layers (no row_of page: skind comes from global)
  static constexpr int SMEM = 2 * REG;  // doubles
};

// nhalf half-sweeps, colour h & 1 in half-sweep h; grid = n = plan entries
// (lean, not all-inside blocks), every CTA resident.
template <int N>
__global__ void __launch_bounds__(kCoopThreads, 4) k_gs_coop(LevelView L, const int4* __restrict__ plan, int n,
                                                            int nhalf, CutTabs cut, unsigned* __restrict__ bar) {
  using S = Stream3<N, kCoopThreads>;
  constexpr int NI = N * N * N, REG = Coop3<N>::REG;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full;
  const int t = threadIdx.x;
  const BlockPlan P = load_plan(plan, blockIdx.x);
  const int slot = P.slot(), kind = P.kind(), pmask = P.phys();
  if (t == 0) {
    mbar_init(&full, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const double h2 = L.h2;
  const int gbase = gs_column_base<N, kCoopThreads>(t);
  const double* blk = L.phi + (size_t)slot * NI;
  for (int h = 0; h < nhalf; ++h) {
    const int c = h & 1, X = 1 - c;
    double* st = sm + X * REG;  // colour X half + the halo layers of this half-sweep
    double* own = sm + c * REG;  // colour c half
    double g[S::PER];
    {
      const double* gs = L.rhs + (size_t)slot * NI + (size_t)c * S::H + gbase;
#pragma unroll
      for (int q = 0; q < S::PER; ++q) g[q] = gs[q * S::FH];
    }
    if (t == 0) {
      // the neighbours' stores (before the grid barrier) are read by the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const int zm = P.nbr(4), zp = P.nbr(5);
      const double* ownc = blk + (size_t)c * S::H;
      const double* s0 = zm >= 0 ? L.phi + (size_t)zm * NI + (size_t)X * S::H + (N - 1) * S::FH : ownc;
      const double* s1 = zp >= 0 ? L.phi + (size_t)zp * NI + (size_t)X * S::H : ownc + (N - 1) * S::FH;
      mbar_arrive_expect_tx(&full, (uint32_t)(2 * S::FH + (h == 0 ? 2 * S::H : 0)) * 8u);
      if (h == 0) {  // both halves, once
        bulk_g2s(sm, blk, S::H * 8, &full);
        bulk_g2s(sm + REG, blk + S::H, S::H * 8, &full);
      }
      bulk_g2s(st + S::OZ, s0, S::FH * 8, &full);
      bulk_g2s(st + S::OZ + S::FH, s1, S::FH * 8, &full);
    }
    gs_issue_async<N, kCoopThreads, false>(L, P, c, st, t);
    cp_async_commit();
    mbar_wait(&full, (uint32_t)(h & 1));
    cp_async_wait<0>();
    __syncthreads();
    if (pmask) {  // block-uniform branch
      gs_phys_faces<N>(L, slot, pmask, c, st, t, kCoopThreads);
      __syncthreads();
    }
    gs_stream_column<N, kCoopThreads, true>(L, st, c, kind, h2, slot, g, t, P.srow(), own);
    if (kind == KIND_IFACE) {  // this block's cut rows (k_gs_cut)
      const int q1 = cut.off[c][slot + 1];
      for (int q = cut.off[c][slot] + t; q < q1; q += kCoopThreads) {
        double v;
        const int a = gs_cut_row<3>(L, cut.ent[c], cut.gbc[c], cut.coef[c], q, v);
        L.phi[a] = v;
        own[a - slot * NI - c * S::H] = v;
      }
    }
    if (h + 1 < nhalf) grid_sync(bar, (unsigned)n);
  }
}

}  // namespace pmgdev

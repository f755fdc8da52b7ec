// stream.cuh -- persistent, TMA-pipelined streaming kernels for lean 3D blocks.
//
// The GS-RB half-sweep of a block needs its other-colour half of phi (N^3/2
// doubles, contiguous in the colour-split layout), its own-colour half of g
// (contiguous) and one face layer per side.  A CTA owns every G-th block of
// the lean list (G = grid size, one or two CTAs per SM) and keeps S blocks in
// flight: one elected warp issues 1D bulk copies (cp.async.bulk, the TMA
// engine) of the two halves and of the z / y face layers into an S-stage
// shared-memory ring, completing on a per-stage mbarrier; the strided x-face
// values are gathered by the threads one block ahead.  The compute of block b
// therefore overlaps the DRAM streaming of blocks b+1 .. b+S-1 without
// holding any of it in registers.
#pragma once
#include "tiles.cuh"
#include "cells.cuh"

namespace pmgdev {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch into L2 (bytes % 16 == 0)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}

// ------------------------------------------------------------------ per-block plan
// Host-built, one int4 pair per lean block of a level (capi.cu upload_stencils):
// a = {slot, kind | physical-face mask << 8 | srow << 14, nbr(-x), nbr(+x)},
// b = {nbr(-y), nbr(+y), nbr(-z), nbr(+z)}   (-1 = physical face; -2 - p =
// coarse-fine face whose cfc page is p, only in the plans of the CF kernels).
struct BlockPlan {
  int4 a, b;
  __device__ __forceinline__ int slot() const { return a.x; }
  __device__ __forceinline__ int kind() const { return a.y & 0xff; }
  __device__ __forceinline__ int phys() const { return (a.y >> 8) & 63; }
  __device__ __forceinline__ int srow() const { return a.y >> 14; }
  __device__ __forceinline__ int nbr(int d) const {
    return d == 0 ? a.z : d == 1 ? a.w : d == 2 ? b.x : d == 3 ? b.y : d == 4 ? b.z : b.w;
  }
};
__device__ __forceinline__ BlockPlan load_plan(const int4* plan, int p) {
  BlockPlan P;
  P.a = __ldg(plan + 2 * p);
  P.b = __ldg(plan + 2 * p + 1);
  return P;
}

// Plan entries of a persistent streaming kernel, staged through a small
// shared-memory ring: threads 0-1 load the entry of local block it + PK into
// registers at iteration it and store it into the ring one iteration later,
// so no warp ever waits on a plan load (it was the top stall of the
// streaming loops).  The entry of block b is read at the end of iteration
// b - S (issue time), after at least one barrier since its store (PK > S).
template <int S>
struct PlanRing {
  static constexpr int PK = S + 2, PR = PK + 1;
  int4* ring;  // [PR][2] in shared memory
  int rev_n = 0;  // > 0: the plan is walked backwards (entry n - 1 - p), see pidx
  int4 held;
  // plan entry of local block b (the CTA's b-th: p = blockIdx.x + b G)
  __device__ __forceinline__ int pidx(int b, int G) const {
    const int p = (int)blockIdx.x + b * G;
    return rev_n ? rev_n - 1 - p : p;
  }
  __device__ __forceinline__ void init(const int4* __restrict__ plan, int nmine, int G) {  // caller syncs
    const int nb = nmine < PK ? nmine : PK;
    for (int q = threadIdx.x; q < 2 * nb; q += blockDim.x)
      ring[((q >> 1) % PR) * 2 + (q & 1)] = __ldg(plan + 2 * pidx(q >> 1, G) + (q & 1));
  }
  __device__ __forceinline__ void advance(const int4* __restrict__ plan, int it, int nmine, int G) {
    if (threadIdx.x < 2) {
      if (it >= 1 && it - 1 + PK < nmine) ring[((it - 1 + PK) % PR) * 2 + threadIdx.x] = held;
      if (it + PK < nmine) held = __ldg(plan + 2 * pidx(it + PK, G) + threadIdx.x);
    }
  }
  __device__ __forceinline__ BlockPlan get(int b) const {
    BlockPlan P;
    P.a = ring[(b % PR) * 2];
    P.b = ring[(b % PR) * 2 + 1];
    return P;
  }
};

// ------------------------------------------------------------------ stage layout
template <int N, int TH = 0>
struct Stream3 {
  static constexpr int HN = N / 2;
  static constexpr int H = N * N * N / 2;
  static constexpr int FH = N * HN;  // z / y face layer of one colour
  static constexpr int THR = TH ? TH : (H < 512 ? H : 512);
  static constexpr int PER = H / THR;
  // doubles per stage: X half, hz[2], hy[2], hx[2] (x rows indexed k*N+j),
  // then H int32 row_of entries of an interface block.  g is not staged: each
  // thread loads its own g values into registers one block ahead.
  static constexpr int OX = 0, OZ = H, OY = OZ + 2 * FH, OXF = OY + 2 * FH;
  static constexpr int ORQ = OXF + 2 * N * N;  // in doubles; H int32 = H/2 doubles
  static constexpr int STAGE = ORQ + H / 2;
  static constexpr uint32_t TX_BYTES = (uint32_t)(H + 2 * FH) * 8u;  // bulk part
  static constexpr int YC = N * HN;  // 16-B chunks of the two y layers (2 sides x N rows x HN/2)
};

// Bulk copies of one block into a stage (one elected thread): the two
// halves and the z layers (physical faces copy the block's own colour-c
// layer; it becomes 2 bc - f1 / f1 after the wait).
template <int N>
__device__ __forceinline__ void gs_issue(const LevelView& L, const BlockPlan& P, int c, double* st,
                                         uint64_t* bar) {
  using S = Stream3<N>;
  constexpr int NI = N * N * N;
  const int X = 1 - c;
  const int slot = P.slot();
  const double* own = L.phi + (size_t)slot * NI + (size_t)c * S::H;
  mbar_arrive_expect_tx(bar, S::TX_BYTES);
  bulk_g2s(st + S::OX, L.phi + (size_t)slot * NI + (size_t)X * S::H, S::H * 8, bar);
  const int zm = P.nbr(4), zp = P.nbr(5);
  const double* s0 = zm >= 0 ? L.phi + (size_t)zm * NI + (size_t)X * S::H + (N - 1) * S::FH : own;
  const double* s1 = zp >= 0 ? L.phi + (size_t)zp * NI + (size_t)X * S::H : own + (N - 1) * S::FH;
  bulk_g2s(st + S::OZ, s0, S::FH * 8, bar);
  bulk_g2s(st + S::OZ + S::FH, s1, S::FH * 8, bar);
}

// x-face row u (0 .. N*N-1): side = u / (N*N/2); the row (j,k) holds a
// colour-c cell on that face.
template <int N>
__device__ __forceinline__ void xface_of(int c, int u, int& side, int& j, int& k) {
  side = u / (N * N / 2);
  const int r = u % (N * N / 2);
  k = r / (N / 2);
  j = 2 * (r % (N / 2)) + ((c + k + side) & 1);
}

// Thread-issued async copies of one block: the strided x-face values (the
// neighbour's X value, or the own value on a physical face) and, for an
// interface block, this thread's row_of entries.
template <int N, int TH, bool ROWQ = true>
__device__ __forceinline__ void gs_issue_async(const LevelView& L, const BlockPlan& P, int c, double* st, int t) {
  using S = Stream3<N, TH>;
  constexpr int NI = N * N * N;
  for (int u = t; u < N * N; u += S::THR) {
    int side, j, k;
    xface_of<N>(c, u, side, j, k);
    const int ns = P.nbr(side);
    const double* src;
    if (ns >= 0)  // -x: neighbour cell (N-1,j,k); +x: (0,j,k); both colour X
      src = L.phi + (size_t)ns * NI + (size_t)(1 - c) * S::H + (size_t)(side ? 0 : S::HN - 1) + S::HN * (j + N * k);
    else
      src = L.phi + (size_t)P.slot() * NI + (size_t)c * S::H + (size_t)(side ? S::HN - 1 : 0) + S::HN * (j + N * k);
    cp_async8(st + S::OXF + side * N * N + k * N + j, src);
  }
  // y layers: 16-B chunks of the x-rows j = N-1 / 0 (neighbour) or own row,
  // issued by the last threads (the first ones carry the x faces)
  for (int u = S::THR - 1 - t; u < S::YC; u += S::THR) {
    constexpr int CR = S::HN / 2;  // chunks per row
    const int side = u / (N * CR), k = (u / CR) % N, ch = u % CR;
    const int ns = P.nbr(2 + side);
    const double* src;
    if (ns >= 0)
      src = L.phi + (size_t)ns * NI + (size_t)(1 - c) * S::H + (size_t)k * S::FH + (side ? 0 : (N - 1) * S::HN);
    else
      src = L.phi + (size_t)P.slot() * NI + (size_t)c * S::H + (size_t)k * S::FH + (side ? (N - 1) * S::HN : 0);
    cp_async16(st + S::OY + side * S::FH + k * S::HN + 2 * ch, src + 2 * ch);
  }
  if (ROWQ && P.kind() == KIND_IFACE) {  // this block's row_of page (colour c), 16-B chunks
    const int32_t* rof = L.row_of + (size_t)P.srow() * NI + (size_t)c * S::H;
    int32_t* rq = reinterpret_cast<int32_t*>(st + S::ORQ);
    for (int q = t; q < S::H / 4; q += S::THR) cp_async16(rq + 4 * q, rof + 4 * q);
  }
}

// CF kernels: the colour-c halves of the cfc pages of the block's coarse-fine
// faces (16-B chunks) into the stage's extra 6 FH doubles; returns their mask.
template <int N, int TH>
__device__ __forceinline__ void cf_issue_async(const LevelView& L, const BlockPlan& P, int c, double* dst, int t) {
  using S = Stream3<N, TH>;
  constexpr int CH = S::FH / 2;
  for (int u = t; u < 6 * CH; u += S::THR) {
    const int f = u / CH, ch = u % CH;
    const int code = P.nbr(f);
    if (code <= -2)
      cp_async16(dst + f * S::FH + 2 * ch, L.cfc + (size_t)(-2 - code) * (2 * S::FH) + (size_t)c * S::FH + 2 * ch);
  }
}
__device__ __forceinline__ int cf_mask_of(const BlockPlan& P) {
  int m = 0;
#pragma unroll
  for (int f = 0; f < 6; ++f) m |= (P.nbr(f) <= -2 ? 1 : 0) << f;
  return m;
}

// Physical faces: the staged own-colour values become ghosts 2 bc - f1
// (Dirichlet) or stay f1 (Neumann), mesh.hpp:538-552.
// CF: faces in cfmask are coarse-fine -- the staged own value f1 becomes
// 1/2 c + 3/4 f1 - 1/4 f2 (mesh.hpp:500-535) with c from the staged cfc page
// (at S::STAGE + dir * FH) and f2 the other-colour value one cell inward.
template <int N, bool CF = false>
__device__ __forceinline__ void gs_phys_faces(const LevelView& L, int slot, int pmask, int c, double* st, int t0,
                                              int nt, int cfmask = 0) {
  using S = Stream3<N>;
  constexpr int NX = N * N;  // x rows (two sides)
  for (int q = t0; q < NX + 4 * S::FH; q += nt) {
    int dir, i, tj;
    int ci, e2;  // CF: position in the face's cfc page, entry of f2 in the staged half
    double* h;
    if (q < NX) {
      int side, j, k;
      xface_of<N>(c, q, side, j, k);
      dir = side;
      i = side ? N - 1 : 0;
      tj = j + N * k;
      h = st + S::OXF + side * N * N + k * N + j;
      ci = tj >> 1;
      e2 = ((side ? N - 2 : 1) + N * tj) >> 1;
    } else {
      const int qq = q - NX;
      const int f = qq / S::FH, r = qq % S::FH;  // f: 0 -y, 1 +y, 2 -z, 3 +z
      dir = f < 2 ? 2 + f : 4 + (f - 2);
      const int m = r % S::HN, a = r / S::HN;  // a = k on y faces, j on z faces
      if (f < 2) {
        const int j = f ? N - 1 : 0;
        i = 2 * m + ((c + j + a) & 1);
        e2 = m + S::HN * ((f ? N - 2 : 1) + N * a);
      } else {
        const int k = f == 3 ? N - 1 : 0;
        i = 2 * m + ((c + a + k) & 1);
        e2 = m + S::HN * (a + N * (f == 3 ? N - 2 : 1));
      }
      tj = i + N * a;
      ci = r;
      h = st + (f < 2 ? S::OY + f * S::FH : S::OZ + (f - 2) * S::FH) + r;
    }
    if (CF && ((cfmask >> dir) & 1)) {
      const double cv = st[S::STAGE + dir * S::FH + ci];
      const double f1 = *h, f2 = st[S::OX + e2];
      *h = 0.5 * cv + 0.75 * f1 - 0.25 * f2;
      continue;
    }
    if (!((pmask >> dir) & 1) || L.bctype[dir] == 1) continue;
    double bcv = 0.0;
    if (!L.bczero) {
      const int bo = L.bcoff[slot * 6 + dir];
      if (bo >= 0) bcv = L.bcval[bo + tj];
    }
    *h = 2.0 * bcv - *h;
  }
}

// Column mapping of the GS half-sweep: thread t owns the PER consecutive
// z-planes k = kq*PER + q of entry column (m, j), so the other-colour values at
// its own entries (the same-entry x neighbour and, one plane up / down, the z
// neighbours) are loaded once as a column of PER + 2 values: 4.5 shared-memory
// loads per cell instead of 6.  Warps still read runs of consecutive doubles.
template <int N, int TH>
__device__ __forceinline__ int gs_column_base(int t) {
  using S = Stream3<N, TH>;
  const int m = t % S::HN, j = (t / S::HN) % N, kq = t / S::FH;
  return m + S::HN * j + S::FH * S::PER * kq;
}
// SKG: the special-row kinds of an interface block come from the global
// skind page (int8, srow) instead of the row_of page staged at ORQ.
template <int N, int TH, bool SKG = false>
__device__ __forceinline__ void gs_stream_column(const LevelView& L, const double* __restrict__ st, int c, int kind,
                                                 double h2, int slot, const double* gcur, int t, int srow = 0,
                                                 double* sdst = nullptr) {
  using S = Stream3<N, TH>;
  constexpr int NI = N * N * N, HN = S::HN, FH = S::FH, PER = S::PER, KS = S::THR / S::FH;
  static_assert(PER * KS == N, "columns cover the block");
  const int m = t % HN, j = (t / HN) % N, kq = t / FH;
  const int eb = m + HN * j + FH * PER * kq;  // entry of q = 0
  const int o0 = (c + j + kq * PER) & 1;       // x offset of q = 0; flips with q
  const int XB = S::OX + eb;
  // the other x neighbour for o = 0 (x-: e - 1 or the -x face) and o = 1 (x+)
  const int bx0 = m > 0 ? XB - 1 : S::OXF + kq * PER * N + j, sx0 = m > 0 ? FH : N;
  const int bx1 = m < HN - 1 ? XB + 1 : S::OXF + N * N + kq * PER * N + j, sx1 = m < HN - 1 ? FH : N;
  const int bym = j > 0 ? XB - HN : S::OY + kq * PER * HN + m, sym = j > 0 ? FH : HN;
  const int byp = j < N - 1 ? XB + HN : S::OY + FH + kq * PER * HN + m, syp = j < N - 1 ? FH : HN;
  double xc[PER + 2];
  xc[0] = st[kq > 0 ? XB - FH : S::OZ + j * HN + m];
#pragma unroll
  for (int q = 0; q < PER; ++q) xc[q + 1] = st[XB + q * FH];
  xc[PER + 1] = st[kq < KS - 1 ? XB + PER * FH : S::OZ + FH + j * HN + m];
  double* __restrict__ dst = L.phi + (size_t)slot * NI + (size_t)c * S::H + eb;
  auto nbrs = [&](int q, double& xm, double& xp, double& ym, double& yp) {
    const int o = o0 ^ (q & 1);
    const double xo = st[o ? bx1 + q * sx1 : bx0 + q * sx0];
    xm = o ? xc[q + 1] : xo;
    xp = o ? xo : xc[q + 1];
    ym = st[bym + q * sym];
    yp = st[byp + q * syp];
  };
  if (kind == KIND_UNIFORM) {  // multigrid.hpp:651-653: (sum of 6 - h^2 g) / 6.0
    double sv[PER], v[PER];
    bool ok = true;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      double xm, xp, ym, yp;
      nbrs(q, xm, xp, ym, yp);
      sv[q] = xm + xp + ym + yp + xc[q] + xc[q + 2] - h2 * gcur[q];
      v[q] = div6_fast(sv[q]);
      ok = ok && div6_in_range(sv[q]);
    }
    if (!ok) {
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] = div6_slow(sv[q]);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) dst[q * FH] = v[q];
    if (sdst) {  // k_gs_coop keeps the block's colour-c half in shared memory
#pragma unroll
      for (int q = 0; q < PER; ++q) sdst[eb + q * FH] = v[q];
    }
  } else {  // interface block (multigrid.hpp:665-684)
    const int32_t* rq = reinterpret_cast<const int32_t*>(st + S::ORQ);
    const int8_t* skg = L.skind + (size_t)srow * NI + (size_t)c * S::H;
    int uni[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) uni[q] = SKG ? (skg[eb + q * FH] == 0 ? -1 : 0) : rq[eb + q * FH];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int r = uni[q];
      double xm, xp, ym, yp;
      nbrs(q, xm, xp, ym, yp);
      if (r < 0) {  // uniform row (:667-672)
        double sv = -h2 * gcur[q];
        sv += xm;
        sv += xp;
        sv += ym;
        sv += yp;
        sv += xc[q];
        sv += xc[q + 2];
        const double v = -sv * (-1.0 / 6.0);
        dst[q * FH] = v;
        if (sdst) sdst[eb + q * FH] = v;
      }  // special rows: cut rows by k_gs_cut, inside rows keep their pin
    }
  }
}

// GS-RB half-sweep of the lean 3D blocks (UNIFORM / IFACE blocks without
// coarse-fine faces, in plan order).  Special rows are left alone: k_gs_cut
// updates the cut rows afterwards, inside rows keep their pin.
// rev: walk the plan backwards.  Alternating the direction between the two
// half-sweeps makes each sweep start on the blocks the previous one wrote
// last -- the ones still in the 126 MB L2.
// CF: the plan may hold blocks with coarse-fine faces (L.cfc set, built).
template <int N, int S_STAGES, int MINB, int TH, bool CF = false>
__global__ void __launch_bounds__(Stream3<N, TH>::THR, MINB) k_gs_stream(LevelView L, int parity,
                                                                        const double* __restrict__ phi_b,
                                                                        const int4* __restrict__ plan, int n,
                                                                        int rev) {
  // PDL: barrier setup and the (static) plan entries happen before waiting
  // for the previous kernel, overlapping its drain
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  using S = Stream3<N, TH>;
  constexpr int NI = N * N * N;
  constexpr int STAGE = S::STAGE + (CF ? 6 * S::FH : 0);
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[S_STAGES];
  __shared__ int meta[S_STAGES][CF ? 3 : 2];
  const int c = parity;
  const int t = threadIdx.x;
  const int G = gridDim.x;
  const int nmine = (int)blockIdx.x < n ? (n - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (nmine == 0) return;
  __shared__ int4 pring[PlanRing<S_STAGES>::PR * 2];
  PlanRing<S_STAGES> R{pring, rev ? n : 0};
  if (t == 0) {
    for (int s = 0; s < S_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  R.init(plan, nmine, G);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  for (int s = 0; s < S_STAGES; ++s) {
    if (s < nmine) {
      const BlockPlan P = R.get(s);
      if (t == 0) gs_issue<N>(L, P, c, sm + s * STAGE, &full[s]);
      if (t == 0) meta[s][0] = P.slot(), meta[s][1] = P.a.y;
      gs_issue_async<N, TH>(L, P, c, sm + s * STAGE, t);
      if (CF) {
        if (t == 0) meta[s][CF ? 2 : 0] = cf_mask_of(P);
        cf_issue_async<N, TH>(L, P, c, sm + s * STAGE + S::STAGE, t);
      }
    }
    cp_async_commit();
  }
  const double h2 = L.h2;
  // S_STAGES == 1 only with at most one block per CTA (the launcher's
  // grid >= n): g of block it+1 is read through meta[] one iteration ahead
  static_assert(S_STAGES >= 1, "stages");
  __syncthreads();  // meta of the first stages
  double gcur[S::PER], gnext[S::PER];
  // this thread's entries: e(q) = gbase + q * FH (column order)
  const int gbase = gs_column_base<N, TH>(t);
  constexpr int gstep = S::FH;
  {
    const double* gsrc = L.rhs + (size_t)meta[0][0] * NI + (size_t)c * S::H + gbase;
#pragma unroll
    for (int q = 0; q < S::PER; ++q) gcur[q] = gsrc[q * gstep];
  }
  for (int it = 0; it < nmine; ++it) {
    const int s = it % S_STAGES;
    double* st = sm + s * STAGE;
    R.advance(plan, it, nmine, G);
    mbar_wait(&full[s], (uint32_t)((it / S_STAGES) & 1));
    cp_async_wait<S_STAGES - 1>();
    __syncthreads();
    const int slot = meta[s][0], flags = meta[s][1];
    const int kind = flags & 0xff, pmask = (flags >> 8) & 63;
    const int cfmask = CF ? meta[s][CF ? 2 : 0] : 0;
    if (S_STAGES > 1 && it + 1 < nmine) {  // this thread's g of the next block, in flight during this one
      const double* gsrc = L.rhs + (size_t)meta[(it + 1) % S_STAGES][0] * NI + (size_t)c * S::H + gbase;
#pragma unroll
      for (int q = 0; q < S::PER; ++q) gnext[q] = gsrc[q * gstep];
    }
    if (pmask | cfmask) {  // block-uniform branch
      gs_phys_faces<N, CF>(L, slot, pmask, c, st, t, blockDim.x, cfmask);
      __syncthreads();
    }
    gs_stream_column<N, TH>(L, st, c, kind, h2, slot, gcur, t);
    __syncthreads();  // stage s consumed
    if (it + S_STAGES < nmine) {
      const BlockPlan pf = R.get(it + S_STAGES);
      if (t == 0) gs_issue<N>(L, pf, c, st, &full[s]);
      if (t == 0) meta[s][0] = pf.slot(), meta[s][1] = pf.a.y;
      gs_issue_async<N, TH>(L, pf, c, st, t);
      if (CF) {
        if (t == 0) meta[s][CF ? 2 : 0] = cf_mask_of(pf);
        cf_issue_async<N, TH>(L, pf, c, st + S::STAGE, t);
      }
    }
    cp_async_commit();
    if (S_STAGES > 1) {
#pragma unroll
      for (int q = 0; q < S::PER; ++q) gcur[q] = gnext[q];
    }
  }
}

// ------------------------------------------------------------------ fused residual + restriction
// residual_level(l) + restrict_level(l) (multigrid.hpp:374-398,510-517,
// 697-722) for a level without coarse-fine faces: one stage holds both colour
// halves of a block's phi and, indexed by the colour of the block's own
// boundary cell, the neighbour (or physical-ghost) value next to every face
// cell.  Thread t owns parent cell (ii,jj,kk) of the block's octant and its
// 2x2x2 children; g comes straight from global memory (coalesced, issued
// before the stage wait).
template <int N>
struct RStream3 {
  static constexpr int HN = N / 2;
  static constexpr int H = N * N * N / 2;
  static constexpr int FH = N * HN;
  static constexpr int THR = HN * HN * HN;  // parents per block
  // doubles: P[2][H], g[2][H], hz[2 side][2 colour][FH], hy[2][2][FH], hx[2][N*N]
  static constexpr int OP = 0, OG = 2 * H, OZ = 4 * H, OY = OZ + 4 * FH, OXF = OY + 4 * FH;
  static constexpr int STAGE = OXF + 2 * N * N;
  static constexpr uint32_t TX_BYTES = (uint32_t)(4 * H + 4 * FH) * 8u;
  static constexpr int YC = 2 * 2 * N * (HN / 2);  // 16-B chunks of the y layers
};

template <int N>
__device__ __forceinline__ void rs_issue(const LevelView& L, const BlockPlan& P, double* st, uint64_t* bar) {
  using S = RStream3<N>;
  constexpr int NI = N * N * N;
  const int slot = P.slot();
  const double* own = L.phi + (size_t)slot * NI;
  mbar_arrive_expect_tx(bar, S::TX_BYTES);
  bulk_g2s(st + S::OP, own, 2 * S::H * 8, bar);
  bulk_g2s(st + S::OG, L.rhs + (size_t)slot * NI, 2 * S::H * 8, bar);
  for (int side = 0; side < 2; ++side) {
    const int ns = P.nbr(4 + side);
    for (int cc = 0; cc < 2; ++cc) {
      const double* src = ns >= 0 ? L.phi + (size_t)ns * NI + (size_t)(1 - cc) * S::H + (side ? 0 : (N - 1) * S::FH)
                                  : own + (size_t)cc * S::H + (side ? (N - 1) * S::FH : 0);
      bulk_g2s(st + S::OZ + (side * 2 + cc) * S::FH, src, S::FH * 8, bar);
    }
  }
}

template <int N, class S = RStream3<N>>
__device__ __forceinline__ void rs_issue_async(const LevelView& L, const BlockPlan& P, double* st) {
  constexpr int NI = N * N * N;
  const int t = threadIdx.x;
  const int slot = P.slot();
  for (int u = t; u < 2 * N * N; u += S::THR) {  // x faces: one value per row (j,k)
    const int side = u / (N * N), r = u % (N * N), k = r / N, j = r % N;
    const int ib = side ? N - 1 : 0;
    const int cb = (ib + j + k) & 1;  // colour of the block's own boundary cell
    const int ns = P.nbr(side);
    const double* src = ns >= 0
                            ? L.phi + (size_t)ns * NI + (size_t)(1 - cb) * S::H + (side ? 0 : S::HN - 1) + S::HN * (j + N * k)
                            : L.phi + (size_t)slot * NI + (size_t)cb * S::H + (ib >> 1) + S::HN * (j + N * k);
    cp_async8(st + S::OXF + side * N * N + k * N + j, src);
  }
  for (int u = t; u < S::YC; u += S::THR) {  // y layers, 16-B chunks
    constexpr int CR = S::HN / 2;
    const int side = u / (2 * N * CR), cc = (u / (N * CR)) % 2, k = (u / CR) % N, ch = u % CR;
    const int ns = P.nbr(2 + side);
    const double* src = ns >= 0 ? L.phi + (size_t)ns * NI + (size_t)(1 - cc) * S::H + (size_t)k * S::FH +
                                      (side ? 0 : (N - 1) * S::HN)
                                : L.phi + (size_t)slot * NI + (size_t)cc * S::H + (size_t)k * S::FH +
                                      (side ? (N - 1) * S::HN : 0);
    cp_async16(st + S::OY + (side * 2 + cc) * S::FH + k * S::HN + 2 * ch, src + 2 * ch);
  }
}

// CF: faces in cfmask are coarse-fine -- the staged own value f1 becomes
// 1/2 c + 3/4 f1 - 1/4 f2 (mesh.hpp:500-535), c from the cfc page staged at
// S::STAGE + dir * 2 FH, f2 the own other-colour value one cell inward.
template <int N, class S = RStream3<N>, bool CF = false>
__device__ __forceinline__ void rs_phys_faces(const LevelView& L, int slot, int pmask, double* st, int t0 = -1,
                                              int nt = 0, int cfmask = 0) {
  if (t0 < 0) t0 = threadIdx.x, nt = blockDim.x;
  for (int q = t0; q < 2 * N * N + 8 * S::FH; q += nt) {
    int dir, tj;
    int cb = 0, e2 = 0;  // CF: colour of the block's own face cell, entry of f2
    double* h;
    if (q < 2 * N * N) {
      const int side = q / (N * N), r = q % (N * N);
      dir = side;
      tj = r % N + N * (r / N);  // j + N k
      h = st + S::OXF + q;
      cb = ((side ? N - 1 : 0) + r % N + r / N) & 1;
      e2 = ((side ? N - 2 : 1) + N * tj) >> 1;
    } else {
      const int qq = q - 2 * N * N;
      const int f = qq / (2 * S::FH), cc = (qq / S::FH) % 2, r = qq % S::FH;  // f: -y +y -z +z
      dir = 2 + f;
      const int m = r % S::HN, a = r / S::HN;
      const int side = f & 1;
      cb = cc;
      if (f < 2) {  // y face: a = k
        const int jb = side ? N - 1 : 0;
        tj = 2 * m + ((cc + jb + a) & 1) + N * a;
        h = st + S::OY + (side * 2 + cc) * S::FH + r;
        e2 = m + S::HN * ((side ? N - 2 : 1) + N * a);
      } else {  // z face: a = j
        const int kb = side ? N - 1 : 0;
        tj = 2 * m + ((cc + a + kb) & 1) + N * a;
        h = st + S::OZ + (side * 2 + cc) * S::FH + r;
        e2 = m + S::HN * (a + N * (side ? N - 2 : 1));
      }
    }
    if (CF && ((cfmask >> dir) & 1)) {
      const double cv = st[S::STAGE + dir * 2 * S::FH + cb * S::FH + (tj >> 1)];
      const double f1 = *h, f2 = st[S::OP + (1 - cb) * S::H + e2];
      *h = 0.5 * cv + 0.75 * f1 - 0.25 * f2;
      continue;
    }
    if (!((pmask >> dir) & 1) || L.bctype[dir] == 1) continue;
    double bcv = 0.0;
    if (!L.bczero) {
      const int bo = L.bcoff[slot * 6 + dir];
      if (bo >= 0) bcv = L.bcval[bo + tj];
    }
    *h = 2.0 * bcv - *h;
  }
}

// RECORD = false: fused residual + restriction into level l-1.
// RECORD = true: leaf-residual record of uniform blocks (record_leaf_residual,
// multigrid.hpp:529-562): per-block max |r|, sum r^2, count into `partial`,
// the last block folds them in slot order (record_finish).
template <int N, int S_STAGES, int MINB, int MODE>
__global__ void __launch_bounds__(RStream3<N>::THR, MINB) k_restrict_stream(LevelView Lf, LevelView Lp,
                                                                           const double* __restrict__ phi_b,
                                                                           const int4* __restrict__ plan, int n,
                                                                           Rec* __restrict__ partial, Rec* rec,
                                                                           unsigned int* counter) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: prologue before the wait
  constexpr bool RECORD = MODE == 1, FASM = MODE == 2;
  using S = RStream3<N>;
  constexpr int NI = N * N * N;
  constexpr int HN = S::HN;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[S_STAGES];
  __shared__ int meta[S_STAGES][2];
  __shared__ double red[72];
  __shared__ bool last;
  const int t = threadIdx.x;
  const int G = gridDim.x;
  const int nmine = (int)blockIdx.x < n ? (n - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (nmine == 0) return;
  __shared__ int4 pring[PlanRing<S_STAGES>::PR * 2];
  PlanRing<S_STAGES> R{pring};
  if (t == 0) {
    for (int s = 0; s < S_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  R.init(plan, nmine, G);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  for (int s = 0; s < S_STAGES; ++s) {
    if (s < nmine) {
      const BlockPlan P = R.get(s);
      if (t == 0) {
        rs_issue<N>(Lf, P, sm + s * S::STAGE, &full[s]);
        meta[s][0] = P.slot(), meta[s][1] = P.a.y;
      }
      rs_issue_async<N>(Lf, P, sm + s * S::STAGE);
    }
    cp_async_commit();
  }
  __syncthreads();  // meta of the first stages
  const int ii = t % HN, jj = (t / HN) % HN, kk = t / (HN * HN);
  const double w = Lf.w;
  double rmx = 0.0, rss = 0.0, rcnt = 0.0;  // RECORD: this CTA's running totals
  for (int it = 0; it < nmine; ++it) {
    const int s = it % S_STAGES;
    double* st = sm + s * S::STAGE;
    R.advance(plan, it, nmine, G);
    const int slot = meta[s][0], flags = meta[s][1];
    const int kind = flags & 0xff, pmask = (flags >> 8) & 63;
    // special-row kinds of the 8 children of an interface block (0 uniform,
    // 1 inside, 2 cut), leaf flag / parent slot and octant: loads in flight
    // across the wait
    int rr[8];
    if (kind == KIND_IFACE) {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const int dx = ch & 1, dy = (ch >> 1) & 1, dz = ch >> 2;
        const int e = ii + HN * ((2 * jj + dy) + N * (2 * kk + dz));
        rr[ch] = Lf.skind[(size_t)(flags >> 14) * NI + (size_t)((dx + dy + dz) & 1) * S::H + e];
      }
    }
    const int Pp = MODE == 0 ? Lf.parent[slot] : 0;
    const int cx = MODE == 0 ? Lf.coords[slot * 3] & 1 : 0, cy = MODE == 0 ? Lf.coords[slot * 3 + 1] & 1 : 0,
              cz = MODE == 0 ? Lf.coords[slot * 3 + 2] & 1 : 0;
    const bool leaf = MODE != 0 ? Lf.leaf[slot] != 0 : false;
    mbar_wait(&full[s], (uint32_t)((it / S_STAGES) & 1));
    cp_async_wait<S_STAGES - 1>();
    __syncthreads();
    if (pmask) {
      rs_phys_faces<N>(Lf, slot, pmask, st);
      __syncthreads();
    }
    const double* P0 = st + S::OP;
    // own values of the 8 children
    double f[8], g[8];
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const int dx = ch & 1, dy = (ch >> 1) & 1, dz = ch >> 2;
      const int e = ii + HN * ((2 * jj + dy) + N * (2 * kk + dz));
      f[ch] = P0[((dx + dy + dz) & 1) * S::H + e];
      g[ch] = st[S::OG + ((dx + dy + dz) & 1) * S::H + e];
    }
    double res[8], ap[8];
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const int dx = ch & 1, dy = (ch >> 1) & 1, dz = ch >> 2;
      const int j = 2 * jj + dy, k = 2 * kk + dz;
      const int cc = (dx + dy + dz) & 1;
      const int e = ii + HN * (j + N * k);
      const double* O = P0 + (1 - cc) * S::H;  // other colour
      double p[6];
      // x-, x+
      if (dx) p[0] = f[ch - 1];
      else p[0] = ii > 0 ? O[e - 1] : st[S::OXF + k * N + j];
      if (!dx) p[1] = f[ch + 1];
      else p[1] = ii < HN - 1 ? O[e + 1] : st[S::OXF + N * N + k * N + j];
      // y-, y+
      if (dy) p[2] = f[ch - 2];
      else p[2] = jj > 0 ? O[e - HN] : st[S::OY + (0 * 2 + cc) * S::FH + k * HN + ii];
      if (!dy) p[3] = f[ch + 2];
      else p[3] = jj < HN - 1 ? O[e + HN] : st[S::OY + (1 * 2 + cc) * S::FH + k * HN + ii];
      // z-, z+
      if (dz) p[4] = f[ch - 4];
      else p[4] = kk > 0 ? O[e - S::FH] : st[S::OZ + (0 * 2 + cc) * S::FH + j * HN + ii];
      if (!dz) p[5] = f[ch + 4];
      else p[5] = kk < HN - 1 ? O[e + S::FH] : st[S::OZ + (1 * 2 + cc) * S::FH + j * HN + ii];
      // uniform row (stencil.hpp:300-322); all-inside blocks have residual 0;
      // parents with a special child in an interface block are recomputed by
      // k_restrict_fix
      double sres = -2.0 * 3 * f[ch];
#pragma unroll
      for (int d = 0; d < 6; ++d) sres += p[d];
      ap[ch] = kind == KIND_ALL_INSIDE ? 0.0 : sres * w;  // L(phi), apply_block (stencil.hpp:300-322)
      // inside rows: residual 0; cut rows: parent recomputed by k_restrict_fix
      res[ch] = (kind == KIND_ALL_INSIDE || (kind == KIND_IFACE && rr[ch] == 1)) ? 0.0 : g[ch] - ap[ch];
    }
    if (FASM) {  // g = L(phi) + R(r) on non-leaf blocks, OLD <- PHI (multigrid.hpp:380-397)
      double* __restrict__ rhs = Lf.rhs + (size_t)slot * NI;
      double* __restrict__ old = Lf.old + (size_t)slot * NI;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const int dx = ch & 1, dy = (ch >> 1) & 1, dz = ch >> 2;
        const size_t a = (size_t)((dx + dy + dz) & 1) * S::H + ii + HN * ((2 * jj + dy) + N * (2 * kk + dz));
        // special rows of interface blocks: inside rows keep r (0 + r), cut rows by k_fas_fix
        if (!leaf && (kind != KIND_IFACE || rr[ch] == 0)) rhs[a] = ap[ch] + g[ch];
        old[a] = f[ch];
      }
    } else if (RECORD) {
      if (leaf && kind == KIND_UNIFORM) {
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          rmx = fmax(rmx, fabs(res[ch]));
          rss += res[ch] * res[ch];
        }
        rcnt += 8.0;
      } else if (leaf && kind == KIND_IFACE) {  // special rows: inside excluded, cut rows by k_record_cut
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          if (rr[ch] != 0) continue;
          rmx = fmax(rmx, fabs(res[ch]));
          rss += res[ch] * res[ch];
          rcnt += 1.0;
        }
      }
    } else {
    // sum of the children in x-fastest order (multigrid.hpp:706-721)
    double sr = 0.0, sf = 0.0;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      sr += res[ch];
      sf += f[ch];
    }
    const int pi = cx * HN + ii, pj = cy * HN + jj, pk = cz * HN + kk;
    const int pc = (pi + pj + pk) & 1, pe = (pi + N * (pj + N * pk)) >> 1;
    const size_t pa = (size_t)Pp * NI + (size_t)pc * S::H + pe;
    // parents with a cut child belong to k_restrict_fix (running concurrently);
    // pinned parents are re-pinned by k_pin_list afterwards
    bool cut = false;
    if (kind == KIND_IFACE) {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) cut = cut || rr[ch] == 2;
    }
    if (!cut) {
      Lp.phi[pa] = sf / 8.0;
      Lp.rhs[pa] = sr / 8.0;
    }
    }
    __syncthreads();  // stage s consumed
    if (it + S_STAGES < nmine) {
      const BlockPlan pf = R.get(it + S_STAGES);
      if (t == 0) {
        rs_issue<N>(Lf, pf, st, &full[s]);
        meta[s][0] = pf.slot(), meta[s][1] = pf.a.y;
      }
      rs_issue_async<N>(Lf, pf, st);
    }
    cp_async_commit();
  }
  if (RECORD)  // this CTA's totals, folded with the other partials by k_record_fold
    record_finish(Lf, partial, rec, nullptr, (int)blockIdx.x, rmx, rss, rcnt, red, &last);
}

// ------------------------------------------------------------------ residual streaming (column mapping)
// residual_level + restrict_level, the FAS right-hand side and the leaf
// record of lean 3D blocks.  Thread t owns the entry column (m, j) on the PER
// consecutive z-planes k = kq*PER + q, in BOTH colours: the cells (2m, j, k)
// and (2m+1, j, k).  The own values of both colours are loaded once as two
// columns, which also hold each cell's same-entry x neighbour and its z
// neighbours, so a cell costs 3 more shared loads (the other x neighbour and
// y-, y+) -- all runs of consecutive doubles across a warp.  The stage holds
// both phi halves (one bulk copy) and the face layers of both colours (the
// RStream3 layout without g); g goes straight from global memory into
// registers, one block ahead.  Per cell r = g - L(phi) with the reference's
// operation order (stencil.hpp:300-322, 336-358).
//   MODE 0: residual + restriction (multigrid.hpp:374-398, 697-722).  A
//           parent's 2x2x2 children are the x pair of two consecutive planes
//           of this thread and of the thread with j + 1 (lane + 8): one
//           shuffle exchange, then the fold in x-fastest order.  Parents with a
//           cut child belong to k_restrict_fix.
//   MODE 1: leaf-residual record (multigrid.hpp:529-562), per-CTA partials.
//   MODE 2: FAS g = L(phi) + r on non-leaf blocks, OLD <- PHI (:380-397).
template <int N, int TT = 512>
struct QStream3 {
  static constexpr int HN = N / 2;
  static constexpr int H = N * N * N / 2;
  static constexpr int FH = N * HN;
  static constexpr int THR = H < TT ? H : TT;
  static constexpr int PER = H / THR;
  static constexpr int KS = THR / FH;  // columns per (m, j): z-plane groups
  // doubles: P[2][H], hz[2 side][2 colour][FH], hy[2][2][FH], hx[2][N*N]
  static constexpr int OP = 0, OZ = 2 * H, OY = OZ + 4 * FH, OXF = OY + 4 * FH;
  static constexpr int STAGE = OXF + 2 * N * N;
  static constexpr uint32_t TX_BYTES = (uint32_t)(2 * H + 4 * FH) * 8u;
  static constexpr int YC = 2 * 2 * N * (HN / 2);  // 16-B chunks of the y layers
};

// CF: the cfc pages (both colours, 2 FH doubles) of the block's coarse-fine
// faces follow the stage at S::STAGE + dir * 2 FH.
template <int N, int TT, bool CF = false>
__device__ __forceinline__ void qs_issue(const LevelView& L, const BlockPlan& P, double* st, uint64_t* bar) {
  using S = QStream3<N, TT>;
  constexpr int NI = N * N * N;
  const double* own = L.phi + (size_t)P.slot() * NI;
  if (CF) {
    const int ncf = __popc((unsigned)cf_mask_of(P));
    mbar_arrive_expect_tx(bar, S::TX_BYTES + (uint32_t)ncf * 2u * S::FH * 8u);
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int code = P.nbr(f);
      if (code <= -2)
        bulk_g2s(st + S::STAGE + f * 2 * S::FH, L.cfc + (size_t)(-2 - code) * (2 * S::FH), 2 * S::FH * 8, bar);
    }
  } else {
    mbar_arrive_expect_tx(bar, S::TX_BYTES);
  }
  bulk_g2s(st + S::OP, own, 2 * S::H * 8, bar);
  for (int side = 0; side < 2; ++side) {
    const int ns = P.nbr(4 + side);
    for (int cc = 0; cc < 2; ++cc) {
      const double* src = ns >= 0 ? L.phi + (size_t)ns * NI + (size_t)(1 - cc) * S::H + (side ? 0 : (N - 1) * S::FH)
                                  : own + (size_t)cc * S::H + (side ? (N - 1) * S::FH : 0);
      bulk_g2s(st + S::OZ + (side * 2 + cc) * S::FH, src, S::FH * 8, bar);
    }
  }
}

// Per-thread body of the column-mapped residual (k_resid_stream): from a
// stage in the QStream3 layout
// (both phi halves + both-colour face layers, physical ghosts already
// formed) the own values col, L(phi) ap and r = g - L(phi) of this thread's
// 2 x PER cells, with the reference's operation order (stencil.hpp:300-322,
// 336-358).  rr: special-row kind per cell (0 uniform, 1 inside, 2 cut).
template <int N, int TT>
__device__ __forceinline__ void qs_cells(const double* __restrict__ st, int kind, double w,
                                         const double (&gcur)[2][QStream3<N, TT>::PER],
                                         const int (&rr)[2][QStream3<N, TT>::PER],
                                         double (&col)[2][QStream3<N, TT>::PER],
                                         double (&res)[2][QStream3<N, TT>::PER],
                                         double (&ap)[2][QStream3<N, TT>::PER], int t) {
  using S = QStream3<N, TT>;
  constexpr int HN = S::HN, H = S::H, FH = S::FH, PER = S::PER, KS = S::KS;
  const int m = t % HN, j = (t / HN) % N, kq = t / FH;
  const int eb = m + HN * j + FH * PER * kq;  // entry of q = 0
  const int jo = (j + kq * PER) & 1;          // o of colour 0 at q = 0; o_c(q) = jo ^ c ^ (q & 1)
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int q = 0; q < PER; ++q) col[c][q] = st[S::OP + c * H + eb + q * FH];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int X = 1 - c;
    const int XB = S::OP + X * H + eb;
    // neighbour bases (index of q = 0) and per-q steps: the other x
    // neighbour for o = 0 (e - 1 or the -x face) and o = 1 (e + 1 or +x),
    // y- / y+ (e -+ HN or the y face of colour c), z halo of colour c
    const int bx0 = m > 0 ? XB - 1 : S::OXF + kq * PER * N + j, sx0 = m > 0 ? FH : N;
    const int bx1 = m < HN - 1 ? XB + 1 : S::OXF + N * N + kq * PER * N + j, sx1 = m < HN - 1 ? FH : N;
    const int bym = j > 0 ? XB - HN : S::OY + (0 * 2 + c) * FH + kq * PER * HN + m, sym = j > 0 ? FH : HN;
    const int byp = j < N - 1 ? XB + HN : S::OY + (1 * 2 + c) * FH + kq * PER * HN + m, syp = j < N - 1 ? FH : HN;
    const double zlo = st[kq > 0 ? XB - FH : S::OZ + (0 * 2 + c) * FH + j * HN + m];
    const double zhi = st[kq < KS - 1 ? XB + PER * FH : S::OZ + (1 * 2 + c) * FH + j * HN + m];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int o = jo ^ c ^ (q & 1);
      const double f = col[c][q];
      const double xo = st[o ? bx1 + q * sx1 : bx0 + q * sx0];
      const double xm = o ? col[X][q] : xo, xp = o ? xo : col[X][q];
      const double ym = st[bym + q * sym], yp = st[byp + q * syp];
      const double zm = q > 0 ? col[X][q - 1] : zlo, zp = q < PER - 1 ? col[X][q + 1] : zhi;
      double sres = -2.0 * 3 * f;  // stencil.hpp:300-322, direction order
      sres += xm;
      sres += xp;
      sres += ym;
      sres += yp;
      sres += zm;
      sres += zp;
      ap[c][q] = kind == KIND_ALL_INSIDE ? 0.0 : sres * w;
      const int r8 = rr[c][q];
      res[c][q] = (kind == KIND_ALL_INSIDE || r8 == 1) ? 0.0 : gcur[c][q] - ap[c][q];
    }
  }
}

// MODE 1 of the column residual: this thread's leaf-record totals
// (record_leaf_residual, multigrid.hpp:529-562); inside rows excluded, cut
// rows recorded from their table (k_record_cut).
template <int PER>
__device__ __forceinline__ void qs_record(bool leaf, int kind, const int (&rr)[2][PER], const double (&res)[2][PER],
                                          double& rmx, double& rss, double& rcnt) {
  if (!leaf || kind == KIND_ALL_INSIDE) return;
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      if (rr[c][q] != 0) continue;
      rmx = fmax(rmx, fabs(res[c][q]));
      rss += res[c][q] * res[c][q];
      rcnt += 1.0;
    }
}

// MODE 0 of the column residual: restriction into the parent (multigrid.hpp:
// 697-722).  A parent's 2x2x2 children are the x pair of two consecutive
// planes of this thread and of the thread with j + 1 (lane + 8): one shuffle
// exchange, then the fold in x-fastest order.  Parents with a cut child
// belong to k_restrict_fix, pinned parents are re-pinned by k_pin_list.
// Every lane of the warp must call it (shuffles).
template <int N, int TT>
__device__ __forceinline__ void qs_restrict(const LevelView& Lp, int Pp, int cx, int cy, int cz,
                                            const int (&rr)[2][QStream3<N, TT>::PER],
                                            const double (&col)[2][QStream3<N, TT>::PER],
                                            const double (&res)[2][QStream3<N, TT>::PER], int t) {
  using S = QStream3<N, TT>;
  constexpr int NI = N * N * N, HN = S::HN, H = S::H, FH = S::FH, PER = S::PER;
  const int m = t % HN, j = (t / HN) % N, kq = t / FH;
  const int jo = (j + kq * PER) & 1;
#pragma unroll
  for (int p2 = 0; p2 < PER / 2; ++p2) {
    double rv[2][2], fv[2][2];  // [dz][dx]
    int cut = 0;
#pragma unroll
    for (int dz = 0; dz < 2; ++dz) {
      const int q = 2 * p2 + dz;
      const int c0 = jo ^ (q & 1);  // colour of the dx = 0 cell (o_c = 0)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int c = c0 ^ dx;
        rv[dz][dx] = c ? res[1][q] : res[0][q];
        fv[dz][dx] = c ? col[1][q] : col[0][q];
        cut |= (c ? rr[1][q] : rr[0][q]) == 2;
      }
    }
    double rn[2][2], fn[2][2];
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        rn[dz][dx] = __shfl_down_sync(0xffffffffu, rv[dz][dx], HN);
        fn[dz][dx] = __shfl_down_sync(0xffffffffu, fv[dz][dx], HN);
      }
    cut |= __shfl_down_sync(0xffffffffu, cut, HN);
    if (!(j & 1) && !cut) {  // multigrid.hpp:706-721: x-fastest order
      double sr = 0.0, sf = 0.0;
      sr += rv[0][0], sf += fv[0][0];
      sr += rv[0][1], sf += fv[0][1];
      sr += rn[0][0], sf += fn[0][0];
      sr += rn[0][1], sf += fn[0][1];
      sr += rv[1][0], sf += fv[1][0];
      sr += rv[1][1], sf += fv[1][1];
      sr += rn[1][0], sf += fn[1][0];
      sr += rn[1][1], sf += fn[1][1];
      const int pi = cx * HN + m, pj = cy * HN + (j >> 1), pk = cz * HN + kq * (PER / 2) + p2;
      const int pc = (pi + pj + pk) & 1, pe = (pi + N * (pj + N * pk)) >> 1;
      const size_t pa = (size_t)Pp * NI + (size_t)pc * H + pe;
      Lp.phi[pa] = sf / 8.0;
      Lp.rhs[pa] = sr / 8.0;
    }
  }
}

template <int N, int S_STAGES, int MINB, int MODE, int TT, bool CF = false>
__global__ void __launch_bounds__(QStream3<N, TT>::THR, MINB) k_resid_stream(LevelView Lf, LevelView Lp,
                                                                        const double* __restrict__ phi_b,
                                                                        const int4* __restrict__ plan, int n,
                                                                        Rec* __restrict__ partial, Rec* rec,
                                                                        unsigned int* counter) {
  pdl_begin();
  using S = QStream3<N, TT>;
  constexpr int NI = N * N * N, HN = S::HN, H = S::H, FH = S::FH, PER = S::PER, KS = S::KS;
  static_assert(S_STAGES >= 2, "g of block it+1 is read through meta[] one iteration ahead");
  static_assert(PER * KS == N && PER % 2 == 0 && 32 % (2 * HN) == 0, "columns of whole z pairs; j + 1 is lane + HN");
  constexpr int STAGE = S::STAGE + (CF ? 12 * FH : 0);
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[S_STAGES];
  __shared__ int meta[S_STAGES][CF ? 3 : 2];
  __shared__ double red[72];
  __shared__ bool last;
  __shared__ int4 pring[PlanRing<S_STAGES>::PR * 2];
  PlanRing<S_STAGES> R{pring};
  const int t = threadIdx.x;
  const int G = gridDim.x;
  const int nmine = (int)blockIdx.x < n ? (n - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (nmine == 0) return;
  if (t == 0) {
    for (int s = 0; s < S_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  R.init(plan, nmine, G);
  __syncthreads();
  for (int s = 0; s < S_STAGES; ++s) {
    if (s < nmine) {
      const BlockPlan P = R.get(s);
      if (t == 0) {
        qs_issue<N, TT, CF>(Lf, P, sm + s * STAGE, &full[s]);
        meta[s][0] = P.slot(), meta[s][1] = P.a.y;
        if (CF) meta[s][CF ? 2 : 0] = cf_mask_of(P);
      }
      rs_issue_async<N, S>(Lf, P, sm + s * STAGE);
    }
    cp_async_commit();
  }
  __syncthreads();  // meta of the first stages
  const int m = t % HN, j = (t / HN) % N, kq = t / FH;
  const int eb = m + HN * j + FH * PER * kq;  // entry of q = 0
  const double w = Lf.w;
  double gcur[2][PER], gnext[2][PER];
  {
    const double* gsrc = Lf.rhs + (size_t)meta[0][0] * NI + eb;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int q = 0; q < PER; ++q) gcur[c][q] = gsrc[c * H + q * FH];
  }
  double rmx = 0.0, rss = 0.0, rcnt = 0.0;  // MODE 1: this CTA's running totals
  for (int it = 0; it < nmine; ++it) {
    const int s = it % S_STAGES;
    double* st = sm + s * STAGE;
    R.advance(plan, it, nmine, G);
    const int slot = meta[s][0], flags = meta[s][1];
    const int kind = flags & 0xff, pmask = (flags >> 8) & 63;
    const int cfmask = CF ? meta[s][CF ? 2 : 0] : 0;
    // per-block scalars and the special-row kinds, in flight across the wait
    int rr[2][PER];
    if (kind == KIND_IFACE) {
      const int8_t* sk = Lf.skind + (size_t)(flags >> 14) * NI + eb;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < PER; ++q) rr[c][q] = sk[c * H + q * FH];
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < PER; ++q) rr[c][q] = 0;
    }
    const int Pp = MODE == 0 ? Lf.parent[slot] : 0;
    const int cx = MODE == 0 ? Lf.coords[slot * 3] & 1 : 0, cy = MODE == 0 ? Lf.coords[slot * 3 + 1] & 1 : 0,
              cz = MODE == 0 ? Lf.coords[slot * 3 + 2] & 1 : 0;
    const bool leaf = MODE != 0 ? Lf.leaf[slot] != 0 : false;
    mbar_wait(&full[s], (uint32_t)((it / S_STAGES) & 1));
    cp_async_wait<S_STAGES - 1>();
    __syncthreads();
    if (it + 1 < nmine) {  // this thread's g of the next block, in flight during this one
      const double* gsrc = Lf.rhs + (size_t)meta[(it + 1) % S_STAGES][0] * NI + eb;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < PER; ++q) gnext[c][q] = gsrc[c * H + q * FH];
    }
    if (pmask | cfmask) {  // block-uniform branch
      rs_phys_faces<N, S, CF>(Lf, slot, pmask, st, -1, 0, cfmask);
      __syncthreads();
    }
    double col[2][PER], res[2][PER], ap[2][PER];
    qs_cells<N, TT>(st, kind, w, gcur, rr, col, res, ap, t);
    if (MODE == 1) {
      qs_record<PER>(leaf, kind, rr, res, rmx, rss, rcnt);
    } else if (MODE == 2) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const size_t a = (size_t)slot * NI + (size_t)c * H + eb + q * FH;
          // special rows of interface blocks: inside rows keep r (0 + r), cut rows by k_fas_fix
          if (!leaf && (kind != KIND_IFACE || rr[c][q] == 0)) Lf.rhs[a] = ap[c][q] + gcur[c][q];
          Lf.old[a] = col[c][q];
        }
    }
    __syncthreads();  // stage s consumed
    if (it + S_STAGES < nmine) {
      const BlockPlan pf = R.get(it + S_STAGES);
      if (t == 0) {
        qs_issue<N, TT, CF>(Lf, pf, st, &full[s]);
        meta[s][0] = pf.slot(), meta[s][1] = pf.a.y;
        if (CF) meta[s][CF ? 2 : 0] = cf_mask_of(pf);
      }
      rs_issue_async<N, S>(Lf, pf, st);
    }
    cp_async_commit();
    if (MODE == 0) qs_restrict<N, TT>(Lp, Pp, cx, cy, cz, rr, col, res, t);
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int q = 0; q < PER; ++q) gcur[c][q] = gnext[c][q];
  }
  if (MODE == 1)  // this CTA's totals, folded with the other partials by k_record_fold
    record_finish(Lf, partial, rec, nullptr, (int)blockIdx.x, rmx, rss, rcnt, red, &last);
}

// Gather-entry evaluation (capi.cu cell_entry): the cell's value, its 2D
// neighbour values (physical ghosts 2 bc - f1 / f1) and L(phi) at the cell --
// uniform row (-2D self + sum p) w, special row center self + sum (nb p [+ bc phi_b])
// from the level's row-coefficient table, 0 for an inside row -- with the
// reference's operation order (stencil.hpp:290-359).
template <int D>
__device__ __forceinline__ double entry_apply(const LevelView& L, const int4& e0, const int4& e1,
                                              const double* __restrict__ gb, int a, double& self, bool& inside) {
  const int code = e0.x;
  const int na[6] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z};
  self = L.phi[a];
  double p[2 * D];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) p[d] = na[d] >= 0 ? L.phi[na[d]] : (na[d] == -1 ? self : 2.0 * gb[d] - self);
  inside = code <= -3;
  if (inside) return 0.0;
  if (code < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return s * L.w;
  }
  const double2* c2 = reinterpret_cast<const double2*>(L.r_coef) + (size_t)code * 8;
  double cf[14];
#pragma unroll
  for (int u = 0; u < 7; ++u) {
    const double2 v = c2[u];
    cf[2 * u] = v.x;
    cf[2 * u + 1] = v.y;
  }
  const int bm = (int)cf[13];
  double s = cf[0] * self;
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) {
    s += cf[1 + d] * p[d];
    if ((bm >> d) & 1) s += cf[7 + d];
  }
  return s;
}

// Parents of the fused restriction that k_restrict_stream cannot finish: a
// cut child in an interface block.  Eight threads per parent, one per child,
// each from its gather entry (two dependent round trips); lane 0 of the group
// sums them in the reference's x-fastest order (multigrid.hpp:706-721).
// Pinned parents are left to k_pin_list.
template <int D, int N>
__global__ void __launch_bounds__(128) k_restrict_fix(LevelView Lf, LevelView Lp, const int2* __restrict__ list,
                                                     const int32_t* __restrict__ tab,
                                                     const double* __restrict__ gbc, int n) {
  pdl_begin();
  using G = Geo<D, N>;
  constexpr int HN = N / 2, NC = 1 << D;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = gid / NC;
  double r = 0.0, f = 0.0;
  if (q < n) {
    const int4 e0 = reinterpret_cast<const int4*>(tab)[2 * gid];
    const int4 e1 = reinterpret_cast<const int4*>(tab)[2 * gid + 1];
    const int a = e1.w;
    bool inside;
    const double ap = entry_apply<D>(Lf, e0, e1, gbc + (size_t)gid * 6, a, f, inside);
    r = inside ? 0.0 : Lf.rhs[a] - ap;
  }
  const int base = threadIdx.x & ~(NC - 1) & 31;
  double sr = 0.0, sf = 0.0;
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    sr += __shfl_sync(0xffffffffu, r, base + u);
    sf += __shfl_sync(0xffffffffu, f, base + u);
  }
  if (q >= n || gid % NC != 0) return;
  const int slot = list[q].x, t = list[q].y;
  const int ii = t % HN, jj = (t / HN) % HN, kk = D == 3 ? t / (HN * HN) : 0;
  const int P = Lf.parent[slot];
  int cp[3] = {0, 0, 0};
  for (int a2 = 0; a2 < D; ++a2) cp[a2] = (Lf.coords[slot * D + a2] & 1) * HN;
  const int pi = cp[0] + ii, pj = cp[1] + jj, pk = cp[2] + kk;
  const size_t pa = (size_t)P * G::NI + (size_t)(G::colour(pi, pj, pk) * G::H + G::entry(pi, pj, pk));
  Lp.phi[pa] = sf / (double)NC;
  Lp.rhs[pa] = sr / (double)NC;
}

// apply_pins (stencil.hpp:225-237) over a list of (cell address, object) pairs
// the list and phi_b are static: loaded before griddepcontrol.wait (PDL)
static __global__ void __launch_bounds__(256) k_pin_list(double* __restrict__ phi, const double* __restrict__ phi_b,
                                                 const int2* __restrict__ list, int n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  int2 e = make_int2(0, 0);
  double v = 0.0;
  if (q < n) {
    e = list[q];
    v = phi_b[e.y];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (q < n) phi[e.x] = v;
}

// Cut rows of the lean interface blocks after the streaming sweep
// (multigrid.hpp:674-684), from a host-built table: per row the cell address,
// the row index and the six neighbour addresses (-1: Neumann ghost f1,
// -2: Dirichlet ghost 2 bc - f1 with bc in gbc), so a thread needs two
// dependent round trips.  One thread per cut row of the active colour.
// gs_cut_row: one row of the table; returns the cell address, `out` its new value
template <int D>
__device__ __forceinline__ int gs_cut_row(const LevelView& L, const int32_t* __restrict__ ent,
                                          const double* __restrict__ gbc, const double* __restrict__ coef, int q,
                                          double& out) {
  const int4 e0 = reinterpret_cast<const int4*>(ent)[2 * q];
  const int4 e1 = reinterpret_cast<const int4*>(ent)[2 * q + 1];
  const double2* cf2 = reinterpret_cast<const double2*>(coef) + (size_t)q * 8;
  double cf[14];
#pragma unroll
  for (int u = 0; u < 7; ++u) {
    const double2 v = cf2[u];
    cf[2 * u] = v.x;
    cf[2 * u + 1] = v.y;
  }
  const int a = e0.x;
  const int na[6] = {e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
  const int bm = (int)cf[13];
  const double self = L.phi[a];
  double num = L.rhs[a];
  double p[2 * D];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d)
    p[d] = na[d] >= 0 ? L.phi[na[d]] : (na[d] == -1 ? self : 2.0 * gbc[(size_t)q * 6 + d] - self);
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) {
    num -= cf[1 + d] * p[d];
    if ((bm >> d) & 1) num -= cf[7 + d];
  }
  out = num / cf[0];
  return a;
}

template <int D>
__global__ void __launch_bounds__(128) k_gs_cut(LevelView L, const int32_t* __restrict__ ent,
                                               const double* __restrict__ gbc, const double* __restrict__ coef,
                                               int n) {
  pdl_begin();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double v;
  const int a = gs_cut_row<D>(L, ent, gbc, coef, q, v);
  L.phi[a] = v;
}

// k_gs_cut over two tables (the cut rows of the blocks without / with
// coarse-fine faces) in one launch.
template <int D>
__global__ void __launch_bounds__(128) k_gs_cut2(LevelView L, const int32_t* __restrict__ ent0,
                                                const double* __restrict__ gbc0, const double* __restrict__ coef0,
                                                int n0, const int32_t* __restrict__ ent1,
                                                const double* __restrict__ gbc1, const double* __restrict__ coef1,
                                                int n1) {
  pdl_begin();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n0 + n1) return;
  const bool first = q < n0;
  double v;
  const int a = gs_cut_row<D>(L, first ? ent0 : ent1, first ? gbc0 : gbc1, first ? coef0 : coef1, first ? q : q - n0, v);
  L.phi[a] = v;
}

// ------------------------------------------------------------------ prolongation
// prolong_correction / prolong_full (multigrid.hpp:422-438, 724-783) for 3D
// fine blocks whose parent octant neighbourhood has no coarse-fine face.  A
// stage holds the fine block's phi (bulk copy; not needed for FULL) and the
// parent's phi and old on the octant plus its face-adjacent one-cell halo in
// natural 10^3 order (cp.async); a prep pass turns them into the delta tile
// (physical-face ghosts 2 bc - f1 evaluated for phi and old separately, as the
// reference's filled ghosts are).  Inside cells are interpolated too and
// re-pinned by k_pin_list afterwards (they always hold their pin).
template <int N, int TH = 0>
struct PStream3 {
  static constexpr int HN = N / 2;
  static constexpr int H = N * N * N / 2;
  static constexpr int PE = HN + 2, PS = PE * PE * PE;
  static constexpr int THR = TH ? TH : (H < 512 ? H : 512);
  static constexpr int PER = H / THR;
  static constexpr int OF = 0, ORP = 2 * H, ORO = ORP + PS;
  static constexpr int STAGE = ORO + PS;
};

// plan entry: {fine slot, parent slot, octant bits, parent neighbour across the
// octant's outer face per axis (-1 physical; CF kernels: -2 - p = a coarse-fine
// face of the parent whose cfc / cfold page is p), kind, edge}
//
// Tile element q (natural 10^3 order over the octant and its one-cell halo)
// of this thread, decoded once per kernel: the thread owns q = t + e*THR.
// `ax`/`side`: the axis on which the element leaves the octant (-1: inside;
// edges and corners are never read and are skipped).  Whether it also
// leaves the parent block depends only on the octant bit of that axis.
struct PElem {
  int q;          // tile index, -1: none
  int t3[3];      // octant-relative coordinates, -1 .. HN
  int ax, side;   // halo axis / side (0: -1, 1: HN), ax -1 inside
};
template <int N>
__device__ __forceinline__ PElem pr_elem(int q) {
  constexpr int HN = N / 2, PE = HN + 2, PS = PE * PE * PE;
  PElem E;
  E.q = -1;
  E.ax = -1;
  E.side = 0;
  E.t3[0] = E.t3[1] = E.t3[2] = 0;
  if (q >= PS) return E;
  const int t3[3] = {q % PE - 1, (q / PE) % PE - 1, q / (PE * PE) - 1};
  int out = 0;
  for (int d = 0; d < 3; ++d) {
    E.t3[d] = t3[d];
    if (t3[d] < 0 || t3[d] >= HN) ++out, E.ax = d, E.side = t3[d] >= HN;
  }
  if (out > 1) return E;  // edges / corners are never read
  E.q = q;
  return E;
}
// parent-block cell of element E for octant `oct`: block (P or the
// neighbour across the parent face, -1 physical) and colour-split address.
// Scalar coordinates (no runtime-indexed arrays: they went to local memory).
template <int N>
__device__ __forceinline__ size_t pr_addr(const PElem& E, int oct, int P, const int* pn, int& phys, int& x0,
                                          int& x1, int& x2) {
  constexpr int NI = N * N * N, HN = N / 2, H = NI / 2;
  x0 = (oct & 1) * HN + E.t3[0];
  x1 = ((oct >> 1) & 1) * HN + E.t3[1];
  x2 = ((oct >> 2) & 1) * HN + E.t3[2];
  int blk = P;
  phys = 0;
  const int ax = E.ax;
  if (ax >= 0 && ((oct >> ax) & 1) == E.side) {  // leaves the parent block
    const int nb = ax == 0 ? pn[0] : ax == 1 ? pn[1] : pn[2];
    int v;
    if (nb >= 0) {
      blk = nb;
      v = E.side ? 0 : N - 1;
    } else {  // physical (or coarse-fine) face: the parent's own boundary cell, made a ghost after the wait
      v = E.side ? N - 1 : 0;
      phys = nb == -1 ? 1 : 2;
    }
    x0 = ax == 0 ? v : x0;
    x1 = ax == 1 ? v : x1;
    x2 = ax == 2 ? v : x2;
  }
  return (size_t)blk * NI + (size_t)(((x0 + x1 + x2) & 1) * H) + (size_t)((x0 + N * (x1 + N * x2)) >> 1);
}

template <int N, bool FULL, int NE, int TH = 0>
__device__ __forceinline__ void pr_issue_async(const LevelView& Lp, const int4& a, const int4& b, double* st,
                                               const PElem* E) {
  using S = PStream3<N, TH>;
  const int pn[3] = {a.w, b.x, b.y};
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    if (E[e].q < 0) continue;
    int phys, x0, x1, x2;
    const size_t ad = pr_addr<N>(E[e], a.z, a.y, pn, phys, x0, x1, x2);
    cp_async8(st + S::ORP + E[e].q, Lp.phi + ad);
    if (!FULL) cp_async8(st + S::ORO + E[e].q, Lp.old + ad);
  }
}

// dead >= 0: the caller overwrites every cell of that colour next (the
// V-cycle's first post-smoothing half-sweep, multigrid.hpp:491-498), so in
// blocks without a physical / coarse-fine face -- where no ghost reads a cell
// of that colour -- those cells are neither read nor written.
// rev: walk the plan backwards, so that the first post-smoothing half-sweep
// (forward) starts on the blocks written last (still in L2).
// CF: a parent face may be coarse-fine (Lp.cfc set and built): its PHI ghost is
// 1/2 c + 3/4 f1 - 1/4 f2 from level l-1's cfc page and the two parent cells
// in the tile, its OLD ghost the cfold snapshot (multigrid.hpp:394-396).
template <int N, int S_STAGES, int MINB, bool FULL, int TH = 0, bool CF = false>
__global__ void __launch_bounds__(PStream3<N, TH>::THR, MINB) k_prolong_stream(LevelView Lf, LevelView Lp,
                                                                          const int4* __restrict__ plan, int n,
                                                                          int dead, int rev) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: prologue before the wait
  using S = PStream3<N, TH>;
  constexpr int NI = N * N * N, HN = S::HN, PE = S::PE;
  constexpr int NE = (S::PS + S::THR - 1) / S::THR;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[S_STAGES];
  __shared__ int4 meta[S_STAGES][2];
  const int t = threadIdx.x;
  const int G = gridDim.x;
  const int nmine = (int)blockIdx.x < n ? (n - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (nmine == 0) return;
  PElem E[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) E[e] = pr_elem<N>(t + e * S::THR);
  if (t == 0) {
    for (int s = 0; s < S_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // plan entry of the next block to issue, loaded one block ahead (its
  // latency overlaps the current block instead of delaying the next issue)
  int4 qa = make_int4(0, 0, 0, 0), qb = qa;
  auto fetch = [&](int idx) {
    int p = blockIdx.x + idx * G;
    if (rev) p = n - 1 - p;
    qa = __ldg(plan + 2 * p);
    qb = __ldg(plan + 2 * p + 1);
  };
  auto issue = [&](int s) {
    const int4 a = qa, b = qb;
    double* st = sm + s * S::STAGE;
    if (t == 0) {
      meta[s][0] = a;
      meta[s][1] = b;
      if (FULL) {
        mbar_arrive_expect_tx(&full[s], 0);
      } else if (dead >= 0 && !b.w) {  // the live colour only
        const int lc = 1 - dead;
        mbar_arrive_expect_tx(&full[s], S::H * 8);
        bulk_g2s(st + S::OF + lc * S::H, Lf.phi + (size_t)a.x * NI + (size_t)lc * S::H, S::H * 8, &full[s]);
      } else {
        mbar_arrive_expect_tx(&full[s], 2 * S::H * 8);
        bulk_g2s(st + S::OF, Lf.phi + (size_t)a.x * NI, 2 * S::H * 8, &full[s]);
      }
    }
    pr_issue_async<N, FULL, NE, TH>(Lp, a, b, st, E);
  };
  for (int s = 0; s < S_STAGES; ++s) {
    if (s < nmine) {
      fetch(s);
      issue(s);
    }
    cp_async_commit();
  }
  if (S_STAGES < nmine) fetch(S_STAGES);
  // fine-cell geometry of this thread: the column of PER consecutive fine
  // planes k = kz*PER + q of entry column (m, j), both colours -- the cells
  // (2m, j, k) and (2m+1, j, k), parent (m, j/2, k/2).  The column's parents
  // span PER/2 planes, so the tile is read once per parent plane (centre, x-,
  // x+, y) plus the plane below and above (the z neighbours): 2 + 2 PER loads
  // for 2 PER fine cells.
  constexpr int KZ = S::THR / (HN * N);  // columns along z
  static_assert(KZ * S::PER == N && S::PER % 2 == 0, "columns of whole parent planes");
  constexpr int PPL = S::PER / 2;  // parent planes per column
  const int m = t % HN, j = (t / HN) % N, kz = t / (HN * N);
  const int ebase = m + HN * j + HN * N * S::PER * kz;  // entry of q = 0
  const int pz0 = PPL * kz;                            // first parent plane
  const int ctr0 = ((pz0 + 1) * PE + (j >> 1) + 1) * PE + m + 1;
  const int dyo = (j & 1) ? PE : -PE;
  for (int it = 0; it < nmine; ++it) {
    const int s = it % S_STAGES;
    double* st = sm + s * S::STAGE;
    mbar_wait(&full[s], (uint32_t)((it / S_STAGES) & 1));
    cp_async_wait<S_STAGES - 1>();
    __syncthreads();
    const int4 a = meta[s][0], b = meta[s][1];
    const int slot = a.x, P = a.y, oct = a.z;
    const int pn[3] = {a.w, b.x, b.y};
    // prep: delta (or phi for FULL) in place of the raw phi tile; physical-face
    // ghosts of phi and old evaluated separately (mesh.hpp:538-552)
    double dv[NE];  // CF: every element's delta first (coarse-fine ghosts read raw tile values), then the stores
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      if (E[e].q < 0) continue;
      const int q = E[e].q;
      double vp = st[S::ORP + q], vo = FULL ? 0.0 : st[S::ORO + q];
      if (E[e].ax >= 0 && ((oct >> E[e].ax) & 1) == E[e].side) {
        const int ax = E[e].ax;
        const int code = ax == 0 ? pn[0] : ax == 1 ? pn[1] : pn[2];
        if (CF && code <= -2) {
          int phys, x0, x1, x2;
          (void)pr_addr<N>(E[e], oct, P, pn, phys, x0, x1, x2);
          const int tj = ax == 0 ? x1 + N * x2 : ax == 1 ? x0 + N * x2 : x0 + N * x1;
          const size_t page = (size_t)(-2 - code) * (N * N);
          const double cv = Lp.cfc[page + (size_t)(((x0 + x1 + x2) & 1) * (N * N / 2) + (tj >> 1))];
          // f2: the parent cell one further inward, two tile elements from the ghost
          const int str = ax == 0 ? 1 : ax == 1 ? PE : PE * PE;
          const double f2 = st[S::ORP + q + (E[e].side ? -2 * str : 2 * str)];
          vp = 0.5 * cv + 0.75 * vp - 0.25 * f2;
          if (!FULL) vo = Lp.cfold[page + tj];
        } else if (code < 0) {
          const int dir = 2 * ax + E[e].side;
          if (Lp.bctype[dir] != 1) {
            int phys, x0, x1, x2;
            (void)pr_addr<N>(E[e], oct, P, pn, phys, x0, x1, x2);
            const int bo = Lp.bcoff[P * 6 + dir];
            const int tj = ax == 0 ? x1 + N * x2 : ax == 1 ? x0 + N * x2 : x0 + N * x1;
            const double bcv = bo < 0 ? 0.0 : Lp.bcval[bo + tj];
            vp = 2.0 * bcv - vp;
            vo = 2.0 * bcv - vo;
          }
        }
      }
      if (CF) dv[e] = FULL ? vp : vp - vo;
      else st[S::ORP + q] = FULL ? vp : vp - vo;
    }
    if (CF) {
      __syncthreads();  // all raw reads done
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (E[e].q >= 0) st[S::ORP + E[e].q] = dv[e];
    }
    __syncthreads();
    const double* Dt = st + S::ORP;
    double* __restrict__ dst = Lf.phi + (size_t)slot * NI;
    const int skipc = (!FULL && dead >= 0 && !b.w) ? dead : -1;
    double zc[PPL + 2], xm[PPL], xp[PPL], yv[PPL];
#pragma unroll
    for (int u = 0; u < PPL + 2; ++u) zc[u] = Dt[ctr0 + (u - 1) * PE * PE];
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
      xm[u] = Dt[ctr0 + u * PE * PE - 1];
      xp[u] = Dt[ctr0 + u * PE * PE + 1];
      yv[u] = Dt[ctr0 + u * PE * PE + dyo];
    }
#pragma unroll
    for (int q = 0; q < S::PER; ++q) {
      const int u = q >> 1;  // parent plane of fine plane k = kz*PER + q (k parity = q parity)
      const double dc = zc[u + 1], dy = yv[u];
      const double dz = zc[(q & 1) ? u + 2 : u];
      const int c0 = (j + q) & 1;  // colour of i = 2m (x neighbour -1); i = 2m+1 has +1
      const int e = ebase + q * HN * N;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = h ? 1 - c0 : c0;
        if (c == skipc) continue;
        double v = (1.0 - 0.25 * 3) * dc;  // multigrid.hpp:742-752
        v += 0.25 * (h ? xp[u] : xm[u]);
        v += 0.25 * dy;
        v += 0.25 * dz;
        const size_t ad = (size_t)c * S::H + e;
        dst[ad] = FULL ? v : st[S::OF + ad] + v;
      }
    }
    __syncthreads();  // stage s consumed
    if (it + S_STAGES < nmine) {
      issue(s);
      if (it + S_STAGES + 1 < nmine) fetch(it + S_STAGES + 1);
    }
    cp_async_commit();
  }
}

// Leaf-residual record of the cut rows (the k_gs_cut tables of both colours):
// r = g - (center phi + sum nb p + sum bc phi_b) (stencil.hpp:344-358); one
// partial (max, sum r^2, count) per CTA into `partial`.
template <int D>
__global__ void __launch_bounds__(256) k_record_cut(LevelView L, const double* __restrict__ phi_b,
                                                   const int32_t* __restrict__ ent0, const double* __restrict__ gbc0,
                                                   int n0, const int32_t* __restrict__ ent1,
                                                   const double* __restrict__ gbc1, int n1, int ni,
                                                   Rec* __restrict__ partial) {
  pdl_begin();
  __shared__ double red[72];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0, ss = 0.0, cnt = 0.0;
  if (q < n0 + n1) {
    const int qq = q < n0 ? q : q - n0;
    const int32_t* ent = q < n0 ? ent0 : ent1;
    const double* gbc = q < n0 ? gbc0 : gbc1;
    const int4 e0 = reinterpret_cast<const int4*>(ent)[2 * qq];
    const int4 e1 = reinterpret_cast<const int4*>(ent)[2 * qq + 1];
    const int a = e0.x, r = e0.y;
    if (L.leaf[a / ni]) {
      // gather-entry form of this cut row: code r, then its neighbour addresses
      const int4 f0 = make_int4(r, e0.z, e0.w, e1.x), f1 = make_int4(e1.y, e1.z, e1.w, 0);
      double self;
      bool inside;
      const double ap = entry_apply<D>(L, f0, f1, gbc + (size_t)qq * 6, a, self, inside);
      const double rv = L.rhs[a] - ap;
      mx = fabs(rv);
      ss = rv * rv;
      cnt = 1.0;
    }
  }
  mx = block_max(mx, red);
  ss = block_sum(ss, red);
  cnt = block_sum(cnt, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x].max = mx;
    partial[blockIdx.x].sumsq = ss;
    partial[blockIdx.x].count = (long long)cnt;
  }
}

// rec = fold of partial[0 .. n) in index order (combine_records' per-level record)
// fin != nullptr: this is the cycle's last record -- thread 0 also forms the
// CycleStats over all levels (k_combine's loop, multigrid.hpp:564-575, with
// this level's totals in place) and writes stats, diag and status to the
// mapped host buffer, so the cycle graph ends here (no combine kernel, no
// device-to-host copy node).
struct FinishArgs {
  const Rec* rec;     // all level records, [0 .. nlev]
  int nlev, level;    // level being folded
  double* outbuf;     // device: stats[2], diag[2], status
  double* host_out;   // mapped pinned image of outbuf
};
static __global__ void __launch_bounds__(1024) k_record_fold(const Rec* __restrict__ partial, int n, Rec* out,
                                                             FinishArgs fin) {
  pdl_begin();
  __shared__ double red[3][32];
  __shared__ double lrec[3][kMaxLevels + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  // the other levels' records for the finish, in flight with the partials
  if (fin.host_out && (int)threadIdx.x <= fin.nlev && (int)threadIdx.x <= kMaxLevels) {
    const Rec r = fin.rec[threadIdx.x];
    lrec[0][threadIdx.x] = r.max;
    lrec[1][threadIdx.x] = r.sumsq;
    lrec[2][threadIdx.x] = (double)r.count;
  }
  double mx = 0.0, ss = 0.0, cc = 0.0;
  for (int b = threadIdx.x; b < n; b += blockDim.x) {
    const Rec r = partial[b];
    mx = fmax(mx, r.max);
    ss += r.sumsq;
    cc += (double)r.count;
  }
  // one barrier: warp butterflies, then thread 0 folds the warps in order (fixed order: deterministic)
  mx = warp_max(mx);
  ss = warp_sum(ss);
  cc = warp_sum(cc);
  if (lane == 0) {
    red[0][wid] = mx;
    red[1][wid] = ss;
    red[2][wid] = cc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mx = 0.0, ss = 0.0, cc = 0.0;
    for (int w = 0; w < nw; ++w) {
      mx = fmax(mx, red[0][w]);
      ss += red[1][w];
      cc += red[2][w];
    }
    out->max = mx;
    out->sumsq = ss;
    out->count = (long long)cc;
    if (fin.host_out) {
      double m = 0, s = 0;
      long long c = 0;
      for (int l = 0; l <= fin.nlev; ++l) {
        const bool me = l == fin.level;
        m = fmax(m, me ? mx : lrec[0][l]);
        s += me ? ss : lrec[1][l];
        c += me ? (long long)cc : (long long)lrec[2][l];
      }
      const double l2 = c > 0 ? sqrt(s / (double)c) : 0.0;
      fin.outbuf[0] = m;
      fin.outbuf[1] = l2;
      fin.host_out[0] = m;
      fin.host_out[1] = l2;
      fin.host_out[2] = fin.outbuf[2];
      fin.host_out[3] = fin.outbuf[3];
      fin.host_out[4] = fin.outbuf[4];
    }
  }
}

// FAS right-hand side of the cut rows of the streamed blocks (the k_gs_cut
// tables of both colours): g = L(phi) + r on non-leaf blocks (multigrid.hpp:388-392)
template <int D, int N>
__global__ void __launch_bounds__(128) k_fas_fix(LevelView L, const int32_t* __restrict__ ent0,
                                                const double* __restrict__ gbc0, int n0,
                                                const int32_t* __restrict__ ent1,
                                                const double* __restrict__ gbc1, int n1) {
  pdl_begin();
  using G = Geo<D, N>;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n0 + n1) return;
  const int qq = q < n0 ? q : q - n0;
  const int32_t* ent = q < n0 ? ent0 : ent1;
  const double* gbc = q < n0 ? gbc0 : gbc1;
  const int4 e0 = reinterpret_cast<const int4*>(ent)[2 * qq];
  const int4 e1 = reinterpret_cast<const int4*>(ent)[2 * qq + 1];
  const int a = e0.x;
  if (L.leaf[a / G::NI]) return;
  const int4 f0 = make_int4(e0.y, e0.z, e0.w, e1.x), f1 = make_int4(e1.y, e1.z, e1.w, 0);
  double self;
  bool inside;
  const double out = entry_apply<D>(L, f0, f1, gbc + (size_t)qq * 6, a, self, inside);
  L.rhs[a] = out + L.rhs[a];
}

}  // namespace pmgdev

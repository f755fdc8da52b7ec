// brick.cuh -- instruction-lean leaf-residual record (record_leaf_residual,
// multigrid.hpp:529-562) over lean 3D blocks (N = 16).
//
// Same stage ring as k_resid_stream (QStream3 layout: both phi halves by one
// TMA bulk copy, the face layers of both colours by bulk copies / cp.async),
// but a thread mapping built for 16-byte shared-memory accesses:
//
//   warp p (8 warps per block) owns the z-planes k = 2p, 2p + 1; lane L owns
//   the x-quarter q = L % 4 (cells i = 4q .. 4q+3) of the rows j = L / 4 and
//   j + 8 in both planes: 16 cells.
//
// The four cells of a quarter-row are the entries e, e+1 (e = 8 j + 2 q +
// 128 k) of both colour halves, so the own values, and the y and z
// neighbours of all four cells, come as pairs of doubles (LDS.128) whose
// addresses run contiguously across the warp (no bank conflicts); only the
// two x neighbours beyond the quarter are single loads.  Every value needed
// by a cell is one register away, so a cell costs ~20 instructions instead
// of ~80 in the column kernel (k_resid_stream in record mode was issue- and
// latency-bound, not HBM-bound: 41.6 M warp instructions for one 256^3
// record; this kernel: 26 M, 85 -> 68 us).
//
// g goes straight from global memory (16-byte loads, issued before the stage
// wait).  HBM latency under full load is several microseconds, more than two
// shared-memory stages cover, so phi and g of the block S + 1 ahead are
// prefetched into L2 (cp.async.bulk.prefetch.L2): the bytes in flight live in
// L2, the stage copies and g loads then hit L2.
// Arithmetic and its order are the reference's (stencil.hpp:300-322,
// 336-358), so every residual is bit-identical to the other residual kernels.
#pragma once
#include "stream.cuh"

namespace pmgdev {

constexpr int kBrickThreads = 256;

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ldg2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void stg2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// Residuals of one quarter-row (4 cells x 0..3 at row j, plane k) from the
// stage: own values f[4], L(phi) ap[4] and r[4] = g - L(phi).
// ca = colour of cell x = 0 (= (j + k) & 1); e = entry of cell 0 within a half.
template <int N>
__device__ __forceinline__ void brick_row(const double* __restrict__ st, int q, int j, int k, double w,
                                          const double (&g)[4], double (&f)[4], double (&ap)[4], double (&r)[4]) {
  using S = QStream3<N, 512>;
  constexpr int H = S::H, HN = S::HN, FH = S::FH;
  const int ca = (j + k) & 1, cb = 1 - ca;
  const int e = HN * j + 2 * q + FH * k;
  // own: cells 0, 2 (colour ca) and 1, 3 (colour cb)
  const double2 A = lds2(st + S::OP + ca * H + e), B = lds2(st + S::OP + cb * H + e);
  f[0] = A.x, f[1] = B.x, f[2] = A.y, f[3] = B.y;
  // x neighbours beyond the quarter: cell -1 (colour cb, entry e - 1) and 4 (ca, e + 2)
  const double xl = st[q > 0 ? S::OP + cb * H + e - 1 : S::OXF + k * N + j];
  const double xr = st[q < 3 ? S::OP + ca * H + e + 2 : S::OXF + N * N + k * N + j];
  // y / z neighbours: the same entries of the other colour in rows j -+ 1 /
  // planes k -+ 1, or the face layer indexed by the colour of the own cell
  // (ca for cells 0, 2; cb for cells 1, 3)
  const int ym0 = j > 0 ? S::OP + cb * H + e - HN : S::OY + (0 * 2 + ca) * FH + k * HN + 2 * q;
  const int ym1 = j > 0 ? S::OP + ca * H + e - HN : S::OY + (0 * 2 + cb) * FH + k * HN + 2 * q;
  const int yp0 = j < N - 1 ? S::OP + cb * H + e + HN : S::OY + (1 * 2 + ca) * FH + k * HN + 2 * q;
  const int yp1 = j < N - 1 ? S::OP + ca * H + e + HN : S::OY + (1 * 2 + cb) * FH + k * HN + 2 * q;
  const int zm0 = k > 0 ? S::OP + cb * H + e - FH : S::OZ + (0 * 2 + ca) * FH + j * HN + 2 * q;
  const int zm1 = k > 0 ? S::OP + ca * H + e - FH : S::OZ + (0 * 2 + cb) * FH + j * HN + 2 * q;
  const int zp0 = k < N - 1 ? S::OP + cb * H + e + FH : S::OZ + (1 * 2 + ca) * FH + j * HN + 2 * q;
  const int zp1 = k < N - 1 ? S::OP + ca * H + e + FH : S::OZ + (1 * 2 + cb) * FH + j * HN + 2 * q;
  const double2 YM0 = lds2(st + ym0), YM1 = lds2(st + ym1), YP0 = lds2(st + yp0), YP1 = lds2(st + yp1);
  const double2 ZM0 = lds2(st + zm0), ZM1 = lds2(st + zm1), ZP0 = lds2(st + zp0), ZP1 = lds2(st + zp1);
  const double xm[4] = {xl, f[0], f[1], f[2]}, xp[4] = {f[1], f[2], f[3], xr};
  const double ym[4] = {YM0.x, YM1.x, YM0.y, YM1.y}, yp[4] = {YP0.x, YP1.x, YP0.y, YP1.y};
  const double zm[4] = {ZM0.x, ZM1.x, ZM0.y, ZM1.y}, zp[4] = {ZP0.x, ZP1.x, ZP0.y, ZP1.y};
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    double s = -2.0 * 3 * f[x];  // stencil.hpp:300-322, direction order
    s += xm[x];
    s += xp[x];
    s += ym[x];
    s += yp[x];
    s += zm[x];
    s += zp[x];
    ap[x] = s * w;
    r[x] = g[x] - ap[x];
  }
}

// One partial (max |r|, sum r^2, count) per CTA into partial[blockIdx.x],
// folded with the cut-row partials by k_record_fold.
template <int N, int S_STAGES>
__global__ void __launch_bounds__(kBrickThreads, 2)
    k_record_brick(LevelView Lf, const int4* __restrict__ plan, int n, Rec* __restrict__ partial) {
  pdl_begin();
  using S = QStream3<N, 512>;  // stage layout only (the 512 is the column kernel's thread count)
  constexpr int NI = N * N * N, H = S::H, HN = S::HN, FH = S::FH;
  static_assert(N == 16, "the lane mapping covers 16^3 blocks with 8 warps");
  constexpr int THR = kBrickThreads, PL = 2;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[S_STAGES];
  __shared__ int meta[S_STAGES][2];
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
  auto issue = [&](const BlockPlan& P, int s) {
    double* st = sm + s * S::STAGE;
    if (t == 0) {
      qs_issue<N, 512>(Lf, P, st, &full[s]);
      meta[s][0] = P.slot(), meta[s][1] = P.a.y;
    }
    // x / y face values (rs_issue_async's layout), 512-thread pattern spread over 256
    for (int u = t; u < 2 * N * N; u += THR) {
      const int side = u / (N * N), rr = u % (N * N), k = rr / N, j = rr % N;
      const int ib = side ? N - 1 : 0;
      const int cbb = (ib + j + k) & 1;
      const int ns = P.nbr(side);
      const double* src = ns >= 0 ? Lf.phi + (size_t)ns * NI + (size_t)(1 - cbb) * H + (side ? 0 : HN - 1) + HN * (j + N * k)
                                  : Lf.phi + (size_t)P.slot() * NI + (size_t)cbb * H + (ib >> 1) + HN * (j + N * k);
      cp_async8(st + S::OXF + side * N * N + k * N + j, src);
    }
    for (int u = t; u < S::YC; u += THR) {
      constexpr int CR = HN / 2;
      const int side = u / (2 * N * CR), cc = (u / (N * CR)) % 2, k = (u / CR) % N, ch = u % CR;
      const int ns = P.nbr(2 + side);
      const double* src = ns >= 0 ? Lf.phi + (size_t)ns * NI + (size_t)(1 - cc) * H + (size_t)k * FH + (side ? 0 : (N - 1) * HN)
                                  : Lf.phi + (size_t)P.slot() * NI + (size_t)cc * H + (size_t)k * FH + (side ? (N - 1) * HN : 0);
      cp_async16(st + S::OY + (side * 2 + cc) * FH + k * HN + 2 * ch, src + 2 * ch);
    }
  };
  for (int s = 0; s < S_STAGES; ++s) {
    if (s < nmine) issue(R.get(s), s);
    cp_async_commit();
  }
  if (t == 0)  // g of the staged blocks and everything of block S into L2 (see the loop)
    for (int b = 0; b <= S_STAGES && b < nmine; ++b) {
      const int pslot = R.get(b).slot();
      if (b == S_STAGES) l2_prefetch(Lf.phi + (size_t)pslot * NI, NI * 8);
      l2_prefetch(Lf.rhs + (size_t)pslot * NI, NI * 8);
    }
  __syncthreads();  // meta of the first stages
  const int lane = t & 31, p = t >> 5;
  const int q = lane & 3, j0 = lane >> 2;  // rows j0 and j0 + 8
  const double w = Lf.w;
  double rmx = 0.0, rss = 0.0;
  int rcnt = 0;
  for (int it = 0; it < nmine; ++it) {
    const int s = it % S_STAGES;
    double* st = sm + s * S::STAGE;
    R.advance(plan, it, nmine, G);
    const int slot = meta[s][0], flags = meta[s][1];
    const int kind = flags & 0xff, pmask = (flags >> 8) & 63;
    // g of this thread's 16 cells [row][plane][x], in flight across the wait
    double g[2][PL][4];
    const double* gb = Lf.rhs + (size_t)slot * NI;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < PL; ++b) {
        const int j = j0 + 8 * a, k = PL * p + b;
        const int ca = (j + k) & 1, e = HN * j + 2 * q + FH * k;
        const double2 A = ldg2(gb + ca * H + e), B = ldg2(gb + (1 - ca) * H + e);
        g[a][b][0] = A.x, g[a][b][1] = B.x, g[a][b][2] = A.y, g[a][b][3] = B.y;
      }
    // special-row kinds of an interface block (0 uniform, 1 inside, 2 cut)
    int rk[2][PL][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < PL; ++b)
#pragma unroll
        for (int x = 0; x < 4; ++x) rk[a][b][x] = 0;
    if (kind == KIND_IFACE) {
      const int8_t* sk = Lf.skind + (size_t)(flags >> 14) * NI;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < PL; ++b) {
          const int j = j0 + 8 * a, k = PL * p + b;
          const int ca = (j + k) & 1, e = HN * j + 2 * q + FH * k;
          rk[a][b][0] = sk[ca * H + e], rk[a][b][1] = sk[(1 - ca) * H + e];
          rk[a][b][2] = sk[ca * H + e + 1], rk[a][b][3] = sk[(1 - ca) * H + e + 1];
        }
    }
    const bool leaf = Lf.leaf[slot] != 0;
    mbar_wait(&full[s], (uint32_t)((it / S_STAGES) & 1));
    cp_async_wait<S_STAGES - 1>();
    __syncthreads();
    // phi and g of the block S + 1 ahead into L2: HBM latency under load is
    // several microseconds, more than the stage ring can cover in shared memory
    if (t == 0 && it + S_STAGES + 1 < nmine) {
      const int pslot = R.get(it + S_STAGES + 1).slot();
      l2_prefetch(Lf.phi + (size_t)pslot * NI, NI * 8);
      l2_prefetch(Lf.rhs + (size_t)pslot * NI, NI * 8);
    }
    if (pmask) {  // block-uniform branch: physical faces become ghosts
      rs_phys_faces<N, S>(Lf, slot, pmask, st);
      __syncthreads();
    }
    double rv[2][PL][4];
    const bool rec = leaf && kind != KIND_ALL_INSIDE;  // block-uniform
    if (rec) {
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < PL; ++b) {
          double f[4], ap[4];
          brick_row<N>(st, q, j0 + 8 * a, PL * p + b, w, g[a][b], f, ap, rv[a][b]);
        }
    }
    __syncthreads();  // stage s consumed
    if (it + S_STAGES < nmine) issue(R.get(it + S_STAGES), s);
    cp_async_commit();
    {  // record_leaf_residual (multigrid.hpp:529-562): inside rows excluded, cut rows by k_record_cut
      // the reference's std::max(mx, |r|) is (mx < |r|) ? |r| : mx
      if (rec && kind == KIND_UNIFORM) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < PL; ++b)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const double v = rv[a][b][x], av = fabs(v);
              rmx = rmx < av ? av : rmx;
              rss += v * v;
            }
        rcnt += 8 * PL;
      } else if (rec) {  // interface block
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < PL; ++b)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              if (rk[a][b][x] != 0) continue;
              const double v = rv[a][b][x], av = fabs(v);
              rmx = rmx < av ? av : rmx;
              rss += v * v;
              ++rcnt;
            }
      }
    }
  }
  record_finish(Lf, partial, nullptr, nullptr, (int)blockIdx.x, rmx, rss, (double)rcnt, red, &last);
}

}  // namespace pmgdev

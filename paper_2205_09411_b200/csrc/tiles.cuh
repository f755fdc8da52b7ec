// tiles.cuh -- CTA-per-block kernels with the block and its face halo staged
// in shared memory.
//
// A "colour tile" holds the cells of ONE colour of a padded (N+2)^D block in
// colour-split form: padded row (jp,kp) keeps its N/2+1 cells of that colour at
// slot ip>>1, so a tile is (N+2)^(D-1) * (N/2+1) doubles (23.3 KB for N=16).
// The face-ghost cells of the tile's colour are filled once per face cell with
// the reference's fill formulas (phi_ghost, mesh.hpp:471-554); corners and
// edges are never read (face ghosts only, as in the reference).  Every kernel
// then runs branch-free stencil arithmetic from shared memory, in exactly the
// operation order of the per-cell reference code (cells.cuh), so results stay
// bit-identical.
#pragma once
#include "kernels.cuh"

namespace pmgdev {

template <int D, int N>
struct Tile {
  static constexpr int P = N + 2;
  static constexpr int RW = N / 2 + 1;
  static constexpr int ROWS = D == 2 ? P : P * P;
  static constexpr int SIZE = ROWS * RW;
  // 3D N = 8: 128 threads (two entries each) -- twice as many blocks resident per
  // SM, which is what these latency-bound kernels need (cfg3: 1.29 -> 1.20 ms per cycle)
  static constexpr int THREADS = (D == 3 && N == 8) ? 128 : (Geo<D, N>::H < 256 ? Geo<D, N>::H : 256);
  // resident CTAs per SM asked of the compiler (register cap)
#ifndef PMG_TILE8_MINB
#define PMG_TILE8_MINB 12
#endif
  static constexpr int MINB = (D == 3 && N == 8) ? PMG_TILE8_MINB : 1;
  __device__ __forceinline__ static int idx(int ip, int jp, int kp) {
    return (D == 3 ? kp * P + jp : jp) * RW + (ip >> 1);
  }
};

// Correctly rounded x / 6.0 without the fp64 division sequence: with
// y = RN(1/6), q = RN(x y) is faithful, the remainder r = x - 6q is exact in
// one FMA, and q' = RN(q + r y) = RN(x / 6) (Markstein's correction; x/6 can
// never be a rounding midpoint for a 53-bit x).  Zero, inf, NaN and the
// subnormal range take the plain division, so the result is bit-identical to
// the reference's `/ 6.0` for every input (multigrid.hpp:651-653).
static __device__ __noinline__ double div6_slow(double x) { return x / 6.0; }
// x / 6.0 in three unconditional ops, exact (correctly rounded) whenever
// div6_in_range(x); callers batch the range test and redo the rare rest
// with the IEEE division.
__device__ __forceinline__ double div6_fast(double x) {
  const double y = 0.16666666666666666;  // RN(1/6)
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, 6.0, x);
  return __fma_rn(r, y, q);
}
__device__ __forceinline__ bool div6_in_range(double x) {
  const double ax = fabs(x);
  return (ax > 1e-290 && ax < 1e300) || x == 0.0;
}
__device__ __forceinline__ double div6(double x) {
  const double y = 0.16666666666666666;  // RN(1/6)
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, 6.0, x);
  const double q1 = __fma_rn(r, y, q);
  const double ax = fabs(x);
  if (__builtin_expect(ax > 1e-290 && ax < 1e300, 1)) return q1;
  if (x == 0.0) return q;  // +-0 * RN(1/6) = +-0 = x / 6
  return div6_slow(x);     // subnormal / huge / inf / nan
}

// Face-ghost loader for one face (AXIS, SIDE compile-time): ghost cells of
// colour X next to interior cells of colour 1-X.  r enumerates them.
template <int D, int N, int AXIS, int SIDE>
__device__ __forceinline__ double halo_cell(int& tix, const LevelView& L, const LevelView& Lc,
                                            int slot, int X, int r,
                                            const double* __restrict__ oth) {
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  constexpr int DIR = 2 * AXIS + SIDE;
  constexpr int AC = SIDE ? N - 1 : 0;
  int c3[3] = {0, 0, 0};
  if (D == 2) {
    c3[AXIS] = AC;
    c3[1 - AXIS] = 2 * r + ((1 - X + AC) & 1);
  } else {
    constexpr int A0 = AXIS == 0 ? 1 : 0;  // lower transverse axis
    constexpr int A1 = AXIS == 2 ? 1 : 2;  // higher transverse axis
    const int t1 = r / (N / 2);
    c3[AXIS] = AC;
    c3[A1] = t1;
    c3[A0] = 2 * (r % (N / 2)) + ((1 - X + AC + t1) & 1);
  }
  const int ns = L.nbr[slot * G::F + DIR];
  double gv;
  if (ns >= 0) {  // same-level copy (mesh.hpp:485-498)
    int w3[3] = {c3[0], c3[1], c3[2]};
    w3[AXIS] = SIDE ? 0 : N - 1;
    gv = L.phi[(size_t)ns * G::NI + (size_t)X * G::H + G::entry(w3[0], w3[1], w3[2])];
  } else {
    const double self = oth[G::entry(c3[0], c3[1], c3[2])];
    if (L.cnbr[slot * G::F + DIR] >= 0) {
      int w3[3] = {c3[0], c3[1], c3[2]};
      w3[AXIS] = SIDE ? N - 2 : 1;
      const double f2 = L.phi[(size_t)slot * G::NI + (size_t)X * G::H + G::entry(w3[0], w3[1], w3[2])];
      gv = cf_ghost<D, N>(L, Lc, slot, DIR, c3[0], c3[1], c3[2], self, f2);
    } else if (L.bctype[DIR] == 1) {
      gv = self;
    } else {
      const int bo = L.bcoff[slot * G::F + DIR];
      const double bcv = bo < 0 ? 0.0 : L.bcval[bo + G::tindex(AXIS, c3[0], c3[1], c3[2])];
      gv = 2.0 * bcv - self;
    }
  }
  int p3[3] = {c3[0] + 1, c3[1] + 1, c3[2] + 1};
  p3[AXIS] = SIDE ? N + 1 : 0;
  tix = TT::idx(p3[0], p3[1], p3[2]);
  return gv;
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Interior cells of colour X into tile T as asynchronous 8-byte copies
// (LDGSTS): every load of the block is in flight at once, no register staging.
// The caller waits with cp_async_wait_all() + __syncthreads().
template <int D, int N>
__device__ __forceinline__ void load_tile_interior_async(double* __restrict__ T,
                                                         const double* __restrict__ src, int X) {
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  constexpr int HN = N / 2;
#pragma unroll
  for (int e = threadIdx.x; e < G::H; e += TT::THREADS) {
    const int m = e % HN, rr = e / HN;
    const int j = rr % N, k = D == 3 ? rr / N : 0;
    const int ip = 2 * m + ((X + j + k) & 1) + 1;
    cp_async8(&T[TT::idx(ip, j + 1, k + 1)], src + e);
  }
}

// Face ghosts of colour X (adjacent interior cells have colour 1-X).
template <int D, int N>
__device__ __forceinline__ void load_tile_halo(double* __restrict__ T, const LevelView& L,
                                               const LevelView& Lc, int slot, int X);

// Fill tile T with colour X of block `slot` (interior + face ghosts of colour X).
// The interior goes in asynchronously; the caller must cp_async_wait_all() and
// __syncthreads() before reading T.
template <int D, int N>
__device__ __forceinline__ void load_tile(double* __restrict__ T, const LevelView& L,
                                          const LevelView& Lc, int slot, int X) {
  using G = Geo<D, N>;
  load_tile_interior_async<D, N>(T, L.phi + (size_t)slot * G::NI + (size_t)X * G::H, X);
  load_tile_halo<D, N>(T, L, Lc, slot, X);
}

template <int D, int N>
__device__ __forceinline__ void load_tile_halo(double* __restrict__ T, const LevelView& L,
                                               const LevelView& Lc, int slot, int X) {
  using G = Geo<D, N>;
  // face ghosts of colour X: adjacent interior cell has colour 1-X
  using TT = Tile<D, N>;
  constexpr int HT = G::NT / 2;  // ghost cells of one colour per face
  constexpr int NQ = G::F * HT;
  constexpr int PER = (NQ + TT::THREADS - 1) / TT::THREADS;
  const double* __restrict__ oth = L.phi + (size_t)slot * G::NI + (size_t)(1 - X) * G::H;
  // all gathers of this thread are issued before any shared-memory store
  double v[PER];
  int tix[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int q = threadIdx.x + u * TT::THREADS;
    tix[u] = -1;
    if (q >= NQ) continue;
    const int dir = q / HT, r = q % HT;  // dir is warp-uniform when HT >= 32
    switch (dir) {
      case 0: v[u] = halo_cell<D, N, 0, 0>(tix[u], L, Lc, slot, X, r, oth); break;
      case 1: v[u] = halo_cell<D, N, 0, 1>(tix[u], L, Lc, slot, X, r, oth); break;
      case 2: v[u] = halo_cell<D, N, 1, 0>(tix[u], L, Lc, slot, X, r, oth); break;
      case 3: v[u] = halo_cell<D, N, 1, 1>(tix[u], L, Lc, slot, X, r, oth); break;
      case 4: if (D == 3) v[u] = halo_cell<D, N, 2 % D, 0>(tix[u], L, Lc, slot, X, r, oth); break;
      default: if (D == 3) v[u] = halo_cell<D, N, 2 % D, 1>(tix[u], L, Lc, slot, X, r, oth); break;
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (tix[u] >= 0) T[tix[u]] = v[u];
}

// Neighbour values of interior cell (i,j,k) from the tile of the opposite colour.
template <int D, int N>
__device__ __forceinline__ void tile_nbrs(const double* __restrict__ T, int i, int j, int k,
                                          double* p) {
  using TT = Tile<D, N>;
  const int ip = i + 1, jp = j + 1, kp = k + 1;
  p[0] = T[TT::idx(ip - 1, jp, kp)];
  p[1] = T[TT::idx(ip + 1, jp, kp)];
  p[2] = T[TT::idx(ip, jp - 1, kp)];
  p[3] = T[TT::idx(ip, jp + 1, kp)];
  if (D == 3) {
    p[4] = T[TT::idx(ip, jp, kp - 1)];
    p[5] = T[TT::idx(ip, jp, kp + 1)];
  }
}

// GS update value of cell with neighbours p, rhs g, row r (-1 uniform row in an
// interface block), kind: multigrid.hpp:633-684.
template <int D>
__device__ __forceinline__ double gs_value(const LevelView& L, const double* __restrict__ phi_b,
                                          uint8_t kind, int r, const double* p, double g) {
  const double h2 = L.h2;
  if (kind == KIND_UNIFORM) {
    if (D == 3) return div6(p[0] + p[1] + p[2] + p[3] + p[4] + p[5] - h2 * g);
    return 0.25 * (p[0] + p[1] + p[2] + p[3] - h2 * g);
  }
  if (r < 0) {
    double s = -h2 * g;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return -s * (-1.0 / (2.0 * D));
  }
  double num = g;
  for (int d = 0; d < 2 * D; ++d) {
    num -= L.r_nb[r * 2 * D + d] * p[d];
    const double b = L.r_bc[r * 2 * D + d];
    if (b != 0) num -= b * phi_b[L.r_obj[r * 2 * D + d]];
  }
  return num / L.r_center[r];
}

// L(phi) (apply_block) / residual from self and neighbours; r = row (-1 uniform).
template <int D>
__device__ __forceinline__ double apply_value(const LevelView& L,
                                             const double* __restrict__ phi_b, int r,
                                             double self, const double* p) {
  if (r < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return s * L.w;
  }
  // special row from the level's row-coefficient table (capi.cu
  // build_row_coef: center, nb[6], bc * phi_b[obj] per cut side, side mask),
  // so the row costs one round trip after its code: the same products and
  // order as center*self + sum(nb p + bc phi_b) (stencil.hpp:273-284)
  (void)phi_b;
  const double2* c2 = reinterpret_cast<const double2*>(L.r_coef) + (size_t)r * 8;
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
template <int D>
__device__ __forceinline__ double resid_value(const LevelView& L,
                                             const double* __restrict__ phi_b, int r,
                                             double self, const double* p, double g) {
  if (r < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return g - s * L.w;
  }
  return g - apply_value<D>(L, phi_b, r, self, p);
}

}  // namespace pmgdev

// tile_kernels.cuh -- the CTA-per-block level kernels (one CTA = one block).
//
// Thread/cell mapping: thread t owns the entries e = t + q*THREADS (q < PER)
// of a colour half.  THREADS is a multiple of N/2, so every owned entry has the
// same x-slot m = e % (N/2) and rows advancing by a compile-time stride; the
// tile slot B = rowbase(j,k) + m of an entry is colour independent and all six
// neighbours sit at fixed offsets from it:
//     own colour  : T_c[B + o]
//     x-, x+      : T_{1-c}[B], T_{1-c}[B + 1]
//     y-, y+      : T_{1-c}[B + o -+ RW]
//     z-, z+      : T_{1-c}[B + o -+ RW*P]
// with o = (c + j + k) & 1.  Per-cell index arithmetic disappears, leaving the
// loads and the reference's floating-point operations.
#pragma once
#include "tiles.cuh"

namespace pmgdev {

template <int D, int N>
struct Own {
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  static constexpr int HN = N / 2;
  static constexpr int THR = TT::THREADS;
  static constexpr int PER = G::H / THR;
  static constexpr int RS = THR / HN;  // rows advanced per q step
  static constexpr int RW = TT::RW;
  static constexpr int ZS = D == 3 ? TT::RW * TT::P : 0;  // z stride in a tile
  // row / slot of owned entry q
  __device__ __forceinline__ static void at(int q, int& j, int& k, int& B) {
    const int row = (int)(threadIdx.x / HN) + RS * q;
    j = row % N;
    k = D == 3 ? row / N : 0;
    B = (D == 3 ? ((k + 1) * TT::P + (j + 1)) : (j + 1)) * RW + (int)(threadIdx.x % HN);
  }
};

// self, neighbours of the colour-c cell at slot B (tile Tc own colour, To opposite)
template <int D, int N>
__device__ __forceinline__ void nbrs_at(const double* __restrict__ To, int B, int o, double* p) {
  using O = Own<D, N>;
  p[0] = To[B];
  p[1] = To[B + 1];
  p[2] = To[B + o - O::RW];
  p[3] = To[B + o + O::RW];
  if (D == 3) {
    p[4] = To[B + o - O::ZS];
    p[5] = To[B + o + O::ZS];
  }
}

// ------------------------------------------------------------------ halo, split phases
// Face-ghost cells of colour X owned by this thread, loaded in three phases so
// that no load waits on another avoidable one: (1) the same-level neighbour
// slots, issued before the interior loads; (2) the ghost values (a plain load
// from the neighbour for same-level faces; the fill formula for physical and
// coarse-fine faces); (3) the shared-memory stores.
template <int D, int N>
struct Halo {
  using G = Geo<D, N>;
  static constexpr int HT = G::NT / 2;
  static constexpr int NQ = G::F * HT;
  static constexpr int PER = (NQ + Tile<D, N>::THREADS - 1) / Tile<D, N>::THREADS;
  int ns[PER];   // same-level neighbour slot of the face (-1 none, -2 not mine)
  int cn[PER];   // coarse neighbour slot (coarse-fine face) or -1
  int bo[PER];   // Dirichlet face-value offset or -1 (value 0)
  int tix[PER];
  double v[PER];

  __device__ __forceinline__ void prefetch(const LevelView& L, int slot) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = threadIdx.x + u * Tile<D, N>::THREADS;
      const int f = slot * G::F + q / HT;
      ns[u] = q < NQ ? nbr_slot<D>(L, slot, q / HT) : -2;
      cn[u] = (q < NQ && !L.dense) ? L.cnbr[f] : -1;
      bo[u] = (q < NQ && !L.bczero) ? L.bcoff[f] : -1;
    }
  }
  template <int AXIS, int SIDE>
  __device__ __forceinline__ void one(int u, const LevelView& L, const LevelView& Lc, int slot,
                                      int X, int r) {
    using TT = Tile<D, N>;
    constexpr int DIR = 2 * AXIS + SIDE;
    constexpr int AC = SIDE ? N - 1 : 0;
    int c3[3] = {0, 0, 0};
    if (D == 2) {
      c3[AXIS] = AC;
      c3[1 - AXIS] = 2 * r + ((1 - X + AC) & 1);
    } else {
      constexpr int A0 = AXIS == 0 ? 1 : 0;
      constexpr int A1 = AXIS == 2 ? 1 : 2;
      const int t1 = r / (N / 2);
      c3[AXIS] = AC;
      c3[A1] = t1;
      c3[A0] = 2 * (r % (N / 2)) + ((1 - X + AC + t1) & 1);
    }
    int p3[3] = {c3[0] + 1, c3[1] + 1, c3[2] + 1};
    p3[AXIS] = SIDE ? N + 1 : 0;
    tix[u] = TT::idx(p3[0], p3[1], p3[2]);
    if (ns[u] >= 0) {  // same-level copy (mesh.hpp:485-498)
      int w3[3] = {c3[0], c3[1], c3[2]};
      w3[AXIS] = SIDE ? 0 : N - 1;
      v[u] = L.phi[(size_t)ns[u] * G::NI + (size_t)X * G::H + G::entry(w3[0], w3[1], w3[2])];
      return;
    }
    const double self = L.phi[(size_t)slot * G::NI + (size_t)(1 - X) * G::H + G::entry(c3[0], c3[1], c3[2])];
    if (cn[u] >= 0) {  // coarse-fine (mesh.hpp:500-535)
      int w3[3] = {c3[0], c3[1], c3[2]};
      w3[AXIS] = SIDE ? N - 2 : 1;
      const double f2 = L.phi[(size_t)slot * G::NI + (size_t)X * G::H + G::entry(w3[0], w3[1], w3[2])];
      v[u] = cf_ghost<D, N>(L, Lc, slot, DIR, c3[0], c3[1], c3[2], self, f2);
    } else if (L.bctype[DIR] == 1) {  // Neumann (mesh.hpp:545-546)
      v[u] = self;
    } else {  // Dirichlet (mesh.hpp:548-550)
      const double bcv = bo[u] < 0 ? 0.0 : L.bcval[bo[u] + G::tindex(AXIS, c3[0], c3[1], c3[2])];
      v[u] = 2.0 * bcv - self;
    }
  }
  __device__ __forceinline__ void issue(const LevelView& L, const LevelView& Lc, int slot, int X) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = threadIdx.x + u * Tile<D, N>::THREADS;
      if (q >= NQ) continue;
      const int dir = q / HT, r = q % HT;  // dir is warp-uniform when HT >= 32
      switch (dir) {
        case 0: one<0, 0>(u, L, Lc, slot, X, r); break;
        case 1: one<0, 1>(u, L, Lc, slot, X, r); break;
        case 2: one<1, 0>(u, L, Lc, slot, X, r); break;
        case 3: one<1, 1>(u, L, Lc, slot, X, r); break;
        case 4: if (D == 3) one<2 % D, 0>(u, L, Lc, slot, X, r); break;
        default: if (D == 3) one<2 % D, 1>(u, L, Lc, slot, X, r); break;
      }
    }
  }
  __device__ __forceinline__ void store(double* __restrict__ T) const {
#pragma unroll
    for (int u = 0; u < PER; ++u)
      if (threadIdx.x + u * Tile<D, N>::THREADS < NQ) T[tix[u]] = v[u];
  }
};

// ------------------------------------------------------------------ GS-RB half-sweep
// All loads of the CTA are issued before any is consumed: neighbour slots,
// then the opposite colour and the rhs (registers), then the halo values;
// then one round of shared-memory stores, a barrier, and the updates.
template <int D, int N>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_gs_tile(LevelView L, LevelView Lc,
                                                                 const double* __restrict__ phi_b,
                                                                 int parity,
                                                                 const int32_t* __restrict__ list) {
  pdl_begin();
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  using O = Own<D, N>;
  __shared__ double T[TT::SIZE];
  const int slot = list ? list[blockIdx.x] : blockIdx.x;
  const int c = parity, X = 1 - c;
  const size_t base = (size_t)slot * G::NI;
  Halo<D, N> h;
  h.prefetch(L, slot);
  const uint8_t kind = L.kind[slot];
  const int sr = L.srow[slot];
  const double* __restrict__ src = L.phi + base + (size_t)X * G::H;
  const double* __restrict__ g = L.rhs + base + (size_t)c * G::H;
  double ov[O::PER], gv[O::PER];
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    const int e = threadIdx.x + q * O::THR;
    ov[q] = src[e];
    gv[q] = g[e];
  }
  // interface blocks: the row indices of this thread's cells, prefetched
  int rq[O::PER];
  const int32_t* rowp = sr < 0 ? nullptr : L.row_of + (size_t)sr * G::NI + c * G::H;
#pragma unroll
  for (int q = 0; q < O::PER; ++q) rq[q] = rowp ? rowp[threadIdx.x + q * O::THR] : -1;
  h.issue(L, Lc, slot, X);
  if (kind == KIND_ALL_INSIDE) return;  // whole CTA: no barrier is skipped unevenly
  double* __restrict__ dst = L.phi + base + (size_t)c * G::H;
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    int j, k, B;
    O::at(q, j, k, B);
    T[B + ((X + j + k) & 1)] = ov[q];
  }
  h.store(T);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    int j, k, B;
    O::at(q, j, k, B);
    const int e = threadIdx.x + q * O::THR;
    const int r = rq[q];
    if (r >= 0 && L.r_mask[r] == 1) continue;
    double p[2 * D];
    nbrs_at<D, N>(T, B, (c + j + k) & 1, p);
    dst[e] = gs_value<D>(L, phi_b, kind, r, p, gv[q]);
  }
}

// ------------------------------------------------------------------ lean GS-RB for interior blocks
// Blocks whose stencil is uniform and whose 2D faces all have a same-level
// neighbour (about two thirds of a uniform level) need none of the physical /
// coarse-fine / interface machinery: the halo is a plain gather and the
// update is the constant-coefficient formula.  Fewer registers per thread let
// more CTAs share an SM, which is what hides the DRAM latency here.
template <int D, int N>
struct Lean {
  using G = Geo<D, N>;
  static constexpr int THR = G::H < 512 ? G::H : 512;
  static constexpr int PER = G::H / THR;
  static constexpr int HN = N / 2;
  static constexpr int RS = THR / HN;
  static constexpr int HT = G::NT / 2;
  static constexpr int HQ = G::F * HT;
  static constexpr int HPER = (HQ + THR - 1) / THR;
};

template <int D, int N, int AXIS, int SIDE>
__device__ __forceinline__ double lean_halo(const LevelView& L, int ns, int X, int r, int& tix,
                                            int slot) {
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  constexpr int AC = SIDE ? N - 1 : 0;
  int c3[3] = {0, 0, 0};
  if (D == 2) {
    c3[AXIS] = AC;
    c3[1 - AXIS] = 2 * r + ((1 - X + AC) & 1);
  } else {
    constexpr int A0 = AXIS == 0 ? 1 : 0;
    constexpr int A1 = AXIS == 2 ? 1 : 2;
    const int t1 = r / (N / 2);
    c3[AXIS] = AC;
    c3[A1] = t1;
    c3[A0] = 2 * (r % (N / 2)) + ((1 - X + AC + t1) & 1);
  }
  int p3[3] = {c3[0] + 1, c3[1] + 1, c3[2] + 1};
  p3[AXIS] = SIDE ? N + 1 : 0;
  tix = TT::idx(p3[0], p3[1], p3[2]);
  if (ns < 0) {  // physical face: Dirichlet 2 bc - f1 / Neumann f1 (mesh.hpp:538-552)
    constexpr int DIR = 2 * AXIS + SIDE;
    const double self = L.phi[(size_t)slot * G::NI + (size_t)(1 - X) * G::H + G::entry(c3[0], c3[1], c3[2])];
    if (L.bctype[DIR] == 1) return self;
    double bcv = 0.0;
    if (!L.bczero) {
      const int bo = L.bcoff[slot * G::F + DIR];
      if (bo >= 0) bcv = L.bcval[bo + G::tindex(AXIS, c3[0], c3[1], c3[2])];
    }
    return 2.0 * bcv - self;
  }
  c3[AXIS] = SIDE ? 0 : N - 1;
  return L.phi[(size_t)ns * G::NI + (size_t)X * G::H + G::entry(c3[0], c3[1], c3[2])];
}

template <int D, int N>
__global__ void __launch_bounds__(Lean<D, N>::THR) k_gs_lean(LevelView L, int parity,
                                                            const int32_t* __restrict__ list) {
  pdl_begin();
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  using LN = Lean<D, N>;
  __shared__ double T[TT::SIZE];
  const int slot = list[blockIdx.x];
  const int c = parity, X = 1 - c;
  const int t = threadIdx.x;
  const size_t base = (size_t)slot * G::NI;
  const uint8_t kind = L.kind[slot];
  int ns[LN::HPER];
#pragma unroll
  for (int u = 0; u < LN::HPER; ++u) {
    const int q = t + u * LN::THR;
    ns[u] = q < LN::HQ ? nbr_slot<D>(L, slot, q / LN::HT) : 0;  // -1: physical face
  }
  double ov[LN::PER], gv[LN::PER];
#pragma unroll
  for (int q = 0; q < LN::PER; ++q) {
    ov[q] = L.phi[base + (size_t)X * G::H + t + q * LN::THR];
    gv[q] = L.rhs[base + (size_t)c * G::H + t + q * LN::THR];
  }
  double hv[LN::HPER];
  int hix[LN::HPER];
#pragma unroll
  for (int u = 0; u < LN::HPER; ++u) {
    const int q = t + u * LN::THR;
    hix[u] = -1;
    if (q >= LN::HQ) continue;
    const int dir = q / LN::HT, r = q % LN::HT;
    switch (dir) {
      case 0: hv[u] = lean_halo<D, N, 0, 0>(L, ns[u], X, r, hix[u], slot); break;
      case 1: hv[u] = lean_halo<D, N, 0, 1>(L, ns[u], X, r, hix[u], slot); break;
      case 2: hv[u] = lean_halo<D, N, 1, 0>(L, ns[u], X, r, hix[u], slot); break;
      case 3: hv[u] = lean_halo<D, N, 1, 1>(L, ns[u], X, r, hix[u], slot); break;
      case 4: if (D == 3) hv[u] = lean_halo<D, N, 2 % D, 0>(L, ns[u], X, r, hix[u], slot); break;
      default: if (D == 3) hv[u] = lean_halo<D, N, 2 % D, 1>(L, ns[u], X, r, hix[u], slot); break;
    }
  }
  const int m = t % LN::HN;
  const int row0 = t / LN::HN;
#pragma unroll
  for (int q = 0; q < LN::PER; ++q) {
    const int row = row0 + LN::RS * q;
    const int j = row % N, k = D == 3 ? row / N : 0;
    const int B = (D == 3 ? ((k + 1) * TT::P + (j + 1)) : (j + 1)) * TT::RW + m;
    T[B + ((X + j + k) & 1)] = ov[q];
  }
#pragma unroll
  for (int u = 0; u < LN::HPER; ++u)
    if (hix[u] >= 0) T[hix[u]] = hv[u];
  __syncthreads();
  double* __restrict__ dst = L.phi + base + (size_t)c * G::H;
  const double h2 = L.h2;
  if (kind == KIND_ALL_INSIDE) return;  // every cell pinned
  if (kind == KIND_UNIFORM) {
#pragma unroll
    for (int q = 0; q < LN::PER; ++q) {
      const int row = row0 + LN::RS * q;
      const int j = row % N, k = D == 3 ? row / N : 0;
      const int B = (D == 3 ? ((k + 1) * TT::P + (j + 1)) : (j + 1)) * TT::RW + m;
      const int o = (c + j + k) & 1;
      double v;
      if (D == 3)  // multigrid.hpp:651-653
        v = div6(T[B] + T[B + 1] + T[B + o - TT::RW] + T[B + o + TT::RW] + T[B + o - TT::RW * TT::P] +
                 T[B + o + TT::RW * TT::P] - h2 * gv[q]);
      else  // multigrid.hpp:640-641
        v = 0.25 * (T[B] + T[B + 1] + T[B + o - TT::RW] + T[B + o + TT::RW] - h2 * gv[q]);
      dst[t + q * LN::THR] = v;
    }
    return;
  }
  // interface block: the uniform-row formula of multigrid.hpp:667-672 for
  // every uniform row; special rows are left alone (inside rows keep their
  // pin, cut rows are updated by k_gs_fix, which still reads their old value
  // for a physical-face ghost 2bc - f1)
  const int32_t* __restrict__ rof = L.row_of + (size_t)L.srow[slot] * G::NI + (size_t)c * G::H;
#pragma unroll
  for (int q = 0; q < LN::PER; ++q) {
    if (rof[t + q * LN::THR] >= 0) continue;
    const int row = row0 + LN::RS * q;
    const int j = row % N, k = D == 3 ? row / N : 0;
    const int B = (D == 3 ? ((k + 1) * TT::P + (j + 1)) : (j + 1)) * TT::RW + m;
    const int o = (c + j + k) & 1;
    double sv = -h2 * gv[q];
    sv += T[B];
    sv += T[B + 1];
    sv += T[B + o - TT::RW];
    sv += T[B + o + TT::RW];
    if (D == 3) {
      sv += T[B + o - TT::RW * TT::P];
      sv += T[B + o + TT::RW * TT::P];
    }
    dst[t + q * LN::THR] = -sv * (-1.0 / (2.0 * D));
  }
}

// Cut rows of lean interface blocks (k_gs_lean skips every special row): the
// boundary-modified update of multigrid.hpp:674-684.  One thread per cut cell
// of the active colour; inside rows are never written, so they keep their pin.
template <int D, int N>
__global__ void __launch_bounds__(128) k_gs_fix(LevelView L, LevelView Lc,
                                               const double* __restrict__ phi_b, int parity,
                                               const int2* __restrict__ cells, int n) {
  pdl_begin();
  using G = Geo<D, N>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 se = cells[i];
  gs_cell<D, N>(L, Lc, phi_b, se.x, parity, se.y);
}

// Both colour tiles (interiors + optional halos), register-staged; the caller
// issues its own extra loads between load_both_issue and load_both_store.
template <int D, int N>
struct Both {
  using O = Own<D, N>;
  double v0[O::PER], v1[O::PER];
  Halo<D, N> h0, h1;
  bool halo;
  __device__ __forceinline__ void issue(const LevelView& L, const LevelView& Lc, int slot,
                                        bool with_halo) {
    using G = Geo<D, N>;
    halo = with_halo;
    if (halo) {
      h0.prefetch(L, slot);
      h1.prefetch(L, slot);
    }
    const size_t base = (size_t)slot * G::NI;
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      const int e = threadIdx.x + q * O::THR;
      v0[q] = L.phi[base + e];
      v1[q] = L.phi[base + G::H + e];
    }
    if (halo) {
      h0.issue(L, Lc, slot, 0);
      h1.issue(L, Lc, slot, 1);
    }
  }
  __device__ __forceinline__ void store(double* __restrict__ T0, double* __restrict__ T1) const {
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      int j, k, B;
      O::at(q, j, k, B);
      const int o0 = (j + k) & 1;  // colour 0 sits at B + o0, colour 1 at B + (1 - o0)
      T0[B + o0] = v0[q];
      T1[B + 1 - o0] = v1[q];
    }
    if (halo) {
      h0.store(T0);
      h1.store(T1);
    }
  }
};

template <int D, int N>
__device__ __forceinline__ void load_both(double* __restrict__ T0, double* __restrict__ T1,
                                          const LevelView& L, const LevelView& Lc, int slot,
                                          bool halo) {
  Both<D, N> b;
  b.issue(L, Lc, slot, halo);
  b.store(T0, T1);
}

// ------------------------------------------------------------------ restriction (+ residual)
// Thread t owns an x-pair of fine cells (the two colours of one entry, which
// share a parent cell) -- for D=3 in both rows of a z-pair -- and its y-partner
// row is the lane HN above.  The 2^D children are summed in the reference's
// x-fastest order (multigrid.hpp:706-721) by the even-j lane; parent phi is
// pinned where the parent row is inside (apply_pins(l-1)); the restricted
// residual (or rhs) goes to the parent's rhs slot for k_fas.
template <int D, int N, int MODE>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_restrict_tile(LevelView Lf, LevelView Lfc,
                                                                       LevelView Lp,
                                                                       const double* __restrict__ phi_b,
                                                                       const int32_t* __restrict__ list = nullptr) {
  pdl_begin();
  if (!list && !owned(Lf, blockIdx.x)) return;  // multi-GPU: another rank's block (lists hold own blocks)
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  constexpr int HN = N / 2;
  constexpr int THR = TT::THREADS;
  // D=3: z-pair groups processed per step; D=2: rows per step
  constexpr int ZG = D == 3 ? (THR / (HN * N) > 0 ? THR / (HN * N) : 1) : 1;
  constexpr int RPS = D == 2 ? THR / HN : N;
  constexpr int STEPS = D == 3 ? ((N / 2) + ZG - 1) / ZG : (N + RPS - 1) / RPS;
  __shared__ double T0s[TT::SIZE];
  __shared__ double T1s[TT::SIZE];
  const int slot = list ? list[blockIdx.x] : (int)blockIdx.x;
  const size_t base = (size_t)slot * G::NI;
  const uint8_t kind = Lf.kind[slot];
  const int fsr = Lf.srow[slot];
  const int P = Lf.parent[slot];
  int cp[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) cp[a] = (Lf.coords[slot * D + a] & 1) * HN;
  const int t = threadIdx.x;
  const int m = t % HN;
  const unsigned mask = THR >= 32 ? 0xffffffffu : ((1u << THR) - 1u);
  Both<D, N> both;
  both.issue(Lf, Lfc, slot, MODE == RM_FUSED);
  // every other global value this thread needs, in flight with the fields:
  // the restricted quantity (or g for the residual), the special-row kind of
  // each cell and of the parent cell (skind: only a cut row needs its row index)
  auto where = [&](int step, int& kp, int& jj) {
    if (D == 3) {
      kp = t / (HN * N) + ZG * step;  // z-pair index
      jj = (t / HN) % N;
    } else {
      kp = 0;
      jj = t / HN + RPS * step;
    }
    return D == 3 ? kp < N / 2 : jj < N;
  };
  double gq[STEPS][2][2];
  int8_t skq[STEPS][2][2], psk[STEPS];
  int rwq[STEPS][2][2];
  const int psr = Lp.srow[P];
#pragma unroll
  for (int step = 0; step < STEPS; ++step) {
    int kp, jj;
    const bool active = where(step, kp, jj);
    psk[step] = 0;
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        gq[step][dz][x] = 0.0;
        skq[step][dz][x] = 0;
        rwq[step][dz][x] = -1;
      }
    if (!active) continue;
    for (int dz = 0; dz < (D == 3 ? 2 : 1); ++dz) {
      const int kk = D == 3 ? 2 * kp + dz : 0;
      const int c0 = (jj + kk) & 1;  // colour of i = 2m
      const int e = m + HN * (jj + N * kk);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int cc = x ? 1 - c0 : c0;
        const size_t a = base + (size_t)cc * G::H + e;
        gq[step][dz][x] = MODE == RM_RES ? Lf.res[a] : Lf.rhs[a];
        if (MODE == RM_FUSED && kind != KIND_UNIFORM) {
          skq[step][dz][x] = Lf.skind[(size_t)fsr * G::NI + (size_t)cc * G::H + e];
          rwq[step][dz][x] = Lf.row_of[(size_t)fsr * G::NI + (size_t)cc * G::H + e];
        }
      }
    }
    if (!(jj & 1) && psr >= 0) {
      const int pi = cp[0] + m, pj = cp[1] + (jj >> 1), pk = D == 3 ? cp[2] + kp : 0;
      psk[step] = Lp.skind[(size_t)psr * G::NI + (size_t)(G::colour(pi, pj, pk) * G::H + G::entry(pi, pj, pk))];
    }
  }
  both.store(T0s, T1s);
  cp_async_wait_all();
  __syncthreads();
  auto cell = [&](int jj, int kk, int cc, double g, int sk, int r, double& phi_out) -> double {
    const int B = (D == 3 ? ((kk + 1) * TT::P + (jj + 1)) : (jj + 1)) * TT::RW + m;
    const int o = (cc + jj + kk) & 1;
    const double* Tc = cc ? T1s : T0s;
    const double* To = cc ? T0s : T1s;
    const double self = Tc[B + o];
    phi_out = self;
    if (MODE != RM_FUSED) return g;
    if (sk == 1) return 0.0;
    double p[2 * D];
    nbrs_at<D, N>(To, B, o, p);
    return resid_value<D>(Lf, phi_b, r, self, p, g);
  };
#pragma unroll
  for (int step = 0; step < STEPS; ++step) {
    int kp, jj;
    const bool active = where(step, kp, jj);
    double r_[2][2] = {{0, 0}, {0, 0}}, f_[2][2] = {{0, 0}, {0, 0}};  // [z][x]
    if (active) {
      for (int dz = 0; dz < (D == 3 ? 2 : 1); ++dz) {
        const int kk = D == 3 ? 2 * kp + dz : 0;
        const int c0 = (jj + kk) & 1;  // colour of i = 2m
        r_[dz][0] = cell(jj, kk, c0, gq[step][dz][0], skq[step][dz][0], rwq[step][dz][0], f_[dz][0]);
        r_[dz][1] = cell(jj, kk, 1 - c0, gq[step][dz][1], skq[step][dz][1], rwq[step][dz][1], f_[dz][1]);
      }
    }
    double pr[2][2], pf[2][2];  // the y+1 partner's values
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx) {
        pr[dz][dx] = __shfl_down_sync(mask, r_[dz][dx], HN);
        pf[dz][dx] = __shfl_down_sync(mask, f_[dz][dx], HN);
      }
    if (!active || (jj & 1)) continue;
    // sum = 0; sum += child for children in x-fastest order
    double sr = 0.0, sf = 0.0;
    for (int dz = 0; dz < (D == 3 ? 2 : 1); ++dz) {
      sr += r_[dz][0];
      sf += f_[dz][0];
      sr += r_[dz][1];
      sf += f_[dz][1];
      sr += pr[dz][0];
      sf += pf[dz][0];
      sr += pr[dz][1];
      sf += pf[dz][1];
    }
    const int pi = cp[0] + m, pj = cp[1] + (jj >> 1), pk = D == 3 ? cp[2] + kp : 0;
    const int pc = G::colour(pi, pj, pk), pe = G::entry(pi, pj, pk);
    const size_t pa = (size_t)P * G::NI + (size_t)(pc * G::H + pe);
    double vphi = sf / (double)(1 << D);
    if (psk[step] == 1) vphi = phi_b[Lp.r_pin[Lp.row_of[(size_t)psr * G::NI + (size_t)(pc * G::H + pe)]]];
    Lp.phi[pa] = vphi;
    Lp.rhs[pa] = sr / (double)(1 << D);
  }
}

// ------------------------------------------------------------------ FAS + OLD snapshot
template <int D, int N, bool FAS>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_fas_tile(LevelView L, LevelView Lc,
                                                                  const double* __restrict__ phi_b,
                                                                  const int32_t* __restrict__ list) {
  pdl_begin();
  if (!list && !owned(L, blockIdx.x)) return;  // multi-GPU: another rank's block (lists hold own blocks)
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  using O = Own<D, N>;
  __shared__ double T0[TT::SIZE];
  __shared__ double T1[TT::SIZE];
  const int slot = list ? list[blockIdx.x] : (int)blockIdx.x;
  const size_t base = (size_t)slot * G::NI;
  if (!FAS || L.leaf[slot]) {
    for (int ce = threadIdx.x; ce < G::NI; ce += blockDim.x) L.old[base + ce] = L.phi[base + ce];
    return;
  }
  const uint8_t kind = L.kind[slot];
  const int sr = L.srow[slot];
  Both<D, N> b;
  b.issue(L, Lc, slot, true);
  double rq[2][O::PER];
  int8_t skq[2][O::PER];  // special-row kinds and row indices, in flight with the fields (k_record_tile)
  int rwq[2][O::PER];
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    const int e = threadIdx.x + q * O::THR;
    rq[0][q] = L.rhs[base + e];
    rq[1][q] = L.rhs[base + G::H + e];
    skq[0][q] = kind == KIND_UNIFORM ? (int8_t)0 : L.skind[(size_t)sr * G::NI + e];
    skq[1][q] = kind == KIND_UNIFORM ? (int8_t)0 : L.skind[(size_t)sr * G::NI + G::H + e];
    rwq[0][q] = kind == KIND_UNIFORM ? -1 : L.row_of[(size_t)sr * G::NI + e];
    rwq[1][q] = kind == KIND_UNIFORM ? -1 : L.row_of[(size_t)sr * G::NI + G::H + e];
  }
  b.store(T0, T1);
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    int j, k, B;
    O::at(q, j, k, B);
    const int e = threadIdx.x + q * O::THR;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int o = (c + j + k) & 1;
      const double* Tc = c ? T1 : T0;
      const double* To = c ? T0 : T1;
      const double self = Tc[B + o];
      const int r = rwq[c][q];
      double out;
      if (skq[c][q] == 1) {
        out = 0.0;
      } else {
        double p[2 * D];
        nbrs_at<D, N>(To, B, o, p);
        out = apply_value<D>(L, phi_b, r, self, p);
      }
      const size_t a = base + (size_t)c * G::H + e;
      L.rhs[a] = out + rq[c][q];  // g[c] += r[c] after apply_block (multigrid.hpp:388-392)
      L.old[a] = self;
    }
  }
}

// ------------------------------------------------------------------ prolongation
// The parent's delta = phi - old (or phi for FULL) over the fine block's
// octant plus a one-cell halo is staged once (ghosts via phi_at / old_at).
// A thread's entry e is an x-pair (i = 2m, 2m+1) under one parent column:
// both cells share the centre, y and z terms and differ in the x term.
template <int D, int N, bool FULL>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_prolong_tile(LevelView Lf, LevelView Lp,
                                                                      LevelView Lpp) {
  pdl_begin();
  if (!owned(Lf, blockIdx.x)) return;  // multi-GPU: another rank's block
  using G = Geo<D, N>;
  using O = Own<D, N>;
  constexpr int HN = N / 2;
  constexpr int PE = HN + 2;  // delta tile extent
  constexpr int PS = D == 2 ? PE * PE : PE * PE * PE;
  __shared__ double Dt[PS];
  const int slot = blockIdx.x;
  const size_t base = (size_t)slot * G::NI;
  const int P = Lf.parent[slot];
  int cp[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) cp[a] = (Lf.coords[slot * D + a] & 1) * HN;
  // fine values in flight first
  double fv[2][O::PER];  // [h][q]: h = 0 -> cell i = 2m, h = 1 -> i = 2m+1
  int8_t skq[2][O::PER];  // special-row kind (1 = inside: the cell keeps its pin)
  const uint8_t kind = Lf.kind[slot];
  const int sr = Lf.srow[slot];
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    int j, k, B;
    O::at(q, j, k, B);
    const int e = threadIdx.x + q * O::THR;
    const int c0 = (j + k) & 1;
    fv[0][q] = FULL ? 0.0 : Lf.phi[base + (size_t)c0 * G::H + e];
    fv[1][q] = FULL ? 0.0 : Lf.phi[base + (size_t)(1 - c0) * G::H + e];
    skq[0][q] = kind == KIND_UNIFORM ? (int8_t)0 : Lf.skind[(size_t)sr * G::NI + (size_t)c0 * G::H + e];
    skq[1][q] = kind == KIND_UNIFORM ? (int8_t)0 : Lf.skind[(size_t)sr * G::NI + (size_t)(1 - c0) * G::H + e];
  }
  for (int q = threadIdx.x; q < PS; q += blockDim.x) {
    const int a = q % PE - 1, b = (q / PE) % PE - 1, cc = D == 3 ? q / (PE * PE) - 1 : 0;
    const int out = (a < 0 || a >= HN) + (b < 0 || b >= HN) + (D == 3 && (cc < 0 || cc >= HN));
    if (out > 1) continue;  // edges/corners are never read
    const int pi = cp[0] + a, pj = cp[1] + b, pk = D == 3 ? cp[2] + cc : 0;
    if (FULL)
      Dt[q] = phi_at<D, N>(Lp, Lpp, P, pi, pj, pk);
    else
      Dt[q] = phi_at<D, N>(Lp, Lpp, P, pi, pj, pk) - old_at<D, N>(Lp, P, pi, pj, pk);
  }
  __syncthreads();
  const int m = threadIdx.x % HN;
#pragma unroll
  for (int q = 0; q < O::PER; ++q) {
    int j, k, B;
    O::at(q, j, k, B);
    (void)B;
    const int e = threadIdx.x + q * O::THR;
    const int ty = (j >> 1) + 1, tz = D == 3 ? (k >> 1) + 1 : 0;
    const int sy = (j & 1) ? 1 : -1, sz = (k & 1) ? 1 : -1;
    const int ctr = (D == 3 ? (tz * PE + ty) * PE : ty * PE) + m + 1;
    const double dc = Dt[ctr];
    const double dxm = Dt[ctr - 1], dxp = Dt[ctr + 1];
    const double dy = Dt[ctr + sy * PE];
    const double dz = D == 3 ? Dt[ctr + sz * PE * PE] : 0.0;
    const int c0 = (j + k) & 1;  // colour of i = 2m (x sign -1); i = 2m+1 has +1
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // h = 0: i = 2m, h = 1: i = 2m+1
      const int c = h ? 1 - c0 : c0;
      if (skq[h][q] == 1) continue;
      double v = (1.0 - 0.25 * D) * dc;
      v += 0.25 * (h ? dxp : dxm);
      v += 0.25 * dy;
      if (D == 3) v += 0.25 * dz;
      const size_t a = base + (size_t)c * G::H + e;
      if (FULL)
        Lf.phi[a] = v;
      else
        Lf.phi[a] = fv[h][q] + v;
    }
  }
}

// ------------------------------------------------------------------ residual record
// Per-block partials (max |r|, sum r^2, count) of the leaf cells, written by
// one or two kernels (lean + general block classes, possibly concurrent); the
// CTA that completes the level's count reduces all partials in slot order
// (deterministic, multigrid.hpp:555-561).
// `arrivals` blocks of the level are accounted for by this CTA (1 for the
// one-block-per-CTA kernels; a persistent CTA reports all its blocks at once,
// its totals in partial[slot] and zeros in its other blocks' entries).
__device__ __forceinline__ void record_finish(const LevelView& L, Rec* __restrict__ partial,
                                              Rec* rec, unsigned int* counter, int slot,
                                              double mx, double ss, double cnt, double* sm,
                                              bool* last, unsigned arrivals = 1u) {
  {  // one barrier: warp butterflies, then thread 0 folds the warps in order
     // (the same order as block_max / block_sum)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    mx = warp_max(mx);
    ss = warp_sum(ss);
    cnt = warp_sum(cnt);
    if (lane == 0) {
      sm[wid] = mx;
      sm[24 + wid] = ss;
      sm[48 + wid] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0, s = 0, n = 0;
      for (int w = 0; w < nw; ++w) {
        m = fmax(m, sm[w]);
        s += sm[24 + w];
        n += sm[48 + w];
      }
      mx = m;
      ss = s;
      cnt = n;
    }
  }
  if (threadIdx.x == 0) {
    partial[slot].max = mx;
    partial[slot].sumsq = ss;
    partial[slot].count = (long long)cnt;
    if (counter) {
      __threadfence();
      *last = atomicAdd(counter, arrivals) + arrivals == (unsigned)L.nb;
    } else {
      *last = false;  // folded by k_record_fold
    }
  }
  __syncthreads();
  if (!*last) return;
  __threadfence();
  mx = 0;
  ss = 0;
  double cc = 0;
  for (int b = threadIdx.x; b < L.nb; b += blockDim.x) {
    const volatile Rec* p = partial + b;
    mx = fmax(mx, p->max);
    ss += p->sumsq;
    cc += (double)p->count;
  }
  mx = block_max(mx, sm);
  ss = block_sum(ss, sm);
  cc = block_sum(cc, sm);
  if (threadIdx.x == 0) {
    rec[L.level].max = mx;
    rec[L.level].sumsq = ss;
    rec[L.level].count = (long long)cc;
    *counter = 0;
  }
}

template <int D, int N>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_record_tile(LevelView L, LevelView Lc,
                                                                     const double* __restrict__ phi_b,
                                                                     Rec* __restrict__ partial,
                                                                     Rec* rec, unsigned int* counter,
                                                                     const int32_t* __restrict__ list) {
  pdl_begin();
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  using O = Own<D, N>;
  __shared__ double T0[TT::SIZE];
  __shared__ double T1[TT::SIZE];
  __shared__ double sm[72];
  __shared__ bool last;
  const int slot = list ? list[blockIdx.x] : blockIdx.x;
  const size_t base = (size_t)slot * G::NI;
  double mx = 0, ss = 0, cnt = 0;
  const bool leaf = L.leaf[slot] != 0;
  const uint8_t kind = L.kind[slot];
  const int sr = L.srow[slot];
  double gq[2][O::PER];
  // special-row kinds of this thread's cells (skind: 0 uniform, 1 inside, 2
  // cut), in flight with the fields: only a cut row then needs its row index
  int8_t skq[2][O::PER];
  int rwq[2][O::PER];  // and the row indices (used by the cut rows only)
  if (leaf) {
    Both<D, N> b;
    b.issue(L, Lc, slot, true);
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      const int e = threadIdx.x + q * O::THR;
      gq[0][q] = L.rhs[base + e];
      gq[1][q] = L.rhs[base + G::H + e];
      skq[0][q] = kind == KIND_UNIFORM ? (int8_t)0 : L.skind[(size_t)sr * G::NI + e];
      skq[1][q] = kind == KIND_UNIFORM ? (int8_t)0 : L.skind[(size_t)sr * G::NI + G::H + e];
      rwq[0][q] = kind == KIND_UNIFORM ? -1 : L.row_of[(size_t)sr * G::NI + e];
      rwq[1][q] = kind == KIND_UNIFORM ? -1 : L.row_of[(size_t)sr * G::NI + G::H + e];
    }
    b.store(T0, T1);
  }
  cp_async_wait_all();
  __syncthreads();
  if (leaf) {
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      int j, k, B;
      O::at(q, j, k, B);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (skq[c][q] == 1) continue;
        const int r = rwq[c][q];
        const int o = (c + j + k) & 1;
        double p[2 * D];
        nbrs_at<D, N>(c ? T0 : T1, B, o, p);
        const double self = (c ? T1 : T0)[B + o];
        const double rv = resid_value<D>(L, phi_b, r, self, p, gq[c][q]);
        mx = fmax(mx, fabs(rv));
        ss += rv * rv;
        cnt += 1;
      }
    }
  }
  // without a counter the partials are per list position, folded by k_record_fold
  record_finish(L, partial, rec, counter, counter ? slot : (int)blockIdx.x, mx, ss, cnt, sm, &last);
}

// Lean record for interior uniform blocks: both colours asynchronously into
// shared memory, halos gathered from the same-level neighbours, uniform
// residual g - (sum_6 - 2D phi) w (stencil.hpp:336-342) for every cell.
template <int D, int N>
__global__ void __launch_bounds__(Tile<D, N>::THREADS, Tile<D, N>::MINB) k_record_lean(LevelView L,
                                                                     Rec* __restrict__ partial,
                                                                     Rec* rec, unsigned int* counter,
                                                                     const int32_t* __restrict__ list) {
  pdl_begin();
  using G = Geo<D, N>;
  using TT = Tile<D, N>;
  using O = Own<D, N>;
  using LN = Lean<D, N>;
  constexpr int HPER = (LN::HQ + TT::THREADS - 1) / TT::THREADS;
  __shared__ double T0[TT::SIZE];
  __shared__ double T1[TT::SIZE];
  __shared__ double sm[72];
  __shared__ bool last;
  const int slot = list[blockIdx.x];
  const int t = threadIdx.x;
  const size_t base = (size_t)slot * G::NI;
  double mx = 0, ss = 0, cnt = 0;
  const bool leaf = L.leaf[slot] != 0;
  if (leaf) {
    int ns[HPER];
#pragma unroll
    for (int u = 0; u < HPER; ++u) {
      const int q = t + u * TT::THREADS;
      ns[u] = q < LN::HQ ? nbr_slot<D>(L, slot, q / LN::HT) : 0;  // -1: physical face
    }
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      int j, k, B;
      O::at(q, j, k, B);
      const int e = t + q * O::THR;
      const int o0 = (j + k) & 1;
      cp_async8(&T0[B + o0], L.phi + base + e);
      cp_async8(&T1[B + 1 - o0], L.phi + base + G::H + e);
    }
    double hv[2][HPER];
    int hix[2][HPER];
#pragma unroll
    for (int X = 0; X < 2; ++X)
#pragma unroll
      for (int u = 0; u < HPER; ++u) {
        const int q = t + u * TT::THREADS;
        hix[X][u] = -1;
        if (q >= LN::HQ) continue;
        const int dir = q / LN::HT, r = q % LN::HT;
        switch (dir) {
          case 0: hv[X][u] = lean_halo<D, N, 0, 0>(L, ns[u], X, r, hix[X][u], slot); break;
          case 1: hv[X][u] = lean_halo<D, N, 0, 1>(L, ns[u], X, r, hix[X][u], slot); break;
          case 2: hv[X][u] = lean_halo<D, N, 1, 0>(L, ns[u], X, r, hix[X][u], slot); break;
          case 3: hv[X][u] = lean_halo<D, N, 1, 1>(L, ns[u], X, r, hix[X][u], slot); break;
          case 4: if (D == 3) hv[X][u] = lean_halo<D, N, 2 % D, 0>(L, ns[u], X, r, hix[X][u], slot); break;
          default: if (D == 3) hv[X][u] = lean_halo<D, N, 2 % D, 1>(L, ns[u], X, r, hix[X][u], slot); break;
        }
      }
#pragma unroll
    for (int u = 0; u < HPER; ++u) {
      if (hix[0][u] >= 0) T0[hix[0][u]] = hv[0][u];
      if (hix[1][u] >= 0) T1[hix[1][u]] = hv[1][u];
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (leaf) {
    const double w = L.w;
#pragma unroll
    for (int q = 0; q < O::PER; ++q) {
      int j, k, B;
      O::at(q, j, k, B);
      const int e = t + q * O::THR;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int o = (c + j + k) & 1;
        const double* To = c ? T0 : T1;
        const double self = (c ? T1 : T0)[B + o];
        double s = -2.0 * D * self;
        s += To[B];
        s += To[B + 1];
        s += To[B + o - TT::RW];
        s += To[B + o + TT::RW];
        if (D == 3) {
          s += To[B + o - TT::RW * TT::P];
          s += To[B + o + TT::RW * TT::P];
        }
        const double rv = L.rhs[base + (size_t)c * G::H + e] - s * w;
        mx = fmax(mx, fabs(rv));
        ss += rv * rv;
        cnt += 1;
      }
    }
  }
  // without a counter the partials are per list position, folded by k_record_fold
  record_finish(L, partial, rec, counter, counter ? slot : (int)blockIdx.x, mx, ss, cnt, sm, &last);
}

}  // namespace pmgdev

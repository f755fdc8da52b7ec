// small.cuh -- table-driven per-cell kernels for the small levels.
//
// On a level of at most kSmallLevel blocks the work is a few hundred thousand
// cells that live in L2, and the generic per-cell path is bound by its chain
// of dependent loads (block kind -> interface page -> row -> neighbour slot
// -> value).  The host resolves all of that once (capi.cu build_small_tables):
// per cell, indexed by its colour-split address a,
//   e[0]    row code: r >= 0 cut row, -1 uniform row of a uniform block,
//           -2 uniform row of an interface block, -3 - r inside row r
//   e[1..6] the 2D neighbour addresses (same block or same-level neighbour),
//           -1 Neumann ghost f1, -2 Dirichlet ghost 2 bc - f1 (bc in gbc[6a+d])
//   e[7]    1 if the block is a leaf
// so every operator needs two dependent round trips (entry, then values).
// The arithmetic is the reference's, as in cells.cuh.
#pragma once
#include "kernels.cuh"
#include "tiles.cuh"
#include "cells.cuh"

namespace pmgdev {

// the cell's table entry is static (host-built at setup), its values are not:
// with programmatic dependent launch (PDL) the entry is loaded before
// griddepcontrol.wait, overlapping the previous kernel's drain
template <int D, bool PDL = false>
__device__ __forceinline__ void tab_load(const LevelView& L, const int4* __restrict__ T,
                                         const double* __restrict__ gbc, int a, int& code, int& leaf,
                                         double& self, double* p) {
  const int4 e0 = T[2 * a], e1 = T[2 * a + 1];
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  code = e0.x;
  leaf = e1.w;
  const int na[6] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z};
  self = L.phi[a];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d)
    p[d] = na[d] >= 0 ? L.phi[na[d]] : (na[d] == -1 ? self : 2.0 * gbc[(size_t)a * 6 + d] - self);
}

// The static part of a cell's operator (its table entry, Dirichlet face
// values, a special row's coefficients with bc * phi_b folded), loaded before
// griddepcontrol.wait under PDL; tab_apply evaluates L(phi) at the cell from
// it with the reference's operation order (stencil.hpp:273-322).
template <int D>
struct TabPre {
  int code, leaf;
  int na[2 * D];
  double gb[2 * D], cf[14];
};
template <int D>
__device__ __forceinline__ TabPre<D> tab_pre(const LevelView& L, const int4* __restrict__ T,
                                             const double* __restrict__ gbc, int a) {
  TabPre<D> P;
  const int4 e0 = T[2 * a], e1 = T[2 * a + 1];
  P.code = e0.x;
  P.leaf = e1.w;
  const int na[6] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z};
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) {
    P.na[d] = na[d];
    P.gb[d] = na[d] == -2 ? gbc[(size_t)a * 6 + d] : 0.0;
  }
  if (P.code >= 0) {
    const double2* c2 = reinterpret_cast<const double2*>(L.r_coef) + (size_t)P.code * 8;
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      const double2 v = c2[u];
      P.cf[2 * u] = v.x;
      P.cf[2 * u + 1] = v.y;
    }
  }
  return P;
}
template <int D>
__device__ __forceinline__ void tab_values(const LevelView& L, const TabPre<D>& P, int a, double& self,
                                           double* p) {
  self = L.phi[a];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d)
    p[d] = P.na[d] >= 0 ? L.phi[P.na[d]] : (P.na[d] == -1 ? self : 2.0 * P.gb[d] - self);
}
// L(phi) at a solved cell (code > -3): uniform row (-2D self + sum p) w, special row center self + sum (nb p + bc phi_b)
template <int D>
__device__ __forceinline__ double tab_apply(const LevelView& L, const TabPre<D>& P, double self, const double* p) {
  if (P.code < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return s * L.w;
  }
  const int bm = (int)P.cf[13];
  double s = P.cf[0] * self;
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) {
    s += P.cf[1 + d] * p[d];
    if ((bm >> d) & 1) s += P.cf[7 + d];
  }
  return s;
}

// gsrb_block half-sweep (multigrid.hpp:621-695) of cell gid of the colour
// (gid < nb * H): the body of k_gs_tab.  Everything static -- the cell's
// entry, its Dirichlet face values and a cut row's coefficients (bc * phi_b
// folded, rebuilt with the graphs on set_boundary_value) -- is loaded before
// griddepcontrol.wait (PDL); only phi and g after it.
template <int D, int N, bool PDL = false>
__device__ __forceinline__ void gs_tab_cell(const LevelView& L, const double* __restrict__ phi_b,
                                            const int4* __restrict__ T, const double* __restrict__ gbc, int parity,
                                            int gid) {
  using G = Geo<D, N>;
  if (!owned(L, gid / G::H)) {
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int a = (gid / G::H) * G::NI + parity * G::H + gid % G::H;
  const int4 e0 = T[2 * a], e1 = T[2 * a + 1];
  const int code = e0.x;
  const int na[6] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z};
  double gb[2 * D], cf[14];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) gb[d] = na[d] == -2 ? gbc[(size_t)a * 6 + d] : 0.0;
  if (code >= 0) {
    const double2* c2 = reinterpret_cast<const double2*>(L.r_coef) + (size_t)code * 8;
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      const double2 v = c2[u];
      cf[2 * u] = v.x;
      cf[2 * u + 1] = v.y;
    }
  }
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (code <= -3) return;  // inside: pinned
  const double self = L.phi[a];
  double p[2 * D];
#pragma unroll
  for (int d = 0; d < 2 * D; ++d) p[d] = na[d] >= 0 ? L.phi[na[d]] : (na[d] == -1 ? self : 2.0 * gb[d] - self);
  const double g = L.rhs[a];
  const double h2 = L.h2;
  double nv;
  if (code == -1) {
    if (D == 3)
      nv = div6(p[0] + p[1] + p[2] + p[3] + p[4] + p[5] - h2 * g);  // :651-653
    else
      nv = 0.25 * (p[0] + p[1] + p[2] + p[3] - h2 * g);  // :640-641
  } else if (code == -2) {
    double sv = -h2 * g;  // :668-671
    for (int d = 0; d < 2 * D; ++d) sv += p[d];
    nv = -sv * (-1.0 / (2.0 * D));
  } else {  // :677-683
    const int bm = (int)cf[13];
    double num = g;
#pragma unroll
    for (int d = 0; d < 2 * D; ++d) {
      num -= cf[1 + d] * p[d];
      if ((bm >> d) & 1) num -= cf[7 + d];
    }
    nv = num / cf[0];
  }
  L.phi[a] = nv;
}

template <int D, int N>
__global__ void __launch_bounds__(256) k_gs_tab(LevelView L, const double* __restrict__ phi_b,
                                               const int4* __restrict__ T, const double* __restrict__ gbc,
                                               int parity) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: see tab_load
  using G = Geo<D, N>;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= L.nb * G::H) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  gs_tab_cell<D, N, true>(L, phi_b, T, gbc, parity, gid);
}

// FAS right-hand side g = L(phi) + R(r) on non-leaf blocks, OLD <- PHI
// (multigrid.hpp:380-397) of cell a (a < nb * NI)
template <int D, int N, bool FAS, bool PDL = false>
__device__ __forceinline__ void fas_tab_cell(const LevelView& L, const double* __restrict__ phi_b,
                                             const int4* __restrict__ T, const double* __restrict__ gbc, int a) {
  using G = Geo<D, N>;
  if (!owned(L, a / G::NI)) return;
  if (FAS) {
    const TabPre<D> P = tab_pre<D>(L, T, gbc, a);
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    double self, p[2 * D];
    tab_values<D>(L, P, a, self, p);
    if (!P.leaf) {
      const double out = P.code <= -3 ? 0.0 : tab_apply<D>(L, P, self, p);
      L.rhs[a] = out + L.rhs[a];
    }
    L.old[a] = self;
  } else {
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    L.old[a] = L.phi[a];
  }
}

template <int D, int N, bool FAS>
__global__ void __launch_bounds__(256) k_fas_tab(LevelView L, const double* __restrict__ phi_b,
                                                const int4* __restrict__ T, const double* __restrict__ gbc) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: see tab_load
  using G = Geo<D, N>;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= L.nb * G::NI) return;
  fas_tab_cell<D, N, FAS, true>(L, phi_b, T, gbc, a);
}

// residual + restriction of a small level (multigrid.hpp:374-418, 697-722):
// one thread per child cell, the first lane of each 2^D group sums them in
// x-fastest order, pins the parent (apply_pins(l-1)) and writes it.  gid is
// the child item; every lane of the warp must call it (the group sum is a
// shuffle), items past the level are idle lanes.
template <int D, int N, int MODE, bool PDL = false>
__device__ __forceinline__ void restrict_tab_item(const LevelView& Lf, const LevelView& Lp,
                                                  const double* __restrict__ phi_b, const int4* __restrict__ T,
                                                  const double* __restrict__ gbc, int gid) {
  using G = Geo<D, N>;
  constexpr int NC = G::NC, NQ = G::NI / NC, HN = N / 2;
  const int t = gid / NC, d = gid % NC;
  const int slot = t < Lf.nb * NQ ? t / NQ : 0;
  const bool live = t < Lf.nb * NQ && owned(Lf, slot);
  const int q = live ? t % NQ : 0;
  const int qx = q % HN, qy = (q / HN) % HN, qz = D == 3 ? q / (HN * HN) : 0;
  // static: the parent cell and its pin (the group's first lane) and, fused,
  // the child's operator -- all before griddepcontrol.wait under PDL
  size_t pa = 0;
  bool pinned = false;
  double pin = 0.0;
  if (live && d == 0) {
    const int P = Lf.parent[slot];
    int cp[3] = {0, 0, 0};
    for (int a2 = 0; a2 < D; ++a2) cp[a2] = (Lf.coords[slot * D + a2] & 1) * HN;
    const int pi = cp[0] + qx, pj = cp[1] + qy, pk = D == 3 ? cp[2] + qz : 0;
    pa = (size_t)P * G::NI + (size_t)(G::colour(pi, pj, pk) * G::H + G::entry(pi, pj, pk));
    const int r = row_index<D, N>(Lp, P, G::colour(pi, pj, pk), G::entry(pi, pj, pk));
    if (r >= 0 && Lp.r_mask[r] == 1) pinned = true, pin = phi_b[Lp.r_pin[r]];
  }
  double vphi = 0, vq = 0;
  int a = 0;
  if (live) {
    const int fi = 2 * qx + (d & 1), fj = 2 * qy + ((d >> 1) & 1), fk = D == 3 ? 2 * qz + ((d >> 2) & 1) : 0;
    a = slot * G::NI + G::colour(fi, fj, fk) * G::H + G::entry(fi, fj, fk);
  }
  if (MODE == RM_FUSED) {
    TabPre<D> Pc;
    if (live) Pc = tab_pre<D>(Lf, T, gbc, a);
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (live) {
      double p[2 * D];
      tab_values<D>(Lf, Pc, a, vphi, p);
      vq = Pc.code <= -3 ? 0.0 : Lf.rhs[a] - tab_apply<D>(Lf, Pc, vphi, p);  // stencil.hpp:336-358
    }
  } else {
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (live) {
      vphi = Lf.phi[a];
      vq = MODE == RM_RES ? Lf.res[a] : Lf.rhs[a];
    }
  }
  const int base = threadIdx.x & ~(NC - 1) & 31;
  double sphi = 0, sq = 0;
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    sphi += __shfl_sync(0xffffffffu, vphi, base + u);
    sq += __shfl_sync(0xffffffffu, vq, base + u);
  }
  if (!live || d != 0) return;
  Lp.phi[pa] = pinned ? pin : sphi / (double)NC;
  Lp.rhs[pa] = sq / (double)NC;
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(256) k_restrict_tab(LevelView Lf, LevelView Lp, const double* __restrict__ phi_b,
                                                     const int4* __restrict__ T, const double* __restrict__ gbc) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: see tab_load
  restrict_tab_item<D, N, MODE, true>(Lf, Lp, phi_b, T, gbc, blockIdx.x * blockDim.x + threadIdx.x);
}

// leaf-residual record of cell a of a small level: accumulates into (mx, ss, cnt)
template <int D, int N>
__device__ __forceinline__ void record_tab_cell(const LevelView& L, const double* __restrict__ phi_b,
                                                const int4* __restrict__ T, const double* __restrict__ gbc, int a,
                                                double& mx, double& ss, double& cnt) {
  using G = Geo<D, N>;
  if (!owned(L, a / G::NI)) return;
  int code, leaf;
  double self, p[2 * D];
  tab_load<D>(L, T, gbc, a, code, leaf, self, p);
  if (leaf && code > -3) {
    const double r = resid_value<D>(L, phi_b, code >= 0 ? code : -1, self, p, L.rhs[a]);
    mx = fmax(mx, fabs(r));
    ss += r * r;
    cnt += 1;
  }
}

// leaf-residual record of a small level: per-CTA partials, folded by k_record_fold
template <int D, int N>
__global__ void __launch_bounds__(256) k_record_tab(LevelView L, const double* __restrict__ phi_b,
                                                   const int4* __restrict__ T, const double* __restrict__ gbc,
                                                   Rec* __restrict__ partial) {
  pdl_begin();
  using G = Geo<D, N>;
  __shared__ double red[72];
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0, ss = 0, cnt = 0;
  if (a < L.nb * G::NI) record_tab_cell<D, N>(L, phi_b, T, gbc, a, mx, ss, cnt);
  mx = block_max(mx, red);
  ss = block_sum(ss, red);
  cnt = block_sum(cnt, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x].max = mx;
    partial[blockIdx.x].sumsq = ss;
    partial[blockIdx.x].count = (long long)cnt;
  }
}

}  // namespace pmgdev

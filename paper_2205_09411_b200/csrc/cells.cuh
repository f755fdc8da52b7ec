// cells.cuh -- per-cell operators of the V-cycle, in the reference's exact
// floating-point operation order (the library is built with --fmad=false).
#pragma once
#include "pmg_dev.cuh"

namespace pmgdev {

// Stencil row index of cell (c,e) of block `slot`, or -1 for the uniform row.
template <int D, int N>
__device__ __forceinline__ int row_index(const LevelView& L, int slot, int c, int e) {
  using G = Geo<D, N>;
  const int sr = L.srow[slot];
  if (sr < 0) return -1;
  return L.row_of[(size_t)sr * G::NI + c * G::H + e];
}

template <int D, int N>
__device__ __forceinline__ bool is_inside(const LevelView& L, int slot, int c, int e) {
  const int r = row_index<D, N>(L, slot, c, e);
  return r >= 0 && L.r_mask[r] == 1;
}

// One Gauss-Seidel update of cell (c,e): multigrid.hpp:621-695.
// Returns false (no write) for inside rows.
template <int D, int N>
__device__ __forceinline__ void gs_cell(const LevelView& L, const LevelView& Lc,
                                        const double* __restrict__ phi_b, int slot, int c, int e) {
  using G = Geo<D, N>;
  const uint8_t kind = L.kind[slot];
  if (kind == KIND_ALL_INSIDE) return;
  int i, j, k;
  G::cell_of(c, e, i, j, k);
  const size_t a = (size_t)slot * G::NI + (size_t)(c * G::H + e);
  int r = -1;
  if (kind != KIND_UNIFORM) {
    r = L.row_of[(size_t)L.srow[slot] * G::NI + c * G::H + e];
    if (r >= 0 && L.r_mask[r] == 1) return;  // inside: pinned (multigrid.hpp:675)
  }
  const double self = L.phi[a];
  const double g = L.rhs[a];
  double p[2 * D];
  neighbours<D, N>(L, Lc, slot, i, j, k, self, p);
  const double h2 = L.h2;
  double nv;
  if (kind == KIND_UNIFORM) {
    if (D == 3)
      nv = (p[0] + p[1] + p[2] + p[3] + p[4] + p[5] - h2 * g) / 6.0;  // :651-653
    else
      nv = 0.25 * (p[0] + p[1] + p[2] + p[3] - h2 * g);  // :640-641
  } else if (r < 0) {
    double s = -h2 * g;  // :668-671
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    nv = -s * (-1.0 / (2.0 * D));
  } else {
    double num = g;  // :677-683
    for (int d = 0; d < 2 * D; ++d) {
      num -= L.r_nb[r * 2 * D + d] * p[d];
      const double b = L.r_bc[r * 2 * D + d];
      if (b != 0) num -= b * phi_b[L.r_obj[r * 2 * D + d]];
    }
    nv = num / L.r_center[r];
  }
  L.phi[a] = nv;
}

// L(phi) at cell (c,e) (stencil.hpp:290-322); 0 for inside rows.
template <int D, int N>
__device__ __forceinline__ double apply_cell(const LevelView& L, const LevelView& Lc,
                                             const double* __restrict__ phi_b, int slot, int c,
                                             int e) {
  using G = Geo<D, N>;
  int i, j, k;
  G::cell_of(c, e, i, j, k);
  const size_t a = (size_t)slot * G::NI + (size_t)(c * G::H + e);
  int r = -1;
  if (L.kind[slot] != KIND_UNIFORM) {
    r = L.row_of[(size_t)L.srow[slot] * G::NI + c * G::H + e];
    if (r >= 0 && L.r_mask[r] == 1) return 0.0;
  }
  const double self = L.phi[a];
  double p[2 * D];
  neighbours<D, N>(L, Lc, slot, i, j, k, self, p);
  if (r < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return s * L.w;
  }
  double s = L.r_center[r] * self;  // row_apply, stencil.hpp:274-284
  for (int d = 0; d < 2 * D; ++d) {
    s += L.r_nb[r * 2 * D + d] * p[d];
    const double b = L.r_bc[r * 2 * D + d];
    if (b != 0) s += b * phi_b[L.r_obj[r * 2 * D + d]];
  }
  return s;
}

// r = g - L(phi) at cell (c,e) (stencil.hpp:325-359); 0 for inside rows.
// *inside is set for inside rows (excluded from residual records).
template <int D, int N>
__device__ __forceinline__ double resid_cell(const LevelView& L, const LevelView& Lc,
                                             const double* __restrict__ phi_b, int slot, int c,
                                             int e, bool* inside) {
  using G = Geo<D, N>;
  int i, j, k;
  G::cell_of(c, e, i, j, k);
  const size_t a = (size_t)slot * G::NI + (size_t)(c * G::H + e);
  int r = -1;
  *inside = false;
  if (L.kind[slot] != KIND_UNIFORM) {
    r = L.row_of[(size_t)L.srow[slot] * G::NI + c * G::H + e];
    if (r >= 0 && L.r_mask[r] == 1) {
      *inside = true;
      return 0.0;
    }
  }
  const double self = L.phi[a];
  const double g = L.rhs[a];
  double p[2 * D];
  neighbours<D, N>(L, Lc, slot, i, j, k, self, p);
  if (r < 0) {
    double s = -2.0 * D * self;
    for (int d = 0; d < 2 * D; ++d) s += p[d];
    return g - s * L.w;
  }
  double s = L.r_center[r] * self;
  for (int d = 0; d < 2 * D; ++d) {
    s += L.r_nb[r * 2 * D + d] * p[d];
    const double b = L.r_bc[r * 2 * D + d];
    if (b != 0) s += b * phi_b[L.r_obj[r * 2 * D + d]];
  }
  return g - s;
}

}  // namespace pmgdev

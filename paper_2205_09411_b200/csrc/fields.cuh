// fields.cuh -- post-solve field kernels: the
// boundary-aware staggered gradient of the solution on the faces of every
// leaf cell, face_gradient (fields.hpp:149-232), and its cell-centred
// magnitude.  One thread per face value; ghosts are evaluated with the
// reference's fill formulas (phi_at: same-level copy, coarse-fine
// interpolation, physical faces), cut distances come from the level's row
// table, so the values are the reference's bit for bit.
#pragma once
#include "cells.cuh"
#include "kernels.cuh"

namespace pmgdev {

struct FaceSide {  // detail::SideInfo (fields.hpp:94-100)
  bool solved;
  double d;
  int obj;
  double phi;
};

// detail::side_info (fields.hpp:102-139): cell c (may be a ghost across face
// `axis`) of block `slot`, cut data toward direction `dir`
template <int D, int N>
__device__ __forceinline__ FaceSide face_side(const LevelView& L, const LevelView& Lc, int slot, const int* c,
                                              int axis, int dir) {
  using G = Geo<D, N>;
  FaceSide s;
  s.solved = true;
  s.d = 1.0;
  s.obj = -1;
  const int c0 = c[0], c1 = c[1], c2 = D == 3 ? c[2] : 0;
  s.phi = phi_at<D, N>(L, Lc, slot, c0, c1, c2);
  int use = slot;
  const int ca = axis == 0 ? c0 : axis == 1 ? c1 : c2;
  int l0 = c0, l1 = c1, l2 = c2;
  if (ca < 0 || ca >= N) {
    // ghost side: the same-level neighbour has the cell's stencil data;
    // coarser neighbours and physical faces count as plain cells
    const int opp = 2 * axis + (ca < 0 ? 0 : 1);
    const int nid = L.nbr[slot * G::F + opp];
    if (nid < 0) return s;
    use = nid;
    const int la = ca < 0 ? N - 1 : 0;
    if (axis == 0) l0 = la;
    else if (axis == 1) l1 = la;
    else l2 = la;
  }
  const int loc[3] = {l0, l1, l2};
  const int r = row_index<D, N>(L, use, G::colour(loc[0], loc[1], loc[2]), G::entry(loc[0], loc[1], loc[2]));
  if (r < 0) return s;  // not a boundary block, or a uniform row
  if (L.r_mask[r] == 1) {  // kInside
    s.solved = false;
    s.obj = L.r_pin[r];
    return s;
  }
  s.d = L.r_d[(size_t)r * G::F + dir];
  s.obj = L.r_obj[(size_t)r * G::F + dir];
  return s;
}

// one thread per face value of the leaves of one level (their (level, slot)
// entries; launched per level): faces[q][axis][f + (N+1) * (transverse, minor to major)]
template <int D, int N>
__global__ void __launch_bounds__(256) k_face_gradient(LevelView L, LevelView Lc, const int2* __restrict__ leaves,
                                                      int n_leaves, const double* __restrict__ phi_b,
                                                      double* __restrict__ out) {
  pdl_begin();
  using G = Geo<D, N>;
  constexpr int PA = (N + 1) * (D == 3 ? N * N : N);  // faces per axis
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)n_leaves * D * PA) return;
  const int q = (int)(gid / (D * PA));
  const int axis = (int)(gid / PA % D);
  const int fi = (int)(gid % PA);
  const int2 lv = leaves[q];
  const int f = fi % (N + 1);
  int rest = fi / (N + 1);
  int t[3] = {0, 0, 0};
  for (int k = 0; k < D; ++k) {
    if (k == axis) continue;
    t[k] = rest % N;
    rest /= N;
  }
  const int cl[3] = {axis == 0 ? f - 1 : t[0], axis == 1 ? f - 1 : t[1], axis == 2 ? f - 1 : t[2]};
  const int cr[3] = {axis == 0 ? f : t[0], axis == 1 ? f : t[1], axis == 2 ? f : t[2]};
  const FaceSide left = face_side<D, N>(L, Lc, lv.y, cl, axis, 2 * axis + 1);
  const FaceSide right = face_side<D, N>(L, Lc, lv.y, cr, axis, 2 * axis);
  const double dx = L.dx;
  double g;  // fields.hpp:179-198
  if (!left.solved && !right.solved) {
    g = 0;
  } else if (!right.solved) {
    g = left.d < 1.0 ? (phi_b[left.obj] - left.phi) / (left.d * dx) : (right.phi - left.phi) / dx;
  } else if (!left.solved) {
    g = right.d < 1.0 ? (right.phi - phi_b[right.obj]) / (right.d * dx) : (right.phi - left.phi) / dx;
  } else if (left.d >= 1.0 && right.d >= 1.0) {
    g = (right.phi - left.phi) / dx;
  } else if (left.d < 1.0 && left.d >= 0.5) {
    g = (phi_b[left.obj] - left.phi) / (left.d * dx);
  } else if (right.d < 1.0 && right.d >= 0.5) {
    g = (right.phi - phi_b[right.obj]) / (right.d * dx);
  } else {
    g = 0;  // thin object: the face lies beyond both roots
  }
  out[gid] = g;
}

// cell-centred |grad phi| from the face values (fields.hpp:204-229); inside
// cells 0; mag[q][i + N (j + N k)]
template <int D, int N>
__global__ void __launch_bounds__(256) k_face_magnitude(LevelView L, const int2* __restrict__ leaves, int n_leaves,
                                                       const double* __restrict__ faces, double* __restrict__ mag) {
  pdl_begin();
  using G = Geo<D, N>;
  constexpr int PA = (N + 1) * (D == 3 ? N * N : N);
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)n_leaves * G::NI) return;
  const int q = (int)(gid / G::NI);
  const int ii = (int)(gid % G::NI);
  const int2 lv = leaves[q];
  const int i3[3] = {ii % N, (ii / N) % N, D == 3 ? ii / (N * N) : 0};
  const int r = row_index<D, N>(L, lv.y, G::colour(i3[0], i3[1], i3[2]), G::entry(i3[0], i3[1], i3[2]));
  if (r >= 0 && L.r_mask[r] == 1) {  // inside electrodes the gradient is zeroed
    mag[gid] = 0;
    return;
  }
  double sq = 0;
  for (int axis = 0; axis < D; ++axis) {
    int idx = 0, mul = N + 1;  // FaceField::face_index (fields.hpp:80-89)
    for (int k = 0; k < D; ++k) {
      if (k == axis) continue;
      idx += i3[k] * mul;
      mul *= N;
    }
    const double* v = faces + ((size_t)q * D + axis) * PA;
    const double lo = v[idx + i3[axis]], hi = v[idx + i3[axis] + 1];
    const double c = 0.5 * (lo + hi);
    sq += c * c;
  }
  mag[gid] = sqrt(sq);
}

}  // namespace pmgdev

namespace pmgdev {

// error_norms against the analytic sphere solution (fields.hpp:9-58): per
// leaf solved cell d = phi - exact(cell centre) with exact = phi_b + a log(r/R)
// (2D) or phi_b + a (1 - R/r) (3D), r = |x| (core.hpp:58-67); per CTA
// {max |d|, sum w d^2, sum w} into part[blockIdx.x]; *err = 1 when a solved
// cell lies inside r < R (the reference throws std::domain_error)
template <int D, int N>
__global__ void __launch_bounds__(256) k_error_norms(LevelView L, const int2* __restrict__ leaves,
                                                    const double* __restrict__ origin, int n_leaves, int tag,
                                                    double phi_b, double a, double R, int vw,
                                                    double* __restrict__ part, int* err) {
  pdl_begin();
  using G = Geo<D, N>;
  __shared__ double red[72];
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0, ss = 0, ws = 0;
  if (gid < (long long)n_leaves * G::NI) {
    const int q = (int)(gid / G::NI), ii = (int)(gid % G::NI);
    const int2 lv = leaves[q];
    const int i3[3] = {ii % N, (ii / N) % N, D == 3 ? ii / (N * N) : 0};
    const int r = row_index<D, N>(L, lv.y, G::colour(i3[0], i3[1], i3[2]), G::entry(i3[0], i3[1], i3[2]));
    if (!(r >= 0 && L.r_mask[r] == 1)) {  // pinned cells are excluded
      double s = 0;
      for (int k = 0; k < D; ++k) {
        const double x = origin[(size_t)q * 3 + k] + ((double)i3[k] + 0.5) * L.dx;
        s += x * x;
      }
      const double rr = sqrt(s);
      if (rr < R) *err = 1;
      const double ex = tag == 0 ? phi_b + a * log(rr / R) : phi_b + a * (1.0 - R / rr);
      const double diff = L.phi[G::addr(lv.y, i3[0], i3[1], i3[2])] - ex;
      double w = 1.0;
      if (vw) {
        w = L.dx;
        for (int k = 1; k < D; ++k) w *= L.dx;
      }
      mx = fabs(diff);
      ss = w * diff * diff;
      ws = w;
    }
  }
  mx = block_max(mx, red);
  ss = block_sum(ss, red);
  ws = block_sum(ws, red);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = mx;
    part[3 * blockIdx.x + 1] = ss;
    part[3 * blockIdx.x + 2] = ws;
  }
}

}  // namespace pmgdev

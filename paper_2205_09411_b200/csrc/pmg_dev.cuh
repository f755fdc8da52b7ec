// pmg_dev.cuh -- device-side data layout and cell access for the B200 V-cycle.
//
// HBM layout (one LevelView per refinement level):
//   * blocks of a level occupy consecutive SLOTS in Morton order of their
//     block coordinates (host permutation slot <-> reference block id);
//   * every cell field (phi, rhs, old, res) is unpadded N^D doubles per block,
//     COLOUR-SPLIT: the N^D/2 cells with (i+j+k) even ("red", parity 0) come
//     first, then the odd ("black") ones; inside a colour, cell (i,j,k) sits at
//     entry (i + N j + N^2 k) >> 1.  A red half-sweep therefore streams the
//     black half, the red rhs half and writes the red half: 12 B/cell instead
//     of the 24 B/cell an interleaved layout moves (sector granularity).
//   * NO ghost layers are stored.  The reference refills every face ghost after
//     every half-sweep (multigrid.hpp:501-508) so at every read a ghost equals
//     the fill formula evaluated on the current interior values
//     (mesh.hpp:471-554); we evaluate that formula at the read instead
//     (same-level: the neighbour's cell; physical: 2 bc - f1 / f1; coarse-fine:
//     1/2 c + 3/4 f1 - 1/4 f2 with c the slope-corrected coarse value).  The
//     only ghosts that are snapshots rather than functions of current state --
//     VAR_OLD at coarse-fine faces (multigrid.hpp:394-396) -- are kept in a small
//     per-level table (cfold).
//
// Arithmetic is written in the reference's operation order and the library is
// compiled with --fmad=false, so every per-cell result is bit-identical to the
// CPU reference (only reductions -- record sums, BiCGStab dots -- reassociate).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pmgdev {

// Programmatic dependent launch (every cycle kernel is launched with
// programmatic stream serialization): let the next kernel in the stream be
// scheduled now, then wait until the previous kernel has completed and its
// writes are visible.  Nothing before pdl_begin() may read device data.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

constexpr int kMaxLevels = 24;

enum BlockKind : uint8_t { KIND_UNIFORM = 0, KIND_IFACE = 1, KIND_ALL_INSIDE = 2 };

struct LevelView {
  int nb;     // blocks on this level
  int level;  // 1-based
  double dx, h2, w;  // dx, dx*dx, 1.0/(dx*dx)  (stencil.hpp:300, multigrid.hpp:633)
  const int32_t* nbr;     // [nb*2D] same-level neighbour slot or -1   (mesh.hpp:45)
  const int32_t* cnbr;    // [nb*2D] coarse neighbour slot (level-1) or -1 (mesh.hpp:46)
  const int32_t* coords;  // [nb*D]
  const int32_t* parent;  // [nb] slot on level-1
  const int32_t* child;   // [nb*2^D] slot on level+1 or -1
  const uint8_t* leaf;    // [nb]
  const uint8_t* kind;    // [nb] BlockKind
  const int32_t* srow;    // [nb] interface-block ordinal (row_of page) or -1
  const int32_t* bcoff;   // [nb*2D] offset into bcval (Dirichlet face values) or -1 (= 0.0)
  const double* bcval;
  double* phi;
  double* rhs;
  double* old;
  double* res;
  const int32_t* row_of;  // [n_iface * N^D], colour-split entry order; -1 = uniform row
  const int8_t* skind;    // same layout: 0 uniform row, 1 inside row, 2 cut row
  const double* r_coef;   // [R*16] center, nb[2D], bc*phi_b[2D], cut mask, inside flag
  const double* r_center; // [R]
  const double* r_nb;     // [R*2D]
  const double* r_d;      // [R*2D] cut distances (face_gradient, fields.hpp:96-139)
  const double* r_bc;     // [R*2D]
  const int8_t* r_obj;    // [R*2D]
  const uint8_t* r_mask;  // [R]
  const int8_t* r_pin;    // [R]
  double* cfold;          // AMR: VAR_OLD ghosts on coarse-fine faces
  const int32_t* cfoff;   // [nb*2D] offset into cfold or -1
  // AMR: the slope-corrected coarse value of every coarse-fine ghost (the part
  // of mesh.hpp:500-535 that only reads level l-1), rebuilt by k_cfc_build
  // whenever level l-1 changed; face f of a block at cfoff[...], colour-split:
  // [colour of the adjacent interior cell][transverse index >> 1].  nullptr:
  // evaluate from level l-1 at the read (the launchers opt in, ops_impl.cuh Vt)
  const double* cfc;
  int bctype[6];          // per domain face: 0 Dirichlet, 1 Neumann-zero (mesh.hpp:22-32)
  int dense;              // 1: all (2^(l-1))^D blocks present and slot == Morton code
  int nside;              // blocks per axis on this level (dense levels)
  int bczero;             // 1: no Dirichlet face values on this level (all zero)
  const uint8_t* own;     // multi-GPU: 1 for blocks this rank computes (nullptr: all)
};

__device__ __forceinline__ bool owned(const LevelView& L, int slot) { return !L.own || L.own[slot]; }

// Morton (Z-order) helpers: on a dense level the slot of a block is the
// interleave of its coordinates, so face neighbours need no table lookup.
__device__ __forceinline__ unsigned m_part3(unsigned x) {  // 10 bits -> every 3rd bit
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000ffu;
  x = (x | (x << 8)) & 0x0300f00fu;
  x = (x | (x << 4)) & 0x030c30c3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}
__device__ __forceinline__ unsigned m_comp3(unsigned x) {
  x &= 0x09249249u;
  x = (x | (x >> 2)) & 0x030c30c3u;
  x = (x | (x >> 4)) & 0x0300f00fu;
  x = (x | (x >> 8)) & 0x030000ffu;
  x = (x | (x >> 16)) & 0x3ffu;
  return x;
}
__device__ __forceinline__ unsigned m_part2(unsigned x) {  // 16 bits -> every 2nd bit
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
__device__ __forceinline__ unsigned m_comp2(unsigned x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0f0f0f0fu;
  x = (x | (x >> 4)) & 0x00ff00ffu;
  x = (x | (x >> 8)) & 0xffffu;
  return x;
}
// same-level neighbour slot across face dir of a dense level, -1 at the domain boundary
template <int D>
__device__ __forceinline__ int dense_nbr(int slot, int dir, int nside) {
  const unsigned s = (unsigned)slot;
  int c[3];
  if (D == 3) {
    c[0] = (int)m_comp3(s);
    c[1] = (int)m_comp3(s >> 1);
    c[2] = (int)m_comp3(s >> 2);
  } else {
    c[0] = (int)m_comp2(s);
    c[1] = (int)m_comp2(s >> 1);
  }
  c[dir >> 1] += (dir & 1) ? 1 : -1;
  if (c[dir >> 1] < 0 || c[dir >> 1] >= nside) return -1;
  if (D == 3) return (int)(m_part3(c[0]) | (m_part3(c[1]) << 1) | (m_part3(c[2]) << 2));
  return (int)(m_part2(c[0]) | (m_part2(c[1]) << 1));
}
// neighbour slot via the table, or arithmetically on dense levels
template <int D>
__device__ __forceinline__ int nbr_slot(const LevelView& L, int slot, int dir) {
  return L.dense ? dense_nbr<D>(slot, dir, L.nside) : L.nbr[slot * 2 * D + dir];
}

template <int D>
struct Ipow {
  static constexpr int of(int n) { return D == 2 ? n * n : n * n * n; }
};

template <int D, int N>
struct Geo {
  static constexpr int F = 2 * D;          // faces
  static constexpr int NC = 1 << D;        // children
  static constexpr int NI = Ipow<D>::of(N);  // interior cells per block
  static constexpr int H = NI / 2;         // cells per colour
  static constexpr int HN = N / 2;         // entries per x-row
  static constexpr int NT = D == 2 ? N : N * N;  // cells per face

  // entry e of colour c -> cell (i,j,k)
  __device__ __forceinline__ static void cell_of(int c, int e, int& i, int& j, int& k) {
    const int m = e % HN;
    const int r = e / HN;
    j = r % N;
    k = D == 3 ? r / N : 0;
    i = 2 * m + ((c + j + k) & 1);
  }
  __device__ __forceinline__ static int colour(int i, int j, int k) { return (i + j + k) & 1; }
  __device__ __forceinline__ static int entry(int i, int j, int k) {
    return (i + N * (j + N * k)) >> 1;
  }
  // address of interior cell (i,j,k) of block slot
  __device__ __forceinline__ static size_t addr(int slot, int i, int j, int k) {
    return (size_t)slot * NI + (size_t)(colour(i, j, k) * H + entry(i, j, k));
  }
  // transverse index of a cell on the face with normal `axis` (lower axis fastest)
  __device__ __forceinline__ static int tindex(int axis, int i, int j, int k) {
    if (D == 2) return axis == 0 ? j : i;
    if (axis == 0) return j + N * k;
    if (axis == 1) return i + N * k;
    return i + N * j;
  }
};

template <int D>
__device__ __forceinline__ int get_c(int axis, int i, int j, int k) {
  return axis == 0 ? i : (axis == 1 ? j : k);
}
__device__ __forceinline__ void set_c(int axis, int v, int& i, int& j, int& k) {
  if (axis == 0) i = v;
  else if (axis == 1) j = v;
  else k = v;
}

// Value of a same-level-or-physical face ghost / interior cell of `arr` on
// level L at padded position (i,j,k) (at most one coordinate outside [0,N)).
// Coarse-fine ghosts are NOT handled here (see cf_ghost): by the 2:1 corner
// balance of the tree (mesh.hpp:252-290, 381-402) the transverse reads of a
// coarse-fine interpolation never land on another coarse-fine ghost; the host
// verifies this when the mesh is uploaded.
template <int D, int N>
__device__ __forceinline__ double val_nocf(const LevelView& L, const double* __restrict__ arr,
                                           int slot, int i, int j, int k) {
  using G = Geo<D, N>;
  int axis = -1, side = 0;
  if (i < 0) { axis = 0; side = 0; } else if (i >= N) { axis = 0; side = 1; }
  else if (j < 0) { axis = 1; side = 0; } else if (j >= N) { axis = 1; side = 1; }
  else if (D == 3 && k < 0) { axis = 2; side = 0; } else if (D == 3 && k >= N) { axis = 2; side = 1; }
  if (axis < 0) return arr[G::addr(slot, i, j, k)];
  const int dir = 2 * axis + side;
  const int ns = L.nbr[slot * G::F + dir];
  int ii = i, jj = j, kk = k;
  if (ns >= 0) {
    set_c(axis, side ? 0 : N - 1, ii, jj, kk);
    return arr[G::addr(ns, ii, jj, kk)];
  }
  set_c(axis, side ? N - 1 : 0, ii, jj, kk);
  const double f1 = arr[G::addr(slot, ii, jj, kk)];
  if (L.bctype[dir] == 1) return f1;  // Neumann: ghost = f1 (mesh.hpp:545-546)
  const int bo = L.bcoff[slot * G::F + dir];
  const double bcv = bo < 0 ? 0.0 : L.bcval[bo + G::tindex(axis, ii, jj, kk)];
  return 2.0 * bcv - f1;  // Dirichlet (mesh.hpp:548-550)
}

// Coarse-fine ghost of fine block `slot` (level L, coarse level Lc) across face
// `dir` next to interior cell (i,j,k): mesh.hpp:500-535.  f1 = value of (i,j,k),
// f2 = value of the next cell inward.
template <int D, int N>
__device__ __forceinline__ double cf_coarse(const LevelView& L, const LevelView& Lc, int slot,
                                            int dir, int i, int j, int k) {
  using G = Geo<D, N>;
  const int axis = dir >> 1, side = dir & 1;
  const int cb = L.cnbr[slot * G::F + dir];
  int lc[3] = {0, 0, 0};
  int sgn[3] = {0, 0, 0};
  const int t[3] = {i, j, k};
  for (int a = 0; a < D; ++a) {
    if (a == axis) {
      lc[a] = side ? 0 : N - 1;
    } else {
      const int gk = L.coords[slot * D + a] * N + t[a];
      lc[a] = (gk >> 1) - Lc.coords[cb * D + a] * N;
      sgn[a] = (gk & 1) ? 1 : -1;
    }
  }
  double c = Lc.phi[G::addr(cb, lc[0], lc[1], lc[2])];
  for (int a = 0; a < D; ++a) {
    if (a == axis) continue;
    int up[3] = {lc[0], lc[1], lc[2]}, dn[3] = {lc[0], lc[1], lc[2]};
    up[a] += 1;
    dn[a] -= 1;
    const double vu = val_nocf<D, N>(Lc, Lc.phi, cb, up[0], up[1], up[2]);
    const double vd = val_nocf<D, N>(Lc, Lc.phi, cb, dn[0], dn[1], dn[2]);
    c += (double)sgn[a] * (vu - vd) / 8.0;
  }
  return c;
}
// position of the ghost next to interior cell (i,j,k) inside its face's cfc page
template <int D, int N>
__device__ __forceinline__ int cfc_index(int axis, int i, int j, int k) {
  using G = Geo<D, N>;
  return G::colour(i, j, k) * (G::NT / 2) + (G::tindex(axis, i, j, k) >> 1);
}
template <int D, int N>
__device__ __forceinline__ double cf_ghost(const LevelView& L, const LevelView& Lc, int slot,
                                           int dir, int i, int j, int k, double f1, double f2) {
  using G = Geo<D, N>;
  const double c = L.cfc ? L.cfc[L.cfoff[slot * G::F + dir] + cfc_index<D, N>(dir >> 1, i, j, k)]
                         : cf_coarse<D, N>(L, Lc, slot, dir, i, j, k);
  return 0.5 * c + 0.75 * f1 - 0.25 * f2;
}

// Ghost of PHI across face `dir` of interior cell (i,j,k) whose current value
// is `self` (the filled ghost value the reference would read there).
template <int D, int N>
__device__ __forceinline__ double phi_ghost(const LevelView& L, const LevelView& Lc, int slot,
                                            int dir, int i, int j, int k, double self) {
  using G = Geo<D, N>;
  const int ns = L.nbr[slot * G::F + dir];
  const int axis = dir >> 1, side = dir & 1;
  if (ns >= 0) {
    int ii = i, jj = j, kk = k;
    set_c(axis, side ? 0 : N - 1, ii, jj, kk);
    return L.phi[G::addr(ns, ii, jj, kk)];
  }
  if (L.cnbr[slot * G::F + dir] >= 0) {
    int ii = i, jj = j, kk = k;
    set_c(axis, side ? N - 2 : 1, ii, jj, kk);
    const double f2 = L.phi[G::addr(slot, ii, jj, kk)];
    return cf_ghost<D, N>(L, Lc, slot, dir, i, j, k, self, f2);
  }
  if (L.bctype[dir] == 1) return self;
  const int bo = L.bcoff[slot * G::F + dir];
  const double bcv = bo < 0 ? 0.0 : L.bcval[bo + G::tindex(axis, i, j, k)];
  return 2.0 * bcv - self;
}

// Ghost of OLD (the snapshot taken right after a fill, multigrid.hpp:394-396).
template <int D, int N>
__device__ __forceinline__ double old_ghost(const LevelView& L, int slot, int dir, int i, int j,
                                            int k, double self) {
  using G = Geo<D, N>;
  const int ns = L.nbr[slot * G::F + dir];
  const int axis = dir >> 1, side = dir & 1;
  if (ns >= 0) {
    int ii = i, jj = j, kk = k;
    set_c(axis, side ? 0 : N - 1, ii, jj, kk);
    return L.old[G::addr(ns, ii, jj, kk)];
  }
  const int co = L.cfoff ? L.cfoff[slot * G::F + dir] : -1;
  if (co >= 0) return L.cfold[co + G::tindex(axis, i, j, k)];
  if (L.bctype[dir] == 1) return self;
  const int bo = L.bcoff[slot * G::F + dir];
  const double bcv = bo < 0 ? 0.0 : L.bcval[bo + G::tindex(axis, i, j, k)];
  return 2.0 * bcv - self;
}

// Generic padded read of PHI (interior or face ghost) on level L.
template <int D, int N>
__device__ __forceinline__ double phi_at(const LevelView& L, const LevelView& Lc, int slot, int i,
                                         int j, int k) {
  using G = Geo<D, N>;
  int axis = -1, side = 0;
  if (i < 0) { axis = 0; side = 0; } else if (i >= N) { axis = 0; side = 1; }
  else if (j < 0) { axis = 1; side = 0; } else if (j >= N) { axis = 1; side = 1; }
  else if (D == 3 && k < 0) { axis = 2; side = 0; } else if (D == 3 && k >= N) { axis = 2; side = 1; }
  if (axis < 0) return L.phi[G::addr(slot, i, j, k)];
  int ii = i, jj = j, kk = k;
  set_c(axis, side ? N - 1 : 0, ii, jj, kk);
  const double self = L.phi[G::addr(slot, ii, jj, kk)];
  return phi_ghost<D, N>(L, Lc, slot, 2 * axis + side, ii, jj, kk, self);
}

template <int D, int N>
__device__ __forceinline__ double old_at(const LevelView& L, int slot, int i, int j, int k) {
  using G = Geo<D, N>;
  int axis = -1, side = 0;
  if (i < 0) { axis = 0; side = 0; } else if (i >= N) { axis = 0; side = 1; }
  else if (j < 0) { axis = 1; side = 0; } else if (j >= N) { axis = 1; side = 1; }
  else if (D == 3 && k < 0) { axis = 2; side = 0; } else if (D == 3 && k >= N) { axis = 2; side = 1; }
  if (axis < 0) return L.old[G::addr(slot, i, j, k)];
  int ii = i, jj = j, kk = k;
  set_c(axis, side ? N - 1 : 0, ii, jj, kk);
  const double self = L.old[G::addr(slot, ii, jj, kk)];
  return old_ghost<D, N>(L, slot, 2 * axis + side, ii, jj, kk, self);
}

// The 2D neighbour PHI values of interior cell (i,j,k) in direction order
// {-x,+x,-y,+y,-z,+z} (stencil.hpp:241-248), ghosts evaluated on the fly.
template <int D, int N>
__device__ __forceinline__ void neighbours(const LevelView& L, const LevelView& Lc, int slot,
                                           int i, int j, int k, double self, double* p) {
  using G = Geo<D, N>;
  const int c = G::colour(i, j, k);
  const double* __restrict__ opp = L.phi + (size_t)slot * G::NI + (size_t)(1 - c) * G::H;
  const int e = G::entry(i, j, k);
  const int o = i & 1;
  // x: (i-1)>>1 == e - (o==0), (i+1)>>1 == e + (o==1) within the row
  p[0] = i > 0 ? opp[e - (o == 0 ? 1 : 0)] : phi_ghost<D, N>(L, Lc, slot, 0, i, j, k, self);
  p[1] = i < N - 1 ? opp[e + (o == 1 ? 1 : 0)] : phi_ghost<D, N>(L, Lc, slot, 1, i, j, k, self);
  p[2] = j > 0 ? opp[e - G::HN] : phi_ghost<D, N>(L, Lc, slot, 2, i, j, k, self);
  p[3] = j < N - 1 ? opp[e + G::HN] : phi_ghost<D, N>(L, Lc, slot, 3, i, j, k, self);
  if (D == 3) {
    p[4] = k > 0 ? opp[e - G::HN * N] : phi_ghost<D, N>(L, Lc, slot, 4, i, j, k, self);
    p[5] = k < N - 1 ? opp[e + G::HN * N] : phi_ghost<D, N>(L, Lc, slot, 5, i, j, k, self);
  }
}

}  // namespace pmgdev

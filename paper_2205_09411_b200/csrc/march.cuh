// march.cuh -- 2.5D "column-march" GS-RB half-sweep for 3D uniform-level blocks.
//
// One CTA per block, one thread per (m, j) column of x-pairs (N/2 * N threads),
// marching over the N planes k.  In plane k the thread's pair holds one cell of
// the active colour c, at i = 2m + oc (oc = (c+j+k)&1), and one of the opposite
// colour at 2m + (1-oc).  The neighbours of the active cell are then
//   z-, z+ : the thread's own opposite values of planes k-1, k+1  (registers)
//   x      : its own opposite value, and the one of pair m-1 (oc=0) or m+1 (oc=1)
//   y-, y+ : the opposite values of pair m in rows j-1, j+1
// so only x and y come from a small double-buffered shared-memory plane
// (4 shared accesses per cell instead of 7 for a full 3D tile), and the global
// loads of plane k+2 (opposite colour, rhs, plane ghosts) are in flight while
// plane k is updated.  Face ghosts are evaluated with the fill formulas
// (same-level copy or physical Dirichlet / Neumann), exactly as in the tile
// kernels; levels with coarse-fine faces use the tile kernels instead.
#pragma once
#include "tile_kernels.cuh"

namespace pmgdev {

template <int N>
struct March {
  static constexpr int HN = N / 2;
  static constexpr int THREADS = HN * N;
  static constexpr int RWP = HN + 1;        // slots per plane row
  static constexpr int PSZ = (N + 2) * RWP;  // one plane with x/y ghost slots
  static constexpr int NG = 2 * N;           // ghost values per plane (x: N, y: N)
};

// Opposite-colour face ghost next to active cell (i,j,k) across face dir of
// block slot (same-level neighbour ns, or physical): mesh.hpp:485-498,538-552.
template <int N>
__device__ __forceinline__ double march_ghost(const LevelView& L, int slot, int dir, int ns,
                                              int i, int j, int k, int X) {
  using G = Geo<3, N>;
  const int axis = dir >> 1, side = dir & 1;
  int w[3] = {i, j, k};
  if (ns >= 0) {
    w[axis] = side ? 0 : N - 1;
    return L.phi[(size_t)ns * G::NI + (size_t)X * G::H + G::entry(w[0], w[1], w[2])];
  }
  const double self = L.phi[(size_t)slot * G::NI + (size_t)(1 - X) * G::H + G::entry(i, j, k)];
  if (L.bctype[dir] == 1) return self;
  const int bo = L.bcoff[slot * G::F + dir];
  const double bcv = bo < 0 ? 0.0 : L.bcval[bo + G::tindex(axis, i, j, k)];
  return 2.0 * bcv - self;
}

template <int N>
__global__ void __launch_bounds__(March<N>::THREADS) k_gs_march(LevelView L,
                                                               const double* __restrict__ phi_b,
                                                               int parity) {
  using G = Geo<3, N>;
  using M = March<N>;
  constexpr int HN = M::HN, RWP = M::RWP;
  __shared__ double P[2][M::PSZ];
  __shared__ int ns_s[6];
  const int slot = blockIdx.x;
  const int c = parity, X = 1 - c;
  const int t = threadIdx.x;
  const int m = t % HN, j = t / HN;
  if (t < 6) ns_s[t] = L.nbr[slot * 6 + t];
  const uint8_t kind = L.kind[slot];
  const size_t base = (size_t)slot * G::NI;
  const double* __restrict__ opp = L.phi + base + (size_t)X * G::H;
  const double* __restrict__ gg = L.rhs + base + (size_t)c * G::H;
  double* __restrict__ act = L.phi + base + (size_t)c * G::H;
  // entry of pair (m, j) in plane k: e = m + HN*(j + N*k)
  const int e0 = m + HN * j;
  constexpr int PS = HN * N;  // entries per plane
  // register windows: opposite values of planes k-1 .. k+2, rhs of planes k .. k+2
  double o_m1, o_0, o_1, o_2, g_0, g_1, g_2;
  __syncthreads();  // ns_s
  int nsx[2], nsy[2];
  nsx[0] = ns_s[0];
  nsx[1] = ns_s[1];
  nsy[0] = ns_s[2];
  nsy[1] = ns_s[3];
  // z ghosts (planes -1 and N) of this column
  {
    const int oc0 = (c + j + 0) & 1;
    o_m1 = march_ghost<N>(L, slot, 4, ns_s[4], 2 * m + oc0, j, 0, X);
  }
  o_0 = opp[e0];
  o_1 = opp[e0 + PS];
  g_0 = gg[e0];
  g_1 = gg[e0 + PS];
  // ghost duty for plane k: threads [0, N) -> x ghost of row j=t; [N, 2N) -> y ghosts
  auto ghost_for = [&](int k) -> double {
    if (t < N) {
      const int jj = t, oc = (c + jj + k) & 1;  // oc=0: i=0 active needs x-; oc=1: i=N-1 needs x+
      return oc == 0 ? march_ghost<N>(L, slot, 0, nsx[0], 0, jj, k, X)
                     : march_ghost<N>(L, slot, 1, nsx[1], N - 1, jj, k, X);
    }
    if (t < 2 * N) {
      const int u = t - N;           // [0, N): first HN -> y- face (row 0), next HN -> y+ (row N-1)
      const int side = u / HN, mm = u % HN;
      const int jj = side ? N - 1 : 0;
      const int oc = (c + jj + k) & 1;
      return march_ghost<N>(L, slot, 2 + side, nsy[side], 2 * mm + oc, jj, k, X);
    }
    return 0.0;
  };
  double gh_0 = ghost_for(0), gh_1 = N > 1 ? ghost_for(1) : 0.0, gh_2 = 0.0;
  const int32_t* rowp = kind == KIND_UNIFORM ? nullptr : L.row_of + (size_t)L.srow[slot] * G::NI + c * G::H;
  if (kind == KIND_ALL_INSIDE) return;  // uniform per CTA: no barrier is split
#pragma unroll 2
  for (int k = 0; k < N; ++k) {
    // loads for plane k+2 (in flight during this plane's update)
    if (k + 2 < N) {
      o_2 = opp[e0 + (k + 2) * PS];
      g_2 = gg[e0 + (k + 2) * PS];
      gh_2 = ghost_for(k + 2);
    } else if (k + 2 == N) {
      const int ocN = (c + j + N - 1) & 1;
      o_2 = march_ghost<N>(L, slot, 5, ns_s[5], 2 * m + ocN, j, N - 1, X);  // z+ ghost plane
    }
    double* Pb = P[k & 1];
    const int oc = (c + j + k) & 1, oX = 1 - oc;
    const int row = (j + 1) * RWP;
    Pb[row + m + oX] = o_0;
    if (t < N) {  // x ghost: slot 0 (x-) or HN (x+) of row t
      const int oct = (c + t + k) & 1;
      Pb[(t + 1) * RWP + (oct == 0 ? 0 : HN)] = gh_0;
    } else if (t < 2 * N) {
      const int u = t - N, side = u / HN, mm = u % HN;
      const int jj = side ? N - 1 : 0, octy = (c + jj + k) & 1;
      Pb[(side ? N + 1 : 0) * RWP + mm + octy] = gh_0;
    }
    __syncthreads();
    const int e = e0 + k * PS;
    double p[6];
    p[0] = oc == 0 ? Pb[row + m] : o_0;          // x-
    p[1] = oc == 0 ? o_0 : Pb[row + m + 1];      // x+
    p[2] = Pb[row - RWP + m + oc];               // y-
    p[3] = Pb[row + RWP + m + oc];               // y+
    p[4] = o_m1;                                 // z-
    p[5] = o_1;                                  // z+
    int r = -1;
    bool skip = false;
    if (rowp) {
      r = rowp[e];
      skip = r >= 0 && L.r_mask[r] == 1;
    }
    if (!skip) act[e] = gs_value<3>(L, phi_b, kind, r, p, g_0);
    // advance the windows
    o_m1 = o_0;
    o_0 = o_1;
    o_1 = o_2;
    g_0 = g_1;
    g_1 = g_2;
    gh_0 = gh_1;
    gh_1 = gh_2;
  }
}

}  // namespace pmgdev

// kernels.cuh -- the sm_100a kernels of the V-cycle / FMG hot path.
//
//   k_gs            half-sweep of one colour               multigrid.hpp:365-370,621-695 (+ fills)
//   k_residual      r = g - L phi                          stencil.hpp:325-359
//   k_restrict      2^D-average of phi and r (or rhs) into the parent, pins
//                   fused; FUSED variant computes r on the fly (residual_level +
//                   restrict_level in one pass)            multigrid.hpp:374-418,697-722; stencil.hpp:225-237
//   k_fas           g_c = L_c(phi_c) + R(r), old = phi      multigrid.hpp:383-397
//   k_cfold_list    VAR_OLD ghost snapshot on coarse-fine faces (AMR)   multigrid.hpp:394-396
//   k_prolong       phi += interp(phi_c - old_c) / phi = interp(phi_c)  multigrid.hpp:422-438,724-783
//   k_record        leaf residual max / sum r^2 / count, fixed-order reduction  multigrid.hpp:529-562
//   k_pins          phi = phi_b at inside rows             stencil.hpp:225-237
//   k_coarse        Jacobi-BiCGStab on the level-1 system (+ GS-RB fallback) multigrid.hpp:194-280,442-472,586-619
//   k_combine       CycleStats from the level records      multigrid.hpp:564-575
#pragma once
#include "cells.cuh"

namespace pmgdev {

struct Rec {
  double max;
  double sumsq;
  long long count;
};

constexpr int kThreads = 256;

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sumll(long long v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum: fixed butterfly inside warps, warp partials summed
// in warp order.  Result returned to every thread.  smem >= 33 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < nw; ++w) s += smem[w];
    smem[32] = s;
  }
  __syncthreads();
  return smem[32];
}
__device__ __forceinline__ void block_sum2(double& a, double& b, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    smem[wid] = a;
    smem[32 + wid] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0, t = 0;
    for (int w = 0; w < nw; ++w) {
      s += smem[w];
      t += smem[32 + w];
    }
    smem[64] = s;
    smem[65] = t;
  }
  __syncthreads();
  a = smem[64];
  b = smem[65];
}
__device__ __forceinline__ double block_max(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < nw; ++w) s = fmax(s, smem[w]);
    smem[32] = s;
  }
  __syncthreads();
  return smem[32];
}

// ---------------------------------------------------------------- GS-RB
template <int D, int N>
__global__ void __launch_bounds__(kThreads) k_gs(LevelView L, LevelView Lc,
                                                 const double* __restrict__ phi_b, int parity) {
  pdl_begin();
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L.nb * G::H) return;
  const int slot = (int)(t / G::H);
  const int e = (int)(t % G::H);
  if (!owned(L, slot)) return;
  gs_cell<D, N>(L, Lc, phi_b, slot, parity, e);
}

// ---------------------------------------------------------------- residual
template <int D, int N>
__global__ void __launch_bounds__(kThreads) k_residual(LevelView L, LevelView Lc,
                                                       const double* __restrict__ phi_b) {
  pdl_begin();
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L.nb * G::NI) return;
  const int slot = (int)(t / G::NI);
  const int ce = (int)(t % G::NI);
  if (!owned(L, slot)) return;
  bool ins;
  L.res[(size_t)slot * G::NI + ce] =
      resid_cell<D, N>(L, Lc, phi_b, slot, ce / G::H, ce % G::H, &ins);
}

// ---------------------------------------------------------------- restriction
enum RestrictMode { RM_RES = 0, RM_RHS = 1, RM_FUSED = 2 };

// One thread per parent cell covered by a fine block: sum of the 2^D children
// in x-fastest order, / 2^D (multigrid.hpp:697-722); phi is then pinned where
// the parent row is inside (apply_pins(l-1), stencil.hpp:225-237).  The second
// restricted quantity (r, or rhs on the first FMG descent) is written to the
// parent's rhs slot: k_fas turns it into g_c = L_c(phi_c) + R(r).
template <int D, int N, int MODE>
__global__ void __launch_bounds__(kThreads) k_restrict(LevelView Lf, LevelView Lfc,
                                                       LevelView Lp,
                                                       const double* __restrict__ phi_b) {
  pdl_begin();
  // 2^D threads per parent cell, one per child (its residual is a chain of
  // dependent loads); the group's first lane sums them in x-fastest order
  using G = Geo<D, N>;
  constexpr int NC = G::NC;
  constexpr int NQ = G::NI / NC;  // parent cells per fine block
  constexpr int HN = N / 2;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long t = gid / NC;
  const int d = (int)(gid % NC);
  const int slot = t < (long long)Lf.nb * NQ ? (int)(t / NQ) : 0;
  const bool live = t < (long long)Lf.nb * NQ && owned(Lf, slot);
  const int q = live ? (int)(t % NQ) : 0;
  const int qx = q % HN, qy = (q / HN) % HN, qz = D == 3 ? q / (HN * HN) : 0;
  double vphi = 0, vq = 0;
  if (live) {
    const int fi = 2 * qx + (d & 1), fj = 2 * qy + ((d >> 1) & 1), fk = D == 3 ? 2 * qz + ((d >> 2) & 1) : 0;
    const int c = G::colour(fi, fj, fk), e = G::entry(fi, fj, fk);
    const size_t a = (size_t)slot * G::NI + (size_t)(c * G::H + e);
    vphi = Lf.phi[a];
    if (MODE == RM_RES) {
      vq = Lf.res[a];
    } else if (MODE == RM_RHS) {
      vq = Lf.rhs[a];
    } else {
      bool ins;
      vq = resid_cell<D, N>(Lf, Lfc, phi_b, slot, c, e, &ins);
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
  const int P = Lf.parent[slot];
  int cp[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) cp[a] = (Lf.coords[slot * D + a] & 1) * HN;
  const int pi = cp[0] + qx, pj = cp[1] + qy, pk = D == 3 ? cp[2] + qz : 0;
  const int pc = G::colour(pi, pj, pk), pe = G::entry(pi, pj, pk);
  const size_t pa = (size_t)P * G::NI + (size_t)(pc * G::H + pe);
  double pv = sphi / (double)(1 << D);
  const int r = row_index<D, N>(Lp, P, pc, pe);
  if (r >= 0 && Lp.r_mask[r] == 1) pv = phi_b[Lp.r_pin[r]];
  Lp.phi[pa] = pv;
  Lp.rhs[pa] = sq / (double)(1 << D);
}

// ---------------------------------------------------------------- FAS RHS + OLD snapshot
template <int D, int N, bool FAS>
__global__ void __launch_bounds__(kThreads) k_fas(LevelView L, LevelView Lc,
                                                  const double* __restrict__ phi_b) {
  pdl_begin();
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L.nb * G::NI) return;
  const int slot = (int)(t / G::NI);
  const int ce = (int)(t % G::NI);
  if (!owned(L, slot)) return;
  const size_t a = (size_t)slot * G::NI + ce;
  if (FAS && !L.leaf[slot]) {
    const double out = apply_cell<D, N>(L, Lc, phi_b, slot, ce / G::H, ce % G::H);
    L.rhs[a] = out + L.rhs[a];  // g[c] += r[c] after apply_block (multigrid.hpp:388-392)
  }
  L.old[a] = L.phi[a];
}

// VAR_OLD ghosts on coarse-fine faces, evaluated right after the fill that
// precedes the snapshot (multigrid.hpp:394-396): one thread per ghost of the
// level's listed coarse-fine faces; L carries the cfc table.
template <int D, int N>
__global__ void __launch_bounds__(256) k_cfold_list(LevelView L, LevelView Lc, const int2* __restrict__ faces,
                                                    int n_faces) {
  pdl_begin();
  using G = Geo<D, N>;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_faces * G::NT) return;
  const int2 f = faces[t / G::NT];
  const int tt = t % G::NT;
  const int slot = f.x, dir = f.y, axis = dir >> 1, side = dir & 1;
  if (!owned(L, slot)) return;
  int c3[3] = {0, 0, 0};
  int u = tt;
  for (int a = 0; a < D; ++a) {
    if (a == axis) continue;
    c3[a] = u % N;
    u /= N;
  }
  c3[axis] = side ? N - 1 : 0;
  const double self = L.phi[G::addr(slot, c3[0], c3[1], c3[2])];
  L.cfold[L.cfoff[slot * G::F + dir] + tt] = phi_ghost<D, N>(L, Lc, slot, dir, c3[0], c3[1], c3[2], self);
}

// The level's cfc table (pmg_dev.cuh LevelView::cfc): one thread per ghost of
// the listed coarse-fine faces.  Only level l-1 is read.  Each face comes with
// a host-built descriptor (capi.cu set_mesh: fine slot, dir, page offset,
// coarse slot, position inside the coarse block, the coarse block's transverse
// neighbours), so a thread's loads are the descriptor and then the five
// coarse values: cf_coarse's arithmetic (mesh.hpp:500-531) without its chain
// of table lookups.  A transverse read that leaves the coarse block across a
// physical face takes the generic path (val_nocf).
template <int D, int N>
__global__ void __launch_bounds__(256) k_cfc_build(LevelView L, LevelView Lc, const int4* __restrict__ desc,
                                                   int n_faces, double* __restrict__ out) {
  pdl_begin();
  using G = Geo<D, N>;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_faces * G::NT) return;
  const int4 d0 = __ldg(desc + 2 * (t / G::NT)), d1 = __ldg(desc + 2 * (t / G::NT) + 1);
  const int tt = t % G::NT;
  if (!owned(L, d0.x)) return;  // multi-GPU: another rank's block (its coarse side may not be backed here)
  const int dir = d0.y & 7, axis = dir >> 1, side = dir & 1;
  const int cb = d0.w;
  const int hb[2] = {(d0.y >> 3) & 1, (d0.y >> 4) & 1};
  const int nn[4] = {d1.x, d1.y, d1.z, d1.w};
  int c3[3] = {0, 0, 0};  // the fine block's interior cell next to the ghost
  int lc[3] = {0, 0, 0};  // the coarse cell behind the ghost
  int sgn[3] = {0, 0, 0};
  int ua[3] = {0, 0, 0};  // transverse ordinal of axis a
  {
    int u = tt, k = 0;
    for (int a = 0; a < D; ++a) {
      if (a == axis) continue;
      c3[a] = u % N;
      u /= N;
      const int gk = hb[k] * N + c3[a];
      lc[a] = gk >> 1;
      sgn[a] = (gk & 1) ? 1 : -1;
      ua[a] = k++;
    }
  }
  c3[axis] = side ? N - 1 : 0;
  lc[axis] = side ? 0 : N - 1;
  double c = Lc.phi[G::addr(cb, lc[0], lc[1], lc[2])];
  for (int a = 0; a < D; ++a) {
    if (a == axis) continue;
    double v[2];
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      int q[3] = {lc[0], lc[1], lc[2]};
      q[a] += sd ? 1 : -1;
      if (q[a] >= 0 && q[a] < N) {
        v[sd] = Lc.phi[G::addr(cb, q[0], q[1], q[2])];
      } else {
        const int ns = nn[2 * ua[a] + sd];
        if (ns >= 0) {
          q[a] = sd ? 0 : N - 1;
          v[sd] = Lc.phi[G::addr(ns, q[0], q[1], q[2])];
        } else {
          v[sd] = val_nocf<D, N>(Lc, Lc.phi, cb, q[0], q[1], q[2]);  // physical face of the coarse block
        }
      }
    }
    c += (double)sgn[a] * (v[1] - v[0]) / 8.0;
  }
  out[d0.z + cfc_index<D, N>(axis, c3[0], c3[1], c3[2])] = c;
}

// ---------------------------------------------------------------- prolongation
// fine cell t (t < nb * NI); the body of k_prolong.  PDL: the static lookups
// (inside test, parent, octant) come before griddepcontrol.wait, the field
// values after it
template <int D, int N, bool FULL, bool PDL = false>
__device__ __forceinline__ void prolong_cell(const LevelView& Lf, const LevelView& Lp, const LevelView& Lpp,
                                             long long t) {
  using G = Geo<D, N>;
  const int slot = (int)(t / G::NI);
  const int ce = (int)(t % G::NI);
  const int c = ce / G::H, e = ce % G::H;
  bool skip = !owned(Lf, slot);
  if (!skip && Lf.kind[slot] != KIND_UNIFORM) {
    const int r = Lf.row_of[(size_t)Lf.srow[slot] * G::NI + ce];
    skip = r >= 0 && Lf.r_mask[r] == 1;  // inside cells are skipped
  }
  int fc[3];
  G::cell_of(c, e, fc[0], fc[1], fc[2]);
  const int P = skip ? 0 : Lf.parent[slot];
  int pc[3] = {0, 0, 0}, sg[3] = {0, 0, 0};
  for (int a = 0; a < D && !skip; ++a) {
    const int gk = ((Lf.coords[slot * D + a] & 1) ? N : 0) + fc[a];
    pc[a] = gk >> 1;
    sg[a] = (gk & 1) ? 1 : -1;
  }
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (skip) return;
  const size_t fa = (size_t)slot * G::NI + ce;
  if (FULL) {
    double val = (1.0 - 0.25 * D) * phi_at<D, N>(Lp, Lpp, P, pc[0], pc[1], pc[2]);
    for (int a = 0; a < D; ++a) {
      int q[3] = {pc[0], pc[1], pc[2]};
      q[a] += sg[a];
      val += 0.25 * phi_at<D, N>(Lp, Lpp, P, q[0], q[1], q[2]);
    }
    Lf.phi[fa] = val;
  } else {
    const double d0 = phi_at<D, N>(Lp, Lpp, P, pc[0], pc[1], pc[2]) -
                      old_at<D, N>(Lp, P, pc[0], pc[1], pc[2]);
    double corr = (1.0 - 0.25 * D) * d0;
    for (int a = 0; a < D; ++a) {
      int q[3] = {pc[0], pc[1], pc[2]};
      q[a] += sg[a];
      corr += 0.25 * (phi_at<D, N>(Lp, Lpp, P, q[0], q[1], q[2]) - old_at<D, N>(Lp, P, q[0], q[1], q[2]));
    }
    Lf.phi[fa] += corr;
  }
}

template <int D, int N, bool FULL>
__global__ void __launch_bounds__(kThreads) k_prolong(LevelView Lf, LevelView Lp, LevelView Lpp) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL: see prolong_cell
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)Lf.nb * G::NI) return;
  prolong_cell<D, N, FULL, true>(Lf, Lp, Lpp, t);
}

// ---------------------------------------------------------------- pins
template <int D, int N>
__global__ void __launch_bounds__(kThreads) k_pins(LevelView L, const double* __restrict__ phi_b) {
  pdl_begin();
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L.nb * G::NI) return;
  const int slot = (int)(t / G::NI);
  if (L.srow[slot] < 0 || !owned(L, slot)) return;
  const int ce = (int)(t % G::NI);
  const int r = L.row_of[(size_t)L.srow[slot] * G::NI + ce];
  if (r >= 0 && L.r_mask[r] == 1) L.phi[(size_t)slot * G::NI + ce] = phi_b[L.r_pin[r]];
}

// ---------------------------------------------------------------- residual record
// One CTA per block: per-block (max |r|, sum r^2, count) over solved cells of
// leaf blocks, then the last CTA reduces the partials in slot order
// (deterministic, multigrid.hpp:555-561) into rec[level].
template <int D, int N>
__global__ void __launch_bounds__(kThreads) k_record(LevelView L, LevelView Lc,
                                                     const double* __restrict__ phi_b,
                                                     Rec* __restrict__ partial, Rec* rec,
                                                     unsigned int* counter) {
  pdl_begin();
  using G = Geo<D, N>;
  __shared__ double sm[72];
  __shared__ bool last;
  const int slot = blockIdx.x;
  double mx = 0, ss = 0;
  long long cnt = 0;
  if (L.leaf[slot] && owned(L, slot)) {
    for (int ce = threadIdx.x; ce < G::NI; ce += blockDim.x) {
      bool ins;
      const double r = resid_cell<D, N>(L, Lc, phi_b, slot, ce / G::H, ce % G::H, &ins);
      if (ins) continue;
      mx = fmax(mx, fabs(r));
      ss += r * r;
      cnt += 1;
    }
  }
  mx = block_max(mx, sm);
  ss = block_sum(ss, sm);
  const double cd = block_sum((double)cnt, sm);
  if (threadIdx.x == 0) {
    partial[slot].max = mx;
    partial[slot].sumsq = ss;
    partial[slot].count = (long long)cd;
    __threadfence();
    const unsigned int done = atomicAdd(counter, 1u);
    last = done == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  mx = 0;
  ss = 0;
  double cc = 0;
  // fixed strided ownership, then fixed tree: deterministic
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
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

// CycleStats from the level records (multigrid.hpp:564-575).
// Per special row of a level, the folded coefficients the gather-entry
// kernels read: center, nb[6], bc * phi_b[obj] per cut direction (formed as
// the reference forms it, stencil.hpp:344-358), the cut mask, inside flag.
static __global__ void __launch_bounds__(256) k_row_coef(int R, int F, const double* __restrict__ center,
                                                         const double* __restrict__ nb, const double* __restrict__ bc,
                                                         const int8_t* __restrict__ obj,
                                                         const uint8_t* __restrict__ mask,
                                                         const double* __restrict__ phi_b, double* __restrict__ out) {
  pdl_begin();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double e[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) e[k] = 0.0;
  e[0] = center[r];
  int bm = 0;
  for (int f = 0; f < F; ++f) {
    e[1 + f] = nb[(size_t)r * F + f];
    const double b = bc[(size_t)r * F + f];
    if (b != 0) {
      bm |= 1 << f;
      e[7 + f] = b * phi_b[obj[(size_t)r * F + f]];
    }
  }
  e[13] = (double)bm;
  e[14] = mask[r] == 1 ? 1.0 : 0.0;  // PMG_INSIDE
  double2* o = reinterpret_cast<double2*>(out + (size_t)r * 16);
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k] = make_double2(e[2 * k], e[2 * k + 1]);
}

// One CTA per interface block of a level (list: StencilSet page, first row,
// level row, row count): the block's rows copied into the level's row arrays
// and its row_of page in the colour-split cell order with level row numbers,
// plus the special-row kind of every cell (0 uniform, 1 inside, 2 cut).
static __global__ void __launch_bounds__(256) k_level_rows(
    const int4* __restrict__ list, int N, int D, int F, const int32_t* __restrict__ rowof,
    const double* __restrict__ center, const double* __restrict__ nb, const double* __restrict__ bc,
    const double* __restrict__ dd, const int8_t* __restrict__ obj, const uint8_t* __restrict__ mask,
    const int8_t* __restrict__ pin, int32_t* __restrict__ o_rowof, int8_t* __restrict__ o_skind,
    double* __restrict__ o_center, double* __restrict__ o_nb, double* __restrict__ o_bc, double* __restrict__ o_d,
    int8_t* __restrict__ o_obj, uint8_t* __restrict__ o_mask, int8_t* __restrict__ o_pin) {
  pdl_begin();
  const int4 e = list[blockIdx.x];  // {page, src row, dst row, count}
  const int NI = D == 2 ? N * N : N * N * N, H = NI / 2;
  const int32_t* src = rowof + (size_t)e.x * NI;
  int32_t* dpg = o_rowof + (size_t)blockIdx.x * NI;
  int8_t* spg = o_skind + (size_t)blockIdx.x * NI;
  for (int ii = threadIdx.x; ii < NI; ii += blockDim.x) {
    const int r = src[ii];
    const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
    const int a = ((i + j + k) & 1) * H + (ii >> 1);
    dpg[a] = r < 0 ? -1 : e.z + r;
    spg[a] = r < 0 ? 0 : (mask[e.y + r] == 1 ? 1 : 2);  // PMG_INSIDE
  }
  for (int q = threadIdx.x; q < e.w; q += blockDim.x) {
    const size_t sr = (size_t)e.y + q, dr = (size_t)e.z + q;
    o_center[dr] = center[sr];
    o_mask[dr] = mask[sr];
    o_pin[dr] = pin[sr];
    for (int f = 0; f < F; ++f) {
      o_nb[dr * F + f] = nb[sr * F + f];
      o_bc[dr * F + f] = bc[sr * F + f];
      o_d[dr * F + f] = dd[sr * F + f];
      o_obj[dr * F + f] = obj[sr * F + f];
    }
  }
}

static __global__ void k_combine(const Rec* __restrict__ rec, int nlev, double* out) {
  pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double m = 0, s = 0;
  long long c = 0;
  for (int l = 0; l <= nlev; ++l) {
    m = fmax(m, rec[l].max);
    s += rec[l].sumsq;
    c += rec[l].count;
  }
  out[0] = m;
  out[1] = c > 0 ? sqrt(s / (double)c) : 0.0;
}

// ---------------------------------------------------------------- coarse solve
struct CoarseDev {
  int n, nnz, n_obj;
  const int32_t* rp;
  const int32_t* ci;
  const double* val;
  const double* dinv;
  const double* c0;
  const double* cobj;   // [n_obj * n]
  const int32_t* uaddr; // unknown -> cell address in level-1 arrays (slot 0)
  double* scratch;      // 10 * n
  double rel_tol;
  int max_iters;
  int fallback_ok;      // n <= 8^D + 1
  int record;           // level 1 is a leaf (single-level mesh)
};

__device__ __forceinline__ void spmv_rows(const CoarseDev& C, const double* __restrict__ x,
                                          double* __restrict__ y) {
  for (int u = threadIdx.x; u < C.n; u += blockDim.x) {
    double s = 0;
    for (int q = C.rp[u]; q < C.rp[u + 1]; ++q) s += C.val[q] * x[C.ci[q]];
    y[u] = s;
  }
}

// Single-CTA Jacobi-BiCGStab, a line-by-line replica of detail::bicgstab
// (multigrid.hpp:208-280) with deterministic block reductions; then write-back,
// the GS-RB fallback of :586-601 when allowed, pins and the level-1 record.
// status[0] = 0 ok / 3 stall; diag[0] = rel, diag[1] = iters.
template <int D, int N>
__global__ void __launch_bounds__(1024) k_coarse(LevelView L, CoarseDev C,
                                                 const double* __restrict__ phi_b, Rec* rec,
                                                 int* status, double* diag) {
  pdl_begin();
  using G = Geo<D, N>;
  __shared__ double sm[72];
  const int n = C.n;
  double* b = C.scratch;
  double* x = b + n;
  double* r = x + n;
  double* r0 = r + n;
  double* p = r0 + n;
  double* v = p + n;
  double* s = v + n;
  double* t = s + n;
  double* ph = t + n;
  double* sh = ph + n;
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    const int ua = C.uaddr[u];
    double bu = L.rhs[ua] + C.c0[u];
    for (int o = 0; o < C.n_obj; ++o) bu += C.cobj[(size_t)o * n + u] * phi_b[o];
    b[u] = bu;
    x[u] = L.phi[ua];
    p[u] = 0;
    v[u] = 0;
  }
  __syncthreads();
  spmv_rows(C, x, r);
  __syncthreads();
  double acc = 0;
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    const double ru = b[u] - r[u];
    r[u] = ru;
    r0[u] = ru;
    acc += ru * ru;
  }
  const double norm0 = sqrt(block_sum(acc, sm));
  bool converged = false;
  double rel = 1.0;
  int iters = 0;
  if (norm0 == 0 || norm0 < 1e-300) {
    converged = true;
    rel = 0;
  } else {
    const double target = C.rel_tol * norm0;
    double rho = 1, alpha = 1, omega = 1;
    for (int it = 0; it < C.max_iters; ++it) {
      acc = 0;
      for (int u = threadIdx.x; u < n; u += blockDim.x) acc += r0[u] * r[u];
      const double rho1 = block_sum(acc, sm);
      if (rho1 == 0) break;
      if (it == 0) {
        for (int u = threadIdx.x; u < n; u += blockDim.x) {
          p[u] = r[u];
          ph[u] = C.dinv[u] * p[u];
        }
      } else {
        const double beta = (rho1 / rho) * (alpha / omega);
        for (int u = threadIdx.x; u < n; u += blockDim.x) {
          p[u] = r[u] + beta * (p[u] - omega * v[u]);
          ph[u] = C.dinv[u] * p[u];
        }
      }
      __syncthreads();
      spmv_rows(C, ph, v);
      __syncthreads();
      acc = 0;
      for (int u = threadIdx.x; u < n; u += blockDim.x) acc += r0[u] * v[u];
      const double r0v = block_sum(acc, sm);
      if (r0v == 0) break;
      alpha = rho1 / r0v;
      acc = 0;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        const double su = r[u] - alpha * v[u];
        s[u] = su;
        acc += su * su;
      }
      const double ns = sqrt(block_sum(acc, sm));
      if (ns <= target) {
        for (int u = threadIdx.x; u < n; u += blockDim.x) x[u] += alpha * ph[u];
        converged = true;
        iters = it + 1;
        rel = ns / norm0;
        break;
      }
      for (int u = threadIdx.x; u < n; u += blockDim.x) sh[u] = C.dinv[u] * s[u];
      __syncthreads();
      spmv_rows(C, sh, t);
      __syncthreads();
      double ts = 0, tt = 0;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        ts += t[u] * s[u];
        tt += t[u] * t[u];
      }
      block_sum2(ts, tt, sm);
      if (tt == 0) break;
      omega = ts / tt;
      acc = 0;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        x[u] += alpha * ph[u] + omega * sh[u];
        const double ru = s[u] - omega * t[u];
        r[u] = ru;
        acc += ru * ru;
      }
      rho = rho1;
      iters = it + 1;
      rel = sqrt(block_sum(acc, sm)) / norm0;
      if (rel <= C.rel_tol) {
        converged = true;
        break;
      }
      if (omega == 0) break;
    }
  }
  __syncthreads();
  // write_back (multigrid.hpp:577-582)
  const bool wb = converged || C.fallback_ok;
  if (wb)
    for (int u = threadIdx.x; u < n; u += blockDim.x) L.phi[C.uaddr[u]] = x[u];
  __syncthreads();
  if (threadIdx.x == 0) {
    status[0] = (converged || C.fallback_ok) ? 0 : 3;
    diag[0] = rel;
    diag[1] = (double)iters;
  }
  if (!converged && C.fallback_ok) {
    // gsrb_fallback (multigrid.hpp:586-601) on the single level-1 block
    double r0m = -1;
    bool ok = false;
    for (int it = 0; it < 20000 && !ok; ++it) {
      for (int par = 0; par < 2; ++par) {
        for (int e = threadIdx.x; e < G::H; e += blockDim.x) gs_cell<D, N>(L, L, phi_b, 0, par, e);
        __syncthreads();
      }
      if (it % 50 == 0) {
        double m = 0;
        for (int ce = threadIdx.x; ce < G::NI; ce += blockDim.x) {
          bool ins;
          const double rr = resid_cell<D, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
          if (!ins) m = fmax(m, fabs(rr));
        }
        m = block_max(m, sm);
        if (r0m < 0) r0m = m;
        if (m <= C.rel_tol * r0m || m < 1e-300) ok = true;
      }
    }
    if (!ok && threadIdx.x == 0) status[0] = 4;
    __syncthreads();
  }
  // pins (multigrid.hpp:469)
  if (L.srow[0] >= 0)
    for (int ce = threadIdx.x; ce < G::NI; ce += blockDim.x) {
      const int rr = L.row_of[(size_t)L.srow[0] * G::NI + ce];
      if (rr >= 0 && L.r_mask[rr] == 1) L.phi[ce] = phi_b[L.r_pin[rr]];
    }
  __syncthreads();
  // record_leaf_residual(1) (multigrid.hpp:471)
  double mx = 0, ss = 0, cnt = 0;
  if (L.leaf[0]) {
    for (int ce = threadIdx.x; ce < G::NI; ce += blockDim.x) {
      bool ins;
      const double rr = resid_cell<D, N>(L, L, phi_b, 0, ce / G::H, ce % G::H, &ins);
      if (ins) continue;
      mx = fmax(mx, fabs(rr));
      ss += rr * rr;
      cnt += 1;
    }
  }
  mx = block_max(mx, sm);
  ss = block_sum(ss, sm);
  cnt = block_sum(cnt, sm);
  if (threadIdx.x == 0) {
    rec[1].max = mx;
    rec[1].sumsq = ss;
    rec[1].count = (long long)cnt;
  }
}

// ---------------------------------------------------------------- field I/O
// layout 0: padded (N+2)^D per block (reference Block::data slice, mesh.hpp:47)
// layout 1: interior N^D per block, x fastest
template <int D, int N>
// own: a partitioned rank's blocks (nullptr: every block); the others are not
// written (their storage may not even be mapped, dist.h)
__global__ void __launch_bounds__(kThreads) k_scatter(int nb, double* __restrict__ dst,
                                                      const double* __restrict__ src,
                                                      const int32_t* __restrict__ slot_id,
                                                      int layout, const uint8_t* __restrict__ own) {
  pdl_begin();
  using G = Geo<D, N>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nb * G::NI) return;
  const int slot = (int)(t / G::NI);
  if (own && !own[slot]) return;
  const int ii = (int)(t % G::NI);
  const int i = ii % N, j = (ii / N) % N, k = D == 3 ? ii / (N * N) : 0;
  const long long id = slot_id[slot];
  double v;
  if (layout == 0) {
    const int s1 = N + 2;
    const long long S = D == 2 ? (long long)s1 * s1 : (long long)s1 * s1 * s1;
    v = src[id * S + (i + 1) + (j + 1) * s1 + (D == 3 ? (long long)(k + 1) * s1 * s1 : 0)];
  } else {
    v = src[id * G::NI + ii];
  }
  dst[G::addr(slot, i, j, k)] = v;
}

// var 0 = PHI (ghosts evaluated), 3 = OLD (ghosts evaluated), else ghosts = 0
template <int D, int N>
__global__ void __launch_bounds__(kThreads) k_gather(LevelView L, LevelView Lc, int var,
                                                     double* __restrict__ dst,
                                                     const int32_t* __restrict__ slot_id,
                                                     int layout) {
  pdl_begin();
  using G = Geo<D, N>;
  const int s1 = N + 2;
  const int S = D == 2 ? s1 * s1 : s1 * s1 * s1;
  const int per = layout == 0 ? S : G::NI;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L.nb * per) return;
  const int slot = (int)(t / per);
  const int q = (int)(t % per);
  int i, j, k;
  if (layout == 0) {
    i = q % s1 - 1;
    j = (q / s1) % s1 - 1;
    k = D == 3 ? q / (s1 * s1) - 1 : 0;
  } else {
    i = q % N;
    j = (q / N) % N;
    k = D == 3 ? q / (N * N) : 0;
  }
  const int out = (i < 0 || i >= N) + (j < 0 || j >= N) + (D == 3 && (k < 0 || k >= N));
  double v = 0.0;
  if (!owned(L, slot)) {  // a partitioned rank reports its own blocks (others: 0)
  } else if (out == 0) {
    const double* arr = var == 0 ? L.phi : var == 1 ? L.rhs : var == 2 ? L.res : L.old;
    v = arr ? arr[G::addr(slot, i, j, k)] : 0.0;
  } else if (out == 1) {
    if (var == 0) v = phi_at<D, N>(L, Lc, slot, i, j, k);
    else if (var == 3) v = old_at<D, N>(L, slot, i, j, k);
  }
  dst[(long long)slot_id[slot] * per + q] = v;
}

}  // namespace pmgdev
